"""Batched contexts (dts_create_batch, include/dts.h): B independent images in one context.
Each image's result must equal the fp64 oracle on that image alone ("eight 4K images" are
independent problems; reading R4 restarts every recurrence at an image's first row) within the
north-star tolerance, and the separate single-image contexts of the CUDA path to fp32 rounding."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import random_problem, target_range  # noqa: E402

TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def problems(B, H, W, C, Ct, seed):
    ps = [random_problem(H, W, C, Ct, seed=seed + 17 * b) for b in range(B)]
    g = np.stack([p[0] for p in ps])
    t = np.stack([p[1] for p in ps])
    c = np.stack([p[2] for p in ps])
    return ps, g, t, c


def batch_solve(g, t, c, ss, sr, N, lam, iters, **kw):
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    with dts.Solver(gd, ss, sr, N, batched=True) as s:
        s.solve(td, cd, lam, iters, out=out, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def single_solve(g, t, c, ss, sr, N, lam, iters):
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    with dts.Solver(gd, ss, sr, N) as s:
        s.solve(td, cd, lam, iters, out=out)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("B,H,W,C,Ct,N", [(3, 70, 97, 3, 1, 3), (4, 40, 300, 3, 3, 3), (2, 129, 64, 1, 2, 2),
                                          (5, 33, 45, 3, 4, 3), (3, 50, 80, 3, 1, 5)])
def test_batch_equals_oracle_per_image(B, H, W, C, Ct, N):
    ps, g, t, c = problems(B, H, W, C, Ct, seed=B * 100 + H)
    got = batch_solve(g, t, c, 12.0, 0.3, N, 0.99, 4)
    for b, (gb, tb, cb) in enumerate(ps):
        ref = oracle.solve(gb, tb, cb, 12.0, 0.3, N, 0.99, 4)
        err = float(np.max(np.abs(got[b] - ref)))
        assert err <= TOL * target_range(tb), (b, err)


@pytest.mark.parametrize("Ct", [1, 3])
def test_batch_matches_single_contexts_tall(Ct):
    """Images whose stack is taller than one cluster column holds (C_t = 3: 10240 rows): the
    batched plan runs image-high strips; every image must match its own context to fp32
    rounding (same arithmetic, the cut coefficient is an exact 0)."""
    B, H, W = 4, 2600, 160
    ps, g, t, c = problems(B, H, W, 3, Ct, seed=7)
    got = batch_solve(g, t, c, 30.0, 0.1, 3, 0.99, 3)
    for b, (gb, tb, cb) in enumerate(ps):
        one = single_solve(gb, tb, cb, 30.0, 0.1, 3, 0.99, 3)
        np.testing.assert_allclose(got[b], one, rtol=0, atol=2e-6 * target_range(tb))


def test_batch_tall_image_against_oracle():
    """C3-high images (2 x 2160 rows, C_t = 3, the batched strip plan) at a reduced width:
    image 1 against the oracle, every element."""
    B, H, W = 2, 2160, 48
    ps, g, t, c = problems(B, H, W, 3, 3, seed=11)
    got = batch_solve(g, t, c, 30.0, 0.1, 3, 0.99, 2)
    gb, tb, cb = ps[1]
    ref = oracle.solve(gb, tb, cb, 30.0, 0.1, 3, 0.99, 2)
    assert float(np.max(np.abs(got[1] - ref))) <= TOL * target_range(tb)


def test_batch_of_one_is_dts_create():
    (gb, tb, cb), = [random_problem(90, 70, 3, 1, seed=3)]
    got = batch_solve(gb[None], tb[None], cb[None], 8.0, 0.2, 3, 0.99, 5)[0]
    one = single_solve(gb, tb, cb, 8.0, 0.2, 3, 0.99, 5)
    np.testing.assert_array_equal(got, one)


def test_batch_support_and_distances_cut_between_images():
    """dts_debug_read on a batched context: d_y is +inf at every image's first row and the
    support of each image equals its own context's."""
    B, H, W = 3, 25, 31
    ps, g, _, _ = problems(B, H, W, 3, 1, seed=5)
    with dts.Solver(torch.from_numpy(g).cuda(), 8.0, 0.2, 3, batched=True) as s:
        dy = s.read(dts.DTS_BUF_DY)
        sup = s.read(dts.DTS_BUF_SUPPORT)
    assert dy.shape == (B * H, W)
    for b, (gb, _, _) in enumerate(ps):
        assert np.all(np.isinf(dy[b * H]))
        with dts.Solver(torch.from_numpy(gb).cuda(), 8.0, 0.2, 3) as s1:
            np.testing.assert_array_equal(dy[b * H:(b + 1) * H], s1.read(dts.DTS_BUF_DY))
            np.testing.assert_allclose(sup[b * H:(b + 1) * H], s1.read(dts.DTS_BUF_SUPPORT), rtol=1e-6)


def test_batch_residual_is_max_over_images():
    B, H, W = 3, 40, 50
    ps, g, t, c = problems(B, H, W, 3, 1, seed=9)
    r_b = torch.zeros(3, device="cuda")
    batch_solve(g, t, c, 8.0, 0.2, 3, 0.99, 3, resid_inf_out=r_b)
    per = []
    for gb, tb, cb in ps:
        r = torch.zeros(3, device="cuda")
        gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (gb, tb, cb))
        with dts.Solver(gd, 8.0, 0.2, 3) as s:
            s.solve(td, cd, 0.99, 3, out=torch.empty_like(td), resid_inf_out=r)
        per.append(r.cpu().numpy())
    np.testing.assert_allclose(r_b.cpu().numpy(), np.max(per, axis=0), rtol=1e-6)


def test_batch_confidence_matches_single():
    B, H, W = 2, 60, 70
    ps, g, t, _ = problems(B, H, W, 3, 1, seed=13)
    gd, td = torch.from_numpy(g).cuda(), torch.from_numpy(t).cuda()
    with dts.Solver(gd, 8.0, 0.2, 3, batched=True) as s:
        conf = s.confidence(td, 0.25).cpu().numpy()
    for b, (gb, tb, _) in enumerate(ps):
        with dts.Solver(torch.from_numpy(gb).cuda(), 8.0, 0.2, 3) as s1:
            one = s1.confidence(torch.from_numpy(tb).cuda(), 0.25).cpu().numpy()
        np.testing.assert_allclose(conf[b], one, rtol=0, atol=1e-5)


def test_batch_argument_errors():
    g = torch.zeros(2, 8, 8, 3, device="cuda")
    lib = dts.load_library()
    import ctypes
    ctx = ctypes.c_void_p()
    for B, H in ((0, 8), (2, 0), (-1, 8)):
        assert lib.dts_create_batch(g.data_ptr(), B, H, 8, 3, 8.0, 0.2, 3, None, ctypes.byref(ctx)) != 0
        assert ctx.value is None
    assert lib.dts_create_batch(g.data_ptr(), 1 << 20, 1 << 20, 8, 3, 8.0, 0.2, 3, None, ctypes.byref(ctx)) == \
        2  # DTS_E_SHAPE


@pytest.mark.parametrize("rows", [12, 16])
def test_three_channel_segment_lengths(rows):
    """C_t = 3 column kernel at 12- and 16-row warp segments (option col_rows; the batched C3
    plan takes 12): parity with the oracle, batched and single."""
    B, H, W = 2, 700, 150
    ps, g, t, c = problems(B, H, W, 3, 3, seed=rows)
    with dts.options(col_rows=rows):
        with dts.Solver(torch.from_numpy(g).cuda(), 10.0, 0.2, 3, batched=True) as s:
            assert dts.debug_col_plan(s.ctx, 3)["Ls"] == rows
        got = batch_solve(g, t, c, 10.0, 0.2, 3, 0.99, 3)
        one = single_solve(*ps[0], 10.0, 0.2, 3, 0.99, 3)
    for b, (gb, tb, cb) in enumerate(ps):
        ref = oracle.solve(gb, tb, cb, 10.0, 0.2, 3, 0.99, 3)
        assert float(np.max(np.abs(got[b] - ref))) <= TOL * target_range(tb)
    assert float(np.max(np.abs(one - oracle.solve(*ps[0], 10.0, 0.2, 3, 0.99, 3)))) <= TOL * target_range(ps[0][1])


def test_batch_host_pointers_match_device():
    """dts_create_batch / dts_solve with numpy (host) arrays: the library stages them; same
    result as device tensors."""
    B, H, W = 3, 50, 70
    ps, g, t, c = problems(B, H, W, 3, 2, seed=31)
    dev = batch_solve(g, t, c, 8.0, 0.2, 3, 0.99, 4)
    ctx = dts.dts_create_batch(np.ascontiguousarray(g), 8.0, 0.2, 3)
    try:
        out = np.empty_like(t)
        dts.dts_solve(ctx, np.ascontiguousarray(t), np.ascontiguousarray(c), 0.99, 4, out)
    finally:
        dts.dts_destroy(ctx)
    np.testing.assert_array_equal(out.astype(np.float64), dev)

