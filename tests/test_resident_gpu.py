"""GPU parity of the SMEM-resident solve (k_resident.cu: the whole iteration loop of a C_t = 1
solve in one cooperative launch, the image held in the shared memory of one CTA per tile, only
the filter carries crossing tiles) and of the per-iteration residual output
(dts_solve_opts.resid_inf_out), against the fp64 oracle (O6 and its
diagnostics, pinned in tests/test_oracle_pins.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs, random_problem, target_range  # noqa: E402

TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def solve(g, t, c, ss, sr, N, lam, iters, resident=1, resid=False, **opts):
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    r = torch.full((max(iters, 1),), -1.0, device="cuda") if resid else None
    with dts.options(resident=resident), dts.Solver(gd, ss, sr, N) as s:
        if resid:
            opts["resid_inf_out"] = r
        s.solve(td, cd, lam, iters, out=out, **opts)
        launches = dts.dts_launch_count(s.ctx)
    torch.cuda.synchronize()
    res = out.cpu().numpy().astype(np.float64)
    return (res, r.cpu().numpy()[:iters].astype(np.float64), launches) if resid else (res, launches)


# shapes around the kernel's tiling: one tile (C0-like, tiny, single row / column), tile widths
# 128 / 64 / 32 with ragged last tile columns and rows, tall-narrow and wide-short grids, a single
# tile row or column (no exchange along one axis), and the largest tilings that fit 148 SMs
SHAPES = [(1, 1), (1, 7), (7, 1), (2, 2), (48, 64), (3, 513), (31, 33), (33, 31), (61, 97), (5, 130),
          (130, 5), (257, 3), (700, 130), (1000, 37), (129, 1025), (47, 1536), (1000, 1400), (1024, 1376),
          (1500, 1000), (3000, 700), (6000, 100), (90, 4700), (1300, 1800)]


def fits(H, W, sms=148):
    """Mirror of plan_resident's capacity rule (k_resident.cu): some tile width TW in {128, 64,
    32} with TC = ceil(W / TW) tile columns and TR <= sms / TC tile rows of TH <= 96 / 192 / 384."""
    for tw, thmax in ((128, 96), (64, 192), (32, 384)):
        tc = -(-W // tw)
        if tc > sms:
            continue
        th = -(-H // (sms // tc))
        if th <= thmax:
            return True
    return False


@pytest.mark.parametrize("H,W", SHAPES)
def test_resident_parity(H, W):
    g, t, c = random_problem(H, W, 3, 1, seed=11 * H + W)
    iters = 4 if H * W > 200000 else 7
    ref = oracle.solve(g, t, c, 5.0, 0.2, 3, 0.99, iters)
    got, launches = solve(g, t, c, 5.0, 0.2, 3, 0.99, iters)
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)
    if fits(H, W):
        assert launches <= 8  # create (<= 5 launches) + prologue + the resident kernel


@pytest.mark.parametrize("N", [1, 2, 4])
def test_resident_pass_counts(N):
    g, t, c = random_problem(300, 410, 3, 1, seed=N + 40)
    ref = oracle.solve(g, t, c, 9.0, 0.15, N, 0.99, 5)
    got, _ = solve(g, t, c, 9.0, 0.15, N, 0.99, 5)
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_resident_paper_shapes(name):
    """The paper's stereo (C1) and 16x SR (C2) shapes, full iteration count."""
    cfg = CONFIGS[name]
    g, t, c = make_inputs(name)
    ref = oracle.solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
    got, launches = solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)
    # same result as the per-pass kernels to fp32 rounding
    other, launches2 = solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters, resident=0)
    assert np.max(np.abs(got - other)) <= 1e-5 * target_range(t)
    assert launches2 > 6 * cfg.iters > launches


def test_resident_options_step_and_support_mode():
    g, t, c = random_problem(200, 300, 3, 1, seed=3)
    ref = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.5, 6, step=0.7, support_mode=1)
    got, _ = solve(g, t, c, 6.0, 0.2, 3, 0.5, 6, step=0.7, support_mode=1)
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)


def test_resident_repeats_bit_identical():
    """Race stress: ten solves through one context (epoch-tagged flags reused across launches)
    and interleaved solves of a second context give bit-identical outputs."""
    g, t, c = random_problem(1000, 1400, 3, 1, seed=8)
    g2, t2, c2 = random_problem(333, 999, 3, 1, seed=9)
    dev = [torch.from_numpy(a).cuda() for a in (g, t, c, g2, t2, c2)]
    outs, outs2 = [], []
    with dts.Solver(dev[0], 16.0, 0.1, 3) as s, dts.Solver(dev[3], 8.0, 0.2, 3) as s2:
        for k in range(10):
            o = torch.empty_like(dev[1])
            s.solve(dev[1], dev[2], 0.99, 3 + (k % 2), out=o)
            outs.append(o)
            o2 = torch.empty_like(dev[4])
            s2.solve(dev[4], dev[5], 0.99, 5, out=o2)
            outs2.append(o2)
    torch.cuda.synchronize()
    for group in (outs[0::2], outs[1::2], outs2):
        ref = group[0].cpu().numpy()
        assert np.isfinite(ref).all()
        for o in group[1:]:
            assert np.array_equal(o.cpu().numpy(), ref)


# ---------------------------------------------------------------- K8: per-iteration residual
@pytest.mark.parametrize("resident", [1, 0])
@pytest.mark.parametrize("H,W,Ct", [(48, 64, 1), (300, 410, 1), (70, 90, 3)])
def test_residual_output_matches_oracle(H, W, Ct, resident):
    """resid_inf_out[k] = ||g_k||_inf of the Eq. (3) gradient at iterate k (reading R13),
    against the oracle's pinned diagnostic; on both solve paths (and the multi-channel one)."""
    g, t, c = random_problem(H, W, 3, Ct, seed=H + W + Ct)
    iters = 12
    _, diag = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.99, iters, diagnostics=True)
    got, r, _ = solve(g, t, c, 6.0, 0.2, 3, 0.99, iters, resident=resident, resid=True)
    ref = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.99, iters)
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)  # the residual path solves the same
    assert np.all(r >= 0)
    np.testing.assert_allclose(r, diag[:, 0], rtol=0, atol=TOL * target_range(t))
    assert np.all(np.diff(r) <= 1e-6 * r[0])  # non-increasing (R13), at fp32 resolution


def test_residual_output_host_buffer_and_c1():
    cfg = CONFIGS["C1"]
    g, t, c = make_inputs("C1")
    _, diag = oracle.solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters, diagnostics=True)
    r = np.full(cfg.iters, -1.0, np.float32)  # a HOST buffer: the library copies into it and syncs
    with dts.Solver(torch.from_numpy(g).cuda(), cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
        o = torch.empty(t.shape, device="cuda")
        s.solve(torch.from_numpy(t).cuda(), torch.from_numpy(c).cuda(), cfg.lam, cfg.iters, out=o, resid_inf_out=r)
    np.testing.assert_allclose(r, diag[:, 0], rtol=0, atol=TOL * target_range(t))
