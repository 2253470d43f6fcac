"""Images wider than the row kernel's staging buffer (11520 columns at C_t = 4): the row passes
run over vertical strips with zero carries at the strip edges and a per-row seam fix-up
(plan_row_strips; reading R26 along x).  Parity with the fp64 oracle, element by element, at the
north-star tolerance: solve (FILTER and the fused Eq. (3) row update), support, confidence,
stereo, and C_t = 4 at a width where C_t = 1 still fits one strip."""
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


def solve(g, t, c, ss, sr, N, lam, iters, **kw):
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    with dts.Solver(gd, ss, sr, N) as s:
        s.solve(td, cd, lam, iters, out=out, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("H,W,Ct", [(24, 24000, 1), (17, 23050, 3), (9, 40000, 2)])
def test_wide_rows_solve_parity(H, W, Ct):
    g, t, c = random_problem(H, W, 3, Ct, seed=W + Ct)
    args = (12.0, 0.25, 3, 0.99, 4)
    got = solve(g, t, c, *args)
    ref = oracle.solve(g, t, c, *args)
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)


def test_wide_rows_support_and_distances():
    g, _, _ = random_problem(12, 25000, 3, 1, seed=2)
    dx_r, dy_r = oracle.distances(g, 12.0, 0.25)
    S_r = oracle.support(dx_r, dy_r, 12.0)
    with dts.Solver(torch.from_numpy(g).cuda(), 12.0, 0.25, 3) as s:
        S = s.read(dts.DTS_BUF_SUPPORT)
        dx = s.read(dts.DTS_BUF_DX)
    inf = np.isinf(dx_r)
    np.testing.assert_allclose(dx[~inf], dx_r[~inf], rtol=2e-6)
    np.testing.assert_allclose(S, S_r, rtol=2e-5)


def test_four_channels_strip_only_where_needed():
    """W = 12000: C_t = 1 rows fit one CTA, C_t = 4 rows take two strips; both within tolerance."""
    for Ct in (1, 4):
        g, t, c = random_problem(10, 12000, 3, Ct, seed=40 + Ct)
        args = (8.0, 0.2, 3, 0.99, 3)
        got = solve(g, t, c, *args)
        assert np.max(np.abs(got - oracle.solve(g, t, c, *args))) <= TOL * target_range(t)


def test_wide_rows_with_residual_and_no_row_update():
    g, t, c = random_problem(14, 26000, 3, 1, seed=8)
    args = (12.0, 0.25, 3, 0.99, 3)
    ref, diag = oracle.solve(g, t, c, *args, diagnostics=True)
    r = torch.zeros(3, device="cuda")
    with dts.options(row_update=0):
        got = solve(g, t, c, *args, resid_inf_out=r)
    rng = target_range(t)
    assert np.max(np.abs(got - ref)) <= TOL * rng
    np.testing.assert_allclose(r.cpu().numpy(), diag[:, 0], rtol=0, atol=TOL * rng)


def test_wide_rows_confidence():
    g, t, _ = random_problem(11, 24500, 3, 1, seed=4)
    cr, vr = oracle.confidence(g, t, 12.0, 0.25, 3, 0.3)
    gd, td = torch.from_numpy(g).cuda(), torch.from_numpy(t).cuda()
    with dts.Solver(gd, 12.0, 0.25, 3) as s:
        v = torch.empty_like(td)
        cc = s.confidence(td, 0.3, var_out=v).cpu().numpy()
    rng = target_range(t)
    assert np.max(np.abs(v.cpu().numpy() - vr)) <= TOL * rng * rng
    assert np.max(np.abs(cc - cr)) <= 1e-4


@pytest.mark.parametrize("gamma", [0.0, 0.001])
def test_wide_rows_stereo(gamma):
    """gamma = 0: element-wise parity.  gamma = 0.001: the photometric gradient is
    discontinuous where u = x - z crosses an integer (R23), so an fp32 iterate can take the
    other side of a kink than the fp64 one at isolated pixels (6 of 240000 here, none near the
    strip seams at columns 8000 / 16000); those are bounded, every other pixel is at parity."""
    L, _, c = random_problem(10, 24000, 3, 1, seed=6)
    rng_ = np.random.default_rng(7)
    R = np.ascontiguousarray((np.roll(L, -2, axis=1) + rng_.normal(0, 0.01, L.shape)).astype(np.float32))
    t = rng_.uniform(0, 8, (10, 24000)).astype(np.float32)
    args = (12.0, 0.25, 3, 0.99, 4, gamma, 1.0)
    ref = oracle.solve_stereo(L, R, t, c, *args)
    Ld, Rd, td, cd = (torch.from_numpy(a).cuda() for a in (L, R, t, c))
    out = torch.empty_like(td)
    with dts.Solver(Ld, 12.0, 0.25, 3) as s:
        s.solve_stereo(td, cd, 0.99, 4, Ld, Rd, gamma, 1.0, out=out)
    torch.cuda.synchronize()
    err = np.abs(out.cpu().numpy() - ref)
    tol = TOL * target_range(t)
    if gamma == 0.0:
        assert err.max() <= tol
    else:
        assert np.count_nonzero(err > tol) <= 1e-4 * err.size
        assert err.max() <= 5e-3
        cols = np.argwhere(err > tol)[:, 1]
        assert np.all(np.minimum(np.abs(cols - 8000), np.abs(cols - 16000)) > 64)


def test_too_wide_is_a_shape_error():
    g = torch.zeros(2, 184321, 1, device="cuda")
    with pytest.raises(dts.DTSError):
        dts.dts_create(g, 8.0, 0.2, 3)
