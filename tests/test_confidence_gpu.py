"""GPU parity of dts_confidence (Eq. 7) against the fp64 oracle O7
on the same seeded fp32 inputs.  Tolerances (R22): |V_gpu - V| <= tol_V =
1e-4 * range(t)^2 (V is in squared target units: the north star's 1e-4 x range, squared),
and c = exp(-V / 2 sigma_c^2) within that tolerance carried through Eq. (7) to first
order: |c_gpu - c| <= c tol_V / (2 sigma_c^2) + 1e-6."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs, random_problem, target_range  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def gpu_conf(g, t, ss, sr, N, sc, host=False):
    if host:
        c = np.empty_like(t)
        v = np.empty_like(t)
        with dts.Solver(g, ss, sr, N) as s:
            s.confidence(np.ascontiguousarray(t), sc, out=c, var_out=v)
        return c.astype(np.float64), v.astype(np.float64)
    gd, td = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t))
    c = torch.empty_like(td)
    v = torch.empty_like(td)
    with dts.Solver(gd, ss, sr, N) as s:
        s.confidence(td, sc, out=c, var_out=v)
    torch.cuda.synchronize()
    return c.cpu().numpy().astype(np.float64), v.cpu().numpy().astype(np.float64)


def check(g, t, ss, sr, N, sc, **kw):
    cr, vr = oracle.confidence(g, t, ss, sr, N, sc)
    c, v = gpu_conf(g, t, ss, sr, N, sc, **kw)
    rng = max(target_range(t), 1e-30)
    tol_v = 1e-4 * rng * rng
    assert np.all(np.isfinite(c)) and np.all(v >= 0) and np.all((c > 0) & (c <= 1))
    assert np.max(np.abs(v - vr)) <= tol_v, np.max(np.abs(v - vr)) / rng ** 2
    assert np.all(np.abs(c - cr) <= cr * tol_v / (2 * sc * sc) + 1e-6), np.max(np.abs(c - cr))


@pytest.mark.parametrize("H,W", [(1, 1), (1, 9), (9, 1), (48, 64), (61, 97), (700, 130), (2600, 35), (13, 3000)])
def test_confidence_shapes(H, W):
    g, t, _ = random_problem(H, W, 3, 1, seed=H + 2 * W)
    check(g, t, 6.0, 0.2, 3, 0.3)


@pytest.mark.parametrize("name,sc", [("C1", 16.0), ("C2", 0.5)])
def test_confidence_configs(name, sc):
    """Disparity (C1, range ~264, sigma_c = 16 disparity units as SPEC S:210) and depth (C2)."""
    cfg = CONFIGS[name]
    g, t, _ = make_inputs(name)
    check(g, t, cfg.sigma_s, cfg.sigma_r, cfg.N, sc)


def test_confidence_offset_target_and_constant():
    g, t, _ = random_problem(80, 90, 3, 1, seed=9)
    check(g, (t + 1000.0).astype(np.float32), 5.0, 0.2, 3, 0.5)  # |t| >> range: shift-invariant path
    tc = np.full((80, 90), 7.5, np.float32)
    c, v = gpu_conf(g, tc, 5.0, 0.2, 3, 0.5)
    assert np.all(v == 0) and np.all(c == 1)


def test_confidence_host_pointers_match_device():
    g, t, _ = random_problem(70, 50, 3, 1, seed=13)
    a = gpu_conf(g, t, 5.0, 0.2, 3, 0.4)
    b = gpu_conf(g, t, 5.0, 0.2, 3, 0.4, host=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_confidence_argument_errors():
    g, t, _ = random_problem(10, 12, 3, 1, seed=1)
    gd, td = (torch.from_numpy(a).cuda() for a in (g, t))
    c = torch.empty_like(td)
    with dts.Solver(gd, 5.0, 0.2, 3) as s:
        for bad in (0.0, -1.0, float("nan"), float("inf")):
            with pytest.raises(dts.DTSError) as ei:
                dts.dts_confidence(s.ctx, td, bad, c)
            assert ei.value.status == 1
        with pytest.raises(dts.DTSError) as ei:
            dts.dts_confidence(s.ctx, td, 0.5, td)  # conf_out aliases target
        assert ei.value.status == 1


def test_confidence_then_solve():
    """The paper's stereo pipeline order: confidence of the target feeds the solve."""
    cfg = CONFIGS["C0"]
    g, t, _ = make_inputs("C0")
    cr, _ = oracle.confidence(g, t, cfg.sigma_s, cfg.sigma_r, cfg.N, 0.2)
    ref = oracle.solve(g, t, cr.astype(np.float32), cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
    gd, td = (torch.from_numpy(a).cuda() for a in (g, t))
    with dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
        c = s.confidence(td, 0.2)
        out = s.solve(td, c, cfg.lam, cfg.iters)
    torch.cuda.synchronize()
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= 1e-4 * target_range(t)


def test_confidence_per_plane_over_row_strips():
    """Too tall for the two-plane cluster column kernel (C_t = 2 holds <= 5120 rows): the passes
    run plane by plane, over row strips with the seam fix-up (forced: col_strips = 2)."""
    g, t, _ = random_problem(5400, 160, 3, 1, seed=5)
    with dts.options(col_strips=2):
        with dts.Solver(torch.from_numpy(g).cuda(), 6.0, 0.2, 3) as s:
            assert dts.debug_strips(s.ctx)["strips"] == 2
        check(g, t, 6.0, 0.2, 3, 0.3)


def test_confidence_taller_than_a_cluster():
    g, t, _ = random_problem(11000, 40, 3, 1, seed=8)
    check(g, t, 6.0, 0.2, 3, 0.3)
