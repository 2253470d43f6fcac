"""GPU parity of the per-iteration residual output (dts_solve_opts.resid_inf_out, SURVEY 2.3
K8): resid[k] = ||g_k||_inf of the Eq. (3) gradient at iterate k (reading R13),
computed on the device inside the update kernels, against the oracle's diagnostic (pinned in
tests/test_oracle_pins.py against the dense operator)."""
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


def solve_with_resid(g, t, c, ss, sr, N, lam, iters, **opts):
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    r = torch.full((max(iters, 1),), -1.0, device="cuda")
    with dts.Solver(gd, ss, sr, N) as s:
        s.solve(td, cd, lam, iters, out=out, resid_inf_out=r, **opts)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), r.cpu().numpy()[:iters].astype(np.float64)


@pytest.mark.parametrize("H,W,Ct", [(48, 64, 1), (300, 410, 1), (70, 90, 3), (1000, 37, 1), (33, 2000, 2)])
def test_residual_output_matches_oracle(H, W, Ct):
    """On the cluster column path and (tall narrow shape) the decoupled one, C_t = 1..3."""
    g, t, c = random_problem(H, W, 3, Ct, seed=H + W + Ct)
    iters = 12
    ref, diag = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.99, iters, diagnostics=True)
    got, r = solve_with_resid(g, t, c, 6.0, 0.2, 3, 0.99, iters)
    rng = target_range(t)
    assert np.max(np.abs(got - ref)) <= TOL * rng  # the residual path solves the same problem
    assert np.all(r >= 0)
    np.testing.assert_allclose(r, diag[:, 0], rtol=0, atol=TOL * rng)
    assert np.all(np.diff(r) <= 1e-6 * r[0])  # non-increasing (R13), at fp32 resolution


def test_residual_output_decoupled_kernel_and_step_option():
    g, t, c = random_problem(200, 150, 3, 1, seed=5)
    _, diag = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.5, 8, step=0.7, diagnostics=True)
    with dts.options(col_kernel=1):
        _, r = solve_with_resid(g, t, c, 6.0, 0.2, 3, 0.5, 8, step=0.7)
    np.testing.assert_allclose(r, diag[:, 0], rtol=0, atol=TOL * target_range(t))


def test_residual_output_host_buffer_c1():
    """C1 (the stereo shape), all 50 iterations, into a HOST buffer."""
    cfg = CONFIGS["C1"]
    g, t, c = make_inputs("C1")
    _, diag = oracle.solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters, diagnostics=True)
    r = np.full(cfg.iters, -1.0, np.float32)  # host memory: the library copies into it and syncs
    with dts.Solver(torch.from_numpy(g).cuda(), cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
        o = torch.empty(t.shape, device="cuda")
        s.solve(torch.from_numpy(t).cuda(), torch.from_numpy(c).cuda(), cfg.lam, cfg.iters, out=o, resid_inf_out=r)
    np.testing.assert_allclose(r, diag[:, 0], rtol=0, atol=TOL * target_range(t))


def test_residual_output_box_context():
    g, t, c = random_problem(60, 80, 3, 1, seed=9)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    r = torch.zeros(5, device="cuda")
    with dts.Solver(gd, 6.0, 0.2, 3, filter=dts.DTS_FILTER_BOX) as s:
        o = torch.empty_like(td)
        s.solve(td, cd, 0.99, 5, out=o, resid_inf_out=r)
    torch.cuda.synchronize()
    rr = r.cpu().numpy()
    assert np.all(rr > 0) and np.all(np.isfinite(rr))
    assert np.all(np.diff(rr) <= 1e-6 * rr[0])


def test_paper_shapes_c1_c2_parity():
    """C1 and C2 (the paper's stereo and 16x SR shapes) at full iteration counts."""
    for name in ("C1", "C2"):
        cfg = CONFIGS[name]
        g, t, c = make_inputs(name)
        ref = oracle.solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
        got, _ = solve_with_resid(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
        assert np.max(np.abs(got - ref)) <= TOL * target_range(t), name
