"""Pins for the fp64 oracle (CPU only).  Each test checks the oracle against
something other than itself: values hand-derived in tests/golden (cited there),
closed forms, dense triangular matrices built from their product formulas
(tests/dense.py), brute-force sums, invariants and the paper's stated
reductions.  Chosen so that a dropped term, wrong sign, wrong index (A[k] vs
A[k+1]), transposed operand or wrong pass order fails at least one test."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests import dense
from synth import make_inputs, random_problem, target_range

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
SS = GOLD["sigma_s"]  # a = 1/2


def const_guide(H, W, C=3, v=0.3):
    return np.full((H, W, C), v, np.float32)


# ------------------------------------------------------------------ O1
def test_distances_spec_examples():
    dx, dy = oracle.distances(const_guide(1, 5), 8.0, 0.2)
    np.testing.assert_array_equal(dx[0], GOLD["distances_spec"]["constant_row_dx"])
    assert np.all(np.isinf(dy))
    g = np.array([[[0.0], [1.0]]], np.float32)
    dx, _ = oracle.distances(g, 0.5, 0.5)
    np.testing.assert_allclose(dx[0], GOLD["distances_spec"]["ramp_dx"], rtol=1e-15)


def test_distances_hand_2x2():
    e = GOLD["distances_2x2"]
    g = np.array(e["guide"], np.float32)[:, :, None]
    dx, dy = oracle.distances(g, e["sigma_s"], e["sigma_r"])
    np.testing.assert_allclose(dx, np.array(e["dx"]), rtol=1e-6)
    np.testing.assert_allclose(dy, np.array(e["dy"]), rtol=1e-6)


def test_distances_invariants():
    rng = np.random.default_rng(1)
    g1 = rng.uniform(0, 1, (7, 9, 2)).astype(np.float32)
    g2 = rng.uniform(0, 1, (7, 9, 3)).astype(np.float32)
    ss, sr = 5.0, 0.3
    dx1, dy1 = oracle.distances(g1, ss, sr)
    dx2, dy2 = oracle.distances(g2, ss, sr)
    dx12, dy12 = oracle.distances(np.concatenate([g1, g2], 2), ss, sr)
    fin = np.isfinite(dx12)
    # squared increments add over channels (L2 isometry)
    np.testing.assert_allclose((dx12 ** 2 - 1)[fin], ((dx1 ** 2 - 1) + (dx2 ** 2 - 1))[fin], rtol=1e-12)
    fin = np.isfinite(dy12)
    np.testing.assert_allclose((dy12 ** 2 - 1)[fin], ((dy1 ** 2 - 1) + (dy2 ** 2 - 1))[fin], rtol=1e-12)
    # vertical distances are horizontal distances of the transposed guide
    dxt, dyt = oracle.distances(np.ascontiguousarray(g1.transpose(1, 0, 2)), ss, sr)
    np.testing.assert_array_equal(dy1, dxt.T)
    np.testing.assert_array_equal(dx1, dyt.T)
    # monotone DT: every finite increment >= 1; sentinels exactly on first column / row
    assert np.all(dx1[:, 1:] >= 1) and np.all(np.isinf(dx1[:, 0]))
    assert np.all(dy1[1:] >= 1) and np.all(np.isinf(dy1[0]))
    # sigma scaling enters only through sigma_s / sigma_r
    dxs, _ = oracle.distances(g1, 2 * ss, 2 * sr)
    np.testing.assert_allclose(dxs, dx1, rtol=1e-14)


# ------------------------------------------------------------------ O2
@pytest.mark.parametrize("N", [1, 2, 3, 5])
def test_sigma_schedule(N):
    s = oracle.sigmas(16.0, N)
    assert math.isclose(float(np.sum(s ** 2)), 256.0, rel_tol=1e-12)  # variances add to sigma_s^2
    np.testing.assert_allclose(s[:-1] / s[1:], 2.0, rtol=1e-12)       # halving per pass
    if N == 1:
        assert math.isclose(s[0], 16.0, rel_tol=1e-14)


# ------------------------------------------------------------------ O3
def test_rf1d_worked_example():
    e = GOLD["impulse_1x5"]
    A = np.array([0, .5, .5, .5, .5])
    np.testing.assert_allclose(oracle.rf1d(e["x"], A), e["dtf"], rtol=0, atol=1e-16)


@pytest.mark.parametrize("n", [1, 2, 3, 8, 13])
def test_rf1d_equals_dense_triangular(n):
    rng = np.random.default_rng(n)
    A = rng.uniform(0, 0.95, n)
    A[0] = 0.0
    x = rng.normal(size=n)
    np.testing.assert_allclose(oracle.rf1d(x, A), dense.pass1d(A) @ x, rtol=1e-13, atol=1e-14)


def test_rf1d_row_stochastic_and_edge_free_kernel():
    rng = np.random.default_rng(3)
    A = rng.uniform(0, 0.99, 50)
    A[0] = 0
    np.testing.assert_allclose(oracle.rf1d(np.full(50, 2.5), A), 2.5, rtol=1e-14)
    a, n = 0.8, 801
    A = np.full(n, a)
    A[0] = 0
    x = np.zeros(n)
    x[n // 2] = 1.0
    z = oracle.rf1d(x, A)
    half = 200
    np.testing.assert_allclose(z[n // 2 - half:n // 2 + half + 1], dense.edge_free_kernel(a, half),
                               rtol=1e-12, atol=1e-18)


# ------------------------------------------------------------------ O4
def test_dtf_worked_examples():
    g = const_guide(1, 5)
    dx, dy = oracle.distances(g, SS, 0.1)
    np.testing.assert_allclose(oracle.dtf(np.array([[0, 0, 1, 0, 0.]]), dx, dy, SS, 1)[0],
                               GOLD["impulse_1x5"]["dtf"], atol=1e-15)
    g = const_guide(2, 2)
    dx, dy = oracle.distances(g, SS, 0.1)
    np.testing.assert_allclose(oracle.dtf(np.array(GOLD["dtf_2x2"]["t"], float), dx, dy, SS, 1),
                               GOLD["dtf_2x2"]["dtf"], atol=1e-15)
    g = const_guide(1, 2)
    dx, dy = oracle.distances(g, SS, 0.1)
    K = np.stack([oracle.dtf(np.array([[1., 0]]), dx, dy, SS, 1)[0],
                  oracle.dtf(np.array([[0., 1]]), dx, dy, SS, 1)[0]], 1)
    np.testing.assert_allclose(K, GOLD["pair_1x2"]["K"], atol=1e-15)


@pytest.mark.parametrize("H,W,N", [(1, 6, 2), (5, 1, 1), (4, 5, 3), (6, 7, 3), (3, 3, 4)])
def test_dtf_equals_dense_operator(H, W, N):
    rng = np.random.default_rng(H * 100 + W)
    dx = rng.uniform(1, 4, (H, W))
    dy = rng.uniform(1, 4, (H, W))
    dx[:, 0] = np.inf
    dy[0, :] = np.inf
    ss = 3.0
    K = dense.dtf_operator(dx, dy, oracle.sigmas(ss, N))
    assert np.all(K >= -1e-15)
    np.testing.assert_allclose(K.sum(1), 1.0, rtol=1e-13)              # row-stochastic
    X = rng.normal(size=(2, H, W))
    Y = oracle.dtf(X, dx, dy, ss, N)
    for ch in range(2):
        np.testing.assert_allclose(Y[ch].ravel(), K @ X[ch].ravel(), rtol=1e-12, atol=1e-13)


def test_dtf_order_rows_then_columns_matters():
    """Pass order is part of the definition (reading R6): columns-first differs."""
    rng = np.random.default_rng(5)
    dx = rng.uniform(1, 5, (4, 4)); dx[:, 0] = np.inf
    dy = rng.uniform(1, 5, (4, 4)); dy[0] = np.inf
    s = oracle.sigmas(3.0, 1)
    Kr = dense.dtf_operator(dx, dy, s)
    Ax = np.exp(-np.sqrt(2) * dx / s[0]); Ay = np.exp(-np.sqrt(2) * dy / s[0])
    Kc = dense.row_operator(Ax) @ dense.col_operator(Ay)
    X = rng.normal(size=(4, 4))
    Y = oracle.dtf(X, dx, dy, 3.0, 1).ravel()
    np.testing.assert_allclose(Y, Kr @ X.ravel(), rtol=1e-12)
    assert np.max(np.abs(Y - Kc @ X.ravel())) > 1e-6


def test_dtf_edge_free_cascade_closed_form():
    """Edge-free guide: the N-pass cascade is the convolution of the per-pass kernels
    (1-a_i)/(1+a_i) a_i^|k|; its variance is sum 2 a_i/(1-a_i)^2 ~= sigma_s^2 (R5)."""
    ss, N, n = 16.0, 3, 2001
    sig = oracle.sigmas(ss, N)
    a = np.exp(-np.sqrt(2) / sig)
    dx = np.ones((1, n)); dx[0, 0] = np.inf
    dy = np.full((1, n), np.inf)
    x = np.zeros((1, n)); x[0, n // 2] = 1
    z = oracle.dtf(x, dx, dy, ss, N)[0]
    half = 700
    h = np.array([1.0])
    for ai in a:
        h = np.convolve(h, dense.edge_free_kernel(ai, half))
    c = len(h) // 2
    h = h[c - 300:c + 301]
    np.testing.assert_allclose(z[n // 2 - 300:n // 2 + 301], h, rtol=1e-9, atol=1e-17)
    k = np.arange(-(n // 2), n // 2 + 1)
    var = float(np.sum(z * k ** 2))
    assert math.isclose(var, float(np.sum(2 * a / (1 - a) ** 2)), rel_tol=1e-9)
    assert abs(var - ss ** 2) / ss ** 2 < 0.01   # 255.50 vs 256 at sigma_s = 16
    # 2-D edge-free: impulse response is the outer product of the 1-D cascades
    m = 81
    g = const_guide(m, m)
    dx2, dy2 = oracle.distances(g, 3.0, 0.1)
    X = np.zeros((m, m)); X[m // 2, m // 2] = 1
    Z = oracle.dtf(X, dx2, dy2, 3.0, 2)
    X1 = np.zeros((1, m)); X1[0, m // 2] = 1
    z1 = oracle.dtf(X1, dx2[:1], np.full((1, m), np.inf), 3.0, 2)[0]
    np.testing.assert_allclose(Z, np.outer(z1, z1), rtol=1e-9, atol=1e-16)


def test_dtf_decoupling_exact():
    """Tiny sigma_r: a^d across a strong edge underflows to exactly 0 (BASELINE north star),
    so the left region's result is bit-identical whatever is on the right."""
    H, W = 10, 16
    g = np.zeros((H, W, 3), np.float32); g[:, W // 2:] = 1.0
    dx, dy = oracle.distances(g, 8.0, 1e-3)
    rng = np.random.default_rng(0)
    X1 = rng.normal(size=(H, W)); X2 = X1.copy(); X2[:, W // 2:] = rng.normal(size=(H, W // 2)) * 100
    Y1 = oracle.dtf(X1, dx, dy, 8.0, 3)
    Y2 = oracle.dtf(X2, dx, dy, 8.0, 3)
    np.testing.assert_array_equal(Y1[:, :W // 2], Y2[:, :W // 2])
    Yc = oracle.dtf(np.ascontiguousarray(X1[:, :W // 2]), dx[:, :W // 2], dy[:, :W // 2], 8.0, 3)
    np.testing.assert_allclose(Y1[:, :W // 2], Yc, rtol=1e-14, atol=1e-15)


# ------------------------------------------------------------------ O5
def brute_support(dx, dy, ss):
    H, W = dx.shape
    sx = np.zeros((H, W)); sy = np.zeros((H, W))
    for r in range(H):
        ct = np.concatenate([[0.0], np.cumsum(dx[r, 1:])])
        sx[r] = np.exp(-np.sqrt(2) * np.abs(ct[:, None] - ct[None, :]) / ss).sum(1)
    for c in range(W):
        ct = np.concatenate([[0.0], np.cumsum(dy[1:, c])])
        sy[:, c] = np.exp(-np.sqrt(2) * np.abs(ct[:, None] - ct[None, :]) / ss).sum(1)
    return sx * sy


def test_support_worked_and_closed_form():
    dx, dy = oracle.distances(const_guide(1, 2), SS, 0.1)
    np.testing.assert_allclose(oracle.support(dx, dy, SS)[0], GOLD["pair_1x2"]["S"], atol=1e-15)
    dx, dy = oracle.distances(const_guide(2, 2), SS, 0.1)
    np.testing.assert_allclose(oracle.support(dx, dy, SS), GOLD["dtf_2x2"]["S"], atol=1e-15)
    W, ss = 40, 6.0
    a = math.exp(-math.sqrt(2) / ss)
    dx, dy = oracle.distances(const_guide(1, W), ss, 0.1)
    n = np.arange(W)
    closed = (1 + a - a ** (n + 1) - a ** (W - n)) / (1 - a)
    np.testing.assert_allclose(oracle.support(dx, dy, ss)[0], closed, rtol=1e-13)


def test_support_brute_force_and_mode():
    g, _, _ = random_problem(9, 11, 3, 1, seed=4)
    dx, dy = oracle.distances(g, 4.0, 0.2)
    S = oracle.support(dx, dy, 4.0)
    np.testing.assert_allclose(S, brute_support(dx, dy, 4.0), rtol=1e-12)
    assert np.all(S >= 1.0)
    np.testing.assert_array_equal(oracle.support(dx, dy, 4.0, mode=1), 1.0)


# ------------------------------------------------------------------ O6
def test_solve_worked_1x2():
    e = GOLD["solve_1x2"]
    g = const_guide(1, 2)
    t = np.array([e["t"]], np.float32); c = np.array([e["c"]], np.float32)
    z1, diag = oracle.solve(g, t, c, SS, 0.1, 1, e["lambda"], 1, step=e["step"], diagnostics=True)
    np.testing.assert_allclose(z1[0], e["z_iter1"], atol=1e-15)
    assert math.isclose(diag[0, 0], max(abs(v) for v in e["g_iter1"]), rel_tol=1e-14)
    zc = oracle.solve(g, t, c, SS, 0.1, 1, e["lambda"], 3000, step=e["step"])
    np.testing.assert_allclose(zc[0], e["z_converged"], atol=1e-13)


def test_solve_zero_iterations_is_target():
    g, t, c = random_problem(5, 7, 3, 2, seed=1)
    np.testing.assert_array_equal(oracle.solve(g, t, c, 4.0, 0.2, 3, 0.99, 0), t.astype(np.float64))


def test_solve_constant_target_stays_constant():
    g, _, c = random_problem(12, 9, 3, 1, seed=2)
    t = np.full((12, 9), 3.25, np.float32)
    z = oracle.solve(g, t, c, 4.0, 0.2, 3, 0.99, 50)
    np.testing.assert_allclose(z, 3.25, rtol=1e-13)


def test_solve_c0_is_filter():
    """c = 0 reduces DTS to DT filtering; with step = 1/lambda one step gives DTF(t)."""
    g, t, _ = random_problem(8, 10, 3, 1, seed=3)
    c = np.zeros((8, 10), np.float32)
    lam = 1 / 0.99
    z = oracle.solve(g, t, c, 5.0, 0.2, 3, lam, 1, step=0.99)
    dx, dy = oracle.distances(g, 5.0, 0.2)
    K = dense.dtf_operator(dx, dy, oracle.sigmas(5.0, 3))
    np.testing.assert_allclose(z.ravel(), K @ t.astype(np.float64).ravel(), rtol=1e-12, atol=1e-13)


def test_solve_two_steps_dense():
    """Two iterations of Eq. (3) written with the dense operator and brute-force support:
    pins the sign of both terms, chat = c/S, the step and z-bar recomputation."""
    g, t, c = random_problem(5, 6, 3, 1, seed=6, conf_lo=0.2)
    ss, sr, lam, step = 3.0, 0.3, 0.9, 0.99
    dx, dy = oracle.distances(g, ss, sr)
    K = dense.dtf_operator(dx, dy, oracle.sigmas(ss, 3))
    chat = (c.astype(np.float64) / brute_support(dx, dy, ss)).ravel()
    tt = t.astype(np.float64).ravel()
    z = tt.copy()
    for _ in range(2):
        z = z - step * (lam * (z - K @ z) + chat * (z - tt))
    np.testing.assert_allclose(oracle.solve(g, t, c, ss, sr, 3, lam, 2, step=step).ravel(), z,
                               rtol=1e-12, atol=1e-13)


def test_solve_fixed_point_eq4():
    """Eq. (4): the limit solves (lambda (I - K) + diag(chat)) z = chat t."""
    g, t, c = random_problem(6, 8, 3, 1, seed=7, conf_lo=0.5)
    ss, sr, lam = 2.0, 0.3, 0.99
    dx, dy = oracle.distances(g, ss, sr)
    K = dense.dtf_operator(dx, dy, oracle.sigmas(ss, 3))
    chat = (c.astype(np.float64) / brute_support(dx, dy, ss)).ravel()
    M = lam * (np.eye(48) - K) + np.diag(chat)
    zstar = np.linalg.solve(M, chat * t.astype(np.float64).ravel())
    z, diag = oracle.solve(g, t, c, ss, sr, 3, lam, 4000, diagnostics=True)
    np.testing.assert_allclose(z.ravel(), zstar, rtol=1e-9, atol=1e-10)
    assert diag[-1, 0] <= 1e-3 * (lam + 1)   # S:249 residual bound


def test_solve_residual_norms_monotone():
    """Reading R13: ||g||_inf and ||g||_2 never increase (asserted); Eq. (2) objectives
    are only reported."""
    g, t, c = make_inputs("C0")
    _, diag = oracle.solve(g, t, c, 8.0, 0.2, 3, 1.0, 60, diagnostics=True)
    ginf, g2 = diag[:, 0], diag[:, 1]
    assert np.all(np.diff(ginf) <= 1e-12 * ginf[0])
    assert np.all(np.diff(g2) <= 1e-12 * g2[0])
    assert ginf[-1] < 0.5 * ginf[0]


def test_solve_channels_independent():
    g, t, c = random_problem(7, 9, 3, 3, seed=8)
    z = oracle.solve(g, t, c, 4.0, 0.2, 3, 0.99, 5)
    for ch in range(3):
        z1 = oracle.solve(g, np.ascontiguousarray(t[..., ch]), c, 4.0, 0.2, 3, 0.99, 5)
        np.testing.assert_array_equal(z[..., ch], z1)


def test_solve_decoupled_regions():
    H, W = 10, 14
    g = np.zeros((H, W, 3), np.float32); g[:, W // 2:] = 1
    rng = np.random.default_rng(9)
    t = rng.uniform(0, 1, (H, W)).astype(np.float32)
    t2 = t.copy(); t2[:, W // 2:] = 50
    c = rng.uniform(0.1, 1, (H, W)).astype(np.float32)
    z1 = oracle.solve(g, t, c, 8.0, 1e-3, 3, 0.99, 20)
    z2 = oracle.solve(g, t2, c, 8.0, 1e-3, 3, 0.99, 20)
    np.testing.assert_array_equal(z1[:, :W // 2], z2[:, :W // 2])


def test_solve_thread_count_invariant():
    g, t, c = make_inputs("C0")
    n0 = oracle.num_threads()
    z8 = oracle.solve(g, t, c, 8.0, 0.2, 3, 1.0, 5)
    oracle.set_threads(1)
    try:
        z1 = oracle.solve(g, t, c, 8.0, 0.2, 3, 1.0, 5)
    finally:
        oracle.set_threads(n0)
    np.testing.assert_array_equal(z8, z1)


# ---------------------------------------------------------------- O7: Eq. (7) confidence
def test_confidence_dense_operator():
    """V = K t^2 - (K t)^2 with K built from the closed-form L/U products (tests/dense.py),
    independent of the recurrences; c = exp(-V / 2 sigma_c^2)."""
    g, t, _ = random_problem(5, 4, 3, 1, seed=21)
    ss, sr, N, sc = 3.0, 0.4, 2, 0.7
    dx, dy = oracle.distances(g, ss, sr)
    K = dense.dtf_operator(dx, dy, oracle.sigmas(ss, N))
    tv = t.astype(np.float64).ravel()
    V = np.maximum(K @ (tv * tv) - (K @ tv) ** 2, 0.0).reshape(t.shape)
    c, v = oracle.confidence(g, t, ss, sr, N, sc)
    np.testing.assert_allclose(v, V, rtol=0, atol=1e-13)
    np.testing.assert_allclose(c, np.exp(-V / (2 * sc * sc)), rtol=0, atol=1e-13)
    assert np.all(v >= 0) and np.all((c > 0) & (c <= 1))


def test_confidence_edge_free_alternating_closed_form():
    """Constant guide, N = 1, a row alternating {0, 2}: at interior pixels the one-pass kernel
    h[k] = (1-a)/(1+a) a^|k| gives mean 1 + s r^(1/2) and mean of squares 2 + 2 s r^(1/2) with
    r = ((1-a)/(1+a))^4, so V = 1 - ((1-a)/(1+a))^4 (SPEC's 'V -> 1 for wide windows' is a -> 1).
    Choosing sigma_c^2 = V / 2 then gives c = e^-1 (Eq. 7 arithmetic)."""
    W = 801
    g = const_guide(1, W)
    t = np.tile(np.array([0.0, 2.0], np.float32), W // 2 + 1)[:W][None, :]
    ss = 9.0
    a = math.exp(-math.sqrt(2.0) / ss)  # N = 1: sigma_1 = sigma_s, d = 1
    Vexp = 1.0 - ((1 - a) / (1 + a)) ** 4
    sc = math.sqrt(Vexp / 2)
    c, v = oracle.confidence(g, t, ss, 0.3, 1, sc)
    mid = slice(300, 501)
    np.testing.assert_allclose(v[0, mid], Vexp, rtol=0, atol=1e-12)
    np.testing.assert_allclose(c[0, mid], math.exp(-1.0), rtol=0, atol=1e-12)


def test_confidence_constant_target_and_range():
    g, _, _ = random_problem(20, 30, 3, 1, seed=4)
    t = np.full((20, 30), 3.25, np.float32)
    c, v = oracle.confidence(g, t, 5.0, 0.2, 3, 0.5)
    assert np.max(v) <= 1e-12 and np.max(np.abs(c - 1.0)) <= 1e-12
    g, t, _ = random_problem(25, 33, 3, 1, seed=5)
    c, v = oracle.confidence(g, t, 5.0, 0.2, 3, 0.5)
    assert np.all(v >= 0) and np.all((c > 0) & (c <= 1))
    c2, _ = oracle.confidence(g, t, 5.0, 0.2, 3, 1.0)  # larger sigma_c: never less confident
    assert np.all(c2 >= c)


def test_confidence_decoupled_regions_exact():
    """A guide edge with tiny sigma_r underflows A to exactly 0: region A's variance is
    bit-identical whatever the target in region B."""
    H, W = 12, 20
    g = np.zeros((H, W, 3), np.float32)
    g[:, W // 2:] = 1.0
    rng = np.random.default_rng(3)
    t1 = rng.uniform(0, 1, (H, W)).astype(np.float32)
    t2 = t1.copy()
    t2[:, W // 2:] = rng.uniform(5, 9, (H, W - W // 2)).astype(np.float32)
    _, v1 = oracle.confidence(g, t1, 6.0, 1e-3, 3, 0.5)
    _, v2 = oracle.confidence(g, t2, 6.0, 1e-3, 3, 0.5)
    assert np.array_equal(v1[:, :W // 2], v2[:, :W // 2])


# ---------------------------------------------------------------- O8: Eq. (10) stereo
def test_stereo_reduces_to_solve_for_large_eps():
    """gamma = 0 and eps >> |z - t|: rho'(r) = r / sqrt(r^2 + eps^2) = r / eps (1 + O(r^2/eps^2)),
    so with confidence c * eps the stereo iteration is the O6 iteration with c."""
    g, t, c = random_problem(14, 17, 3, 1, seed=31)
    eps = 1e7
    ref = oracle.solve(g, t, c, 5.0, 0.2, 3, 0.99, 6)
    got = oracle.solve_stereo(g, g, t, (c.astype(np.float64) * eps).astype(np.float32), 5.0, 0.2, 3, 0.99, 6,
                              gamma=0.0, eps=eps)
    assert np.max(np.abs(got - ref)) <= 1e-6 * target_range(t)


def test_stereo_fixed_point_at_true_disparity():
    """Right image = left image shifted by an integer disparity d*: at z = d* every in-range
    residual I_L(x) - I_R(x - d*) is 0 and out-of-range samples have zero slope, so the
    gradient vanishes and z = t = d* is a fixed point."""
    rng = np.random.default_rng(8)
    H, W, C, dstar = 9, 40, 3, 5
    L = rng.uniform(0, 1, (H, W, C)).astype(np.float32)
    R = np.empty_like(L)
    R[:, :W - dstar] = L[:, dstar:]   # I_R(u) = I_L(u + d*)
    R[:, W - dstar:] = L[:, -1:]
    t = np.full((H, W), float(dstar), np.float32)
    c = np.full((H, W), 0.5, np.float32)
    # eps in the contractive regime (the paper's eps = 1e-3 makes rho' stiff at r = 0: curvature
    # chat / eps > 2 / step, so rounding-level deviations grow until |r| ~ eps; R23)
    got = oracle.solve_stereo(L, R, t, c, 6.0, 0.3, 3, 0.99, 5, gamma=0.3, eps=1.0)
    assert np.max(np.abs(got - dstar)) <= 1e-12


def test_stereo_photometric_gradient_finite_difference():
    """One step with lambda = 0 and c = 0 isolates the photometric gradient:
    z1 = z0 - step gamma dE_p/dz; compare with a central finite difference of the brute-force
    energy E_p(z) = 1/2 sum_k (I_L,k(x) - interp(I_R,k)(x - z))^2 at non-integer u."""
    rng = np.random.default_rng(12)
    H, W, C = 3, 30, 2
    L = rng.uniform(0, 1, (H, W, C)).astype(np.float32)
    R = rng.uniform(0, 1, (H, W, C)).astype(np.float32)
    t = (rng.uniform(2.1, 2.9, (H, W))).astype(np.float32)  # u = x - z never integer, inside for x >= 3
    c = np.zeros((H, W), np.float32)
    gamma, step = 0.7, 0.5
    z1 = oracle.solve_stereo(L, R, t, c, 4.0, 0.3, 1, 0.0, 1, gamma=gamma, step=step)
    gnum = (t.astype(np.float64) - z1) / (step * gamma)

    def energy(r, x, z):
        u = x - z
        out = 0.0
        for k in range(C):
            v = np.interp(u, np.arange(W), R[r, :, k].astype(np.float64))
            out += 0.5 * (float(L[r, x, k]) - v) ** 2
        return out

    h = 1e-6
    for r in range(H):
        for x in range(3, W):
            z = float(t[r, x])
            fd = (energy(r, x, z + h) - energy(r, x, z - h)) / (2 * h)
            assert abs(fd - gnum[r, x]) <= 1e-6, (r, x, fd, gnum[r, x])


def test_stereo_charbonnier_stationarity():
    """gamma = 0, many iterations: the iterate approaches the point where
    lambda (z - K z) + chat rho'(z - t) = 0 (Eq. 4 with the Charbonnier target); K is the dense
    operator of tests/dense.py and rho' the closed form."""
    g, t, c = random_problem(6, 5, 3, 1, seed=6)
    ss, sr, N, lam, eps = 3.0, 0.3, 2, 0.99, 0.5
    z = oracle.solve_stereo(g, g, t, c, ss, sr, N, lam, 3000, gamma=0.0, eps=eps)
    dx, dy = oracle.distances(g, ss, sr)
    K = dense.dtf_operator(dx, dy, oracle.sigmas(ss, N))
    S = oracle.support(dx, dy, ss)
    zv = z.ravel()
    r = zv - t.astype(np.float64).ravel()
    res = lam * (zv - K @ zv) + (c.astype(np.float64).ravel() / S.ravel()) * r / np.sqrt(r * r + eps * eps)
    assert np.max(np.abs(res)) <= 1e-6


# ---------------------------------------------------------------- O9: SR front end
def test_sr_factor_one_identity_and_constant():
    rng = np.random.default_rng(2)
    low = rng.uniform(0.5, 10, (7, 9)).astype(np.float32)
    t, c = oracle.sr_prepare(low, 1)
    assert np.array_equal(t, low.astype(np.float64)) and np.all(c == 1.0)
    t, _ = oracle.sr_prepare(np.full((5, 6), 3.5, np.float32), 4)
    np.testing.assert_allclose(t, 3.5, rtol=0, atol=1e-14)


def test_sr_reproduces_quadratics_in_the_interior():
    """The Catmull-Rom (Keys a = -0.5) kernel reproduces polynomials of degree <= 2; with the
    centre alignment, high-res pixel X samples the low-res polynomial at u = (X + 0.5)/f - 0.5."""
    h, w, f = 12, 14, 3
    jj, ii = np.mgrid[0:h, 0:w].astype(np.float64)
    poly = lambda v, u: 0.3 * u * u - 0.7 * u * v + 0.2 * v * v + 1.5 * u - 2.0 * v + 4.0  # noqa: E731
    low = poly(jj, ii).astype(np.float32)
    t, _ = oracle.sr_prepare(low, f)
    YY, XX = np.mgrid[0:h * f, 0:w * f].astype(np.float64)
    U, V = (XX + 0.5) / f - 0.5, (YY + 0.5) / f - 0.5
    ref = poly(V, U)
    inner = (U >= 1) & (U <= w - 2) & (V >= 1) & (V <= h - 2)  # all 4 taps inside
    np.testing.assert_allclose(t[inner], ref[inner], rtol=0, atol=2e-5)  # fp32 inputs


def test_sr_brute_force_2d_and_interpolation():
    """Against an independent 2-D sum over all low-res pixels with the closed-form kernel
    (indices clamped); odd f puts sample centres on pixels, where the value is the sample."""
    rng = np.random.default_rng(5)
    h, w, f = 5, 6, 3
    low = rng.uniform(0, 1, (h, w)).astype(np.float32)
    t, c = oracle.sr_prepare(low, f)

    def k(x):
        x = abs(x)
        return 1.5 * x ** 3 - 2.5 * x ** 2 + 1 if x < 1 else (-0.5 * x ** 3 + 2.5 * x ** 2 - 4 * x + 2 if x < 2 else 0.0)

    for Y in range(h * f):
        for X in range(w * f):
            u, v = (X + 0.5) / f - 0.5, (Y + 0.5) / f - 0.5
            acc = 0.0
            for j in range(int(np.floor(v)) - 1, int(np.floor(v)) + 3):
                for i in range(int(np.floor(u)) - 1, int(np.floor(u)) + 3):
                    acc += k(v - j) * k(u - i) * float(low[min(max(j, 0), h - 1), min(max(i, 0), w - 1)])
            assert abs(acc - t[Y, X]) <= 1e-12
    for j in range(h):
        for i in range(w):
            Y, X = j * f + (f - 1) // 2, i * f + (f - 1) // 2
            assert abs(t[Y, X] - float(low[j, i])) <= 1e-12 and c[Y, X] == 1.0


def test_sr_bump_confidence_closed_form():
    """f = 4: sigma_b = 1; centres at 4k + 1.5, so pixel (1, 1) is at distance sqrt(0.5) from the
    first centre -> c = exp(-0.25); c is periodic with period f away from the borders."""
    _, c = oracle.sr_prepare(np.zeros((6, 6), np.float32), 4)
    assert abs(c[1, 1] - np.exp(-0.25)) <= 1e-15
    np.testing.assert_allclose(c[4:20, 4:20], np.tile(c[4:8, 4:8], (4, 4)), rtol=0, atol=1e-15)
    assert np.all((c > 0) & (c <= 1))


# ---------------------------------------------------------------------------------------
# O10: box (normalised-convolution) variant (reading R25)

BOX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "box_spec_examples.json")))


def _line_guide(n):
    return np.zeros((1, n), np.float32)


def test_box_spec_worked_examples():
    for key in ("box_mean_constant_guide", "box_mean_radius_zero"):
        ex = BOX[key]
        x = np.array([ex["values"]], np.float64)
        got = oracle.box_dtf(x, _line_guide(x.shape[1]), 1.0, 0.1, 1, radius_scale=ex["radius"])
        np.testing.assert_allclose(got[0], ex["mean"], rtol=0, atol=1e-15)
    for key in ("box_count_constant_guide", "box_count_radius_zero"):
        ex = BOX[key]
        lox, hix, _, _, S = oracle.box_tables(_line_guide(ex["length"]), 1.0, 0.1, 1, radius_scale=ex["radius"])
        assert (lox[0, 0] + hix[0, 0] + 1).tolist() == ex["count"]
        assert S[0].tolist() == ex["count"]  # H = 1: the column count is 1


def test_box_increments_match_the_fp64_distance():
    # q = round(d * 2^16) with d the O1 increment (pinned above), evaluated in fp32
    rng = np.random.default_rng(5)
    g = rng.random((13, 17, 3), dtype=np.float32)
    for ss, sr in ((8.0, 0.1), (64.0, 0.2), (3.0, 2.0)):
        qx, qy = oracle.box_increments(g, ss, sr)
        dx, dy = oracle.distances(g, ss, sr)
        for q, d in ((qx[:, 1:], dx[:, 1:]), (qy[1:], dy[1:])):
            ref = d * 65536.0
            assert np.all(np.abs(q - ref) <= 0.5 + 4e-7 * ref)
        assert np.all(qx[:, 0] == 0) and np.all(qy[0] == 0)
        assert np.all(qx[:, 1:] >= 65536) and np.all(qy[1:] >= 65536)  # d >= 1


def _brute_windows(T, r):
    """Real-valued window of every sample from the DT coordinate T (fp64): the set
    {j : |T_j - T_i| <= r}, checked contiguous; returns (lo_off, hi_off, margin) where
    margin is the distance of the nearest |T_j - T_i| to r (to skip rounding ties)."""
    n = T.size
    lo, hi, margin = np.zeros(n, int), np.zeros(n, int), np.full(n, np.inf)
    for i in range(n):
        dist = np.abs(T - T[i])
        idx = np.nonzero(dist <= r)[0]
        assert idx.size == idx[-1] - idx[0] + 1  # contiguous (T is increasing)
        lo[i], hi[i] = i - idx[0], idx[-1] - i
        margin[i] = np.min(np.abs(dist - r))
    return lo, hi, margin


def test_box_windows_brute_force():
    rng = np.random.default_rng(7)
    g = rng.random((9, 31, 3), dtype=np.float32)
    ss, sr, N = 6.0, 0.6, 3
    dx, dy = oracle.distances(g, ss, sr)
    sig = oracle.sigmas(ss, N)
    lox, hix, loy, hiy, S = oracle.box_tables(g, ss, sr, N)
    checked = 0
    for i in range(N):
        r = np.sqrt(3.0) * sig[i]
        for row in range(9):
            T = np.concatenate([[0.0], np.cumsum(dx[row, 1:])])
            lo, hi, m = _brute_windows(T, r)
            ok = m > 1e-3
            assert np.array_equal(lox[i, row][ok], lo[ok]) and np.array_equal(hix[i, row][ok], hi[ok])
            checked += ok.sum()
        for col in range(31):
            T = np.concatenate([[0.0], np.cumsum(dy[1:, col])])
            lo, hi, m = _brute_windows(T, r)
            ok = m > 1e-3
            assert np.array_equal(loy[i, :, col][ok], lo[ok]) and np.array_equal(hiy[i, :, col][ok], hi[ok])
            checked += ok.sum()
    assert checked > 0.95 * N * 2 * 9 * 31
    # support: counts at r = sqrt(3) sigma_s, multiplied
    r = np.sqrt(3.0) * ss
    cx = np.array([[sum(_brute_windows(np.concatenate([[0.0], np.cumsum(dx[row, 1:])]), r)[k][c] for k in (0, 1)) + 1
                    for c in range(31)] for row in range(9)])
    cy = np.array([[sum(_brute_windows(np.concatenate([[0.0], np.cumsum(dy[1:, col])]), r)[k][row] for k in (0, 1)) + 1
                    for col in range(31)] for row in range(9)])
    np.testing.assert_array_equal(S, cx * cy)


def _box_dense_operator(g, ss, sr, N, radius_scale=np.sqrt(3.0)):
    """Dense matrix of the 2-D box mean built from real-valued brute-force windows:
    K = prod_i (M_y,i M_x,i) (rows then columns per pass)."""
    H, W = g.shape[:2]
    dx, dy = oracle.distances(g, ss, sr)
    sig = oracle.sigmas(ss, N)
    K = np.eye(H * W)
    margin = np.inf
    for i in range(N):
        r = radius_scale * sig[i]
        Mx, My = np.zeros((H * W, H * W)), np.zeros((H * W, H * W))
        for row in range(H):
            lo, hi, m = _brute_windows(np.concatenate([[0.0], np.cumsum(dx[row, 1:])]), r)
            margin = min(margin, m.min())
            for c in range(W):
                Mx[row * W + c, row * W + c - lo[c]: row * W + c + hi[c] + 1] = 1.0 / (lo[c] + hi[c] + 1)
        for col in range(W):
            lo, hi, m = _brute_windows(np.concatenate([[0.0], np.cumsum(dy[1:, col])]), r)
            margin = min(margin, m.min())
            for rr in range(H):
                for j in range(rr - lo[rr], rr + hi[rr] + 1):
                    My[rr * W + col, j * W + col] = 1.0 / (lo[rr] + hi[rr] + 1)
        K = My @ Mx @ K
    return K, margin


@pytest.mark.parametrize("H,W,N", [(7, 9, 1), (6, 11, 3)])
def test_box_dtf_equals_dense_operator(H, W, N):
    rng = np.random.default_rng(H * 100 + W)
    g = rng.random((H, W, 2), dtype=np.float32)
    K, margin = _box_dense_operator(g, 4.0, 0.8, N)
    assert margin > 1e-4  # no rounding tie on this instance
    x = rng.standard_normal((2, H, W))
    got = oracle.box_dtf(x, g, 4.0, 0.8, N)
    for ch in range(2):
        np.testing.assert_allclose(got[ch].ravel(), K @ x[ch].ravel(), rtol=0, atol=1e-13)
    np.testing.assert_allclose(K.sum(axis=1), 1.0, atol=1e-13)  # normalised: row-stochastic


def test_box_two_region_spec_example():
    ex = BOX["two_region"]
    H, W, s = ex["H"], ex["W"], ex["split"]
    g = np.zeros((H, W, 3), np.float32)
    g[:, s:] = 1.0
    x = np.where(np.arange(W)[None, :] < s, ex["left"], ex["right"]) * np.ones((H, 1))
    got = oracle.box_dtf(x, g, ex["sigma_s"], ex["sigma_r"], 1)
    np.testing.assert_array_equal(got, x)  # no window crosses the edge: exact
    _, _, _, _, S = oracle.box_tables(g, ex["sigma_s"], ex["sigma_r"], 1)
    h = ex["half_width"]

    def counts(n):
        i = np.arange(n)
        return np.minimum(i, h) + np.minimum(n - 1 - i, h) + 1

    cx = np.concatenate([counts(s), counts(W - s)])
    np.testing.assert_array_equal(S, counts(H)[:, None] * cx[None, :])


def test_box_constant_values_any_guide():
    rng = np.random.default_rng(11)
    g = rng.random((12, 15, 3), dtype=np.float32)
    got = oracle.box_dtf(np.full((12, 15), 0.375), g, 5.0, 0.3, 3)
    np.testing.assert_allclose(got, 0.375, rtol=0, atol=1e-15)


def test_box_solve_equals_dense_iteration():
    rng = np.random.default_rng(13)
    H, W, N = 6, 8, 2
    g = rng.random((H, W, 3), dtype=np.float32)
    t = rng.random((H, W), dtype=np.float32)
    c = rng.uniform(0.1, 1.0, (H, W)).astype(np.float32)
    lam, step, iters = 0.99, 0.99, 4
    K, margin = _box_dense_operator(g, 3.0, 0.5, N)
    assert margin > 1e-4
    _, _, _, _, S = oracle.box_tables(g, 3.0, 0.5, N)
    chat = c.astype(np.float64).ravel() / S.ravel()
    z = t.astype(np.float64).ravel()
    T = z.copy()
    for _ in range(iters):
        z = z - step * (lam * (z - K @ z) + chat * (z - T))  # Eq. (3)
    got = oracle.solve_box(g, t, c, 3.0, 0.5, N, lam, iters, step=step)
    np.testing.assert_allclose(got.ravel(), z, rtol=0, atol=1e-12)
    # support mode 1: S = 1
    z = T.copy()
    for _ in range(iters):
        z = z - step * (lam * (z - K @ z) + c.astype(np.float64).ravel() * (z - T))
    got = oracle.solve_box(g, t, c, 3.0, 0.5, N, lam, iters, step=step, support_mode=1)
    np.testing.assert_allclose(got.ravel(), z, rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------------------
# Round 2: pins for the parts the round-1 review found unpinned (VERDICT r1 "What's weak" 1)

def _dense_diag(K, chat, t, lam, step, iters):
    """O6 diagnostics written out with the dense operator (reading R13):
    per k, at Z^k: [max |g|, ||g||_2, lam/2 ||Z - zbar||^2 + 1/2 sum chat (Z - T)^2,
    lam/2 Z.(Z - zbar) + 1/2 sum chat (Z - T)^2], g = lam (Z - zbar) + chat (Z - T)."""
    z = t.copy()
    rows, signs = [], []
    for _ in range(iters):
        zb = K @ z
        gk = lam * (z - zb) + chat * (z - t)
        data = 0.5 * float(np.sum(chat * (z - t) ** 2))
        rows.append([float(np.max(np.abs(gk))), float(np.sqrt(np.sum(gk * gk))),
                     0.5 * lam * float(np.sum((z - zb) ** 2)) + data,
                     0.5 * lam * float(z @ (z - zb)) + data])
        signs.append(float(np.max(gk)) < float(np.max(np.abs(gk))))  # the most negative g dominates
        z = z - step * gk
    return np.array(rows), signs


def test_solve_diagnostics_equal_dense_values():
    """The four O6 diagnostics against their definitions evaluated with the dense operator K
    (tests/dense.py) and the brute-force support, over three iterations (k = 0 has Z = T, so the
    data terms of F_hat and E_q are pinned from k = 1 on).  The target is run with both signs, so
    on at least one iterate the most negative gradient outweighs the most positive one: a
    ||g||_inf taken without |.| fails there; ||g||_2 without the square or the root fails."""
    g, t, c = random_problem(5, 6, 3, 1, seed=6, conf_lo=0.2)
    ss, sr, lam, step, iters = 3.0, 0.3, 0.9, 0.99, 3
    dx, dy = oracle.distances(g, ss, sr)
    K = dense.dtf_operator(dx, dy, oracle.sigmas(ss, 3))
    chat = (c.astype(np.float64) / brute_support(dx, dy, ss)).ravel()
    negative_dominant = 0
    for sign in (1.0, -1.0):
        ts = (sign * t).astype(np.float32)
        want, signs = _dense_diag(K, chat, ts.astype(np.float64).ravel(), lam, step, iters)
        negative_dominant += sum(signs)
        _, diag = oracle.solve(g, ts, c, ss, sr, 3, lam, iters, step=step, diagnostics=True)
        np.testing.assert_allclose(diag, want, rtol=1e-11, atol=1e-15)
        assert np.all(want[1:, 2] != want[1:, 3])  # F_hat and E_q differ once Z != T
    assert negative_dominant >= 1


def test_solve_diagnostics_two_channels_and_support_off():
    """Diagnostics sum over every channel (reading R14) and follow support_mode 1 (chat = c)."""
    g, t, c = random_problem(4, 5, 3, 2, seed=12, conf_lo=0.3)
    ss, sr, lam, step, iters = 2.5, 0.4, 0.99, 0.99, 2
    dx, dy = oracle.distances(g, ss, sr)
    K = dense.dtf_operator(dx, dy, oracle.sigmas(ss, 3))
    KK = np.kron(np.eye(2), K)
    for mode, S in ((0, brute_support(dx, dy, ss)), (1, np.ones(dx.shape))):
        chat = np.tile((c.astype(np.float64) / S).ravel(), 2)
        tt = np.concatenate([t[..., 0].astype(np.float64).ravel(), t[..., 1].astype(np.float64).ravel()])
        want, _ = _dense_diag(KK, chat, tt, lam, step, iters)
        _, diag = oracle.solve(g, t, c, ss, sr, 3, lam, iters, step=step, support_mode=mode, diagnostics=True)
        np.testing.assert_allclose(diag, want, rtol=1e-11, atol=1e-15)


def test_confidence_clamp_of_rounding_residues():
    """Reading R22: V = DTF(z^2) - DTF(z)^2 is clamped at 0.  A constant target that is not a
    dyadic fraction leaves rounding residues of either sign in the two filtered planes; the
    clamp must turn every negative one into exactly 0, so with a tiny sigma_c the confidence
    never exceeds 1 (without the clamp exp(-V / 2 sigma_c^2) > 1 wherever V < 0)."""
    g, _, _ = random_problem(16, 21, 3, 1, seed=11)
    t = np.full((16, 21), 0.1, np.float32)
    z = float(t[0, 0])
    K = dense.dtf_operator(*oracle.distances(g, 5.0, 0.2), oracle.sigmas(5.0, 3))
    zz = np.full(t.size, z)
    resid = (K @ (zz * zz)) - (K @ zz) ** 2  # rounding residues of the dense form
    assert np.max(np.abs(resid)) < 1e-15
    c, v = oracle.confidence(g, t, 5.0, 0.2, 3, 1e-9)
    assert np.all(v >= 0.0) and np.all(v < 1e-15)
    assert np.all(c <= 1.0)
    assert np.sum(v == 0.0) >= 0.2 * v.size  # the clamped residues (about half of them)


def test_box_radius_is_floored_on_a_tie():
    """Reading R25: R = floor(r 2^16).  Constant guide: every increment is q = 2^16 exactly, so
    T_j - T_i = 2^16 |j - i|.  With r = 2 - 2^-17 (N = 1, radius_scale 1: r = sigma_s), r 2^16 =
    131071.5: floor keeps +-1 pixel (131072 > 131071), ceil or round would keep +-2."""
    ss = 2.0 - 2.0 ** -17
    assert oracle.box_radius(1.0, ss) == 131071
    H, W = 6, 9
    lox, hix, loy, hiy, S = oracle.box_tables(const_guide(H, W), ss, 0.2, 1, radius_scale=1.0)
    i = np.arange(W)
    np.testing.assert_array_equal(lox[0], np.broadcast_to(np.minimum(i, 1), (H, W)))
    np.testing.assert_array_equal(hix[0], np.broadcast_to(np.minimum(W - 1 - i, 1), (H, W)))
    j = np.arange(H)[:, None]
    np.testing.assert_array_equal(loy[0], np.broadcast_to(np.minimum(j, 1), (H, W)))
    np.testing.assert_array_equal(hiy[0], np.broadcast_to(np.minimum(H - 1 - j, 1), (H, W)))
    cx = np.minimum(i, 1) + np.minimum(W - 1 - i, 1) + 1
    cy = np.minimum(j, 1) + np.minimum(H - 1 - j, 1) + 1
    np.testing.assert_array_equal(S, cy * cx[None, :])
