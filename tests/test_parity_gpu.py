"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by
element on the same seeded fp32 inputs.  Tolerance (BASELINE.json north star):
max |gpu - oracle| <= 1e-4 * (max(t) - min(t)) after the full solve (reading R15)."""
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


def gpu_solve(g, t, c, ss, sr, N, lam, iters, host=False, **opts):
    if host:
        out = np.empty_like(t)
        with dts.Solver(g, ss, sr, N) as s:
            s.solve(t, c, lam, iters, out=out, **opts)
        return out.astype(np.float64)
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    with dts.Solver(gd, ss, sr, N) as s:
        s.solve(td, cd, lam, iters, out=out, **opts)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def check(g, t, c, ss, sr, N, lam, iters, **kw):
    ref = oracle.solve(g, t, c, ss, sr, N, lam, iters)
    got = gpu_solve(g, t, c, ss, sr, N, lam, iters, **kw)
    rng = max(target_range(t), 1e-30)
    err = float(np.max(np.abs(got - ref))) if got.size else 0.0
    assert np.all(np.isfinite(got))
    assert err <= TOL * rng, f"max err {err:.3e} > {TOL * rng:.3e}"
    return err / rng


# ---------------------------------------------------------------- K1 / K5 pieces
@pytest.mark.parametrize("H,W,C", [(1, 1, 1), (7, 5, 3), (48, 64, 3), (33, 70, 16), (20, 1000, 2)])
def test_guide_derivative_parity(H, W, C):
    g, _, _ = random_problem(H, W, C, 1, seed=H + W)
    dx_r, dy_r = oracle.distances(g, 8.0, 0.2)
    with dts.Solver(torch.from_numpy(g).cuda(), 8.0, 0.2, 3) as s:
        dx, dy = s.read(dts.DTS_BUF_DX), s.read(dts.DTS_BUF_DY)
    for got, ref in ((dx, dx_r), (dy, dy_r)):
        inf = np.isinf(ref)
        assert np.array_equal(np.isinf(got), inf)
        np.testing.assert_allclose(got[~inf], ref[~inf], rtol=2e-6)


@pytest.mark.parametrize("H,W", [(1, 1), (1, 9), (9, 1), (48, 64), (300, 41), (1500, 70), (13, 3000)])
def test_support_parity(H, W):
    g, _, _ = random_problem(H, W, 3, 1, seed=H * W)
    dx_r, dy_r = oracle.distances(g, 6.0, 0.3)
    S_r = oracle.support(dx_r, dy_r, 6.0)
    with dts.Solver(torch.from_numpy(g).cuda(), 6.0, 0.3, 3) as s:
        S = s.read(dts.DTS_BUF_SUPPORT)
    np.testing.assert_allclose(S, S_r, rtol=2e-5)


# ---------------------------------------------------------------- full solves
def test_c0_parity():
    cfg = CONFIGS["C0"]
    g, t, c = make_inputs("C0")
    rel = check(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
    assert rel < 1e-5


SHAPES = [(1, 1), (1, 7), (7, 1), (2, 2), (31, 33), (33, 31), (32, 32), (61, 97), (5, 130), (130, 5),
          (257, 3), (3, 1031), (17, 4099), (3, 10000), (2, 18000), (1000, 37), (2600, 35), (5000, 40),
          (12000, 33)]


@pytest.mark.parametrize("H,W", SHAPES)
def test_edge_shapes_parity(H, W):
    g, t, c = random_problem(H, W, 3, 1, seed=7 * H + W)
    iters = 3 if H * W > 100000 else 6
    check(g, t, c, 5.0, 0.2, 3, 0.99, iters)


@pytest.mark.parametrize("Ct", [2, 3, 4])
@pytest.mark.parametrize("H,W", [(9, 13), (70, 300), (1200, 64)])
def test_multichannel_parity(Ct, H, W):
    g, t, c = random_problem(H, W, 3, Ct, seed=Ct * 1000 + H)
    check(g, t, c, 6.0, 0.15, 3, 0.99, 4)


@pytest.mark.parametrize("N", [1, 2, 5])
def test_pass_count_parity(N):
    g, t, c = random_problem(40, 50, 3, 1, seed=N)
    check(g, t, c, 7.0, 0.25, N, 0.99, 5)


def test_support_mode_unweighted():
    g, t, c = random_problem(30, 40, 3, 1, seed=11)
    ref = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.99, 5, support_mode=1)
    got = gpu_solve(g, t, c, 6.0, 0.2, 3, 0.99, 5, support_mode=1)
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)


def test_step_option():
    g, t, c = random_problem(20, 30, 3, 1, seed=12)
    ref = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.5, 4, step=0.7)
    got = gpu_solve(g, t, c, 6.0, 0.2, 3, 0.5, 4, step=0.7)
    assert np.max(np.abs(got - ref)) <= TOL * target_range(t)


def test_zero_iterations_exact():
    g, t, c = random_problem(11, 13, 3, 3, seed=2)
    got = gpu_solve(g, t, c, 5.0, 0.2, 3, 0.99, 0)
    assert np.array_equal(got, t.astype(np.float64))


def test_constant_target_stays_constant():
    g, _, c = random_problem(200, 300, 3, 1, seed=3)
    t = np.full((200, 300), 7.5, np.float32)
    got = gpu_solve(g, t, c, 8.0, 0.2, 3, 0.99, 20)
    assert np.max(np.abs(got - 7.5)) <= 1e-6 * 7.5


def test_c0_reduces_to_filter():
    """c = 0, step = 1/lambda, one iteration -> the domain-transform filter output."""
    g, t, _ = random_problem(60, 80, 3, 1, seed=4)
    c = np.zeros((60, 80), np.float32)
    dx, dy = oracle.distances(g, 6.0, 0.2)
    ref = oracle.dtf(t.astype(np.float64), dx, dy, 6.0, 3)
    got = gpu_solve(g, t, c, 6.0, 0.2, 3, 1 / 0.99, 1)
    assert np.max(np.abs(got - ref)) <= 1e-6 * target_range(t)


def test_decoupled_regions_bit_identical():
    H, W = 64, 96
    g = np.zeros((H, W, 3), np.float32)
    g[:, W // 2:] = 1
    rng = np.random.default_rng(5)
    t = rng.uniform(0, 1, (H, W)).astype(np.float32)
    t2 = t.copy()
    t2[:, W // 2:] = 100
    c = rng.uniform(0.1, 1, (H, W)).astype(np.float32)
    a = gpu_solve(g, t, c, 8.0, 1e-3, 3, 0.99, 10)
    b = gpu_solve(g, t2, c, 8.0, 1e-3, 3, 0.99, 10)
    assert np.array_equal(a[:, :W // 2], b[:, :W // 2])


def test_deterministic_and_host_pointer_path():
    g, t, c = random_problem(100, 150, 3, 1, seed=6)
    a = gpu_solve(g, t, c, 8.0, 0.2, 3, 0.99, 7)
    b = gpu_solve(g, t, c, 8.0, 0.2, 3, 0.99, 7)
    h = gpu_solve(g, t, c, 8.0, 0.2, 3, 0.99, 7, host=True)
    assert np.array_equal(a, b)
    assert np.array_equal(a, h)


def test_multichannel_equals_single_channel():
    g, t, c = random_problem(50, 70, 3, 3, seed=8)
    z = gpu_solve(g, t, c, 6.0, 0.2, 3, 0.99, 5)
    for ch in range(3):
        z1 = gpu_solve(g, np.ascontiguousarray(t[..., ch]), c, 6.0, 0.2, 3, 0.99, 5)
        np.testing.assert_allclose(z[..., ch], z1, rtol=0, atol=1e-6 * target_range(t))


def test_residual_decreases_on_gpu():
    """Reading R13 on the CUDA path: ||g||_inf of Eq. (3) evaluated by the oracle's
    DTF at the GPU iterates is non-increasing (to fp32 noise)."""
    g, t, c = make_inputs("C0")
    cfg = CONFIGS["C0"]
    dx, dy = oracle.distances(g, cfg.sigma_s, cfg.sigma_r)
    chat = c / oracle.support(dx, dy, cfg.sigma_s)
    prev = None
    for k in [1, 2, 4, 8, 16]:
        z = gpu_solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, k)
        zb = oracle.dtf(z, dx, dy, cfg.sigma_s, cfg.N)
        gn = float(np.max(np.abs(cfg.lam * (z - zb) + chat * (z - t))))
        if prev is not None:
            assert gn <= prev * (1 + 1e-4)
        prev = gn


def test_invalid_arguments():
    g, t, c = random_problem(8, 9, 3, 1, seed=9)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    with dts.Solver(gd, 5.0, 0.2, 3) as s:
        out = torch.empty_like(td)
        for lam, it in [(1.1, 3), (-0.1, 3), (float("nan"), 3), (0.99, -1)]:
            with pytest.raises(dts.DTSError) as ei:
                dts.dts_solve(s.ctx, td, cd, lam, it, out)
            assert ei.value.status == 1
        with pytest.raises(dts.DTSError) as ei:
            dts.dts_solve(s.ctx, td, cd, 0.99, 3, td)  # out aliases target
        assert ei.value.status == 1
        bad = cd.clone()
        bad[0, 0] = 2.0
        with pytest.raises(dts.DTSError) as ei:
            dts.dts_solve_ex(s.ctx, td, bad, 0.99, 3, out, check_inputs=True)
        assert ei.value.status == 4
        bad[0, 0] = float("nan")
        with pytest.raises(dts.DTSError) as ei:
            dts.dts_solve_ex(s.ctx, td, bad, 0.99, 3, out, check_inputs=True)
        assert ei.value.status == 3


def test_profile_counters():
    g, t, c = random_problem(64, 128, 3, 1, seed=10)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    with dts.Solver(gd, 5.0, 0.2, 3) as s:
        n0 = dts.dts_launch_count(s.ctx)
        assert n0 == 5  # deriv + bottom-link row fill + support row + support col + column coefficient A1
        dts.dts_profile_enable(s.ctx, True)
        s.solve(td, cd, 0.99, 4)
        st = dts.dts_profile_read(s.ctx)
        n1 = dts.dts_launch_count(s.ctx)
    # 3 row passes + 3 column passes per iteration; the Eq. (3) step is fused into the
    # next iteration's first row pass (row_update) + one closing update kernel, or fused
    # into the last column pass (col_update), or a separate streaming kernel (update)
    assert st["row_pass"]["launches"] + st["row_update"]["launches"] == 12
    assert st["col_pass"]["launches"] + st["col_update"]["launches"] == 12
    assert st["update"]["launches"] + st["col_update"]["launches"] + st["row_update"]["launches"] == 4
    assert st["prologue"]["launches"] == 1
    assert n1 == n0 + 1 + 4 * 6 + st["update"]["launches"]
    assert st["row_pass"]["total_ms"] > 0


# ---------------------------------------------------------------- BASELINE.json configs
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_parity(name):
    cfg = CONFIGS[name]
    g, t, c = make_inputs(name)
    check(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)


def test_c3_one_image_parity():
    cfg = CONFIGS["C3"]
    g, t, c = make_inputs("C3", image=5)
    check(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)


@pytest.mark.slow
def test_c4_full_parity():
    """The bench workload at full size (10000 x 10000, 16-band guide, 20 iterations),
    in the launch configuration bench.py times, against the full fp64 oracle."""
    cfg = CONFIGS["C4"]
    g, t, c = make_inputs("C4")
    check(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)


@pytest.mark.parametrize("H,W,Ct", [(48, 64, 1), (33, 31, 1), (700, 130, 1), (300, 90, 3), (61, 97, 2)])
def test_fallback_column_kernel_parity(H, W, Ct):
    """The decoupled band-tuple column kernel (used when a column does not fit a cluster)
    forced for ordinary shapes (option col_kernel = 1), Eq. (3) in its write-out."""
    g, t, c = random_problem(H, W, 3, Ct, seed=H + 3 * W)
    with dts.options(col_kernel=1):
        check(g, t, c, 6.0, 0.2, 3, 0.99, 5)


@pytest.mark.parametrize("H,W,Ct", [(48, 64, 1), (700, 130, 1), (300, 90, 3), (2600, 35, 1)])
def test_separate_update_kernel_parity(H, W, Ct):
    """The cluster column kernel with the Eq. (3) step as its own streaming kernel every
    iteration (option row_update = 0) instead of inside the next row pass."""
    g, t, c = random_problem(H, W, 3, Ct, seed=H + 5 * W)
    with dts.options(row_update=0):
        check(g, t, c, 6.0, 0.2, 3, 0.99, 5)


def test_repeated_solves_replay_a_graph():
    """A repeated identical solve is captured once and replayed as a CUDA graph: results are
    bit-identical to the eager launches, and the launch counter advances the same way."""
    g, t, c = random_problem(200, 300, 3, 1, seed=21)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    outs = []
    with dts.Solver(gd, 6.0, 0.2, 3) as s:
        counts = []
        for _ in range(4):  # eager, capture + launch, replay, replay
            o = torch.empty_like(td)
            n0 = dts.dts_launch_count(s.ctx)
            s.solve(td, cd, 0.99, 5, out=o)
            counts.append(dts.dts_launch_count(s.ctx) - n0)
            outs.append(o)
    torch.cuda.synchronize()
    ref = outs[0].cpu().numpy()
    for o in outs[1:]:
        assert np.array_equal(o.cpu().numpy(), ref)
    # prologue + 5 iterations x (3 row + 3 column passes) + the closing update; iterations
    # 2-5 take the previous Eq. (3) step in their first row pass
    assert len(set(counts)) == 1 and counts[0] == 1 + 5 * 6 + 1


def test_concurrent_contexts_on_two_threads():
    """Two host threads, each with its own context and stream, solving repeatedly (eager,
    graph capture, replay) at the same time: every result equals the single-threaded one.
    Covers the process-wide state (function attributes, profiler, plan caches)."""
    import threading
    probs = [random_problem(300, 410, 3, 1, seed=31), random_problem(520, 260, 3, 2, seed=32)]
    refs = [gpu_solve(g, t, c, 7.0, 0.2, 3, 0.99, 6) for g, t, c in probs]
    outs, errs = [[], []], []

    def worker(k):
        try:
            torch.cuda.set_device(0)
            g, t, c = probs[k]
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
                with dts.Solver(gd, 7.0, 0.2, 3, stream=stream.cuda_stream) as s:
                    for _ in range(4):
                        o = torch.empty_like(td)
                        s.solve(td, cd, 0.99, 6, out=o, stream=stream.cuda_stream)
                        stream.synchronize()
                        outs[k].append(o.cpu().numpy().astype(np.float64))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for th in ths:
        th.start()
    for th in ths:
        th.join(timeout=120)
    assert not errs, errs[0]
    for k in range(2):
        assert len(outs[k]) == 4
        for o in outs[k]:
            assert np.array_equal(o, refs[k])


def _random_cases(n, seed):
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        H = int(rng.choice([1, 2, 31, 33, 64, 65, 127, 200, 333, 641, 700]))
        W = int(rng.choice([1, 3, 32, 33, 63, 96, 129, 257, 500, 700]))
        cases.append((H, W, int(rng.integers(1, 4)), float(rng.uniform(2.0, 40.0)), float(rng.uniform(0.05, 1.0)),
                      int(rng.integers(1, 5)), int(rng.integers(1, 9)), int(rng.integers(0, 1 << 30))))
    return cases


@pytest.mark.parametrize("H,W,Ct,ss,sr,N,iters,seed", _random_cases(24, 2026))
def test_random_shapes_parity(H, W, Ct, ss, sr, N, iters, seed):
    """Seeded random sweep of shapes (ragged tails, single rows / columns), target channels,
    sigmas, pass counts and iteration counts through the default path, against the oracle."""
    g, t, c = random_problem(H, W, 3, Ct, seed=seed % 100000)
    check(g, t, c, ss, sr, N, 0.99, iters)


@pytest.mark.parametrize("H,W,Ct", [(25000, 33, 1), (16000, 40, 1), (6400, 20, 3)])
def test_tall_images_parity(H, W, Ct):
    """Columns longer than a cluster holds (10240 rows at C_t = 1): the decoupled column
    kernel, near the per-context row limit stated in include/dts.h."""
    g, t, c = random_problem(H, W, 3, Ct, seed=H)
    check(g, t, c, 8.0, 0.2, 3, 0.99, 3)


def test_too_tall_image_is_a_shape_error():
    g, t, c = random_problem(60000, 8, 3, 1, seed=1)
    with pytest.raises(dts.DTSError) as ei:
        with dts.Solver(torch.from_numpy(g).cuda(), 8.0, 0.2, 3):
            pass
    assert "DTS_E_SHAPE" in str(ei.value)


@pytest.mark.parametrize("H,W,Ct", [(1500, 330, 1), (9000, 200, 1), (2160, 390, 3), (700, 70, 2), (1300, 4100, 1)])
def test_repeat_solves_bit_identical(H, W, Ct):
    """Race stress for the cluster column kernels (per-warp TMA issue, no end-of-tile
    barrier, link coefficient behind the next segment's mbarrier): their arithmetic order is
    fixed, so a shared-memory hazard shows up as a run-to-run difference.  Shapes: several
    CTAs per cluster with a ragged last segment, 15 CTAs per cluster, C_t = 3 and 2 on the
    16-row-segment variant.  Ten eager solves each, outputs compared bit for bit."""
    g, t, c = random_problem(H, W, 3, Ct, seed=H + W + Ct)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    outs = []
    with dts.options(graphs=0), dts.Solver(gd, 8.0, 0.1, 3) as s:
        for _ in range(10):
            o = torch.empty_like(td)
            s.solve(td, cd, 0.99, 3, out=o)
            outs.append(o)
    torch.cuda.synchronize()
    ref = outs[0].cpu().numpy()
    assert np.isfinite(ref).all()
    for o in outs[1:]:
        assert np.array_equal(o.cpu().numpy(), ref)


def test_forty_row_segments_parity():
    """C_t = 1 images with several cluster tile rounds per column pass take the 16-warp x
    40-row-segment instantiation of the cluster kernel (plan_col); a wide image reaches it.
    Parity with the oracle, and again with the 32-row kernel forced (option col_rows = 32)."""
    g, t, c = random_problem(1300, 4100, 3, 1, seed=77)
    check(g, t, c, 6.0, 0.15, 3, 0.99, 3)
    with dts.options(col_rows=32):
        check(g, t, c, 6.0, 0.15, 3, 0.99, 3)


def test_guide_beyond_2_31_elements():
    """SURVEY 7 / 8(c) 64-bit indexing: a guide of more than 2^31 elements (10000 x 13500 x 16 =
    2.16e9 floats, 8.6 GB); d_x and d_y of the last rows (element offsets past 2^31) against O1
    evaluated on those rows (d_x of a row depends on that row only, d_y on it and the row above)."""
    H, W, C = 10000, 13500, 16
    assert H * W * C > 2 ** 31
    gen = torch.Generator(device="cuda").manual_seed(5)
    g = torch.rand((H, W, C), device="cuda", generator=gen, dtype=torch.float32)
    rows = [0, 1, H // 2, H - 2, H - 1]
    with dts.Solver(g, 8.0, 0.2, 3) as s:
        dx, dy = s.read(dts.DTS_BUF_DX), s.read(dts.DTS_BUF_DY)
    for r in rows:
        lo = max(r - 1, 0)
        sl = g[lo:r + 1].cpu().numpy()
        dx_r, dy_r = oracle.distances(sl, 8.0, 0.2)
        for got, ref in ((dx[r], dx_r[r - lo]), (dy[r], dy_r[r - lo])):
            inf = np.isinf(ref)  # the +inf sentinels: column 0 of d_x, row 0 of d_y
            assert np.array_equal(np.isinf(got), inf)
            np.testing.assert_allclose(got[~inf], ref[~inf], rtol=2e-6)
    del g
    torch.cuda.empty_cache()


def _seam_fix_launches(g, t, c, ss, sr, N, lam, iters):
    """Solve; also returns the number of row strips the context planned (0: none)."""
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    with dts.Solver(gd, ss, sr, N) as s:
        s.solve(td, cd, lam, iters, out=out)
        nst = dts.debug_strips(s.ctx)["strips"]
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), nst


@pytest.mark.parametrize("H,W,ss", [(3000, 4000, 6.0), (2900, 3000, 9.0), (1300, 4100, 4.0)])
def test_row_strip_column_passes_parity(H, W, ss):
    """Tall, wide single-context images run their C_t = 1 column passes over row strips with
    small clusters (all 148 SMs) and a seam fix-up (plan_strips, reading R26 on one GPU): parity
    with the oracle, and with the unstripped path (option col_strips = 0) to fp32 rounding."""
    g, t, c = random_problem(H, W, 3, 1, seed=H + W)
    ref = oracle.solve(g, t, c, ss, 0.2, 3, 0.99, 3)
    got, nfix = _seam_fix_launches(g, t, c, ss, 0.2, 3, 0.99, 3)
    rng = target_range(t)
    assert np.max(np.abs(got - ref)) <= TOL * rng
    with dts.options(col_strips=0):
        plain, nfix0 = _seam_fix_launches(g, t, c, ss, 0.2, 3, 0.99, 3)
    assert nfix0 == 0
    assert np.max(np.abs(got - plain)) <= 1e-5 * rng
    if H == 3000:
        assert nfix > 1  # this shape takes row strips


@pytest.mark.parametrize("opts", [{"row_update": 0}, {"graphs": 0}])
def test_row_strips_with_separate_update_and_residual(opts):
    """Row strips with the seam carries taken by the update kernel (row_update = 0) and by the
    row update + closing update (default), with the residual output requested."""
    g, t, c = random_problem(3000, 4000, 3, 1, seed=77)
    ref, diag = oracle.solve(g, t, c, 6.0, 0.2, 3, 0.99, 4, diagnostics=True)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    r = torch.zeros(4, device="cuda")
    with dts.options(**opts), dts.Solver(gd, 6.0, 0.2, 3) as s:
        s.solve(td, cd, 0.99, 4, out=out, resid_inf_out=r)
        s.solve(td, cd, 0.99, 4, out=out)  # plain (row update) on the same context
    torch.cuda.synchronize()
    rng = target_range(t)
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= TOL * rng
    np.testing.assert_allclose(r.cpu().numpy(), diag[:, 0], rtol=0, atol=TOL * rng)


@pytest.mark.parametrize("H,W,Ct,strips", [(12000, 64, 1, True), (6000, 48, 3, True), (8000, 40, 2, True),
                                            (5400, 36, 4, False), (300, 200, 4, False)])
def test_columns_taller_than_a_cluster_run_over_strips(H, W, Ct, strips):
    """Columns no cluster holds (C_t = 1 above 10240 rows, C_t = 2 above 7168, C_t = 3 above 5632)
    run over row strips chosen at the first solve, with the seam fix-up, instead of the decoupled
    kernel;
    C_t = 4 (no cluster instance) runs as two C_t = 2 halves.  Parity with the oracle."""
    g, t, c = random_problem(H, W, 3, Ct, seed=H + W + Ct)
    args = (6.0, 0.2, 3, 0.99, 3)
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    with dts.Solver(gd, 6.0, 0.2, 3) as s:
        plan = dts.debug_col_plan(s.ctx, Ct if Ct < 4 else 2)
        out = torch.empty_like(td)
        s.solve(td, cd, 0.99, 3, out=out)
    torch.cuda.synchronize()
    assert plan["kind"] == 1
    assert (plan["HS"] > 0) == strips
    ref = oracle.solve(g, t, c, *args)
    assert np.max(np.abs(out.cpu().numpy().astype(np.float64) - ref)) <= TOL * target_range(t)


@pytest.mark.parametrize("H,W,Ct,oop", [(3000, 4000, 1, 0), (3000, 4000, 1, 2), (700, 900, 1, 2), (500, 600, 3, 2)])
def test_column_passes_in_and_out_of_place(H, W, Ct, oop):
    """Option col_oop: column passes in place (0), over row strips out of place (1, default) or
    every cluster-kernel pass out of place (2) give the same output, bit for bit (the next row
    pass reads whichever buffer the column pass wrote)."""
    g, t, c = random_problem(H, W, 3, Ct, seed=91 + H)
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    outs = []
    for o in (1, oop):
        out = torch.empty_like(td)
        with dts.options(col_oop=o), dts.Solver(gd, 6.0, 0.2, 3) as s:
            s.solve(td, cd, 0.99, 4, out=out)
            nst = dts.debug_strips(s.ctx)["strips"]
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert (nst > 1) == (H == 3000)
    np.testing.assert_array_equal(outs[0], outs[1])
