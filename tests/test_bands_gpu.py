"""Row-band (multi-GPU) algebra on ONE GPU: P ranks run as P host threads of this
process, each with its own band context and stream, exchanging column-pass tuples
through the loopback transport (the same library path as NCCL except the copy).
The concatenated band outputs must match the fp64 oracle (tolerance of the north
star) and the single-context GPU solve (reading R18: equal up to fp32 rounding)."""
import threading

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


def solve_bands(g, t, c, ss, sr, N, lam, iters, P):
    H = g.shape[0]
    comms = dts.dts_comm_init_loopback(P)
    outs, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            r0, r1 = dts.band_rows(H, P, r)
            a, b = dts.band_guide_rows(H, r0, r1)
            with torch.cuda.stream(stream):
                gd = torch.from_numpy(np.ascontiguousarray(g[a:b])).cuda()
                td = torch.from_numpy(np.ascontiguousarray(t[r0:r1])).cuda()
                cd = torch.from_numpy(np.ascontiguousarray(c[r0:r1])).cuda()
                out = torch.empty_like(td)
            ctx = dts.dts_create_band(gd, H, r0, r1 - r0, ss, sr, N, comm=comms[r], stream=stream.cuda_stream)
            dts.dts_solve(ctx, td, cd, lam, iters, out, stream=stream.cuda_stream)
            stream.synchronize()
            outs[r] = out.cpu().numpy()
            dts.dts_destroy(ctx)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(P)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=120)
    assert not any(th.is_alive() for th in threads), "band ranks did not finish"
    for cm in comms:
        dts.dts_comm_destroy(cm)
    if errs:
        raise errs[0]
    return np.concatenate(outs, 0).astype(np.float64)


def single(g, t, c, ss, sr, N, lam, iters):
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    with dts.Solver(gd, ss, sr, N) as s:
        s.solve(td, cd, lam, iters, out=out)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("H,W,Ct", [(60, 70, 1), (517, 130, 1), (301, 45, 3), (3000, 100, 1), (2100, 70, 3)])
def test_bands_match_oracle_and_single(P, H, W, Ct):
    g, t, c = random_problem(H, W, 3, Ct, seed=P * 100 + H)
    args = (5.0, 0.2, 3, 0.99, 6)
    ref = oracle.solve(g, t, c, *args)
    got = solve_bands(g, t, c, *args, P=P)
    one = single(g, t, c, *args)
    rng = target_range(t)
    assert np.max(np.abs(got - ref)) <= 1e-4 * rng
    assert np.max(np.abs(got - one)) <= 1e-5 * rng


def test_bands_c1_shape():
    cfg = CONFIGS["C1"]
    g, t, c = make_inputs("C1")
    args = (cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, 10)
    ref = oracle.solve(g, t, c, *args)
    got = solve_bands(g, t, c, *args, P=4)
    assert np.max(np.abs(got - ref)) <= 1e-4 * target_range(t)


def test_single_band_comm_equals_plain_context():
    """P = 1 through the band machinery (TUPLE, exchange, compose, APPLY)."""
    g, t, c = random_problem(90, 66, 3, 1, seed=5)
    args = (5.0, 0.2, 3, 0.99, 4)
    got = solve_bands(g, t, c, *args, P=1)
    one = single(g, t, c, *args)
    assert np.max(np.abs(got - one)) <= 1e-5 * target_range(t)


def test_nccl_transport_single_rank():
    """The NCCL transport itself (dlopen of the process's libnccl, ncclCommInitRank,
    ncclAllGather on the launch stream) with one rank owning every row."""
    g, t, c = random_problem(120, 90, 3, 1, seed=7)
    args = (5.0, 0.2, 3, 0.99, 5)
    uid = dts.dts_comm_unique_id()
    comm = dts.dts_comm_init(uid, 0, 1)
    try:
        gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
        out = torch.empty_like(td)
        ctx = dts.dts_create_band(gd, 120, 0, 120, 5.0, 0.2, 3, comm=comm)
        dts.dts_solve(ctx, td, cd, 0.99, 5, out)
        torch.cuda.synchronize()
        dts.dts_destroy(ctx)
    finally:
        dts.dts_comm_destroy(comm)
    one = single(g, t, c, *args)
    assert np.max(np.abs(out.cpu().numpy() - one)) <= 1e-5 * target_range(t)


def test_bands_legacy_kernel_matches():
    """The decoupled band-tuple kernel (option band_scheme = 2) and the cluster TUPLE / APPLY
    kernels give the same banded solve (fp32 rounding)."""
    g, t, c = random_problem(1500, 96, 3, 1, seed=11)
    args = (9.0, 0.3, 3, 0.99, 4)
    with dts.options(band_scheme=1):
        a = solve_bands(g, t, c, *args, P=2)
    with dts.options(band_scheme=2):
        b = solve_bands(g, t, c, *args, P=2)
    assert np.max(np.abs(a - b)) <= 1e-5 * target_range(t)


@pytest.mark.parametrize("P", [2, 3])
def test_bands_edge_scheme_matches_tuple_scheme(P):
    """Bands of >= 2L rows use the edge fix-up scheme (zero-carry pass + corrections on the L
    rows at each edge); option band_scheme = 1 forces the exact TUPLE / APPLY composition.  The
    two agree to fp32 rounding, and both match the oracle."""
    g, t, c = random_problem(900, 80, 3, 1, seed=17 + P)
    args = (5.0, 0.2, 3, 0.99, 5)
    a = solve_bands(g, t, c, *args, P=P)
    with dts.options(band_scheme=1):
        b = solve_bands(g, t, c, *args, P=P)
    rng = target_range(t)
    assert np.max(np.abs(a - b)) <= 1e-5 * rng
    assert np.max(np.abs(a - oracle.solve(g, t, c, *args))) <= 1e-4 * rng


def test_bands_straddling_the_edge_threshold():
    """band heights that differ by one row around 2L + 1 must still run the same
    scheme on every rank (H = 113 over 2 ranks: 56 and 57 rows; sigma_s = 5, N = 3)."""
    g, t, c = random_problem(113, 70, 3, 1, seed=5)
    args = (5.0, 0.2, 3, 0.99, 4)
    rng = target_range(t)
    ref = oracle.solve(g, t, c, *args)
    for scheme in (0, 1, 2):
        with dts.options(band_scheme=scheme):
            a = solve_bands(g, t, c, *args, P=2)
        assert np.max(np.abs(a - ref)) <= 1e-4 * rng, scheme


@pytest.mark.parametrize("Ct", [1, 3])
def test_bands_overlapped_exchange_is_bit_identical(Ct):
    """Edge scheme with the all-gather overlapped (default: the next row pass runs on the
    band's interior rows while the exchange is in flight, then the edge fix-up and the 2L edge
    rows) against the serial order (option band_overlap = 0): the same kernels on the same
    rows, so the same bits; and parity with the oracle."""
    g, t, c = random_problem(1200, 90, 3, Ct, seed=23 + Ct)
    args = (6.0, 0.2, 3, 0.99, 5)
    a = solve_bands(g, t, c, *args, P=3)
    with dts.options(band_overlap=0):
        b = solve_bands(g, t, c, *args, P=3)
    np.testing.assert_array_equal(a, b)
    assert np.max(np.abs(a - oracle.solve(g, t, c, *args))) <= 1e-4 * target_range(t)
