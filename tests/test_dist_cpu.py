"""Multi-rank host logic on CPU (gloo, world_size 2): band partition and halos, the
unique-id broadcast bench.py performs, and the row-band exchange protocol (tuples
all-gathered in rank order, carries composed, bands finished) -- checked against the
dense triangular form of a full column pass (tests/dense.py), in fp64."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1805_04590_b200 as dts
from synth import make_inputs
from tests import bandalg, dense


@pytest.mark.parametrize("H,P", [(10000, 1), (10000, 2), (10000, 8), (1000, 3), (7, 4), (5, 5)])
def test_band_partition(H, P):
    rows = [dts.band_rows(H, P, r) for r in range(P)]
    assert rows[0][0] == 0 and rows[-1][1] == H
    for (a, b), (c, d) in zip(rows, rows[1:]):
        assert b == c and a < b
    sizes = [b - a for a, b in rows]
    assert max(sizes) - min(sizes) <= 1
    for r, (a, b) in enumerate(rows):
        assert a == r * H // P
        ga, gb = dts.band_guide_rows(H, a, b)
        assert ga == max(a - 1, 0) and gb == min(b + 1, H)


def test_band_inputs_are_rows_of_the_full_image():
    g, t, c = make_inputs("C1")
    for r0, r1 in [(0, 251), (250, 500), (999, 1000)]:
        g2, t2, c2 = make_inputs("C1", rows=(r0, r1))
        assert np.array_equal(g2, g[r0:r1]) and np.array_equal(t2, t[r0:r1]) and np.array_equal(c2, c[r0:r1])


def test_band_algebra_single_process():
    rng = np.random.default_rng(0)
    H = 57
    A = rng.uniform(0.2, 0.98, H)
    A[0] = 0.0
    x = rng.normal(size=H)
    ref = dense.pass1d(A) @ x
    for P in (1, 2, 3, 5):
        cuts = [k * H // P for k in range(P + 1)]
        tuples, parts = [], []
        for k in range(P):
            lo, hi = cuts[k], cuts[k + 1]
            tup, pr = bandalg.band_parts(x, A, lo, hi, A[hi] if hi < H else 0.0)
            tuples.append(tup)
            parts.append(pr)
        c, e = bandalg.compose(tuples)
        got = np.concatenate([bandalg.finish(parts[k], c[k], e[k]) for k in range(P)])
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # (1) unique-id broadcast as bench.py does it (rank 0's bytes reach every rank)
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid.copy_(torch.arange(128, dtype=torch.uint8) * 7)
        dist.broadcast(uid, 0)
        ok_uid = bool(torch.equal(uid, torch.arange(128, dtype=torch.uint8) * 7))
        # (2) the exchange: every rank summarises its band of 16 columns, tuples are
        #     all-gathered in rank order, carries composed, bands finished
        H, Wc = 41, 16
        rng = np.random.default_rng(123)
        A = rng.uniform(0.1, 0.97, (H, Wc))
        A[0] = 0.0
        X = rng.normal(size=(H, Wc))
        r0, r1 = dts.band_rows(H, world, rank)
        tup = np.zeros((Wc, 5))
        parts = []
        for col in range(Wc):
            t, pr = bandalg.band_parts(X[:, col], A[:, col], r0, r1, A[r1, col] if r1 < H else 0.0)
            tup[col] = t
            parts.append(pr)
        send = torch.from_numpy(tup.copy())
        recv = [torch.zeros_like(send) for _ in range(world)]
        dist.all_gather(recv, send)
        gathered = np.stack([t.numpy() for t in recv], 0)  # [P][Wc][5]
        band_out = np.zeros((r1 - r0, Wc))
        for col in range(Wc):
            c, e = bandalg.compose([gathered[k, col] for k in range(world)])
            band_out[:, col] = bandalg.finish(parts[col], c[rank], e[rank])
        outs = [None] * world
        dist.all_gather_object(outs, band_out)
        if rank == 0:
            full = np.concatenate(outs, 0)
            ref = np.stack([dense.pass1d(A[:, col]) @ X[:, col] for col in range(Wc)], 1)
            q.put((ok_uid, float(np.max(np.abs(full - ref)))))
        else:
            q.put((ok_uid, 0.0))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[0] for r in res)
    assert max(r[1] for r in res) <= 1e-12


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_edge_scheme_algebra(P):
    """The edge fix-up scheme of the row-band column pass: with bands of >= 2L rows,
    zero-carry passes + corrections c Gamma (top L rows) and e Theta (bottom L rows), with
    c = y0 at the last row of the band above and e = z0 at the first row of the band below
    + y0(this band's last row) Gamma_0(below), equal the full column pass to below 2^-26."""
    rng = np.random.default_rng(P)
    H = 480
    amax = 0.7  # every coefficient <= a_i (d >= 1); L = 51 rows
    A = rng.uniform(0.3, amax, H)
    A[0] = 0.0
    x = rng.normal(size=H)
    ref = dense.pass1d(A) @ x
    L = int(np.ceil(np.log(2.0 ** -26) / np.log(amax)))
    assert 2 * L + 1 <= H // P
    cuts = [k * H // P for k in range(P + 1)]
    got = bandalg.edge_scheme(x, A, cuts, L)
    assert np.max(np.abs(got - ref)) <= 2.0 ** -24 * np.max(np.abs(x))


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_edge_scheme_cut_variant(P):
    """The edge scheme run on the single-context column kernel: the zero-carry pass cuts the
    link below the band (a_H = 0), so row H - 1 of its output is y0 and row 0 is z0; the
    bottom correction is (z_H - y0(H - 1)) Theta_k with the uncut Theta.  Equals the full
    column pass to below 2^-26, like the exported-value scheme."""
    rng = np.random.default_rng(10 + P)
    H = 480
    amax = 0.7
    A = rng.uniform(0.3, amax, H)
    A[0] = 0.0
    x = rng.normal(size=H)
    ref = dense.pass1d(A) @ x
    L = int(np.ceil(np.log(2.0 ** -26) / np.log(amax)))
    cuts = [k * H // P for k in range(P + 1)]
    got = bandalg.edge_scheme_cut(x, A, cuts, L)
    assert np.max(np.abs(got - ref)) <= 2.0 ** -24 * np.max(np.abs(x))
    # the changed bottom carry matters: with the exported-value scheme's carry the bands
    # would not join
    if P > 1:
        bad = bandalg.edge_scheme_cut(x, A, cuts, L, fix_carry=False)
        assert np.max(np.abs(bad - ref)) > 1e-3 * np.max(np.abs(x))


def test_edge_scheme_support_variant():
    """The support's edge scheme: s = P + Q - 1 (P[k] = 1 + a_k P[k-1], Q[k] = 1 + a_{k+1} Q[k+1]),
    zero-carry s0 per band, carries c = s0 at the last row of the band above (P carry) and
    e = s0 at the first row of the band below (Q carry), corrections c G_k and e Theta_k."""
    rng = np.random.default_rng(9)
    H, P, amax = 360, 3, 0.85
    a = rng.uniform(0.2, amax, H)
    a[0] = 0.0
    Pf, Qf = np.zeros(H), np.zeros(H)
    for k in range(H):
        Pf[k] = 1 + (a[k] * Pf[k - 1] if k > 0 else 0.0)
    for k in range(H - 1, -1, -1):
        Qf[k] = 1 + (a[k + 1] * Qf[k + 1] if k + 1 < H else 0.0)
    ref = Pf + Qf - 1
    L = int(np.ceil(np.log(2.0 ** -26) / np.log(amax)))
    cuts = [k * H // P for k in range(P + 1)]
    s0, prof = [], []
    for k in range(P):
        lo, hi = cuts[k], cuts[k + 1]
        n = hi - lo
        p0, q0 = np.zeros(n), np.zeros(n)
        for i in range(n):
            p0[i] = 1 + (a[lo + i] * p0[i - 1] if i > 0 else 0.0)
        for i in range(n - 1, -1, -1):
            q0[i] = 1 + (a[lo + i + 1] * q0[i + 1] if i + 1 < n else 0.0)
        s0.append(p0 + q0 - 1)
        below = a[hi] if hi < H else 0.0
        G, _, theta = bandalg.edge_profiles(a, lo, hi, below, L)
        prof.append((G, theta))
    out = []
    for k in range(P):
        s = s0[k].copy()
        c = s0[k - 1][-1] if k > 0 else 0.0
        e = s0[k + 1][0] if k + 1 < P else 0.0
        s[:L] += c * prof[k][0]
        s[-L:] += e * prof[k][1]
        out.append(s)
    got = np.concatenate(out)
    assert np.max(np.abs(got - ref)) <= 2.0 ** -22 * np.max(np.abs(ref))
