#!/usr/bin/env python
"""DTS benchmark (driver contract).  One JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Workload: BASELINE.json config C4 -- the 100-MP, 16-band
satellite-scale guide, 1-channel target, sigma_s = 64, sigma_r = 0.2, N = 3 passes,
lambda = 0.99, 20 iterations.  One STEP is the whole hot path over one input:
dts_create (guide derivative K1 + support K5) + dts_solve (prologue K6 + 20 x [3 row passes
K2 (the first fused with the previous iteration's Eq. (3) step), 3 column passes K3] + one
closing Eq. (3) update K4) + dts_destroy.  Metric: Mpix*iterations per second (pixels x
iterations / step time).

`value` times the step with inputs resident in HBM, the library's per-launch profiler OFF
(CUDA events on the launch stream, barrier + synchronize on both sides, max over ranks); a
second, profiled pass gives the per-kernel table and the roofline of the dominant kernel.
`e2e` times the same step through the C ABI with page-locked HOST buffers: H2D of the guide,
target and confidence and D2H of the output happen inside the timed region.
--gpus N > 1 without torchrun re-launches this script under torch.distributed.run with N
ranks (one per GPU): C4 is split into row bands (NCCL exchange of column-pass carries), C3 by
image (each rank's images in one dts_create_batch context); rank 0 checks the gathered banded
output against a single-context solve (untimed).
--impl reference times the fp64 CPU oracle (oracle/) on a bounded row-band sample of the same
workload; that and the cpu_baseline / parity legs are the only places this script executes
oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, make_inputs, target_range  # noqa: E402

METRIC = "DTS Mpix·iter/s at 1/2/4/8 B200; achieved HBM GB/s vs peak"
UNIT = "Mpix·iter/s"
CPU_SAMPLE_ROWS = {"C0": 48, "C1": 1000, "C2": 1024, "C3": 256, "C4": 384}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the NEXT rows, the other configs and the sweeps")
    ap.add_argument("--bands", action="store_true",
                    help="row-band mode even on one rank (exercises the NCCL transport at N=1)")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="library option (dts_set_option) for experiments; recorded in config.options")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload_desc(cfg):
    return (f"{cfg.name}: {cfg.batch}x {cfg.W}x{cfg.H} guide with {cfg.Cg} channels, {cfg.Ct}-channel target, "
            f"sigma_s={cfg.sigma_s:g}, sigma_r={cfg.sigma_r:g}, N={cfg.N} passes, lambda={cfg.lam:g}, "
            f"{cfg.iters} iterations")


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run, one rank per GPU."""
    import torch
    if torch.cuda.device_count() < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} GPU(s) visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ CPU oracle leg
def cpu_oracle_sample(cfg, steps=1, warmup=0):
    """The oracle, as it stands, on a bounded sample: the first CPU_SAMPLE_ROWS rows
    (full width, all channels) of the workload's image 0, all iterations."""
    import oracle
    rows = min(CPU_SAMPLE_ROWS.get(cfg.name, 256), cfg.H)
    g, t, c = make_inputs(cfg.name, rows=(0, rows))
    mpix_iter = rows * cfg.W * cfg.iters / 1e6
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        oracle.solve(g, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return {"value": mpix_iter / statistics.median(times), "unit": UNIT, "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"rows [0,{rows}) x {cfg.W} cols of {cfg.name} image 0 ({cfg.Cg}-channel guide), "
                      f"{cfg.iters} iterations = {mpix_iter:.1f} Mpix*iter per run; fp64 C oracle, OpenMP, "
                      f"includes distances + support + solve",
            "seconds_per_run": statistics.median(times)}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cb = cpu_oracle_sample(cfg, steps=max(args.steps, 1), warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * cb["seconds_per_run"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "sample": cb["sample"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                mx.append(float(parts[2].split()[0]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers for the GPU leg
class Timer:
    """CUDA-event timing of fn() x steps on `stream`, synchronised (and max-reduced) across ranks."""

    def __init__(self, torch, stream, dev, world):
        self.torch, self.stream, self.dev, self.world = torch, stream, dev, world

    def barrier(self):
        if self.world > 1:
            import torch.distributed as tdist
            tdist.barrier()

    def __call__(self, fn, steps):
        torch = self.torch
        torch.cuda.synchronize()
        self.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for _ in range(steps):
            fn()
        e1.record(self.stream)
        e1.synchronize()
        torch.cuda.synchronize()
        self.barrier()
        ms = e0.elapsed_time(e1)
        if self.world > 1:
            import torch.distributed as tdist
            tt = torch.tensor([ms], device=self.dev)
            tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms


def kernel_table(stats, steps, step_ms, peak):
    fams = {k: v for k, v in stats.items() if v["launches"] > 0}
    out = {}
    for k, v in fams.items():
        gbs = v["bytes_per_launch"] / (v["avg_ms"] / 1e3) / 1e9 if v["avg_ms"] > 0 else 0.0
        out[k] = {"launches_per_step": v["launches"] / steps, "avg_ms": v["avg_ms"],
                  "bytes_per_launch": v["bytes_per_launch"], "gbs": gbs, "frac_of_peak": gbs / peak,
                  "share_of_step": (v["total_ms"] / steps) / step_ms if step_ms > 0 else 0.0}
    return out


def dominant(table, solve_only=True):
    create = ("guide_deriv", "link_fill", "support_row", "support_col", "edge_profiles", "box_windows")
    cand = {k: v for k, v in table.items() if not (solve_only and k in create)}
    name = max(cand, key=lambda k: cand[k]["share_of_step"])
    return name, cand[name]


# ------------------------------------------------------------------ extras (rank 0, one GPU)
def extra_configs(dts, torch, dev, stream, timer, peak):
    """Every paper-shaped workload besides the headline (north star "Reporting"; VERDICT r1 item
    5): C1 stereo shape, C2 16x SR, C3 8 x 4K 3-channel.  Per
    config: create + solve + destroy per step (profiler off; C3: one batched context for its
    images, and per-image contexts beside it), the dominant solve kernel's
    fraction of the HBM peak (profiled step) and parity of image 0 against the fp64 oracle."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    res = {}
    for name in ("C1", "C2", "C3"):
        cfg = CONFIGS[name]
        if cfg.batch > 1:
            with ThreadPoolExecutor(min(cfg.batch, os.cpu_count() or 1)) as ex:
                host = list(ex.map(lambda i: make_inputs(name, image=i), range(cfg.batch)))
        else:
            host = [make_inputs(name)]
        devin = [tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in x) for x in host]
        outs = [torch.empty_like(t) for _, t, _ in devin]
        batched = cfg.batch > 1  # one context for all images (dts_create_batch)
        if batched:
            bin_ = tuple(torch.stack([x[j] for x in devin]) for j in range(3))
            bout = torch.empty_like(bin_[1])

        def step_per_image():
            for (g, t, c), o in zip(devin, outs):
                ctx = dts.dts_create(g, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)
                dts.dts_solve(ctx, t, c, cfg.lam, cfg.iters, o, stream=stream.cuda_stream)
                dts.dts_destroy(ctx)

        def step_batched():
            ctx = dts.dts_create_batch(bin_[0], cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)
            dts.dts_solve(ctx, bin_[1], bin_[2], cfg.lam, cfg.iters, bout, stream=stream.cuda_stream)
            dts.dts_destroy(ctx)

        step = step_batched if batched else step_per_image
        step()
        steps = 3
        ms = timer(step, steps) / steps
        ms_per_image_ctx = None
        if batched:
            step_per_image()
            ms_per_image_ctx = timer(step_per_image, steps) / steps
        # solve only, first (eager) solve of a fresh context and a repeat (graph replay): the
        # batched context of every image, else image 0's
        if batched:
            ctx = dts.dts_create_batch(bin_[0], cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)
            g0, t0, c0, o0, px_solve = *bin_, bout, cfg.pixels
        else:
            (g0, t0, c0), o0, px_solve = devin[0], outs[0], cfg.H * cfg.W
            ctx = dts.dts_create(g0, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)
        first = timer(lambda: dts.dts_solve(ctx, t0, c0, cfg.lam, cfg.iters, o0, stream=stream.cuda_stream), 1)
        dts.dts_solve(ctx, t0, c0, cfg.lam, cfg.iters, o0, stream=stream.cuda_stream)
        rep = timer(lambda: dts.dts_solve(ctx, t0, c0, cfg.lam, cfg.iters, o0, stream=stream.cuda_stream), 3) / 3
        dts.dts_destroy(ctx)
        dts.dts_profile_enable(0, True)
        step()
        table = kernel_table(dts.dts_profile_read(0), 1, ms, peak)
        dts.dts_profile_enable(0, False)
        kname, k = dominant(table)
        t_or = time.perf_counter()
        ref = oracle.solve(host[0][0], host[0][1], host[0][2], cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, cfg.iters)
        t_or = time.perf_counter() - t_or
        step()  # outputs of a plain step for the parity check
        torch.cuda.synchronize()
        got0 = (bout[0] if batched else outs[0]).cpu().numpy().astype(np.float64)
        err = float(np.max(np.abs(got0 - ref)))
        rng = float(target_range(host[0][1]))
        res[name] = {"workload": workload_desc(cfg),
                     "mpix_iter_per_s": cfg.pixels * cfg.iters / 1e6 / (ms / 1e3), "ms_per_step": ms,
                     "step": ("dts_create_batch + dts_solve + dts_destroy, one context for all images" if batched
                              else "dts_create + dts_solve + dts_destroy"),
                     "solve_only": "all images (batched context)" if batched else "image 0",
                     "solve_only_first_ms": first, "solve_only_repeat_ms": rep,
                     "solve_only_first_mpix_iter_per_s": px_solve * cfg.iters / 1e6 / (first / 1e3),
                     "solve_only_repeat_mpix_iter_per_s": px_solve * cfg.iters / 1e6 / (rep / 1e3),
                     "dominant_kernel": {"name": kname, "avg_ms": k["avg_ms"], "gbs": k["gbs"],
                                         "frac_of_peak": k["frac_of_peak"], "share_of_step": k["share_of_step"]},
                     "kernels": {kk: {"avg_ms": v["avg_ms"], "frac_of_peak": v["frac_of_peak"],
                                      "launches_per_step": v["launches_per_step"]} for kk, v in table.items()},
                     "parity": {"vs": "fp64 oracle (O6), image 0, full solve", "max_abs_err": err,
                                "tol_abs": 1e-4 * rng, "max_abs_err_over_range": err / rng, "ok": err <= 1e-4 * rng,
                                "oracle_seconds": t_or}}
        if batched:
            res[name]["per_image_contexts"] = {"ms_per_step": ms_per_image_ctx,
                                               "mpix_iter_per_s": cfg.pixels * cfg.iters / 1e6 / (ms_per_image_ctx / 1e3)}
            del bin_, bout
        del devin, outs
    return res


def sweeps(dts, torch, dev, stream, timer):
    """The paper's scaling claims on the C1 shape: run time nearly independent of sigma_s and
    sigma_r and linear in the iteration count; and linear in the pixel count
     over 0.35-100 Mpixel.  Solve time (eager first solve of a fresh context, and a repeat)
    per setting."""
    cfg = CONFIGS["C1"]
    g, t, c = make_inputs("C1")
    gd, td, cd = (torch.from_numpy(a).to(dev) for a in (g, t, c))
    o = torch.empty_like(td)

    def solve_ms(ss, sr, iters):
        ctx = dts.dts_create(gd, ss, sr, cfg.N, stream=stream.cuda_stream)
        first = timer(lambda: dts.dts_solve(ctx, td, cd, cfg.lam, iters, o, stream=stream.cuda_stream), 1)
        dts.dts_solve(ctx, td, cd, cfg.lam, iters, o, stream=stream.cuda_stream)
        rep = timer(lambda: dts.dts_solve(ctx, td, cd, cfg.lam, iters, o, stream=stream.cuda_stream), 3) / 3
        dts.dts_destroy(ctx)
        return first, rep

    out = {"shape": "C1 1400 x 1000, 1-channel target, N = 3, lambda = 0.99", "sigma_s": {}, "sigma_r": {},
           "iterations": {}}
    for ss in (16.0, 32.0, 128.0, 256.0):
        f, r = solve_ms(ss, 0.1, cfg.iters)
        out["sigma_s"][f"{ss:g}"] = {"first_ms": f, "repeat_ms": r}
    for sr in (0.1, 0.3, 0.5, 0.7, 0.9):
        f, r = solve_ms(16.0, sr, cfg.iters)
        out["sigma_r"][f"{sr:g}"] = {"first_ms": f, "repeat_ms": r}
    its = (10, 25, 50, 100, 200)
    for it in its:
        f, r = solve_ms(16.0, 0.1, it)
        out["iterations"][str(it)] = {"first_ms": f, "repeat_ms": r}
    for key in ("sigma_s", "sigma_r"):
        v = [x["first_ms"] for x in out[key].values()]
        out[key]["max_over_min_first"] = max(v) / min(v)
    y = np.array([out["iterations"][str(i)]["first_ms"] for i in its])
    A = np.stack([np.ones(len(its)), np.array(its, float)], 1)
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    fit = A @ coef
    out["iterations"]["linear_fit_first"] = {"ms_at_0": float(coef[0]), "ms_per_iteration": float(coef[1]),
                                             "r2": float(1 - np.sum((y - fit) ** 2) / np.sum((y - y.mean()) ** 2))}
    # run time against the pixel count ("linear in the number of pixels"): device-generated
    # images from 0.35 to 100 Mpixel (3-channel guide, 20 iterations), the median of three eager
    # solves (graph replay off) after a warm-up solve on the same context
    del gd, td, cd, o
    out["pixels"] = {"shape": "H x W random 3-channel guide with a step edge, 1-channel target, sigma_s = 16, "
                            "sigma_r = 0.1, N = 3, 20 iterations, median of 3 eager solves"}
    graphs0 = dts.dts_get_option("graphs")
    dts.dts_set_option("graphs", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    for H, W in ((500, 700), (1000, 1400), (2000, 2800), (4000, 5600), (7071, 10000), (10000, 10000)):
        gq = torch.rand(H, W, 3, device=dev, generator=gen) * 0.05
        gq[H // 3:, W // 3:, :] += 0.5
        tq = torch.rand(H, W, device=dev, generator=gen)
        cq = torch.rand(H, W, device=dev, generator=gen)
        oq = torch.empty_like(tq)
        ctx = dts.dts_create(gq, 16.0, 0.1, 3, stream=stream.cuda_stream)
        dts.dts_solve(ctx, tq, cq, 0.99, 20, oq, stream=stream.cuda_stream)  # warm-up
        ts = sorted(timer(lambda: dts.dts_solve(ctx, tq, cq, 0.99, 20, oq, stream=stream.cuda_stream), 1)
                    for _ in range(3))
        dts.dts_destroy(ctx)
        out["pixels"][f"{H}x{W}"] = {"mpix": H * W / 1e6, "ms": ts[1], "ms_all": ts,
                                     "mpix_iter_per_s": H * W * 20 / 1e6 / (ts[1] / 1e3)}
        del gq, tq, cq, oq
    dts.dts_set_option("graphs", graphs0)
    sizes = [v for k, v in out["pixels"].items() if isinstance(v, dict)]
    xp = np.array([v["mpix"] for v in sizes])
    yp = np.array([v["ms"] for v in sizes])
    A = np.stack([np.ones(len(xp)), xp], 1)
    coef, *_ = np.linalg.lstsq(A, yp, rcond=None)
    fit = A @ coef
    out["pixels"]["linear_fit"] = {"ms_at_0": float(coef[0]), "ms_per_mpix": float(coef[1]),
                                   "r2": float(1 - np.sum((yp - fit) ** 2) / np.sum((yp - yp.mean()) ** 2))}
    return out


def next_rows(dts, torch, dev, stream, timer, cfg, dev_in, peak):
    """SURVEY 8(f) rows on the headline workload / the C1 shape (unchanged from round 1)."""
    extras = {}
    g0, t0, c0 = dev_in[0]
    if cfg.Ct == 1:
        conf_out = torch.empty_like(t0)
        var_out = torch.empty_like(t0)
        ctx = dts.dts_create(g0, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)
        sc = 0.5 * float(t0.max().item() - t0.min().item())  # sigma_c: half the target range (R22)
        dts.dts_confidence(ctx, t0, sc, conf_out, var_out, stream=stream.cuda_stream)  # warm-up
        reps = 3
        c_ms = timer(lambda: dts.dts_confidence(ctx, t0, sc, conf_out, var_out, stream=stream.cuda_stream), reps)
        dts.dts_destroy(ctx)
        c_ms /= reps
        px = t0.numel()
        cbytes = px * (28.0 + 40.0 * cfg.N)  # t in, [t, t^2] out; N x (row + col, C_t = 2); X in, c + V out
        extras["confidence"] = {"what": "dts_confidence (Eq. 7): DT(t^2) - DT(t)^2 -> c, same guide", "sigma_c": sc,
                                "ms": c_ms, "mpix_per_s": px / 1e6 / (c_ms / 1e3),
                                "gbs_algorithmic": cbytes / (c_ms / 1e3) / 1e9,
                                "frac": cbytes / (c_ms / 1e3) / 1e9 / peak}
    bout = torch.empty_like(t0)

    def box_step():
        bctx = dts.dts_create_ex(g0, cfg.sigma_s, cfg.sigma_r, cfg.N, dts.DTS_FILTER_BOX, stream=stream.cuda_stream)
        dts.dts_solve(bctx, t0, c0, cfg.lam, cfg.iters, bout, stream=stream.cuda_stream)
        dts.dts_destroy(bctx)

    box_step()
    b_ms = timer(box_step, 2) / 2
    dts.dts_profile_enable(0, True)
    box_step()
    bstats = dts.dts_profile_read(0)
    dts.dts_profile_enable(0, False)
    bpx = t0.shape[0] * t0.shape[1]
    extras["box"] = {"what": "dts_create_ex(DTS_FILTER_BOX) + dts_solve + dts_destroy: the box-window edge-aware "
                             "mean (reading R25), same guide / target / confidence / iterations",
                     "ms_per_step": b_ms, "mpix_iter_per_s": bpx * cfg.iters / 1e6 / (b_ms / 1e3), "kernels": {}}
    for name in ("box_windows", "box_row", "box_col", "update", "prologue"):
        v = bstats.get(name)
        if v and v["launches"]:
            gbs = v["bytes_per_launch"] / (v["avg_ms"] / 1e3) / 1e9
            extras["box"]["kernels"][name] = {"launches": v["launches"], "avg_ms": v["avg_ms"], "gbs": gbs,
                                              "frac": gbs / peak}
    # Eq. (10) stereo refinement, C1 shape, the paper's gamma = eps = 0.001 (parity: tests/test_stereo_gpu.py)
    c1 = CONFIGS["C1"]
    Lh, th, ch = make_inputs("C1")
    rng = np.random.default_rng(1)
    Rh = (np.roll(Lh, -16, axis=1) + rng.normal(0, 0.01, Lh.shape)).astype(np.float32)
    Ld, Rd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (Lh, Rh, th, ch))
    sout = torch.empty_like(td)
    sctx = dts.dts_create(Ld, c1.sigma_s, c1.sigma_r, c1.N, stream=stream.cuda_stream)
    run = lambda: dts.dts_solve_stereo(sctx, td, cd, c1.lam, c1.iters, sout, Ld, Rd, 0.001, 0.001,  # noqa: E731
                                       stream=stream.cuda_stream)
    s_first = timer(run, 1)
    run()  # the second identical call captures the launch sequence as a CUDA graph
    reps = 3
    s_ms = timer(run, reps) / reps
    dts.dts_destroy(sctx)
    spx = c1.H * c1.W
    extras["stereo"] = {"what": "dts_solve_stereo (Eq. 10, Charbonnier target, gamma = eps = 0.001) on C1 "
                                "(1400 x 1000, 3-channel pair: right = left shifted 16 px + noise)",
                        "iterations": c1.iters, "first_ms": s_first, "ms": s_ms,
                        "mpix_iter_per_s": spx * c1.iters / 1e6 / (s_ms / 1e3)}
    low = torch.rand(64, 86, device=dev) * 9.5 + 0.5
    st_o, sc_o = torch.empty(1024, 1376, device=dev), torch.empty(1024, 1376, device=dev)
    runp = lambda: dts.dts_sr_prepare(low, 16, st_o, sc_o, stream=stream.cuda_stream)  # noqa: E731
    runp()
    p_ms = timer(runp, 10) / 10
    extras["sr_prepare"] = {"what": "dts_sr_prepare: bicubic x16 target + bump confidence, 86x64 -> 1376x1024",
                            "ms": p_ms, "mpix_per_s": 1376 * 1024 / 1e6 / (p_ms / 1e3)}
    return extras


# ------------------------------------------------------------------ GPU leg
def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)

    # the JSON line is the only thing on stdout: libraries (NCCL prints its version at communicator
    # init) write to stderr while this leg runs
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)

    import torch
    import paper_1805_04590_b200 as dts

    opts = {}
    for o in args.option:
        k, v = o.split("=")
        dts.dts_set_option(k, int(v))
        opts[k] = int(v)
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)
    launched = "WORLD_SIZE" in os.environ  # under torchrun (any N)
    tdist = None
    if world > 1 or (launched and args.bands):
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    # units of this rank: images (batched configs: no collective on the data path) or a
    # row band of the single image (column-pass carries exchanged with NCCL)
    comm = None
    band = None
    if cfg.batch > 1:
        if cfg.batch % world:
            raise SystemExit(f"{cfg.batch} images do not split over {world} ranks")
        per = cfg.batch // world
        images = list(range(rank * per, (rank + 1) * per))
        inputs = [make_inputs(cfg.name, image=i) for i in images]
        if per > 1:  # one batched context for this rank's images (dts_create_batch)
            inputs = [tuple(np.ascontiguousarray(np.stack([x[j] for x in inputs])) for j in range(3))]
    elif world > 1 or args.bands:
        r0, r1 = dts.band_rows(cfg.H, world, rank)
        a, b = dts.band_guide_rows(cfg.H, r0, r1)
        g, t, c = make_inputs(cfg.name, rows=(a, b))
        inputs = [(g, np.ascontiguousarray(t[r0 - a:r1 - a]), np.ascontiguousarray(c[r0 - a:r1 - a]))]
        band = (r0, r1)
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(dts.dts_comm_unique_id()), dtype=torch.uint8))
        if world > 1:
            tdist.broadcast(uid, 0)
        comm = dts.dts_comm_init(bytes(uid.cpu().numpy().tobytes()), rank, world)
    else:
        inputs = [make_inputs(cfg.name)]
    batched = cfg.batch > 1 and cfg.batch // world > 1
    pixels_rank = (cfg.batch // world) * cfg.H * cfg.W if cfg.batch > 1 else sum(t.shape[0] * t.shape[1]
                                                                                for _, t, _ in inputs)

    stream = torch.cuda.Stream(device=dev)
    timer = Timer(torch, stream, dev, world)
    dev_in = [tuple(torch.from_numpy(a).to(dev) for a in x) for x in inputs]
    outs = [torch.empty_like(t) for _, t, _ in dev_in]

    def make_ctx(g):
        if batched:
            return dts.dts_create_batch(g, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)
        if band is not None:
            return dts.dts_create_band(g, cfg.H, band[0], band[1] - band[0], cfg.sigma_s, cfg.sigma_r, cfg.N,
                                       comm=comm, stream=stream.cuda_stream)
        return dts.dts_create(g, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)

    def step_device():
        for (g, t, c), o in zip(dev_in, outs):
            ctx = make_ctx(g)
            dts.dts_solve(ctx, t, c, cfg.lam, cfg.iters, o, stream=stream.cuda_stream)
            dts.dts_destroy(ctx)

    for _ in range(max(args.warmup, 0)):
        step_device()
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs, profiler OFF, clocks sampled ----
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    ms = timer(step_device, args.steps)
    clk = clocks.stop() if clocks else None
    ms_step = ms / args.steps
    mpix_iter_total = pixels_rank * world * cfg.iters / 1e6
    value = mpix_iter_total / (ms_step / 1e3)

    # ---- second pass with the per-launch profiler: kernel table, roofline, launch count ----
    psteps = max(1, min(args.steps, 3))
    dts.dts_profile_enable(0, True)
    p_ms = timer(step_device, psteps) / psteps
    kstats = dts.dts_profile_read(0)
    dts.dts_profile_enable(0, False)
    peak, peak_src = measured_peaks()
    table = kernel_table(kstats, psteps, p_ms, peak)
    launches_per_step = sum(v["launches_per_step"] for v in table.values())
    create_fams = ("guide_deriv", "link_fill", "support_row", "support_col", "edge_profiles")
    create_ms = sum(v["avg_ms"] * v["launches_per_step"] for k, v in table.items() if k in create_fams)
    split = {"create_ms": create_ms, "solve_ms": ms_step - create_ms,
             "solve_mpix_iter_per_s": mpix_iter_total / ((ms_step - create_ms) / 1e3),
             "note": "create_ms = event time of the create-time kernels per step (profiled pass); solve_ms = the "
                     "unprofiled step time minus create_ms"}

    # ---- banded runs: gathered output against a single-context solve (untimed) ----
    parity = None
    if band is not None:
        step_device()
        torch.cuda.synchronize()
        mine = outs[0]
        if world > 1:
            if rank == 0:
                parts = [mine]
                for r in range(1, world):
                    a_, b_ = dts.band_rows(cfg.H, world, r)
                    buf = torch.empty((b_ - a_, cfg.W), dtype=torch.float32, device=dev)
                    tdist.recv(buf, r)
                    parts.append(buf)
                full = torch.cat(parts, 0)
            else:
                tdist.send(mine, 0)
        else:
            full = mine
        if rank == 0:
            gf, tf, cf = make_inputs(cfg.name)
            gfd, tfd, cfd = (torch.from_numpy(a).to(dev) for a in (gf, tf, cf))
            ref = torch.empty_like(tfd)
            ctx = dts.dts_create(gfd, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)
            dts.dts_solve(ctx, tfd, cfd, cfg.lam, cfg.iters, ref, stream=stream.cuda_stream)
            dts.dts_destroy(ctx)
            torch.cuda.synchronize()
            err = float((full - ref).abs().max().item())
            rng = float(target_range(tf))
            parity = {"vs": "single-context solve of the whole image on rank 0's GPU", "max_abs_diff": err,
                      "max_abs_diff_over_range": err / rng, "tol_over_range": 1e-5, "ok": err <= 1e-5 * rng}
            del gfd, tfd, cfd, ref, full

    # ---- e2e: the same step through the C ABI with pinned HOST buffers ----
    e2e = None
    if not args.no_e2e:
        host_in = [tuple(torch.from_numpy(a).pin_memory() for a in x) for x in inputs]
        host_out = [torch.empty(t.shape, dtype=torch.float32, pin_memory=True) for _, t, _ in host_in]
        h2d = sum(g.numel() * 4 + t.numel() * 4 + c.numel() * 4 for g, t, c in host_in)
        d2h = sum(o.numel() * 4 for o in host_out)

        def step_host():
            for (g, t, c), o in zip(host_in, host_out):
                ctx = make_ctx(g)
                dts.dts_solve(ctx, t, c, cfg.lam, cfg.iters, o, stream=stream.cuda_stream)
                dts.dts_destroy(ctx)

        step_host()  # warm the staging buffers
        e_steps = max(1, min(args.steps, 3))
        e_ms = timer(step_host, e_steps)
        e2e = {"value": mpix_iter_total / (e_ms / e_steps / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": d2h * world, "ms_per_step": e_ms / e_steps,
               "check_max_abs_vs_device": float((host_out[0].to(dev) - outs[0]).abs().max().item())}
        del host_in, host_out

    extras = {}
    if world == 1 and band is None and not args.no_extras:
        if cfg.batch == 1:
            extras.update(next_rows(dts, torch, dev, stream, timer, cfg, dev_in, peak))
        del dev_in, outs
        torch.cuda.empty_cache()
        extras["configs"] = extra_configs(dts, torch, dev, stream, timer, peak)
        extras["sweeps"] = sweeps(dts, torch, dev, stream, timer)

    if rank != 0:
        if comm:
            dts.dts_comm_destroy(comm)
        tdist.destroy_process_group()
        return 0

    # ---- roofline of the dominant solve kernel ----
    dom_name, dom = dominant(table)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        ent = tj.get(cfg.name, {}).get(dom_name)
        if ent:
            traffic = ent.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": dom["gbs"], "peak": peak, "unit": "GB/s",
                "frac": dom["gbs"] / peak, "traffic": traffic, "peak_source": peak_src,
                "bytes_per_launch": dom["bytes_per_launch"], "avg_launch_ms": dom["avg_ms"],
                "share_of_step": dom["share_of_step"]}
    step_bytes = sum(v["bytes_per_launch"] * v["launches_per_step"] for v in table.values())
    roofline["step_gbs_algorithmic"] = step_bytes / (ms_step / 1e3) / 1e9 * world
    roofline["step_frac_algorithmic"] = roofline["step_gbs_algorithmic"] / (peak * world)

    cpu = None
    if not args.no_cpu and world == 1:
        cb = cpu_oracle_sample(cfg)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    scaling = "weak" if cfg.batch > 1 else "strong"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "pixels": cfg.pixels, "iterations": cfg.iters,
                       "step": ("dts_create_batch (one context for this rank's images) + dts_solve + dts_destroy"
                                if batched else "dts_create + dts_solve + dts_destroy") +
                               " (guide derivative, support, prologue, "
                               f"{cfg.iters} x (3 row + 3 column pass kernels), closing update)",
                       "l2": "inputs larger than L2 (6.4 GB guide, 0.4 GB per state plane): no flush needed"
                             if cfg.name == "C4" else "L2 not flushed between steps",
                       "parallelism": (f"image split x{world}" if cfg.batch > 1 else
                                       (f"row bands x{world} (NCCL all-gather of column-pass edge records)"
                                        if band is not None else "single GPU")),
                       "profiler": "off in the timed region; kernels / roofline from a second, profiled pass",
                       **({"options": opts} if opts else {})},
            "roofline": roofline,
            "kernels": table,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(round(launches_per_step * args.steps)),
            "gpu_launches_per_step": launches_per_step, "clocks": clk, "split": split, "parity": parity,
            "profiled_ms_per_step": p_ms, "extras": extras}
    sys.stdout.flush()
    os.write(json_fd, (json.dumps(line) + "\n").encode())
    if comm:
        dts.dts_comm_destroy(comm)
    if tdist is not None:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
