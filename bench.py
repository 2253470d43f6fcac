#!/usr/bin/env python
"""DTS benchmark (driver contract).  One JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Workload: BASELINE.json config C4 -- the 100-MP, 16-band
satellite-scale guide, 1-channel target, sigma_s = 64, sigma_r = 0.2, N = 3 passes,
lambda = 0.99, 20 iterations.  One STEP is the whole hot path over one input:
dts_create (guide derivative K1 + support K5) + dts_solve (prologue K6 + 20 x
[3 row passes K2, 2 column passes K3, 1 column pass fused with the update K4]) +
dts_destroy.  Metric: Mpix*iterations per second (pixels x iterations / step time).

`value` times the step with inputs resident in HBM (CUDA events on the launch
stream, barrier + synchronize on both sides, max over ranks).  `e2e` times the
same step through the C ABI with page-locked HOST buffers: H2D of the guide,
target and confidence and D2H of the output happen inside the timed region.
--impl reference times the fp64 CPU oracle (oracle/) on a bounded row-band sample
of the same workload; that is the only other place this script executes oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, make_inputs  # noqa: E402

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
    ap.add_argument("--bands", action="store_true",
                    help="row-band mode even on one rank (exercises the NCCL transport at N=1)")
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
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
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


# ------------------------------------------------------------------ GPU leg
def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import paper_1805_04590_b200 as dts

    rank, world, local = dist_env()
    launched = "WORLD_SIZE" in os.environ  # under torchrun (any N)
    if world > 1 or (launched and args.bands):
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    # units of this rank: images (batched configs: no collective on the data path) or a
    # row band of the single image (one all-gather of band tuples per column pass)
    comm = None
    band = None
    scaling = "strong"  # the total work is fixed; N GPUs share it
    if cfg.batch > 1:
        if cfg.batch % world:
            raise SystemExit(f"{cfg.batch} images do not split over {world} ranks")
        per = cfg.batch // world
        images = list(range(rank * per, (rank + 1) * per))
        inputs = [make_inputs(cfg.name, image=i) for i in images]
    elif world > 1 or args.bands:
        import torch.distributed as tdist
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
    pixels_rank = sum(t.shape[0] * t.shape[1] for _, t, _ in inputs)

    stream = torch.cuda.Stream(device=dev)
    dev_in = [tuple(torch.from_numpy(a).to(dev) for a in x) for x in inputs]
    outs = [torch.empty_like(t) for _, t, _ in dev_in]

    def make_ctx(g):
        if band is not None:
            return dts.dts_create_band(g, cfg.H, band[0], band[1] - band[0], cfg.sigma_s, cfg.sigma_r, cfg.N,
                                       comm=comm, stream=stream.cuda_stream)
        return dts.dts_create(g, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=stream.cuda_stream)

    def step_device():
        for (g, t, c), o in zip(dev_in, outs):
            ctx = make_ctx(g)
            dts.dts_solve(ctx, t, c, cfg.lam, cfg.iters, o, stream=stream.cuda_stream)
            dts.dts_destroy(ctx)

    def barrier():
        if world > 1:
            import torch.distributed as tdist
            tdist.barrier()

    def timed(fn, steps):
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            import torch.distributed as tdist
            tt = torch.tensor([ms], device=dev)
            tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs), per-kernel events + clock sampling ----
    dts.dts_profile_enable(0, True)
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    # the library counts its own launches per context; count them for one step
    ms = timed(step_device, args.steps)
    clk = clocks.stop() if clocks else None
    kstats = dts.dts_profile_read(0)
    dts.dts_profile_enable(0, False)
    launches = sum(v["launches"] for v in kstats.values())

    ms_step = ms / args.steps
    mpix_iter_total = pixels_rank * world * cfg.iters / 1e6
    value = mpix_iter_total / (ms_step / 1e3)
    # SURVEY 8(d) defines the metric on dts_solve and reports dts_create separately: the
    # create-time kernels' event time per step, and the solve as the rest of the step
    create_fams = ("guide_deriv", "link_fill", "support_row", "support_col", "edge_profiles")
    create_ms = sum(v["total_ms"] for k, v in kstats.items() if k in create_fams) / args.steps
    solve_ms = ms_step - create_ms
    split = {"create_ms": create_ms, "solve_ms": solve_ms,
             "solve_mpix_iter_per_s": mpix_iter_total / (solve_ms / 1e3),
             "note": "create_ms = event time of the create-time kernels per step (guide derivative with the "
                     "pass-1 column coefficient, support passes); solve_ms = step time minus create_ms"}

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
        e_ms = timed(step_host, max(1, min(args.steps, 3)))
        e_steps = max(1, min(args.steps, 3))
        e2e = {"value": mpix_iter_total / (e_ms / e_steps / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / e_steps,
               "check_max_abs_vs_device": float((host_out[0].to(dev) - outs[0]).abs().max().item())}

    # ---- Eq. (7) confidence on the same guide/target (single image, N = 1) ----
    extras = {}
    if world == 1 and band is None and cfg.batch == 1 and cfg.Ct == 1:
        g0, t0, _ = dev_in[0]
        conf_out = torch.empty_like(t0)
        var_out = torch.empty_like(t0)
        ctx = make_ctx(g0)
        sc = 0.5 * float(t0.max().item() - t0.min().item())  # sigma_c: half the target range (R22)
        dts.dts_confidence(ctx, t0, sc, conf_out, var_out, stream=stream.cuda_stream)  # warm-up
        reps = 3
        c_ms = timed(lambda: dts.dts_confidence(ctx, t0, sc, conf_out, var_out, stream=stream.cuda_stream), reps)
        dts.dts_destroy(ctx)
        c_ms /= reps
        px = t0.numel()
        cbytes = px * (28.0 + 40.0 * cfg.N)  # t in, [t, t^2] out; N x (row + col, C_t = 2); X in, c + V out
        # (on C4 the column passes run plane by plane: +4 B/pixel each, not counted as algorithmic)
        peak_c, _ = measured_peaks()
        extras["confidence"] = {"what": "dts_confidence (Eq. 7): DT(t^2) - DT(t)^2 -> c, same guide", "sigma_c": sc,
                                "ms": c_ms, "mpix_per_s": px / 1e6 / (c_ms / 1e3),
                                "gbs_algorithmic": cbytes / (c_ms / 1e3) / 1e9,
                                "frac": cbytes / (c_ms / 1e3) / 1e9 / peak_c}

    # ---- the box (normalised-convolution) variant on the same workload ----
    if world == 1 and band is None and cfg.batch == 1:
        g0, t0, c0 = dev_in[0]
        bout = torch.empty_like(t0)

        def box_step():
            bctx = dts.dts_create_ex(g0, cfg.sigma_s, cfg.sigma_r, cfg.N, dts.DTS_FILTER_BOX, stream=stream.cuda_stream)
            dts.dts_solve(bctx, t0, c0, cfg.lam, cfg.iters, bout, stream=stream.cuda_stream)
            dts.dts_destroy(bctx)

        box_step()
        dts.dts_profile_enable(0, True)
        b_ms = timed(box_step, 2) / 2
        bstats = dts.dts_profile_read(0)
        dts.dts_profile_enable(0, False)
        peak_b, _ = measured_peaks()
        bpx = t0.shape[0] * t0.shape[1]
        extras["box"] = {"what": "dts_create_ex(DTS_FILTER_BOX) + dts_solve + dts_destroy: the box-window edge-aware "
                                 "mean (reading R25), same guide / target / confidence / iterations",
                         "ms_per_step": b_ms, "mpix_iter_per_s": bpx * cfg.iters / 1e6 / (b_ms / 1e3),
                         "kernels": {}}
        for name in ("box_windows", "box_row", "box_col", "update", "prologue"):
            v = bstats.get(name)
            if v and v["launches"]:
                avg = v["total_ms"] / v["launches"]
                gbs = v["bytes_per_launch"] / (avg / 1e3) / 1e9
                extras["box"]["kernels"][name] = {"launches": v["launches"], "avg_ms": avg, "gbs": gbs,
                                                  "frac": gbs / peak_b}

    # ---- Eq. (10) stereo refinement, C1 shape (single GPU, rank 0) ----
    if world == 1 and band is None:
        c1 = CONFIGS["C1"]
        Lh, th, ch = make_inputs("C1")
        rng = np.random.default_rng(1)
        Rh = (np.roll(Lh, -16, axis=1) + rng.normal(0, 0.01, Lh.shape)).astype(np.float32)
        Ld, Rd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (Lh, Rh, th, ch))
        sout = torch.empty_like(td)
        sctx = dts.dts_create(Ld, c1.sigma_s, c1.sigma_r, c1.N, stream=stream.cuda_stream)
        run = lambda: dts.dts_solve_stereo(sctx, td, cd, c1.lam, c1.iters, sout, Ld, Rd, 0.001, 0.001,  # noqa: E731
                                           stream=stream.cuda_stream)
        run()
        run()  # the second identical call captures the launch sequence as a CUDA graph
        reps = 3
        s_ms = timed(run, reps) / reps
        dts.dts_destroy(sctx)
        spx = c1.H * c1.W
        sbytes = spx * c1.iters * (6 * 12.0 + 20.0 + 12.0 * c1.Cg) + spx * 28.0
        extras["stereo"] = {"what": "dts_solve_stereo (Eq. 10, Charbonnier target, gamma = eps = 0.001) on C1 "
                                    "(1400 x 1000, 3-channel pair: right = left shifted 16 px + noise)",
                            "iterations": c1.iters, "ms": s_ms,
                            "mpix_iter_per_s": spx * c1.iters / 1e6 / (s_ms / 1e3),
                            "gbs_algorithmic": sbytes / (s_ms / 1e3) / 1e9}

    # ---- depth-SR front end, C2 shape (86 x 64 -> 1376 x 1024, f = 16) ----
    if world == 1 and band is None:
        low = torch.rand(64, 86, device=dev) * 9.5 + 0.5
        st_o, sc_o = torch.empty(1024, 1376, device=dev), torch.empty(1024, 1376, device=dev)
        runp = lambda: dts.dts_sr_prepare(low, 16, st_o, sc_o, stream=stream.cuda_stream)  # noqa: E731
        runp()
        p_ms = timed(runp, 10) / 10
        extras["sr_prepare"] = {"what": "dts_sr_prepare: bicubic x16 target + bump confidence, 86x64 -> 1376x1024",
                                "ms": p_ms, "mpix_per_s": 1376 * 1024 / 1e6 / (p_ms / 1e3)}

    if rank != 0:
        if comm:
            dts.dts_comm_destroy(comm)
        import torch.distributed as tdist
        tdist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel ----
    peak, peak_src = measured_peaks()
    fams = {k: v for k, v in kstats.items() if v["launches"] > 0}
    for v in fams.values():
        v["gbs"] = v["bytes_per_launch"] / (v["avg_ms"] / 1e3) / 1e9 if v["avg_ms"] > 0 else 0.0
        v["share_of_step"] = v["total_ms"] / ms if ms > 0 else 0.0
    dom_name = max(fams, key=lambda k: fams[k]["total_ms"])
    dom = fams[dom_name]
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
                "step_gbs_algorithmic": None}
    # whole-step algorithmic bytes / step time
    step_bytes = sum(v["bytes_per_launch"] * v["launches"] for v in fams.values()) / args.steps
    roofline["step_gbs_algorithmic"] = step_bytes / (ms_step / 1e3) / 1e9 * world

    cpu = None
    if not args.no_cpu and world == 1:
        cb = cpu_oracle_sample(cfg)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "pixels": cfg.pixels, "iterations": cfg.iters,
                       "step": "dts_create + dts_solve + dts_destroy (guide derivative, support, prologue, "
                               f"{cfg.iters} x 6 pass kernels)",
                       "l2": "inputs larger than L2 (6.4 GB guide, 0.4 GB per state plane): no flush needed"
                             if cfg.name == "C4" else "L2 not flushed between steps",
                       "parallelism": (f"image split x{world}" if cfg.batch > 1 else
                                       (f"row bands x{world} (NCCL all-gather of column-pass tuples)"
                                        if world > 1 else "single GPU"))},
            "roofline": roofline,
            "kernels": {k: {kk: v[kk] for kk in ("launches", "avg_ms", "bytes_per_launch", "gbs", "share_of_step")}
                        for k, v in fams.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk, "split": split,
            "extras": extras}
    print(json.dumps(line), flush=True)
    if comm:
        dts.dts_comm_destroy(comm)
    if world > 1 or (launched and args.bands):
        import torch.distributed as tdist
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
