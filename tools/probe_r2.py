"""Round-2 probe: (1) where the C1/C2 solve time goes (eager vs graph replay, per-kernel
event time vs wall time), (2) fp32-vs-fp64 divergence of the stereo solve at the paper's
eps = gamma = 0.001.  Prints JSON lines."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs, target_range  # noqa: E402

torch.cuda.set_device(0)
out = {}


def timing(name):
    cfg = CONFIGS[name]
    g, t, c = make_inputs(name)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    o = torch.empty_like(td)
    s = torch.cuda.Stream()
    res = {}
    with torch.cuda.stream(s):
        ctx = dts.dts_create(gd, cfg.sigma_s, cfg.sigma_r, cfg.N, stream=s.cuda_stream)
        torch.cuda.synchronize()
        for label in ("first", "second", "replay1", "replay2"):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            t0 = time.perf_counter()
            e0.record(s)
            dts.dts_solve(ctx, td, cd, cfg.lam, cfg.iters, o, stream=s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            res[label + "_ms"] = e0.elapsed_time(e1)
            res[label + "_host_ms"] = 1e3 * (time.perf_counter() - t0)
        dts.dts_profile_enable(0, True)
        dts.dts_solve(ctx, td, cd, cfg.lam, cfg.iters, o, stream=s.cuda_stream)
        st = dts.dts_profile_read(0)
        dts.dts_profile_enable(0, False)
        res["kernels"] = {k: {"n": v["launches"], "avg_us": 1e3 * v["avg_ms"]} for k, v in st.items() if v["launches"]}
        res["kernel_sum_ms"] = sum(v["total_ms"] for v in st.values())
        dts.dts_destroy(ctx)
    px = cfg.H * cfg.W
    res["mpix_iter_first"] = px * cfg.iters / 1e6 / (res["first_ms"] / 1e3)
    res["mpix_iter_replay"] = px * cfg.iters / 1e6 / (res["replay2_ms"] / 1e3)
    return res


for name in ("C1", "C2"):
    out[name] = timing(name)
    print(json.dumps({name: out[name]}), flush=True)


# stereo divergence at the paper's constants
def right_image(L, shift, seed):
    rng = np.random.default_rng(seed)
    R = np.roll(L, -shift, axis=1) + rng.normal(0, 0.01, L.shape)
    return np.ascontiguousarray(R.astype(np.float32))


cfg = CONFIGS["C1"]
L, t, c = make_inputs("C1")
R = right_image(L, 16, 1)
rng_t = target_range(t)
Ld, Rd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (L, R, t, c))
res = {}
for iters in (1, 2, 5, 10, 20, 50):
    for eps in (1.0, 0.1, 0.01, 0.001):
        o = torch.empty_like(td)
        with dts.Solver(Ld, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
            s.solve_stereo(td, cd, cfg.lam, iters, Ld, Rd, 0.001, eps, out=o)
        torch.cuda.synchronize()
        got = o.cpu().numpy().astype(np.float64)
        ref = oracle.solve_stereo(L, R, t, c, cfg.sigma_s, cfg.sigma_r, cfg.N, cfg.lam, iters, 0.001, eps)
        d = np.abs(got - ref)
        res[f"it{iters}_eps{eps}"] = {"max": float(d.max()), "max_over_range": float(d.max() / rng_t),
                                     "p999": float(np.quantile(d, 0.999)), "p99": float(np.quantile(d, 0.99)),
                                     "n_over_tol": int(np.sum(d > 1e-4 * rng_t)),
                                     "tol": 1e-4 * rng_t}
        print(json.dumps({f"stereo_it{iters}_eps{eps}": res[f"it{iters}_eps{eps}"]}), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/probe_r2.json", "w") as f:
    json.dump({"timing": out, "stereo": res}, f, indent=1)
