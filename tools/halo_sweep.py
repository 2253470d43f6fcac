"""Dev probe: halo strips vs seam strips on the bench's C4 (or C3 batched) inputs.
Usage: CONFIG=C4|C3 python tools/halo_sweep.py halo:n:cb ...
  halo 1 = halo strips, 0 = seam strips (+ fix-up); n: 0 none, 1 auto, >= 2 forced strips (C4:
  per image; C3: per image of the batch); cb: forced strip cluster size (0 auto).
Prints per configuration the column plan, the strips, the median of 3 unprofiled 20-iteration
(C3: 30) solves with graphs off, the profiled per-kernel averages and the max |difference| from
the unstripped solve."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402

name = os.environ.get("CONFIG", "C4")
cfg = CONFIGS[name]
iters = int(os.environ.get("ITERS", cfg.iters))
batched = cfg.batch > 1
if batched:
    host = [make_inputs(name, image=i) for i in range(cfg.batch)]
    g, t, c = (torch.from_numpy(np.ascontiguousarray(np.stack([h[j] for h in host]))).cuda() for j in range(3))
else:
    g, t, c = (torch.from_numpy(a).cuda() for a in make_inputs(name))
Ct = 1 if t.dim() == (3 if batched else 2) else t.shape[-1]
ref = None


def run(halo, n, cb):
    opts = dict(graphs=0, col_halo=halo, strip_cluster=cb, col_rows=int(os.environ.get("COL_ROWS", "0")))
    if batched:
        opts["batch_strips"] = n
    else:
        opts["col_strips"] = n
    o = torch.empty_like(t)
    with dts.options(**opts), dts.Solver(g, cfg.sigma_s, cfg.sigma_r, cfg.N, batched=batched) as s:
        s.solve(t, c, cfg.lam, iters, out=o)
        plan = dts.debug_col_plan(s.ctx, Ct)
        st = dts.debug_strips(s.ctx)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            s.solve(t, c, cfg.lam, iters, out=o)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        dts.dts_profile_enable(s.ctx, True)
        s.solve(t, c, cfg.lam, iters, out=o)
        torch.cuda.synchronize()
        prof = {k: round(1e3 * v["total_ms"] / max(v["launches"], 1), 1) for k, v in dts.dts_profile_read(s.ctx).items()
                if v["launches"]}
    return o, plan, st, sorted(ts)[1], prof


ref, *_ = run(1, 0, 0)
rng = float(t.max() - t.min())
for a in sys.argv[1:]:
    halo, n, cb = (int(v) for v in a.split(":"))
    try:
        o, plan, st, ms, prof = run(halo, n, cb)
    except dts.DTSError as ex:
        print(json.dumps({"cfg": a, "error": str(ex)}), flush=True)
        continue
    err = float((o - ref).abs().max()) / rng
    print(json.dumps({"cfg": a, "plan": plan, "strips": st, "solve_ms": round(ms, 3),
                      "mpix_iter_per_s": round(cfg.pixels * iters / 1e3 / ms), "err_over_range": err,
                      "avg_us": prof}), flush=True)
