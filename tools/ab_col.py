"""Dev A/B probe: alternate a library option between solves on ONE context (same box, same
process, same data) and report the per-kernel averages of each setting (library profiler on,
graphs off).  Usage: OPT=col_vst VALS=0,1 REPS=4 python tools/ab_col.py [C4|C3|C1]
The shapes are the bench's configs (synth inputs; C3: the batched 8-image context)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
opt = os.environ.get("OPT", "col_vst")
vals = [int(v) for v in os.environ.get("VALS", "0,1").split(",")]
reps = int(os.environ.get("REPS", "4"))
iters = int(os.environ.get("ITERS", "4"))
cfg = CONFIGS[name]
batched = cfg.batch > 1
if batched:
    host = [make_inputs(name, image=i) for i in range(cfg.batch)]
    g, t, c = (torch.from_numpy(np.ascontiguousarray(np.stack([h[j] for h in host]))).cuda() for j in range(3))
else:
    g, t, c = (torch.from_numpy(a).cuda() for a in make_inputs(name))
outs = {v: torch.empty_like(t) for v in vals}
acc = {v: {} for v in vals}
wall = {v: [] for v in vals}
with dts.options(graphs=0), dts.Solver(g, cfg.sigma_s, cfg.sigma_r, cfg.N, batched=batched) as s:
    s.solve(t, c, cfg.lam, iters, out=outs[vals[0]])
    for r in range(reps):
        for v in vals:
            dts.dts_set_option(opt, v)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            s.solve(t, c, cfg.lam, iters, out=outs[v])
            e1.record()
            torch.cuda.synchronize()
            wall[v].append(e0.elapsed_time(e1))
            dts.dts_profile_enable(s.ctx, 1)
            s.solve(t, c, cfg.lam, iters, out=outs[v])
            torch.cuda.synchronize()
            for k, d in dts.dts_profile_read(s.ctx).items():
                if d["launches"]:
                    acc[v].setdefault(k, []).append(1e3 * d["avg_ms"])
            dts.dts_profile_enable(s.ctx, 0)
diff = float((outs[vals[0]] - outs[vals[-1]]).abs().max())
for v in vals:
    print(json.dumps({"opt": opt, "val": v, "solve_ms_median": round(float(np.median(wall[v])), 3),
                      "avg_us_median": {k: round(float(np.median(x)), 1) for k, x in acc[v].items()},
                      "max_abs_diff_first_last": diff}), flush=True)
