"""Solve time of the small (paper-shaped) configs: the SMEM-resident kernel against the per-pass
kernels (eager first solve and graph replay), profiler off.  One JSON line per config."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402

torch.cuda.set_device(0)
for name in sys.argv[1:] or ["C0", "C1", "C2"]:
    cfg = CONFIGS[name]
    g, t, c = make_inputs(name)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    o = torch.empty_like(td)
    res = {"config": name}
    for resident in (1, 0):
        with dts.options(resident=resident), dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
            times = []
            for _ in range(4):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                torch.cuda.synchronize()
                e0.record()
                s.solve(td, cd, cfg.lam, cfg.iters, out=o)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
        key = "resident" if resident else "per_pass"
        res[key + "_ms"] = [round(x, 4) for x in times]
        res[key + "_mpix_iter_first"] = cfg.H * cfg.W * cfg.iters / 1e6 / (times[0] / 1e3)
        res[key + "_mpix_iter_best"] = cfg.H * cfg.W * cfg.iters / 1e6 / (min(times) / 1e3)
    print(json.dumps(res), flush=True)
