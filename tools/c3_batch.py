"""C3 (8 x 4K, C_t = 3) in one batched context: solve time and per-kernel averages, for each
forced strip cluster size given on the command line (0 = the automatic plan).
Usage: python tools/c3_batch.py [cb ...]  (also the launch sequence the C3 ncu captures read)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402

cfg = CONFIGS["C3"]
iters = int(os.environ.get("C3_ITERS", cfg.iters))
host = [make_inputs("C3", image=i) for i in range(cfg.batch)]
g, t, c = (torch.from_numpy(np.ascontiguousarray(np.stack([h[j] for h in host]))).cuda() for j in range(3))
o = torch.empty_like(t)
for cb in [int(a) for a in sys.argv[1:]] or [0]:
    with dts.options(strip_cluster=cb, col_rows=int(os.environ.get("COL_ROWS", "0")),
                     row_two_ctas=int(os.environ.get("ROW_TWO", "1")), pdl=int(os.environ.get("PDL", "1"))):
      try:
        with dts.Solver(g, cfg.sigma_s, cfg.sigma_r, cfg.N, batched=True) as s:
            s.solve(t, c, cfg.lam, iters, out=o)
            plan = dts.debug_col_plan(s.ctx, 3)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(3):
                s.solve(t, c, cfg.lam, iters, out=o)
            e1.record()
            torch.cuda.synchronize()
            dts.dts_profile_enable(s.ctx, True)
            s.solve(t, c, cfg.lam, iters, out=o)
            torch.cuda.synchronize()
            prof = {k: round(v["total_ms"] / max(v["launches"], 1), 4) for k, v in dts.dts_profile_read(s.ctx).items()
                    if v["launches"]}
      except dts.DTSError as ex:
        print(json.dumps({"cb": cb, "error": str(ex)}))
        continue
    print(json.dumps({"cb": cb, "plan": plan, "solve_ms": e0.elapsed_time(e1) / 3,
                      "mpix_iter_per_s": cfg.pixels * iters / 1e3 / (e0.elapsed_time(e1) / 3), "avg_ms": prof}))
