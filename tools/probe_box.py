"""Dev probe: one box-variant solve on the C4 workload (for ncu captures of k_box_row /
k_box_col).  python tools/probe_box.py [iterations]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = CONFIGS["C4"]
g, t, c = (torch.from_numpy(a).cuda() for a in make_inputs("C4"))
out = torch.empty_like(t)
with dts.Solver(g, cfg.sigma_s, cfg.sigma_r, cfg.N, filter=dts.DTS_FILTER_BOX) as s:
    s.solve(t, c, cfg.lam, iters, out=out)
    torch.cuda.synchronize()
    dts.dts_profile_enable(0, True)
    s.solve(t, c, cfg.lam, iters, out=out)
    st = dts.dts_profile_read(0)
    for k, v in st.items():
        if v["launches"]:
            print(k, v["launches"], round(v["avg_ms"], 4))
print("ok")
