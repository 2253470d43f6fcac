"""One C1-shaped SMEM-resident solve (for ncu): create, 1 warm-up solve, 1 profiled solve."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts
from synth import CONFIGS, make_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = CONFIGS[name]
g, t, c = make_inputs(name)
gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
o = torch.empty_like(td)
with dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
    s.solve(td, cd, cfg.lam, iters, out=o)
    s.solve(td, cd, cfg.lam, iters, out=o)
torch.cuda.synchronize()
print("ok")
