"""One eager C1 solve after a warm-up solve (graphs off): the launch sequence profiles/ reads for
the C1 launch-gap breakdown.  Prints the event-timed solve."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts
from synth import CONFIGS, make_inputs
cfg = CONFIGS["C1"]
g, t, c = make_inputs("C1")
gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
o = torch.empty_like(td)
with dts.options(graphs=0), dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
    s.solve(td, cd, cfg.lam, cfg.iters, out=o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    s.solve(td, cd, cfg.lam, cfg.iters, out=o)
    e1.record()
    torch.cuda.synchronize()
print(json.dumps({"c1_eager_solve_ms": e0.elapsed_time(e1), "launches": 1 + 6 * cfg.iters + 1}))
