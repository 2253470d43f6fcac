import os, sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1805_04590_b200 as dts
from synth import CONFIGS, make_inputs
c1 = CONFIGS["C1"]
Lh, th, ch = make_inputs("C1")
Rh = (np.roll(Lh, -16, axis=1) + np.random.default_rng(1).normal(0, 0.01, Lh.shape)).astype(np.float32)
Ld, Rd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (Lh, Rh, th, ch))
out = torch.empty_like(td)
with dts.Solver(Ld, c1.sigma_s, c1.sigma_r, c1.N) as s:
    for _ in range(3):
        s.solve_stereo(td, cd, c1.lam, c1.iters, Ld, Rd, 0.001, 0.001, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        s.solve_stereo(td, cd, c1.lam, c1.iters, Ld, Rd, 0.001, 0.001, out=out)
    e1.record(); torch.cuda.synchronize()
    print(os.environ.get("DTS_NO_GRAPH", "graph"), f"{e0.elapsed_time(e1)/5:.3f} ms per C1 stereo solve (50 iterations)")
