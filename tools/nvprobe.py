import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, paper_1805_04590_b200 as dts
from synth import random_problem, target_range
for (H, W, Ct) in [(64, 64, 2), (448, 64, 2), (449, 64, 2), (900, 64, 2), (1200, 64, 2), (1200, 64, 1), (1200, 32, 2), (600, 33, 3)]:
    g, t, c = random_problem(H, W, 3, Ct, seed=H + W)
    ref = oracle.solve(g, t, c, 6.0, 0.15, 3, 0.99, 2)
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    with dts.Solver(gd, 6.0, 0.15, 3) as s:
        s.solve(td, cd, 0.99, 2, out=out)
    o = out.cpu().numpy()
    err = np.abs(o - ref)
    idx = np.unravel_index(np.argmax(err), err.shape)
    print(H, W, Ct, "err/range", err.max() / target_range(t), "at", idx)
