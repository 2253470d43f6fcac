"""Dev check (env HMIN/HMAX/WMIN/WMAX: the shape ranges): random shapes / channel counts / pass counts / option sets against the fp64 oracle
(the tests' tolerance 1e-4 x range).  Usage: python tools/random_parity.py [cases] [seed]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1805_04590_b200 as dts  # noqa: E402
from synth import random_problem, target_range  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
worst, bad = 0.0, 0
for k in range(cases):
    H = int(rng.integers(int(os.environ.get("HMIN", 1)), int(os.environ.get("HMAX", 700))))
    W = int(rng.integers(int(os.environ.get("WMIN", 1)), int(os.environ.get("WMAX", 700))))
    Ct = int(rng.integers(1, 5))
    Cg = int(rng.choice([1, 3, 4, 8]))
    N = int(rng.integers(1, 5))
    ss = float(rng.choice([2.0, 6.0, 20.0, 64.0]))
    sr = float(rng.choice([0.05, 0.2, 1.0]))
    it = int(rng.integers(0, 6))
    opts = {"col_oop": int(rng.integers(0, 3)), "col_rows": int(rng.choice([0, 0, 12, 16, 32]))}
    if Ct != 3 and opts["col_rows"] in (12, 16):
        opts["col_rows"] = 0
    g, t, c = random_problem(H, W, Cg, Ct, seed=1000 + k)
    ref = oracle.solve(g, t, c, ss, sr, N, 0.99, it)
    gd, td, cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (g, t, c))
    out = torch.empty_like(td)
    try:
        with dts.options(**opts), dts.Solver(gd, ss, sr, N) as s:
            s.solve(td, cd, 0.99, it, out=out)
        torch.cuda.synchronize()
    except dts.DTSError as ex:
        print(f"case {k}: {H}x{W} Cg={Cg} Ct={Ct} N={N} opts={opts}: {ex}", flush=True)
        bad += 1
        continue
    err = float(np.max(np.abs(out.cpu().numpy().astype(np.float64) - ref))) / max(target_range(t), 1e-30)
    worst = max(worst, err)
    flag = "" if err <= 1e-4 else "  <-- FAIL"
    if flag:
        bad += 1
    print(f"case {k}: {H}x{W} Cg={Cg} Ct={Ct} N={N} ss={ss} sr={sr} it={it} opts={opts}: err/range {err:.2e}{flag}",
          flush=True)
print(f"{cases} cases, {bad} failures, worst err/range {worst:.2e}")
