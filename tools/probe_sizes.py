"""Dev probe: column plan, row strips and first-solve time across image sizes (3-channel guide,
C_t = 1, 20 iterations), as extras.sweeps.pixels in bench.py; per-kernel averages."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402

sizes = [(500, 700), (1000, 1400), (2000, 2800), (3000, 4200), (4000, 5600), (5000, 7000), (7071, 10000),
         (10000, 10000)]
if len(sys.argv) > 1:  # "HxW[xCt] ..." on the command line
    sizes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for sz in sizes:
    H, W = sz[0], sz[1]
    Ct = sz[2] if len(sz) > 2 else 1
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    g = torch.rand(H, W, 3, device="cuda", generator=gen) * 0.05
    g[H // 3:, W // 3:, :] += 0.5
    t = torch.rand(H, W, Ct, device="cuda", generator=gen) if Ct > 1 else torch.rand(H, W, device="cuda", generator=gen)
    c = torch.rand(H, W, device="cuda", generator=gen)
    o = torch.empty_like(t)
    NP = int(os.environ.get("NPASS", "3"))
    SS = float(os.environ.get("SIGMA_S", "16"))
    with dts.Solver(g, SS, 0.1, NP) as s:
        s.solve(t, c, 0.99, 20, out=o)
    with dts.options(graphs=0, row_seg=int(os.environ.get("ROW_SEG", "0")),
                     col_split=int(os.environ.get("COL_SPLIT", "0")),
                     col_rows=int(os.environ.get("COL_ROWS", "0"))), dts.Solver(g, SS, 0.1, NP) as s:
        s.solve(t, c, 0.99, 20, out=o)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        s.solve(t, c, 0.99, 20, out=o)
        e1.record()
        torch.cuda.synchronize()
        plan = dts.debug_col_plan(s.ctx, Ct)
        st = dts.debug_strips(s.ctx)
        dts.dts_profile_enable(s.ctx, 1)
        s.solve(t, c, 0.99, 20, out=o)
        torch.cuda.synchronize()
        prof = {k: round(1e3 * v["avg_ms"], 1) for k, v in dts.dts_profile_read(s.ctx).items() if v["launches"]}
    ms = e0.elapsed_time(e1)
    print(json.dumps({"HxW": f"{H}x{W}x{Ct}", "ms": round(ms, 3), "mpix_iter_per_s": round(H * W * 20 / 1e3 / ms),
                      "plan": plan, "strips": st, "avg_us": prof}), flush=True)
