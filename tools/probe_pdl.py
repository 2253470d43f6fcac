"""Dev probe: programmatic dependent launch trigger placement (option pdl: 0 off, 1 auto, 2 at the
kernel start, 3 at the end) across image sizes (3-channel guide, C_t = 1, 20 iterations): median
of three eager solves after a warm-up on the same context, and the first solve of a fresh one."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402

dts.dts_set_option("graphs", 0)
sizes = [(1000, 1400), (2000, 2800), (4000, 5600), (7071, 10000), (10000, 10000)]
for H, W in sizes:
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    g = torch.rand(H, W, 3, device="cuda", generator=gen) * 0.05
    g[H // 3:, W // 3:, :] += 0.5
    t = torch.rand(H, W, device="cuda", generator=gen)
    c = torch.rand(H, W, device="cuda", generator=gen)
    o = torch.empty_like(t)
    res = {"HxW": f"{H}x{W}"}
    for mode in (0, 1, 2):
        dts.dts_set_option("pdl", mode)
        ctx = dts.dts_create(g, 16.0, 0.1, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        dts.dts_solve(ctx, t, c, 0.99, 20, o)
        e1.record()
        torch.cuda.synchronize()
        first = e0.elapsed_time(e1)
        ts = []
        for _ in range(3):
            e0.record()
            dts.dts_solve(ctx, t, c, 0.99, 20, o)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        dts.dts_destroy(ctx)
        res[f"pdl{mode}"] = {"first": round(first, 3), "median": round(sorted(ts)[1], 3)}
    dts.dts_set_option("pdl", 1)
    print(json.dumps(res), flush=True)
    del g, t, c, o
