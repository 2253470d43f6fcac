"""Dev probe: dts_confidence on a C4-shaped problem (10000 x 10000, 16-channel guide) with the
library profiler on: per-family launches and averages."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402

PEAK = 6466.1
H = W = 10000
torch.manual_seed(0)
g = (torch.rand(H, W, 16, device="cuda") * 0.05).contiguous()
g[H // 3:, W // 3:, :] += 0.5
t = torch.rand(H, W, device="cuda")
c = torch.empty_like(t)
with dts.Solver(g, 64.0, 0.2, 3) as s:
    s.confidence(t, 1.0, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3):
        s.confidence(t, 1.0, out=c)
    e1.record()
    torch.cuda.synchronize()
    dts.dts_profile_enable(s.ctx, 1)
    s.confidence(t, 1.0, out=c)
    torch.cuda.synchronize()
    res = {"ms": e0.elapsed_time(e1) / 3}
    for k, v in dts.dts_profile_read(s.ctx).items():
        if v["launches"]:
            gbs = v["bytes_per_launch"] / (v["avg_ms"] / 1e3) / 1e9
            res[k] = {"n": v["launches"], "avg_us": round(1e3 * v["avg_ms"], 2), "frac": round(gbs / PEAK, 4)}
print(json.dumps(res))
