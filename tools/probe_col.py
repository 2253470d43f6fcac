"""Dev probe: time one DTS solve on a C4-sized device-generated problem, per kernel family
(library profiler).  Set DTS_COLV_DEBUG=1 for the streaming column kernel's phase timers."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402

H = int(os.environ.get("H", 10000))
W = int(os.environ.get("W", 10000))
C = int(os.environ.get("C", 16))
Ct = int(os.environ.get("CT", 1))
iters = int(os.environ.get("ITERS", 2))
torch.manual_seed(0)
g = (torch.rand(H, W, C, device="cuda") * 0.05).contiguous()
g[H // 3:, W // 3:, :] += 0.5
t = torch.rand(H, W, Ct, device="cuda").squeeze(-1).contiguous() if Ct > 1 else torch.rand(H, W, device="cuda")
c = torch.rand(H, W, device="cuda")
out = torch.empty_like(t)
with dts.Solver(g, 64.0, 0.2, 3) as s:
    s.solve(t, c, 0.99, iters, out=out)
    torch.cuda.synchronize()
    dts.dts_profile_enable(s.ctx, 1)
    t0 = time.time()
    s.solve(t, c, 0.99, iters, out=out)
    torch.cuda.synchronize()
    print(f"solve {1e3 * (time.time() - t0):.2f} ms wall")
    for k, v in dts.dts_profile_read(s.ctx).items():
        print(k, v)
