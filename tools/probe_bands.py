"""Dev probe: a C4-sized problem split into P row bands (loopback ranks on one GPU), one
solve, library profiler per kernel family.  P=2 by default; DTS_BAND_LEGACY=1 selects the
decoupled band-tuple kernel for the banded column passes."""
import os
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402

H = int(os.environ.get("H", 10000))
W = int(os.environ.get("W", 10000))
P = int(os.environ.get("P", 2))
iters = int(os.environ.get("ITERS", 2))
torch.manual_seed(0)
g = (torch.rand(H, W, 16, device="cuda") * 0.05).contiguous()
t = torch.rand(H, W, device="cuda")
c = torch.rand(H, W, device="cuda")
comms = dts.dts_comm_init_loopback(P)


def run(r, prof):
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    r0, r1 = dts.band_rows(H, P, r)
    a, b = dts.band_guide_rows(H, r0, r1)
    ctx = dts.dts_create_band(g[a:b].contiguous(), H, r0, r1 - r0, 64.0, 0.2, 3, comm=comms[r],
                              stream=stream.cuda_stream)
    out = torch.empty(r1 - r0, W, device="cuda")
    dts.dts_solve(ctx, t[r0:r1].contiguous(), c[r0:r1].contiguous(), 0.99, iters, out, stream=stream.cuda_stream)
    stream.synchronize()
    dts.dts_destroy(ctx)


for prof in (False, True):
    if prof:
        dts.dts_profile_enable(0, True)
    ths = [threading.Thread(target=run, args=(r, prof)) for r in range(P)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
st = dts.dts_profile_read(0)
for k, v in st.items():
    if v["launches"]:
        print(k, v["launches"], round(v["avg_ms"], 4))
