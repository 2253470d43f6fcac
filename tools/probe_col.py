"""Dev probe: per-kernel-family times of a DTS solve on device-generated problems shaped like C4
(10000 x 10000, 16-channel guide, C_t = 1) and one C3 image (3840 x 2160, C_t = 3), library
profiler on.  Prints one JSON line per shape."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts  # noqa: E402

PEAK = 6466.1
shapes = {"C4": (10000, 10000, 16, 1, 64.0, 0.2), "C3": (2160, 3840, 3, 3, 24.0, 0.15)}
iters = int(os.environ.get("ITERS", 4))
for name in (sys.argv[1:] or ["C4", "C3"]):
    H, W, C, Ct, ss, sr = shapes[name]
    torch.manual_seed(0)
    g = (torch.rand(H, W, C, device="cuda") * 0.05).contiguous()
    g[H // 3:, W // 3:, :] += 0.5
    t = torch.rand(H, W, Ct, device="cuda").contiguous() if Ct > 1 else torch.rand(H, W, device="cuda")
    c = torch.rand(H, W, device="cuda")
    out = torch.empty_like(t)
    res = {"shape": name}
    with dts.Solver(g, ss, sr, 3) as s:
        s.solve(t, c, 0.99, iters, out=out)
        torch.cuda.synchronize()
        dts.dts_profile_enable(s.ctx, 1)
        s.solve(t, c, 0.99, iters, out=out)
        torch.cuda.synchronize()
        for k, v in dts.dts_profile_read(s.ctx).items():
            if v["launches"]:
                gbs = v["bytes_per_launch"] / (v["avg_ms"] / 1e3) / 1e9
                res[k] = {"n": v["launches"], "avg_us": round(1e3 * v["avg_ms"], 2), "frac": round(gbs / PEAK, 4)}
        dts.dts_profile_enable(s.ctx, 0)
    print(json.dumps(res), flush=True)
    import ctypes
    lib = dts.load_library()
    lib.dts_debug_strips.restype = ctypes.c_int32
    lib.dts_debug_strips.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int32)] * 4
    hs, cb, gr = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    L3 = (ctypes.c_int32 * 3)()
    with dts.Solver(g, ss, sr, 3) as s2:
        nst = lib.dts_debug_strips(s2.ctx, ctypes.byref(hs), L3, ctypes.byref(cb), ctypes.byref(gr))
    print(json.dumps({"strips": nst, "HS": hs.value, "L": list(L3), "CB": cb.value, "grid": gr.value}), flush=True)
