# column pass + seam fix-up time on C4 for each strip count (1 = auto plan)
for n in 1 4 8 16 32; do
python - << PY
import os, sys, json, ctypes
import torch
sys.path.insert(0, os.getcwd())
import paper_1805_04590_b200 as dts
lib = dts.load_library()
dts.dts_set_option("col_strips", $n)
H, W, C = 10000, 10000, 16
torch.manual_seed(0)
g = (torch.rand(H, W, C, device="cuda") * 0.05).contiguous(); g[H // 3:, W // 3:, :] += 0.5
t = torch.rand(H, W, device="cuda"); c = torch.rand(H, W, device="cuda"); o = torch.empty_like(t)
lib.dts_debug_strips.restype = ctypes.c_int32
lib.dts_debug_strips.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int32)] * 4
with dts.Solver(g, 64.0, 0.2, 3) as s:
    s.solve(t, c, 0.99, 4, out=o); torch.cuda.synchronize()
    dts.dts_profile_enable(s.ctx, 1); s.solve(t, c, 0.99, 4, out=o); st = dts.dts_profile_read(s.ctx); dts.dts_profile_enable(s.ctx, 0)
    hs, cb, gr = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(); L3 = (ctypes.c_int32 * 3)()
    nst = lib.dts_debug_strips(s.ctx, ctypes.byref(hs), L3, ctypes.byref(cb), ctypes.byref(gr))
col = 1e3 * st["col_pass"]["avg_ms"]; sf = 1e3 * st["seam_fix"]["avg_ms"] if st["seam_fix"]["launches"] else 0.0
print(json.dumps({"opt": $n, "strips": nst, "HS": hs.value, "L": list(L3), "CB": cb.value, "grid": gr.value,
                  "col_us": round(col, 1), "seam_us": round(sf, 1), "sum_us": round(col + sf, 1)}))
PY
done
