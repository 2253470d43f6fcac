"""Phase timeline of the SMEM-resident kernel (one CTA's %globaltimer stamps, first iteration)."""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts
from synth import CONFIGS, make_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = CONFIGS[name]
g, t, c = make_inputs(name)
gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
lib = dts.load_library()
lib.dts_debug_resident_timers.argtypes = [ctypes.c_void_p, ctypes.c_int32]
buf = torch.zeros(128, dtype=torch.int64, device="cuda")
o = torch.empty_like(td)
with dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
    s.solve(td, cd, cfg.lam, 2, out=o)
    torch.cuda.synchronize()
    lib.dts_debug_resident_timers(buf.data_ptr(), cta)
    s.solve(td, cd, cfg.lam, 2, out=o)
    torch.cuda.synchronize()
    lib.dts_debug_resident_timers(None, 0)
ts = buf.cpu().numpy().astype(np.int64)
names = {0: "load"}
lab = ["rowC fold", "pub", "comp", "rowA fold", "pub", "comp", "colC fold", "pub", "comp", "colA fold", "pub", "comp", "apply"]
out = []
prev = ts[0]
for i in range(3):
    for j, l in enumerate(lab):
        v = ts[1 + 16 * i + j]
        if v:
            out.append([f"p{i} {l}", round((v - prev) / 1e3, 2)])
            prev = v
if ts[63]:
    out.append(["update", round((ts[63] - prev) / 1e3, 2)])
print(json.dumps({"cfg": name, "cta": cta, "iteration_us": round((ts[63] - ts[0]) / 1e3, 2), "sm_ghz": float((ts[127] - ts[64]) / max(1, ts[63] - ts[0])), "timeline_us": out}))
