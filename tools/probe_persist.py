"""Phase timeline of the persistent solve kernel (block 0's %globaltimer stamps) on C1."""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts
from synth import CONFIGS, make_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = CONFIGS[name]
g, t, c = make_inputs(name)
gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
lib = dts.load_library()
buf = torch.zeros(4096, dtype=torch.int64, device="cuda")
lib.dts_debug_persist_timers.argtypes = [ctypes.c_void_p]
o = torch.empty_like(td)
with dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
    s.solve(td, cd, cfg.lam, iters, out=o)
    torch.cuda.synchronize()
    lib.dts_debug_persist_timers(buf.data_ptr())
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); s.solve(td, cd, cfg.lam, iters, out=o); e1.record(); torch.cuda.synchronize()
    lib.dts_debug_persist_timers(None)
ts = buf.cpu().numpy()
n = 1 + iters * cfg.N * 4
d = np.diff(ts[:n]) / 1e3
lab = ["row", "bar", "col", "bar"]
rows = [[lab[j % 4], round(float(x), 2)] for j, x in enumerate(d)]
print(json.dumps({"name": name, "iters": iters, "solve_ms": e0.elapsed_time(e1), "phases_us": rows[:24],
                  "mean_us": {l: float(np.mean(d[j::4])) for j, l in enumerate(lab[:2])} | {"col": float(np.mean(d[2::4])), "bar2": float(np.mean(d[3::4]))}}))
sub = ts[3000:3007]
print(json.dumps({"col_sub_us": [round(float(x), 2) for x in np.diff(sub) / 1e3], "labels": ["fold", "scan", "pubwaitC", "apply+fold", "pubwaitA", "apply+store"],
                  "col_start_after_kernel_start_us": float((sub[0] - ts[0]) / 1e3)}))
