# C4 pass times: unstripped, strips + separate seam fix-up, strips with the fix-up fused into the next kernel
for cfg in "0 0" "1 0" "1 1"; do set -- $cfg
python - << PY
import os, sys, json
import torch
sys.path.insert(0, os.getcwd())
import paper_1805_04590_b200 as dts
dts.load_library()
dts.dts_set_option("col_strips", $1); dts.dts_set_option("col_strips_fused", $2)
H, W, C = 10000, 10000, 16
torch.manual_seed(0)
g = (torch.rand(H, W, C, device="cuda") * 0.05).contiguous(); g[H // 3:, W // 3:, :] += 0.5
t = torch.rand(H, W, device="cuda"); c = torch.rand(H, W, device="cuda"); o = torch.empty_like(t)
with dts.Solver(g, 64.0, 0.2, 3) as s:
    s.solve(t, c, 0.99, 4, out=o); torch.cuda.synchronize()
    dts.dts_profile_enable(s.ctx, 1); s.solve(t, c, 0.99, 4, out=o); st = dts.dts_profile_read(s.ctx); dts.dts_profile_enable(s.ctx, 0)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); s.solve(t, c, 0.99, 20, out=o); e1.record(); torch.cuda.synchronize()
res = {"strips": $1, "fused": $2, "solve20_ms": round(e0.elapsed_time(e1), 3)}
for k in ("row_pass", "col_pass", "row_update", "seam_fix", "update"):
    if st[k]["launches"]: res[k] = round(1e3 * st[k]["avg_ms"], 1)
print(json.dumps(res))
PY
done
