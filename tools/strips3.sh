# C4: column pass + separate seam fix-up for (strips, forced cluster size)
for cfg in ${CFGS:-8:4 16:0 4:4}; do set -- ${cfg/:/ }
python - << PY
import os, sys, json
import torch
sys.path.insert(0, os.getcwd())
import paper_1805_04590_b200 as dts
dts.load_library()
dts.dts_set_option("col_strips", $1); dts.dts_set_option("strip_cluster", $2)
H, W, C = 10000, 10000, 16
torch.manual_seed(0)
g = (torch.rand(H, W, C, device="cuda") * 0.05).contiguous(); g[H // 3:, W // 3:, :] += 0.5
t = torch.rand(H, W, device="cuda"); c = torch.rand(H, W, device="cuda"); o = torch.empty_like(t)
with dts.Solver(g, 64.0, 0.2, 3) as s:
    info = dts.debug_strips(s.ctx)
    s.solve(t, c, 0.99, 4, out=o); torch.cuda.synchronize()
    dts.dts_profile_enable(s.ctx, 1); s.solve(t, c, 0.99, 4, out=o); st = dts.dts_profile_read(s.ctx); dts.dts_profile_enable(s.ctx, 0)
res = {"strips": $1, "cb": $2, **info}
for k in ("col_pass", "seam_fix"):
    if st[k]["launches"]: res[k] = round(1e3 * st[k]["avg_ms"], 1)
res["sum"] = round(res.get("col_pass", 0) + res.get("seam_fix", 0), 1)
print(json.dumps(res))
PY
done
