# C4 unprofiled solve time (20 iterations) for strip configurations "strips:cluster" (0:0 = unstripped)
for cfg in ${CFGS:-0:0 2:0 4:4 16:0}; do set -- ${cfg/:/ }
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
ts = []
with dts.Solver(g, 64.0, 0.2, 3) as s:
    info = dts.debug_strips(s.ctx)
    s.solve(t, c, 0.99, 20, out=o); torch.cuda.synchronize()
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); s.solve(t, c, 0.99, 20, out=o); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
print(json.dumps({"strips": $1, "cb": $2, "plan": info, "solve20_ms": sorted(ts)}))
PY
done
