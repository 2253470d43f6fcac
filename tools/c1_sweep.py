"""C1 / C2 solve time (first eager solve and graph replay) for column-kernel cluster sizes."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts
from synth import CONFIGS, make_inputs
torch.cuda.set_device(0)
for name in ("C1", "C2"):
    cfg = CONFIGS[name]
    g, t, c = make_inputs(name)
    gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
    o = torch.empty_like(td)
    dts.dts_set_option("col_rows", int(os.environ.get("COL_ROWS", "0")))
    for cb in [int(x) for x in os.environ.get("CBS", "0 1 2 3 4 6").split()]:
        dts.dts_set_option("col_cluster", cb)
        with dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
            ts = []
            for _ in range(4):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(); s.solve(td, cd, cfg.lam, cfg.iters, out=o); e1.record(); torch.cuda.synchronize()
                ts.append(round(e0.elapsed_time(e1), 3))
        print(json.dumps({"cfg": name, "col_rows": dts.dts_get_option("col_rows"), "col_cluster": cb, "ms": ts}),
              flush=True)
    dts.dts_set_option("col_cluster", 0)
    dts.dts_set_option("col_rows", 0)
