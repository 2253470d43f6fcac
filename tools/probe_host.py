"""Host enqueue time vs device time of eager C1 solves (graphs off), per launch."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04590_b200 as dts
from synth import CONFIGS, make_inputs
torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = CONFIGS[name]
g, t, c = make_inputs(name)
gd, td, cd = (torch.from_numpy(a).cuda() for a in (g, t, c))
o = torch.empty_like(td)
res = {}
with dts.options(graphs=0), dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
    s.solve(td, cd, cfg.lam, cfg.iters, out=o)
    torch.cuda.synchronize()
    n0 = dts.dts_launch_count(s.ctx)
    # host-only enqueue rate: block the stream behind a long sleep kernel so launches only queue
    torch.cuda._sleep(int(2e9 * 0.05))  # ~50 ms of device time ahead of the solve
    t0 = time.perf_counter()
    s.solve(td, cd, cfg.lam, cfg.iters, out=o)
    host = time.perf_counter() - t0
    torch.cuda.synchronize()
    n = dts.dts_launch_count(s.ctx) - n0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); s.solve(td, cd, cfg.lam, cfg.iters, out=o); e1.record(); torch.cuda.synchronize()
    res = {"config": name, "launches": n, "host_enqueue_ms": host * 1e3, "host_us_per_launch": host * 1e6 / n,
           "eager_device_ms": e0.elapsed_time(e1)}
with dts.Solver(gd, cfg.sigma_s, cfg.sigma_r, cfg.N) as s:
    for _ in range(3):
        s.solve(td, cd, cfg.lam, cfg.iters, out=o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); s.solve(td, cd, cfg.lam, cfg.iters, out=o); e1.record(); torch.cuda.synchronize()
    res["graph_replay_ms"] = e0.elapsed_time(e1)
print(json.dumps(res))
