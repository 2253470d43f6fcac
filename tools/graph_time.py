import os, sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1805_04590_b200 as dts
for (H, W, C, it) in [(375, 450, 3, 20), (640, 480, 1, 20), (1080, 1920, 3, 20)]:
    g = torch.rand(H, W, C, device='cuda'); t = torch.rand(H, W, device='cuda'); c = torch.rand(H, W, device='cuda')
    with dts.Solver(g, 8.0, 0.1, 3) as s:
        o = torch.empty_like(t)
        for _ in range(3): s.solve(t, c, 0.99, it, out=o)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): s.solve(t, c, 0.99, it, out=o)
        e1.record(); torch.cuda.synchronize()
        print(os.environ.get('DTS_NO_GRAPH', 'graph'), H, W, C, f"{e0.elapsed_time(e1)/20:.3f} ms/solve")
