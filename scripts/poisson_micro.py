import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_11235_b200 as sk
for nx_cfg in [(512, 1024), (64, 128), (4096, 8192)]:
    g = sk.Grid1D.three_block(-200.0, 200.0, nx_cfg[0], nx_cfg[1], 1)
    for k in (2, 3):
        ctx = sk.Context(g, k)
        op = sk.PoissonOperator(ctx)
        rho = torch.randn(g.ncells * (k + 1), dtype=torch.float64, device="cuda") * 1e-5
        for _ in range(3): op.solve(rho)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ctx.stream):
            e0.record(ctx.stream)
            for _ in range(20): op.solve(rho)
            e1.record(ctx.stream)
        torch.cuda.synchronize()
        print(f"N={g.ncells} k={k}: {e0.elapsed_time(e1)/20*1e3:.1f} us per solve (incl. python + 2 allocs)")
        ctx.close()
