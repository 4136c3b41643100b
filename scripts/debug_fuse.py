"""Debug: fused step boundaries against separate sweeps, per batch pattern."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk

kw = dict(k=3, fine_block_cells=32, coarse_block_cells=64, refinement_ratio=1, v_cells=128, mu=1836.0,
          limiter="sldg")
cfg = sk.RunConfig(**kw)


def rel(a, b):
    m = np.abs(b).max()
    return np.abs(a - b).max() / (m if m > 0 else 1)


for pat in ([2], [3], [1, 2], [2, 2], [1, 3], [10, 2], [3, 10]):
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    b.ctx.set_step_fusion(False)
    out = []
    for n in pat:
        a.run_steps(n)
        b.run_steps(n)
        d = [rel(a.field(sp).download(), b.field(sp).download()) for sp in (0, 1)]
        out.append((n, a.step_index(), "%.2e %.2e" % tuple(d), a.shrinks(0), b.shrinks(0)))
    print(pat, out, flush=True)
    a.close(); b.close()
