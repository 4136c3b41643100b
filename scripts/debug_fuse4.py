"""Debug: k=1 fused boundary vs separate sweeps, per step."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk


def rel(a, b):
    m = np.abs(b).max()
    return np.abs(a - b).max() / (m if m > 0 else 1)


for kw in (dict(k=1, fine_block_cells=24, coarse_block_cells=24, refinement_ratio=1, v_cells=48, limiter="sldg"),
           dict(k=1, fine_block_cells=24, coarse_block_cells=24, refinement_ratio=1, v_cells=48, limiter="none"),
           dict(k=2, fine_block_cells=24, coarse_block_cells=24, refinement_ratio=1, v_cells=48, limiter="sldg")):
    cfg = sk.RunConfig(**kw)
    for pat in ([1, 2], [2, 2], [1, 5]):
        a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
        a.ctx.set_step_fusion(True)
        b.ctx.set_step_fusion(False)
        out = []
        for n in pat:
            a.run_steps(n); b.run_steps(n)
            out.append("%d: f %.2e %.2e E %.2e" % (a.step_index(), rel(a.field(0).download(), b.field(0).download()),
                                                   rel(a.field(1).download(), b.field(1).download()),
                                                   np.abs(a.E() - b.E()).max()))
        print(kw["k"], kw["limiter"], pat, out, a.ctx.stats()["inline_troubled"], b.ctx.stats()["inline_troubled"], flush=True)
