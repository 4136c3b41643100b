"""Debug: limiter counters of one fused boundary vs separate sweeps."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk

cfg = sk.RunConfig(k=3, fine_block_cells=32, coarse_block_cells=64, refinement_ratio=1, v_cells=128, mu=1836.0,
                   limiter="sldg")
for pat in ([1, 2], [2, 2], [5, 2]):
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    b.ctx.set_step_fusion(False)
    for n in pat[:-1]:
        a.run_steps(n); b.run_steps(n)
    a.ctx.reset_stats(); b.ctx.reset_stats()
    a.run_steps(pat[-1]); b.run_steps(pat[-1])
    print(pat, "fused", a.ctx.stats(), "\n      sep  ", b.ctx.stats(), flush=True)
