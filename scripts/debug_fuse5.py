"""Debug: fused charge density vs separate sweeps (k = 1)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk

for k in (1, 2):
    cfg = sk.RunConfig(k=k, fine_block_cells=24, coarse_block_cells=24, refinement_ratio=1, v_cells=48, limiter="sldg")
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    a.ctx.set_step_fusion(True)
    b.ctx.set_step_fusion(False)
    a.run_steps(1); b.run_steps(1)
    a.run_steps(2); b.run_steps(2)
    ra, rb = a.rho(), b.rho()
    d = np.abs(ra - rb)
    print("k", k, "rho max", np.abs(rb).max(), "diff max", d.max(), "at", np.argsort(d)[-8:], flush=True)
    print("   ra", ra[np.argsort(d)[-4:]], "\n   rb", rb[np.argsort(d)[-4:]])
