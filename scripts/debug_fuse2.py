"""Debug: where does a fused boundary differ from separate sweeps?"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk


def rel(a, b):
    m = np.abs(b).max()
    return np.abs(a - b).max() / (m if m > 0 else 1)


for kw in (dict(k=3, fine_block_cells=32, coarse_block_cells=64, refinement_ratio=1, v_cells=128, mu=1836.0, limiter="none"),
           dict(k=1, fine_block_cells=32, coarse_block_cells=64, refinement_ratio=1, v_cells=64, limiter="none"),
           dict(k=3, fine_block_cells=256, coarse_block_cells=512, refinement_ratio=1, v_cells=64, mu=1836.0, limiter="none")):
    cfg = sk.RunConfig(**kw)
    p = cfg.k + 1
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    b.ctx.set_step_fusion(False)
    a.run_steps(1); b.run_steps(1)
    a.run_steps(2); b.run_steps(2)
    fa, fb = a.field(0).download(), b.field(0).download()
    nx = cfg.nx
    d = np.abs(fa - fb).reshape(cfg.v_cells * p, nx, p).max(axis=2)
    print(kw["k"], nx, "rel", rel(fa, fb), "E", np.abs(a.E() - b.E()).max(), np.abs(b.E()).max())
    bad_x = np.where(d.max(axis=0) > 1e-10 * np.abs(fb).max())[0]
    bad_v = np.where(d.max(axis=1) > 1e-10 * np.abs(fb).max())[0]
    print("  bad x cells", bad_x[:20], len(bad_x), " bad v rows", bad_v[:10], len(bad_v))
    a.close(); b.close()
