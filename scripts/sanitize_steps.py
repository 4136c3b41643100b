"""A few run() loop bodies of small configurations touching every kernel
family (x/v sweeps with deferred clamps, 3-block ghosts, post limiters,
cut-off shrinks, single-CTA and cluster Poisson, fused step boundaries, exact
mode) with guard zones around every state buffer (SK_GUARD=1): prints and
returns the guard words overwritten. compute-sanitizer is closed on the GPU
pool; tests/test_gpu_parity.py::test_no_out_of_bounds_writes runs this."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CFGS = [
    dict(k=2, fine_block_cells=8, coarse_block_cells=16, refinement_ratio=4, v_cells=24, limiter="sldg"),
    dict(k=3, fine_block_cells=6, coarse_block_cells=12, refinement_ratio=1, v_cells=16, mu=1836.0,
         limiter="meanerr+line"),
    dict(k=3, fine_block_cells=256, coarse_block_cells=512, refinement_ratio=1, v_cells=16, mu=1836.0,
         limiter="sldg"),
    dict(k=1, fine_block_cells=5, coarse_block_cells=7, refinement_ratio=3, v_cells=10, limiter="minmod+simple"),
    dict(k=5, fine_block_cells=4, coarse_block_cells=8, refinement_ratio=2, v_cells=12, limiter="sldg"),
]


def run() -> dict:
    os.environ["SK_GUARD"] = "1"
    import paper_2408_11235_b200 as sk

    bad = {}
    for i, kw in enumerate(CFGS):
        cfg = sk.RunConfig(**kw)
        for exact in (False, True):
            st = sk.SimulationState(cfg, exact=exact)
            st.ctx.set_step_fusion(not exact)
            st.run_steps(3)
            st.run_step()
            st.run_steps(8)
            st.ctx.synchronize()
            bad[(i, exact)] = st.ctx.check_guards()
            st.close()
            st.ctx.close()
    return bad


if __name__ == "__main__":
    out = run()
    print(out)
    sys.exit(1 if any(out.values()) else 0)
