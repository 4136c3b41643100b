"""Run a few steps of custom shapes (for ncu launch lists): nf nc m nv k."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses

import paper_2408_11235_b200 as sk

base = sk.named_config("C3")
for spec in sys.argv[1:]:
    nf, nc, m, nv = (int(x) for x in spec.split(","))
    cfg = dataclasses.replace(base, fine_block_cells=nf, coarse_block_cells=nc, refinement_ratio=m, v_cells=nv)
    st = sk.SimulationState(cfg)
    for _ in range(3):
        st.run_step()
    st.ctx.synchronize()
    print(spec, "ok", flush=True)
    st.close()
