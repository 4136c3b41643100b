"""Troubled/clamped cells per x sweep of a named config vs the fix-list capacity."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = sk.named_config(name)
st = sk.SimulationState(cfg)
for _ in range(5):
    st.run_step()
st.ctx.synchronize()
st.ctx.reset_stats()
n = 10
for _ in range(n):
    st.run_step()
st.ctx.synchronize()
cells = 2 * cfg.v_cells * (cfg.k + 1) * st.ctx.grid.ncells if hasattr(st.ctx, "grid") else None
print(name, "stats over", n, "steps:", st.ctx.stats(), "cells/sweep(both species):", cells)
