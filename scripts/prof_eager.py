"""Eager (no CUDA graph) C3 steps for ncu kernel replay: graph-replayed
windows interact badly with kernel replay (the sweeps' list counters are not
restored per pass), so profile the fixup kernels from plain enqueues."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2408_11235_b200 as sk

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
st = sk.SimulationState(sk.named_config(sys.argv[2] if len(sys.argv) > 2 else "C3"))
for _ in range(steps):
    st.run_step()
st.ctx.synchronize()
print("stats", st.stats())
