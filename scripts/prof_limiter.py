"""Eager C3 steps with a given limiter (ncu target for the post-limiter kernels)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk  # noqa: E402

lim = sys.argv[1] if len(sys.argv) > 1 else "minmod+simple"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
st = sk.SimulationState(dataclasses.replace(sk.named_config("C3"), limiter=lim))
for _ in range(steps):
    st.run_step()
st.ctx.synchronize()
print("ok", st.stats())
