"""Eager steps of a named config (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk  # noqa: E402

st = sk.SimulationState(sk.named_config(sys.argv[1]))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    st.run_step()
st.ctx.synchronize()
print("ok")
