import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2408_11235_b200 as sk
from oracle import Oracle
from tests.test_gpu_parity import cfg_of, FULL_CFGS
from tests.golden.make_golden import STATE_CFGS
O = Oracle()
def rel(a, b):
    m = np.abs(b).max(); return np.abs(a-b).max()/m
for name, kw in list(FULL_CFGS.items()) + [("k3_meanerr_line_m2", STATE_CFGS["k3_meanerr_line_m2"])]:
    cfg = cfg_of(sk, **kw)
    o = O.state(**cfg.oracle_kwargs()); st = sk.SimulationState(cfg)
    print("==", name)
    for s in range(1, 13):
        st.run_step(); o.step()
        fe, fo = st.f_e.download(), o.field(0)
        i = np.argmax(np.abs(fe - fo))
        E, Eo = st.E(), o.E()
        print(f" s{s}: rel_e {rel(fe, fo):.2e} (at {i}: {fe[i]:.3e} vs {fo[i]:.3e}) rel_i {rel(st.f_i.download(), o.field(1)):.2e} |dE| {np.abs(E-Eo).max():.2e} max|E| {np.abs(Eo).max():.2e} stats g {st.stats()['post_troubled']} {st.stats()['inline_troubled']} o {o.stats()['post_troubled']} {o.stats()['inline_troubled']}")
