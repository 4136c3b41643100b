"""C3 fast vs exact mode (exact == the reference bitwise, see
test_c3_full_size_run_matches_reference): per-step E and f differences and
the species masses, to size the fast-mode envelope at full size."""
import numpy as np
import paper_2408_11235_b200 as sk

cfg = sk.named_config("C3")
a, b = sk.SimulationState(cfg, exact=True), sk.SimulationState(cfg)
for s in range(1, 12):
    a.run_step(); b.run_step()
    Ea, Eb = a.E(), b.E()
    row = [s, np.abs(Ea).max(), np.abs(Eb - Ea).max()]
    for sp in (0, 1):
        fa, fb = a.field(sp).download(), b.field(sp).download()
        row += [np.abs(fb - fa).max() / np.abs(fa).max(), fa.sum(), fb.sum() - fa.sum()]
    print("step %2d max|E_exact| %.3e |dE| %.3e | e: rel %.2e sum %.12e dsum %.2e | i: rel %.2e sum %.12e dsum %.2e"
          % tuple(row), flush=True)
print("shrinks", a.shrinks(0), a.shrinks(1), b.shrinks(0), b.shrinks(1))
