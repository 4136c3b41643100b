"""B200-native sLdG scrape-off-layer time step (arXiv 2408.11235).

Drop-in for the reference solver interface in proj/core: the step runs in
hand-written sm_100a kernels behind the C ABI include/sk_b200.h
(lib/libsk_b200.so); `solver` mirrors the reference's free functions and
`sharding` holds the v-sharded multi-GPU plumbing.
"""
from .solver import (  # noqa: F401
    NAMED_CONFIGS, Context, FieldPair, Grid1D, LimiterConfig, NodalField, PoissonOperator,
    RunConfig, SimulationError, SimulationState, SpeciesParams, SweepOptions, VAdjustPolicy,
    advect_v, advect_x, apply_post_limiter, build_shift_matrices, charge_density,
    check_velocity_shrink, electric_energy, matrices_text, named_config, run, run_step,
    shrink_velocity_domain, strang_step)

__version__ = "0.1.0"
