"""B200-native Hermite-leapfrog hot path of arXiv 1808.10481.

The compute path is lib/libhlf_b200.so (hand-written sm_100a CUDA behind the
C-ABI in include/hlf_b200.h); this package is its host-side mirror of the
reference's solver interface (proj/include/hlf)."""
from .solver import (  # noqa: F401
    DUAL, PERIODIC, PRIMARY, REFLECTIVE, ConfigError, CudaError, Grid, Grid1d, Grid2d, Grid3d,
    InstabilityError, InterpOperator, MaxwellTM2d, SchemeConfig, Stepper, Stepper1d, Stepper2d, Stepper3d,
    SCHEME_DUAL_HERMITE, SCHEME_LEAPFROG, SCHEME_MODIFIED, SCHEME_MODIFIED_ADVECTION, build_interp_operator, plan_steps, step_count,
)
