"""B200-native KSE-Parareal for the linear 2D acoustic-advection system (arXiv 1510.02237).

Drop-in for the reference package ``pitwave``'s hot path: the same public
names (reference src/pitwave/__init__.py:8-18), with the fine RK3
predictor, the split FE-FB coarse propagator, the Krylov subspace and the
Parareal sweeps executed by hand-written sm_100a CUDA kernels behind the C
ABI in include/pitwave_b200.h (loaded with ctypes from
``libpitwave_b200.so``).  There is no CPU fallback: device entry points
fail loudly when the library or the GPU is missing.
"""
from .mesh import (ACOUSTIC, SCALAR, ConstantVelocity, Grid2D, SolidBodyRotation, State,
                   build_grid, init_cosine_bump)
from .physics import ModelSpec, damping_coefficients
from .integrators import (MatrixPropagator, PropagatorSpec, SlicePropagator, make_propagator,
                          propagate)
from .parareal import (KSE, ORIGINAL, PitConfig, RunReport, Timings, kse_sweep, parareal_sweep,
                       run_windowed)
from .subspace import Subspace, kse_coarse
from .config import ConfigError, ExperimentConfig, load_config, parse_config

KERNEL_BACKEND = "sm_100a"
__version__ = "0.1.0"
