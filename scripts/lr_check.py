"""Large-rank KSE window: device residuals (current serial-step kernel) and diag ratios."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

from paper_1510_02237_b200 import harness  # noqa: E402
from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator  # noqa: E402
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid  # noqa: E402
from paper_1510_02237_b200.parareal import kse_sweep  # noqa: E402
from paper_1510_02237_b200.physics import ModelSpec  # noqa: E402

n, p, k = 24, 150, 4
grid = build_grid(n, n)
vel = ConstantVelocity(0.1, 0.0)
fspec = make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), grid, 0.5)
cspec = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), grid, 1.0, 4)
span = 2 * fspec.dt
fine, coarse = SlicePropagator(fspec, span), SlicePropagator(cspec, span)
q0 = harness.initial_state("c3", n=n)
for kk in range(1, k + 1):
    ends, res, sub = kse_sweep(q0, fine, coarse, p, kk)
    rat = np.sort(sub.diag_ratios())
    kept = rat[rat > 1e-10]
    dropped = rat[rat <= 1e-10]
    print(os.environ.get("PW_CG_VARIANT", "0"), kk, sub.rank, res[-1],
          "kept min %.3g" % kept.min(), "dropped max %.3g" % (dropped.max() if dropped.size else 0), flush=True)
