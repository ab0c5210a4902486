"""Perturbation floor of a KSE window: the same window with the fast (folded, FMA) kernels
and with the strict reference-operation-order kernels.  The two differ only by ~1e-16
rounding in the propagators, so their per-slice relative L2 distance measures how much
the window amplifies rounding -- the analogue of the reference's numba-vs-numpy floor.

    python scripts/floor_check.py c3 5     # or: c4 1
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1510_02237_b200 import _lib, harness  # noqa: E402
from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator  # noqa: E402
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid  # noqa: E402
from paper_1510_02237_b200.parareal import kse_sweep  # noqa: E402
from paper_1510_02237_b200.physics import ModelSpec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = harness.WORKLOADS[name]
g = build_grid(wl.n, wl.n)
vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
fine = SlicePropagator(make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5), wl.slice_span)
coarse = SlicePropagator(make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 4.0, 16),
                         wl.slice_span)
q0 = torch.as_tensor(harness.initial_state(name)).cuda()
ctx = _lib.Context.get(0)
out = {"config": name, "per_iteration": []}
for k in range(1, kmax + 1):
    a, ra, sa = kse_sweep(q0, fine, coarse, wl.n_p, k, return_device=True)
    ctx.set_strict(True)
    try:
        b, rb, sb = kse_sweep(q0, fine, coarse, wl.n_p, k, return_device=True)
    finally:
        ctx.set_strict(False)
    dev = torch.linalg.norm(a - b, dim=1) / torch.linalg.norm(b, dim=1)
    out["per_iteration"].append({"k": k, "max_rel_l2": float(dev.max()), "median_rel_l2": float(dev.median()),
                                 "residual_rel_diff": abs(ra[-1] - rb[-1]) / abs(rb[-1]),
                                 "ranks": [sa.rank, sb.rank]})
    print(json.dumps(out["per_iteration"][-1]), flush=True)
    del a, b, sa, sb
    torch.cuda.empty_cache()
