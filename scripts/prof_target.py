"""Small, fixed workloads for ncu captures (run plain first, then under ncu).

    python scripts/prof_target.py fine   # 4 fused RK3 launches on the c2 batch
    python scripts/prof_target.py c3k2   # c3 KSE window with K=2 (launch list)
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1510_02237_b200 import harness  # noqa: E402
from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator  # noqa: E402
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid  # noqa: E402
from paper_1510_02237_b200.parareal import kse_sweep  # noqa: E402
from paper_1510_02237_b200.physics import ModelSpec  # noqa: E402


def specs(n):
    g = build_grid(n, n)
    vel = ConstantVelocity(0.1, 0.0)
    f = make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5)
    c = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 4.0, 16)
    return f, c


what = sys.argv[1]
torch.cuda.set_device(0)
if what == "fine":
    f, _ = specs(256)
    x = torch.as_tensor(harness.fine_batch_states(256, 64, 2001)).cuda()
    p = SlicePropagator(f, nsteps=4)
    y = p.apply(x)
    torch.cuda.synchronize()
    print("fine ok", bool(torch.isfinite(y).all()))
elif what == "fine200":  # the bench's c2 propagation: 200 RK3 steps (one persistent launch)
    f, _ = specs(256)
    x = torch.as_tensor(harness.fine_batch_states(256, 64, 2001)).cuda()
    y = SlicePropagator(f, nsteps=200).apply(x)
    torch.cuda.synchronize()
    print("fine200 ok", bool(torch.isfinite(y).all()))
elif what == "coarse":
    _, c = specs(512)
    x = torch.as_tensor(harness.initial_state("c3")).cuda()[None, :].contiguous()
    y = SlicePropagator(c, nsteps=1).apply(x)
    torch.cuda.synchronize()
    print("coarse ok", bool(torch.isfinite(y).all()))
elif what in ("c3k2", "c3k5", "c4k2", "c4k4"):
    cfgname = "c4" if what.startswith("c4") else "c3"
    wl = harness.WORKLOADS[cfgname]
    f, c = specs(wl.n)
    fine, coarse = SlicePropagator(f, wl.slice_span), SlicePropagator(c, wl.slice_span)
    q0 = torch.as_tensor(harness.initial_state(cfgname)).cuda()
    k = {"c3k2": 2, "c3k5": 5, "c4k2": 2, "c4k4": 4}[what]
    if os.environ.get("PW_WARM") == "1":
        kse_sweep(q0, fine, coarse, wl.n_p, k, return_device=True)
        torch.cuda.synchronize()
        print("---- warm")
    ends, res, sub = kse_sweep(q0, fine, coarse, wl.n_p, k, return_device=True)
    torch.cuda.synchronize()
    print("c3k2 ok", res, sub.rank)
