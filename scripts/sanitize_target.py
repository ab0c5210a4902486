"""Reduced-shape workloads for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python scripts/sanitize_target.py march

Each case launches the production kernels of one protocol at a shape small
enough for the sanitizer's replay:
  march   rk3_march_persist_kernel  (per-segment release/acquire step counters,
          cp.async ring, one CTA barrier per tick), 128^2 x 3 states x 6 steps,
          and the per-step march kernel (PW_MARCH_PERSIST=0)
  window  one KSE window at 128^2, P=4, K=2: fefb tiled cooperative coarse G,
          combine_tma_kernel (TMA bulk-copy mbarrier ring), pqr_kernel and the
          rest of the subspace refactorisation, the residual and K7 diagnostics
  peers   pw_prop_apply_to_peers: the peer-store epilogue into two local
          "peer" buffers (the IPC path's kernel, same-process pointers)
Exit code 0 = ran; the sanitizer's own summary line is the verdict.
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1510_02237_b200 import harness  # noqa: E402
from paper_1510_02237_b200.diagnostics import window_diag  # noqa: E402
from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator  # noqa: E402
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid  # noqa: E402
from paper_1510_02237_b200.parareal import kse_sweep  # noqa: E402
from paper_1510_02237_b200.physics import ModelSpec  # noqa: E402


def specs(n):
    g = build_grid(n, n)
    vel = ConstantVelocity(0.1, 0.0)
    f = make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5)
    c = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 4.0, 16)
    return g, f, c


def main(what):
    torch.cuda.set_device(0)
    rng = np.random.default_rng(5)
    if what == "march":
        g, f, _ = specs(128)
        x = torch.as_tensor(rng.standard_normal((3, 3 * 128 * 128))).cuda()
        y = SlicePropagator(f, nsteps=6).apply(x)
        os.environ["PW_MARCH_PERSIST"] = "0"
        z = SlicePropagator(f, nsteps=2).apply(x)
        torch.cuda.synchronize()
        print("march ok", bool(torch.isfinite(y).all() and torch.isfinite(z).all()))
    elif what == "window":
        n = 128
        g, f, c = specs(n)
        span = 1.0 / 8
        fine, coarse = SlicePropagator(f, span), SlicePropagator(c, span)
        q0 = torch.as_tensor(harness.initial_state("c1", n=n)).cuda()
        ends, res, sub = kse_sweep(q0, fine, coarse, 4, 2, return_device=True)
        d = window_diag(fine.ctx, ends[-1].contiguous(), g, [5, 77])
        torch.cuda.synchronize()
        print("window ok", res, sub.rank, d.finite)
    elif what == "peers":
        g, f, _ = specs(256)
        p = SlicePropagator(f, nsteps=1)
        x = torch.as_tensor(rng.standard_normal((2, 3 * 256 * 256))).cuda()
        out = torch.empty_like(x)
        peers = [torch.empty_like(x), torch.empty_like(x)]
        p.apply_to_peers(x, out, [t.data_ptr() for t in peers])
        torch.cuda.synchronize()
        ok = all(torch.equal(out, t) for t in peers)
        print("peers ok", ok)
        if not ok:
            sys.exit(1)
    else:
        raise SystemExit(f"unknown case {what!r}")


if __name__ == "__main__":
    main(sys.argv[1])
