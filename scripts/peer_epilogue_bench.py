"""Cost of the fused peer-store epilogue on one GPU (CUDA events; no profiler).

    python scripts/peer_epilogue_bench.py

One RK3 step over one rank's block of the c3 fine sweep at 8 GPUs (8 slices of
512^2), with the result also needed in 7 more buffers:
  plain   : pw_prop_apply, no peers
  fused   : pw_prop_apply_to_peers, the marching kernel stores every row 8 times
  copies  : pw_prop_apply, then 7 device-to-device copies
Here the 7 "peers" are buffers on the same GPU, so the stores go to local HBM,
not over NVLink: this measures how much of the store traffic the epilogue hides
behind the step's compute, not NVLink bandwidth.
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1510_02237_b200.integrators import RK3, SlicePropagator, make_propagator  # noqa: E402
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid  # noqa: E402
from paper_1510_02237_b200.physics import ModelSpec  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    n, nslice, npeer = 512, 8, 7
    spec = make_propagator(RK3, ModelSpec(ACOUSTIC, ConstantVelocity(0.1, 0.0), 6, 1.0, 0.005, 1.0),
                           build_grid(n, n), 0.5)
    prop = SlicePropagator(spec, nsteps=1)
    x = torch.as_tensor(np.random.default_rng(5).standard_normal((nslice, 3 * n * n))).cuda()
    out = torch.empty_like(x)
    peers = [torch.empty_like(x) for _ in range(npeer)]
    ptrs = [p.data_ptr() for p in peers]

    def plain():
        prop.apply(x, out)

    def fused():
        prop.apply_to_peers(x, out, ptrs)

    def copies():
        prop.apply(x, out)
        for p in peers:
            p.copy_(out)

    fused()
    torch.cuda.synchronize()
    assert all(torch.equal(p, out) for p in peers)
    mb = x.numel() * 8 / 1e6
    t = {name: timeit(fn) for name, fn in (("plain", plain), ("fused", fused), ("copies", copies))}
    print(f"one RK3 step, {nslice} x {n}^2 ({mb:.0f} MB per copy), {npeer} local peer buffers")
    for name, us in t.items():
        print(f"  {name:7s} {us:8.1f} us")
    print(f"  epilogue cost: fused +{t['fused'] - t['plain']:.1f} us, copies +{t['copies'] - t['plain']:.1f} us")


if __name__ == "__main__":
    main()
