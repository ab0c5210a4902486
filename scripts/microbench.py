"""Per-component device timings of the hot path (CUDA events; no profiler).

    python scripts/microbench.py [fine|coarse|qr|combine|all]

fine    : fused RK3 launch over the c2 batch (64 x 256^2), one RK3 step
coarse  : coarse G over one c3 slice (512^2, 2 FE-FB steps x 16 substeps)
qr      : subspace refactorisation at c3 sizes (d = 786432, m = 64..320)
combine : fused correction GEMV (D alpha + Q^T y) at d = 786432, r = 64..310
"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1510_02237_b200 import harness  # noqa: E402
from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator  # noqa: E402
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid  # noqa: E402
from paper_1510_02237_b200.physics import ModelSpec  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def specs(n):
    g = build_grid(n, n)
    vel = ConstantVelocity(0.1, 0.0)
    f = make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5)
    c = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 4.0, 16)
    return f, c


def bench_fine():
    f, _ = specs(256)
    xs = harness.fine_batch_states(256, 64, 2001)
    x = torch.as_tensor(xs).cuda()
    y = torch.empty_like(x)
    # correctness of the selected tile variant against the oracle (2 states, 3 steps)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    from oracle import oracle as orc

    want = orc.SlicePropagator(orc.RK3, 3, nx=256, ny=256, cs=1.0, order=6, nu=0.005, cfl=0.5,
                               velocity=("constant", 0.1, 0.0)).batch(xs[:2])
    got = SlicePropagator(f, nsteps=3).batch(xs[:2])
    err = max(np.linalg.norm(got[b] - want[b]) / np.linalg.norm(want[b]) for b in range(2))
    print(f"variant {os.environ.get('PW_FUSED_VARIANT', '0')}: rel err vs oracle {err:.2e}")
    for steps in (1, 10):
        p = SlicePropagator(f, nsteps=steps)
        t = timeit(lambda: p.apply(x, out=y), reps=5)
        cu = 64 * 256 * 256 * steps / t
        print(f"fine fused: {steps} step(s) {t*1e3:.3f} ms  -> {cu/1e9:.2f} G cell-updates/s, "
              f"{cu*48/1e9:.0f} GB/s algorithmic")


def bench_fine_grid(n, batch):
    """fine RK3 throughput on another grid (c3: 512^2 x 64, c4: 1024^2 x 64)"""
    f, _ = specs(n)
    xs = harness.fine_batch_states(n, batch, 7)
    x = torch.as_tensor(xs).cuda()
    y = torch.empty_like(x)
    p = SlicePropagator(f, nsteps=4)
    t = timeit(lambda: p.apply(x, out=y), reps=5)
    cu = batch * n * n * 4 / t
    print(f"fine fused {n}^2 x {batch}: 4 steps {t*1e3:.3f} ms  -> {cu/1e9:.2f} G cell-updates/s")


def bench_fine_wide():
    """K1 on wide rows (clusters): c4 (1024^2 x 64) and c5 (2048^2 x 16), 20 steps per launch"""
    for n, batch in ((1024, 64), (2048, 16)):
        f, _ = specs(n)
        x = torch.as_tensor(harness.fine_batch_states(n, batch, 7)).cuda()
        y = torch.empty_like(x)
        p = SlicePropagator(f, nsteps=20)
        t = timeit(lambda: p.apply(x, out=y), reps=3)
        cu = batch * n * n * 20 / t
        print(f"fine {n}^2 x {batch}: 20 steps {t*1e3:.3f} ms  -> {cu/1e9:.2f} G cell-updates/s")


def bench_coarse():
    _, c = specs(512)
    x = torch.as_tensor(harness.initial_state("c3")).cuda()[None, :].contiguous()
    y = torch.empty_like(x)
    for steps in (1, 2):
        p = SlicePropagator(c, nsteps=steps)
        t = timeit(lambda: p.apply(x, out=y), reps=10)
        print(f"coarse FE-FB 512^2: {steps} step(s) {t*1e6:.1f} us")
    _, c4 = specs(1024)
    x4 = torch.as_tensor(harness.initial_state("c4")).cuda()[None, :].contiguous()
    y4 = torch.empty_like(x4)
    for steps in (1, 2):
        p = SlicePropagator(c4, nsteps=steps)
        t = timeit(lambda: p.apply(x4, out=y4), reps=10)
        print(f"coarse FE-FB 1024^2: {steps} step(s) {t*1e6:.1f} us")
    p = SlicePropagator(c, nsteps=2)
    xb = x.repeat(64, 1)
    yb = torch.empty_like(xb)
    t = timeit(lambda: p.apply(xb, out=yb), reps=3)
    print(f"coarse FE-FB 512^2 batched x64: 2 steps {t*1e3:.2f} ms")


def bench_qr():
    from paper_1510_02237_b200.subspace import Subspace

    d = 3 * 512 * 512
    rng = np.random.default_rng(0)
    for m in (64, 128, 320):
        s = torch.as_tensor(rng.standard_normal((m, d))).cuda()
        cols = [s[k] for k in range(m)]
        sub = Subspace(d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sub2 = sub.update(cols, cols)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        t0 = time.perf_counter()
        sub2 = sub.update(cols, cols)
        torch.cuda.synchronize()
        t2 = time.perf_counter() - t0
        print(f"subspace update d={d} m={m}: first {t*1e3:.1f} ms, second {t2*1e3:.1f} ms, rank {sub2.rank}")


def bench_combine():
    from paper_1510_02237_b200 import _lib

    d = 3 * 512 * 512
    lib = _lib.load_library()
    print("combine GEMV is timed inside the sweep (see bench parareal phases)")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    if what in ("fine", "all"):
        bench_fine()
    if what in ("fine512", "all"):
        bench_fine_grid(512, 64)
    if what in ("fine1024", "all"):
        bench_fine_grid(1024, 16)
    if what in ("wide", "all"):
        bench_fine_wide()
    if what in ("coarse", "all"):
        bench_coarse()
    if what in ("qr", "all"):
        bench_qr()
