import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1510_02237_b200 import harness
from paper_1510_02237_b200.integrators import RK3, SlicePropagator, make_propagator
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
from paper_1510_02237_b200.physics import ModelSpec
n, batch, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = build_grid(n, n)
spec = make_propagator(RK3, ModelSpec(ACOUSTIC, ConstantVelocity(0.1, 0.0), 6, 1.0, 0.005, 1.0), g, 0.5)
x = torch.randn(batch, 3 * n * n, dtype=torch.float64, device="cuda") * 1e-3
p = SlicePropagator(spec, nsteps=steps)
out = torch.empty_like(x)
for _ in range(2): p.apply(x, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3): p.apply(x, out=out)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(f"n={n} batch={batch} steps={steps} NSEG={os.environ.get('PW_MARCH_NSEG','auto')}: {ms:.2f} ms  {batch*n*n*steps/ms/1e6:.1f} G cell-updates/s")
