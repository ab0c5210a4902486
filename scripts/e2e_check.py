"""Break the bench e2e step into H2D / compute / D2H (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1510_02237_b200 import harness  # noqa: E402
from paper_1510_02237_b200.integrators import RK3, SlicePropagator, make_propagator  # noqa: E402
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid  # noqa: E402
from paper_1510_02237_b200.physics import ModelSpec  # noqa: E402

g = build_grid(256, 256)
spec = make_propagator(RK3, ModelSpec(ACOUSTIC, ConstantVelocity(0.1, 0.0), 6, 1.0, 0.005, 1.0), g, 0.5)
prop = SlicePropagator(spec, nsteps=200)
q = torch.as_tensor(harness.fine_batch_states(256, 64, 2001))
pin = q.pin_memory()
pout = torch.empty_like(pin).pin_memory()
x = pin.cuda()
prop.apply(x)
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


for rep in range(3):
    e = [ev() for _ in range(4)]
    e[0].record()
    xd = pin.to("cuda", non_blocking=True)
    e[1].record()
    yd = prop.apply(xd)
    e[2].record()
    pout.copy_(yd, non_blocking=True)
    e[3].record()
    torch.cuda.synchronize()
    h2d, comp, d2h = (e[i].elapsed_time(e[i + 1]) for i in range(3))
    print(f"h2d {h2d:.2f} ms ({pin.numel() * 8 / h2d / 1e6:.1f} GB/s)  compute {comp:.2f} ms  "
          f"d2h {d2h:.2f} ms ({pin.numel() * 8 / d2h / 1e6:.1f} GB/s)", flush=True)
