"""The exact headline workload (bench.py, BASELINE.json configs[1] = c2) against the oracle.

64 states x 256^2 x 200 RK3 steps (CFL 0.5, order 6, nu 0.005, cs 1, U 0.1),
seeded random-mode inputs (seed 2001, the bench's rank-0 batch), through the
default device path (K1, the TMA-fed persistent row march, march_tma.cu) and
through the previous-generation kernels (PW_MARCH_V2=0: the cp.async persistent march
and its per-step launches, PW_MARCH_PERSIST=0), each state compared with the C
oracle (reference operation order, oracle/pw_oracle.c; integrators.py:126-146,
numba_backend.py:119-128).

Tolerance: 1e-12 relative L2 per state.  The device kernels fold the stencils
and contract to FMA, so they differ from the reference's operation order by
rounding only (~1e-16 per step); 200 steps of a non-expanding operator (spectral
radius 0.99896 per step) keep the accumulated difference
far below 1e-12.
"""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1510_02237_b200 import harness

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

N, BATCH, STEPS, SEED = 256, 64, 200, 2001


@pytest.fixture(scope="module")
def c2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_02237_b200 import _lib

    _lib.Context.get(0).set_strict(False)
    q0 = harness.fine_batch_states(n=N, batch=BATCH, seed=SEED)
    want = orc.SlicePropagator(orc.RK3, STEPS, nx=N, ny=N, cs=harness.CS, order=6, nu=0.005, cfl=0.5,
                               velocity=("constant", harness.VEL_U, harness.VEL_V)).batch(q0)
    return q0, want


def _spec():
    from paper_1510_02237_b200.integrators import RK3, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
    return make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, harness.CS, 0.005, 1.0), build_grid(N, N), 0.5)


def _check(got, want):
    err = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert np.all(np.isfinite(got))
    assert err.max() <= 1e-12, f"worst state {int(err.argmax())}: {err.max():.3e}"
    return err.max()


@pytest.mark.parametrize("env", [{}, {"PW_MARCH_V2": "0"}, {"PW_MARCH_V2": "0", "PW_MARCH_PERSIST": "0"}],
                         ids=["tma-persistent", "cpasync-persistent", "cpasync-per-step"])
def test_bench_workload_every_state_matches_oracle(c2, monkeypatch, env):
    """The default K1 (march_tma.cu) and both previous-generation paths, every state."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    q0, want = c2
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    prop = SlicePropagator(_spec(), nsteps=STEPS)
    x = torch.as_tensor(q0).cuda()
    got = prop.apply(x).cpu().numpy()
    _check(got, want)


def test_bench_workload_drop_in_host_api(c2):
    """The call a reference user makes: SlicePropagator.batch on host numpy (synchronous)."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    q0, want = c2
    got = SlicePropagator(_spec(), nsteps=STEPS).batch(q0)
    _check(got, want)
