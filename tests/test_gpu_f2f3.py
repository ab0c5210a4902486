"""SURVEY 8(f) rows f2 (scalar advection model) and f3 (split RK3-FB) on the device,
against the reference's own propagate() (tests/golden/make_f2f3_golden.py).  Both run
the reference-operation-order kernels (csrc/exact.cu), so the comparison is bitwise."""
import numpy as np
import pytest

from conftest import golden
from paper_1510_02237_b200.integrators import (RK3, SPLIT_RK3_FB, SlicePropagator, make_propagator,
                                               propagate, split_rk3_fb_step)
from paper_1510_02237_b200.mesh import ACOUSTIC, SCALAR, ConstantVelocity, SolidBodyRotation, State, build_grid
from paper_1510_02237_b200.physics import ModelSpec

pytestmark = pytest.mark.gpu

G = build_grid(32, 32, 1.0, 1.0)
SCALAR_CASES = {"const1": ConstantVelocity(1.0, 1.0), "const6": ConstantVelocity(1.0, 1.0),
                "solid5": SolidBodyRotation(np.pi)}
SRK3_CASES = {"damped": ConstantVelocity(0.1, -0.05), "solid": SolidBodyRotation(np.pi)}


@pytest.mark.parametrize("name", sorted(SCALAR_CASES))
def test_scalar_advection_rk3_bitwise(name):
    g = golden("prop_f2f3.npz")
    order, cfl, n = g[f"scalar_{name}_meta"]
    model = ModelSpec(kind=SCALAR, vel=SCALAR_CASES[name], advective_flux_order=int(order))
    spec = make_propagator(RK3, model, G, float(cfl))
    end = propagate(spec, State.unflatten(G, g[f"scalar_{name}_q0"], SCALAR), 0.0, int(n) * spec.dt)
    np.testing.assert_array_equal(end.flatten(), g[f"scalar_{name}_q"])


@pytest.mark.parametrize("name", sorted(SRK3_CASES))
def test_split_rk3_fb_bitwise(name):
    g = golden("prop_f2f3.npz")
    order, nu, nsound, cfl, n = g[f"srk3_{name}_meta"]
    model = ModelSpec(kind=ACOUSTIC, vel=SRK3_CASES[name], advective_flux_order=int(order), sound_speed=1.0,
                      nu_damp=float(nu), damping_timescale=1.0 if nu > 0 else None)
    spec = make_propagator(SPLIT_RK3_FB, model, G, float(cfl), n_sound=int(nsound))
    end = propagate(spec, State.unflatten(G, g[f"srk3_{name}_q0"], ACOUSTIC), 0.0, int(n) * spec.dt)
    np.testing.assert_array_equal(end.flatten(), g[f"srk3_{name}_q"])
    # the single-step entry point is the same map
    one = split_rk3_fb_step(State.unflatten(G, g[f"srk3_{name}_q0"], ACOUSTIC), spec, spec.dt)
    first = SlicePropagator(spec, nsteps=1).batch(g[f"srk3_{name}_q0"][None])[0]
    np.testing.assert_array_equal(one.flatten(), first)


def test_scalar_batch_and_dimension():
    model = ModelSpec(kind=SCALAR, vel=ConstantVelocity(1.0, 0.5), advective_flux_order=3)
    prop = SlicePropagator(make_propagator(RK3, model, G, 0.2), nsteps=4)
    assert prop.dim == 32 * 32
    rng = np.random.default_rng(3)
    xs = rng.standard_normal((3, prop.dim))
    got = prop.batch(xs)
    for b in range(3):
        np.testing.assert_array_equal(got[b], prop(xs[b]))
