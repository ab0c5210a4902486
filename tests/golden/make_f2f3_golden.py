"""Scalar-advection RK3 and split RK3-FB fixtures from the REFERENCE (this container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_f2f3_golden.py

SURVEY.md 8(f) rows f2 (scalar advection model, physics.py:77-80, with constant and
solid-body velocity) and f3 (split_rk3_fb_step, integrators.py:109-120): the
reference's own ``propagate`` on seeded 32^2 states -> prop_f2f3.npz.
"""
from __future__ import annotations

import os

import numpy as np

from pitwave.integrators import RK3, SPLIT_RK3_FB, make_propagator, propagate
from pitwave.kernels import BACKEND_NAME
from pitwave.mesh import ACOUSTIC, SCALAR, ConstantVelocity, SolidBodyRotation, State, build_grid
from pitwave.physics import ModelSpec

assert BACKEND_NAME == "numba"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(909)
    g = build_grid(32, 32, 1.0, 1.0)
    out = {}
    # f2: scalar advection, RK3, orders 1 and 6, constant diagonal and solid-body velocity
    cases = [("const1", ConstantVelocity(1.0, 1.0), 1), ("const6", ConstantVelocity(1.0, 1.0), 6),
             ("solid5", SolidBodyRotation(np.pi), 5)]
    for name, vel, order in cases:
        q0 = rng.standard_normal((1, 32, 32))
        model = ModelSpec(kind=SCALAR, vel=vel, advective_flux_order=order)
        spec = make_propagator(RK3, model, g, 0.3)
        n = 7
        end = propagate(spec, State(g, q0.copy()), 0.0, n * spec.dt)
        out[f"scalar_{name}_q0"] = q0.ravel()
        out[f"scalar_{name}_q"] = end.flatten()
        out[f"scalar_{name}_meta"] = np.array([order, 0.3, n], dtype=np.float64)
    # f3: split RK3-FB, acoustic, with and without damping
    cases = [("damped", ConstantVelocity(0.1, -0.05), 1, 0.1, 6), ("solid", SolidBodyRotation(np.pi), 3, 0.0, 5)]
    for name, vel, order, nu, nsound in cases:
        q0 = rng.standard_normal((3, 32, 32))
        model = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=order, sound_speed=1.0, nu_damp=nu,
                          damping_timescale=1.0 if nu > 0 else None)
        spec = make_propagator(SPLIT_RK3_FB, model, g, 2.0, n_sound=nsound)
        n = 3
        end = propagate(spec, State(g, q0.copy()), 0.0, n * spec.dt)
        out[f"srk3_{name}_q0"] = q0.ravel()
        out[f"srk3_{name}_q"] = end.flatten()
        out[f"srk3_{name}_meta"] = np.array([order, nu, nsound, 2.0, n], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "prop_f2f3.npz"), **out)
    print("wrote prop_f2f3.npz", sorted(out))


if __name__ == "__main__":
    main()
