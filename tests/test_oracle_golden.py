"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

The fixtures were produced by importing the reference (tests/golden/make_golden.py).
Stencil and propagator outputs must match BITWISE (the oracle restates the
numba kernels operation for operation, no FMA contraction); the c1
KSE-Parareal history to 1e-12 relative (BLAS reduction order may differ
between hosts in the subspace matmuls).
"""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as orc
from paper_1510_02237_b200 import harness


def test_rhs_bitwise_all_orders_and_velocities():
    g = golden("rhs.npz")
    n = 16
    dx = 1.0 / n
    for st, want, (velk, order, nu) in zip(g["states"], g["rhs"], g["meta"]):
        vel = ("constant", 0.1, -0.05) if velk == 0 else ("solid_body", np.pi, 0.5, 0.5)
        uf, vf = orc.face_velocities(n, n, velocity=vel)
        a = nu * dx * dx / 0.01 if nu > 0 else 0.0
        got = orc.acoustic_rhs(st, nx=n, ny=n, dx=dx, dy=dx, cs=1.3, order=int(order),
                               a1=a, a2=a, uf=uf, vf=vf)
        np.testing.assert_array_equal(got, want)


def _c2_style_props(n):
    fine = orc.SlicePropagator(orc.RK3, 16, nx=n, ny=n, cs=1.0, order=6, nu=0.005, cfl=0.5,
                               velocity=("constant", 0.1, 0.0))
    coarse = orc.SlicePropagator(orc.SPLIT_FE_FB, 2, nx=n, ny=n, cs=1.0, order=1, nu=0.1, cfl=4.0,
                                 n_sound=16, velocity=("constant", 0.1, 0.0))
    return fine, coarse


def test_propagate_bitwise_constant_velocity():
    g = golden("prop.npz")
    fine, coarse = _c2_style_props(64)
    np.testing.assert_array_equal(fine.batch(g["q0"]), g["fine16"])
    np.testing.assert_array_equal(coarse.batch(g["q0"]), g["coarse2"])


def test_propagate_bitwise_solid_body():
    g = golden("prop.npz")
    vel = ("solid_body", np.pi, 0.5, 0.5)
    fine = orc.SlicePropagator(orc.RK3, 20, nx=32, ny=32, cs=30.0, order=5, nu=0.005, cfl=0.2,
                               velocity=vel)
    coarse = orc.SlicePropagator(orc.SPLIT_FE_FB, 3, nx=32, ny=32, cs=30.0, order=1, nu=0.1,
                                 cfl=4.0, n_sound=4, velocity=vel)
    np.testing.assert_array_equal(fine(g["sb_q0"]), g["sb_fine20"])
    np.testing.assert_array_equal(coarse(g["sb_q0"]), g["sb_coarse3"])


def test_c1_initial_state_generator_matches_fixture():
    g = golden("c1_kse.npz")
    np.testing.assert_array_equal(harness.initial_state("c1"), g["q0"])


def c1_props():
    wl = harness.WORKLOADS["c1"]
    n = wl.n
    fine = orc.SlicePropagator(orc.RK3, wl.fine_steps_per_slice, nx=n, ny=n, cs=harness.CS,
                               order=6, nu=0.005, cfl=0.5, velocity=("constant", 0.1, 0.0))
    coarse = orc.SlicePropagator(orc.SPLIT_FE_FB, wl.coarse_steps_per_slice, nx=n, ny=n,
                                 cs=harness.CS, order=1, nu=0.1, cfl=4.0, n_sound=16,
                                 velocity=("constant", 0.1, 0.0))
    return wl, fine, coarse


def test_c1_kse_history_matches_reference():
    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    hist, ranks = [], []
    ends, res, sub = orc.kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it, history=hist, ranks=ranks)
    assert ranks == list(g["kse_ranks"])
    for k, (got, want) in enumerate(zip(hist, g["kse_hist"])):
        for i in range(wl.n_p):
            rel = np.linalg.norm(got[i] - want[i]) / np.linalg.norm(want[i])
            assert rel <= 1e-12, (k, i, rel)
    np.testing.assert_allclose(res, g["kse_res"], rtol=1e-12)


def test_c1_original_parareal_matches_reference():
    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    ends, res = orc.parareal_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    np.testing.assert_allclose(res, g["orig_res"], rtol=1e-13)
    np.testing.assert_allclose(np.array(ends), g["orig_final"], rtol=0, atol=1e-13)
