"""Known-answer tests of the device propagators (SURVEY 8(c) list), mirroring the
reference's tests/test_integrators.py:41-52 (RK3 = stability polynomial of the dense
RHS matrix), :85-100 (one FB substep against circulant derivative matrices) and
:102-132 (FE-FB against a dense Kronecker-product assembly)."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1510_02237_b200.integrators import (RK3, SPLIT_FE_FB, PropagatorSpec, make_propagator,
                                               rk3_step, split_fe_fb_step)
from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, SolidBodyRotation, State, build_grid
from paper_1510_02237_b200.physics import ModelSpec, damping_coefficients

pytestmark = pytest.mark.gpu


def small_acoustic(nu=0.0, order=6, vel=None, nx=8, cs=2.0, tau=None):
    g = build_grid(nx, nx, 1, 1)
    vel = vel if vel is not None else ConstantVelocity(0.0, 0.0)
    return g, ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=order, sound_speed=cs, nu_damp=nu,
                        damping_timescale=tau)


def rhs_matrix(model, g):
    """Dense matrix of the linear RHS from the oracle's restatement of acoustic_rhs
    (pinned bitwise to the reference by tests/test_oracle_golden.py)."""
    from paper_1510_02237_b200.mesh import face_normal_velocities

    ux, vy = face_normal_velocities(model.vel, g)
    a1, a2 = (damping_coefficients(model.nu_damp, g.dx, g.dy, model.damping_timescale)
              if model.nu_damp > 0 else (0.0, 0.0))
    d = 3 * g.nx * g.ny
    mat = np.empty((d, d))
    for k in range(d):
        e = np.zeros(d)
        e[k] = 1.0
        mat[:, k] = orc.acoustic_rhs(e, nx=g.nx, ny=g.ny, dx=g.dx, dy=g.dy, cs=model.sound_speed,
                                     order=model.advective_flux_order, a1=a1, a2=a2, uf=ux, vf=vy)
    return mat


def circulant_d0(n, h):
    c = np.zeros((n, n))
    for i in range(n):
        c[i, (i + 1) % n] = 0.5 / h
        c[i, (i - 1) % n] = -0.5 / h
    return c


@pytest.mark.parametrize("vel,order", [(SolidBodyRotation(0.7), 3), (ConstantVelocity(0.3, -0.2), 6),
                                       (ConstantVelocity(0.3, 0.0), 5)])
def test_rk3_matches_stability_polynomial(vel, order):
    """Constant velocity runs the folded fused kernel, solid body the reference-order one."""
    g, model = small_acoustic(nu=0.02, tau=1e-2, order=order, vel=vel)
    spec = PropagatorSpec(scheme=RK3, model=model, grid=g, cfl=0.2)
    hl = 0.01 * rhs_matrix(model, g)
    q = np.random.default_rng(7).standard_normal(hl.shape[0])
    expected = q + hl @ q + hl @ (hl @ q) / 2.0 + hl @ (hl @ (hl @ q)) / 6.0
    got = rk3_step(State.unflatten(g, q, ACOUSTIC), spec, 0.01).flatten()
    np.testing.assert_allclose(got, expected, rtol=1e-12, atol=1e-13)


def test_single_fb_substep(rng):
    g, model = small_acoustic(cs=2.0)
    spec = PropagatorSpec(scheme=SPLIT_FE_FB, model=model, grid=g, cfl=0.5, n_sound=1)
    st = State(g, rng.standard_normal((3, 8, 8)))
    dt = spec.dt
    out = split_fe_fb_step(st, spec, dt)
    dxm, dym = circulant_d0(g.nx, g.dx), circulant_d0(g.ny, g.dy)
    u1 = st.u - dt * model.sound_speed * (st.p @ dxm.T)
    v1 = st.v - dt * model.sound_speed * (dym @ st.p)
    p1 = st.p - dt * model.sound_speed * (u1 @ dxm.T + dym @ v1)
    for a, b in ((out.u, u1), (out.v, v1), (out.p, p1)):
        np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-14)


def test_fe_fb_matches_dense_kronecker_assembly():
    g, model = small_acoustic(cs=2.0, nu=0.08, tau=1.0)
    nsub = 3
    spec = make_propagator(SPLIT_FE_FB, model, g, cfl=0.9, n_sound=nsub)
    dt = spec.dt
    tau = dt / nsub
    a1 = model.nu_damp * g.dx ** 2 / tau
    a2 = model.nu_damp * g.dy ** 2 / tau
    dxm = np.kron(np.eye(g.ny), circulant_d0(g.nx, g.dx))
    dym = np.kron(circulant_d0(g.ny, g.dy), np.eye(g.nx))
    n = g.nx * g.ny
    cs = model.sound_speed
    x = g.x_centers()
    u = np.tile(np.sin(2 * np.pi * x), (g.ny, 1)).ravel()
    v = np.zeros(n)
    p = np.zeros(n)
    for _ in range(nsub):
        div = dxm @ u + dym @ v
        un = u + tau * (-cs * (dxm @ p) + a1 * (dxm @ div))
        vn = v + tau * (-cs * (dym @ p) + a2 * (dym @ div))
        p = p + tau * (-cs * (dxm @ un + dym @ vn))
        u, v = un, vn
    st = State.acoustic(g, np.tile(np.sin(2 * np.pi * x), (g.ny, 1)), np.zeros((g.ny, g.nx)),
                        np.zeros((g.ny, g.nx)))
    out = split_fe_fb_step(st, spec, dt)
    np.testing.assert_allclose(out.u.ravel(), u, rtol=0, atol=1e-14)
    np.testing.assert_allclose(out.v.ravel(), v, rtol=0, atol=1e-14)
    np.testing.assert_allclose(out.p.ravel(), p, rtol=0, atol=1e-14)
