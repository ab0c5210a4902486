"""Generate golden fixtures by running the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Imports the reference package ``pitwave`` from /root/reference (read-only,
not available on the GPU box) and writes small .npz fixtures next to this
script.  The fixtures pin the oracle (tests/test_oracle_golden.py) and the
device path (tests/test_gpu_*.py) to the reference's own outputs.

Fixtures
--------
rhs.npz     acoustic_advection_rhs on 16x16 random states: constant and
            solid-body velocity, flux orders 1..6, with/without damping.
prop.npz    propagate() of RK3 and split FE-FB on 64x64 / 32x32 states.
c1_kse.npz  BASELINE c1 (64^2, P=8, K=3) KSE-Parareal via kse_sweep with
            slice-length propagate closures: qn[1:] per iteration, residuals,
            ranks; plus the original-Parareal sweep (residuals + final qn).
small_kse.npz  nx=8 production KSE window (parareal.py test seam) and a
            dense-matrix KSE window.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from pitwave import subspace as ref_sub  # noqa: E402
from pitwave.integrators import RK3, SPLIT_FE_FB, make_propagator, propagate  # noqa: E402
from pitwave.kernels import BACKEND_NAME  # noqa: E402
from pitwave.mesh import ACOUSTIC, ConstantVelocity, SolidBodyRotation, State, build_grid  # noqa: E402
from pitwave.parareal import kse_sweep, parareal_sweep  # noqa: E402
from pitwave.physics import ModelSpec, acoustic_advection_rhs  # noqa: E402

from paper_1510_02237_b200 import harness  # noqa: E402  (seeded generators only)

# fixtures come from the reference's default numba backend; PW_GOLDEN_ANY_BACKEND=1 lets
# make_window_golden.py measure the numba-vs-numpy noise floor with PITWAVE_KERNELS=numpy
assert BACKEND_NAME == "numba" or os.environ.get("PW_GOLDEN_ANY_BACKEND") == "1", \
    "golden fixtures are generated with the reference's default numba backend"


def rhs_cases():
    rng = np.random.default_rng(11)
    out = {}
    g = build_grid(16, 16, 1.0, 1.0)
    cases = []
    for vel_name, vel in (("const", ConstantVelocity(0.1, -0.05)), ("solid", SolidBodyRotation(np.pi))):
        for order in range(1, 7):
            for nu in (0.0, 0.02):
                cases.append((vel_name, vel, order, nu))
    states = []
    outs = []
    meta = []
    for vel_name, vel, order, nu in cases:
        model = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=order, sound_speed=1.3,
                          nu_damp=nu, damping_timescale=0.01 if nu > 0 else None)
        st = State(g, rng.standard_normal((3, 16, 16)))
        states.append(st.flatten())
        outs.append(acoustic_advection_rhs(st, model, g).flatten())
        meta.append((0 if vel_name == "const" else 1, order, nu))
    out["states"] = np.array(states)
    out["rhs"] = np.array(outs)
    out["meta"] = np.array(meta, dtype=np.float64)  # (vel kind, order, nu); cs=1.3, tau=0.01
    return out


def prop_cases():
    out = {}
    n = 64
    g = build_grid(n, n, 1.0, 1.0)
    vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
    fm = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=6, sound_speed=1.0,
                   nu_damp=0.005, damping_timescale=1.0)
    cm = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=1, sound_speed=1.0,
                   nu_damp=0.1, damping_timescale=1.0)
    fine = make_propagator(RK3, fm, g, 0.5)
    coarse = make_propagator(SPLIT_FE_FB, cm, g, 4.0, n_sound=16)
    q0 = harness.fine_batch_states(n=n, batch=2, seed=77)
    out["q0"] = q0
    out["fine16"] = np.array([propagate(fine, State.unflatten(g, q, ACOUSTIC), 0.0, 16 * fine.dt).flatten()
                              for q in q0])
    out["coarse2"] = np.array([propagate(coarse, State.unflatten(g, q, ACOUSTIC), 0.0, 2 * coarse.dt).flatten()
                               for q in q0])
    # solid-body rotation, odd order, 32x32 (the paper's velocity field)
    n2 = 32
    g2 = build_grid(n2, n2, 1.0, 1.0)
    sb = SolidBodyRotation(np.pi)
    fm2 = ModelSpec(kind=ACOUSTIC, vel=sb, advective_flux_order=5, sound_speed=30.0,
                    nu_damp=0.005, damping_timescale=1.0)
    cm2 = ModelSpec(kind=ACOUSTIC, vel=sb, advective_flux_order=1, sound_speed=30.0,
                    nu_damp=0.1, damping_timescale=1.0)
    fine2 = make_propagator(RK3, fm2, g2, 0.2)
    coarse2 = make_propagator(SPLIT_FE_FB, cm2, g2, 4.0, n_sound=4)
    q2 = harness.fine_batch_states(n=n2, batch=1, seed=78)[0]
    out["sb_q0"] = q2
    out["sb_fine20"] = propagate(fine2, State.unflatten(g2, q2, ACOUSTIC), 0.0, 20 * fine2.dt).flatten()
    out["sb_coarse3"] = propagate(coarse2, State.unflatten(g2, q2, ACOUSTIC), 0.0, 3 * coarse2.dt).flatten()
    return out


def slice_closures(wl):
    g = build_grid(wl.n, wl.n, 1.0, 1.0)
    vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
    fm = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=harness.FINE["order"],
                   sound_speed=harness.CS, nu_damp=harness.FINE["nu"], damping_timescale=1.0)
    cm = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=harness.COARSE["order"],
                   sound_speed=harness.CS, nu_damp=harness.COARSE["nu"], damping_timescale=1.0)
    fine = make_propagator(RK3, fm, g, harness.FINE["cfl"])
    coarse = make_propagator(SPLIT_FE_FB, cm, g, harness.COARSE["cfl"], n_sound=harness.COARSE["n_sound"])
    span = wl.slice_span

    def mk(spec):
        def run(vec):
            return propagate(spec, State.unflatten(g, vec, ACOUSTIC), 0.0, span).flatten()
        return run

    return mk(fine), mk(coarse)


def c1_cases():
    wl = harness.WORKLOADS["c1"]
    fine, coarse = slice_closures(wl)
    q0 = harness.initial_state("c1")
    hist = []
    ranks = []
    diag = []
    orig_update = ref_sub.Subspace.update

    def spy_update(self, states, images):
        new = orig_update(self, states, images)
        ranks.append(new.rank)
        return new

    import pitwave.parareal as ref_par
    orig_res = ref_par.iteration_residual

    def spy_res(prev, nxt):
        hist.append(np.stack([np.asarray(v) for v in nxt]))
        return orig_res(prev, nxt)

    ref_sub.Subspace.update = spy_update
    ref_par.iteration_residual = spy_res
    try:
        ends, res, sub = kse_sweep(q0, fine, coarse, wl.n_p, wl.n_it)
    finally:
        ref_sub.Subspace.update = orig_update
        ref_par.iteration_residual = orig_res
    out = {"q0": q0, "kse_hist": np.array(hist), "kse_res": np.array(res),
           "kse_ranks": np.array(ranks)}
    ends_o, res_o = parareal_sweep(q0, fine, coarse, wl.n_p, wl.n_it)
    out["orig_res"] = np.array(res_o)
    out["orig_final"] = np.array(ends_o)
    del diag
    return out


def small_cases():
    # the reference test seam: tests/test_parareal.py:245-265 (nx=8 production KSE window)
    g = build_grid(8, 8, 1, 1)
    model = ModelSpec(kind=ACOUSTIC, vel=SolidBodyRotation(np.pi), advective_flux_order=6,
                      sound_speed=30.0, nu_damp=0.005, damping_timescale=1.0)
    cmodel = ModelSpec(kind=ACOUSTIC, vel=SolidBodyRotation(np.pi), advective_flux_order=1,
                       sound_speed=30.0, nu_damp=0.1, damping_timescale=1.0)
    fine = make_propagator(RK3, model, g, 0.2)
    coarse = make_propagator(SPLIT_FE_FB, cmodel, g, 2.0, n_sound=4)
    from pitwave.parareal import KSE, PitConfig
    cfg = PitConfig(mode=KSE, fine=fine, coarse=coarse, n_p=3, n_it=2)
    fv, cv = cfg.vector_propagators()
    from pitwave.mesh import init_cosine_bump
    bump = init_cosine_bump(g, 0.5, 0.65)
    q0 = State.acoustic(g, bump, np.zeros_like(bump), np.zeros_like(bump)).flatten()
    ends, res, sub = kse_sweep(q0, fv, cv, 3, 2)
    return {"pde8_q0": q0, "pde8_ends": np.array(ends), "pde8_res": np.array(res),
            "pde8_rank": np.array(sub.rank)}


def main():
    np.savez_compressed(os.path.join(HERE, "rhs.npz"), **rhs_cases())
    np.savez_compressed(os.path.join(HERE, "prop.npz"), **prop_cases())
    np.savez_compressed(os.path.join(HERE, "c1_kse.npz"), **c1_cases())
    np.savez_compressed(os.path.join(HERE, "small_kse.npz"), **small_cases())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
