"""Reference noise floors of the reduced-shape KSE windows (this container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_floor_golden.py

SURVEY.md 8(c)'s parity rule: per config and iteration, the device's max relative L2
per slice must be <= max(1e-10, 10 x the reference's OWN reproducibility floor), the
floor being the deviation between two runs of the reference that differ only in its
kernel backend (PITWAVE_KERNELS=numba vs numpy; the order-1 flux rounds differently,
numpy_backend.py:27-28 vs numba_backend.py:17).  This script runs the reference's
kse_sweep on each reduced-shape window the GPU tests use, once per backend (each in
its own process: the backend is chosen at import), and writes per-iteration floors:
max over slices of ||q_numba - q_numpy|| / ||q_numba|| of qn[1:] after every iteration,
and the relative residual difference, to floors.json next to this script.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))

# name -> (n, P, K, initial-state generator, slice span): the shapes of
# tests/test_gpu_sweeps.py (c1 shape P=16, c5-shaped 128^2) and the BASELINE c1 window
CASES = {
    "c1": (64, 8, 3, "c1", 1.0 / 8),
    "c1_shape_p16": (64, 16, 3, "c3", 1.0 / 16),
    "c5_shape_128": (128, 16, 3, "c5", 1.0 / 16),
}


def run_case(name):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    from pitwave import parareal as ref_par
    from pitwave.integrators import RK3, SPLIT_FE_FB, make_propagator, propagate
    from pitwave.mesh import ACOUSTIC, ConstantVelocity, State, build_grid
    from pitwave.physics import ModelSpec

    from paper_1510_02237_b200 import harness

    n, p, k, gen, span = CASES[name]
    g = build_grid(n, n)
    vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
    fm = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=6, sound_speed=1.0, nu_damp=0.005,
                   damping_timescale=1.0)
    cm = ModelSpec(kind=ACOUSTIC, vel=vel, advective_flux_order=1, sound_speed=1.0, nu_damp=0.1,
                   damping_timescale=1.0)
    fine = make_propagator(RK3, fm, g, 0.5)
    coarse = make_propagator(SPLIT_FE_FB, cm, g, 4.0, n_sound=16)

    def mk(spec):
        return lambda v: propagate(spec, State.unflatten(g, v, ACOUSTIC), 0.0, span).flatten()

    q0 = harness.initial_state(gen, n=n)
    hist = []
    orig = ref_par.iteration_residual

    def spy(prev, nxt):
        hist.append(np.stack([np.asarray(v) for v in nxt]))
        return orig(prev, nxt)

    ref_par.iteration_residual = spy
    try:
        _, res, _ = ref_par.kse_sweep(q0, mk(fine), mk(coarse), p, k)
    finally:
        ref_par.iteration_residual = orig
    return np.array(hist), np.array(res)


def main():
    if len(sys.argv) == 3 and sys.argv[1] == "--one":  # child: one backend, all cases
        out = {}
        for name in CASES:
            st, res = run_case(name)
            out[f"{name}_states"] = st
            out[f"{name}_res"] = res
        np.savez(sys.argv[2], **out)
        return
    tmp = {}
    for backend in ("numba", "numpy"):
        path = f"/tmp/pw_floor_{backend}.npz"
        env = dict(os.environ, PITWAVE_KERNELS=backend)
        subprocess.run([sys.executable, __file__, "--one", path], check=True, env=env)
        tmp[backend] = np.load(path)
    floors = {}
    for name in CASES:
        a, b = tmp["numba"][f"{name}_states"], tmp["numpy"][f"{name}_states"]
        per_it = [float(np.max(np.linalg.norm(a[k] - b[k], axis=1) / np.linalg.norm(a[k], axis=1)))
                  for k in range(a.shape[0])]
        ra, rb = tmp["numba"][f"{name}_res"], tmp["numpy"][f"{name}_res"]
        floors[name] = {"state": per_it, "residual": [float(abs(x - y) / abs(x)) for x, y in zip(ra, rb)],
                        "shape": {"n": CASES[name][0], "P": CASES[name][1], "K": CASES[name][2], "init": CASES[name][3]}}
    with open(os.path.join(HERE, "floors.json"), "w") as fh:
        json.dump(floors, fh, indent=1)
    print(json.dumps(floors, indent=1))


if __name__ == "__main__":
    main()
