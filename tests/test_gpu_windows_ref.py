"""c3 / c4 KSE windows against the REFERENCE's own runs of the same windows
(tests/golden/make_window_golden.py: residuals, ranks, per-slice norms and 512
fixed-seed sampled entries per slice of qn[1:] after every iteration).

Tolerance: SURVEY.md 8(c) -- per iteration, the deviation statistic (max over slices
of the relative norm difference and the relative L2 difference of the sampled
entries) must be <= max(1e-10, 10 x the reference's OWN floor), where the floor is
the same statistic between the reference's numba run (<config>_reference.npz) and
its numpy-backend run of the same window (<config>_reference_numpy.npz, same
script with PITWAVE_KERNELS=numpy).  Iterations without a numpy-backend fixture
fall back to the survey's c3 floor (Appendix A) or, for c4, to 1e-5, and say so.
"""
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_1510_02237_b200 import harness

pytestmark = pytest.mark.gpu

# fallbacks when no numpy-backend fixture exists: the survey's c3 stable-G floor
# (Appendix A; another seed, indicative) and the survey's expected c4 level
FALLBACK_FLOOR = {"c3": [2.8e-9, 1.1e-8, 9.0e-9, 3.6e-8, 2.1e-7], "c4": [1e-6] * 4}


def _stat(a_norms, a_samp, b_norms, b_samp):
    d_norm = np.max(np.abs(a_norms - b_norms) / b_norms)
    d_samp = np.max(np.linalg.norm(a_samp - b_samp, axis=1) / np.linalg.norm(b_samp, axis=1))
    return float(max(d_norm, d_samp))


def measured_floor(name):
    """Per-iteration reference floor (numba vs numpy fixture), or the fallback."""
    ref = np.load(os.path.join(GOLDEN, f"{name}_reference.npz"))
    path = os.path.join(GOLDEN, f"{name}_reference_numpy.npz")
    out = list(FALLBACK_FLOOR[name])
    src = ["fallback"] * len(out)
    if os.path.exists(path):
        alt = np.load(path)
        assert np.array_equal(alt["idx"], ref["idx"])
        for k in range(min(len(alt["res"]), len(ref["res"]))):
            out[k] = _stat(alt["norms"][k], alt["samples"][k], ref["norms"][k], ref["samples"][k])
            src[k] = "measured"
    print(f"{name} reference floor per iteration: " +
          ", ".join(f"{f:.2e} ({s})" for f, s in zip(out, src)))
    return out


def bounds(name):
    return [max(1e-10, 10.0 * f) for f in measured_floor(name)]


def props(name):
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    wl = harness.WORKLOADS[name]
    g = build_grid(wl.n, wl.n)
    vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
    fine = make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5)
    coarse = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 4.0, 16)
    return wl, SlicePropagator(fine, wl.slice_span), SlicePropagator(coarse, wl.slice_span)


def check_window(name, tol_per_iteration):
    from paper_1510_02237_b200.parareal import kse_sweep

    path = os.path.join(GOLDEN, f"{name}_reference.npz")
    if not os.path.exists(path):
        pytest.skip(f"{name}_reference.npz not generated")
    g = np.load(path)
    wl, fine, coarse = props(name)
    n_it = len(g["res"])
    q0 = torch.as_tensor(harness.initial_state(name)).cuda()
    idx = torch.as_tensor(g["idx"]).cuda()
    worst = []
    for k in range(1, n_it + 1):
        ends, res, sub = kse_sweep(q0, fine, coarse, wl.n_p, k, return_device=True)
        st = torch.stack(list(ends)) if isinstance(ends, (list, tuple)) else ends
        st = st.reshape(wl.n_p, -1)
        norms = torch.linalg.norm(st, dim=1).cpu().numpy()
        samp = st[:, idx].cpu().numpy()
        want_n, want_s = g["norms"][k - 1], g["samples"][k - 1]
        worst.append(_stat(norms, samp, want_n, want_s))
        d_res = abs(res[-1] - g["res"][k - 1]) / abs(g["res"][k - 1])
        print(f"{name} iteration {k}: rank {sub.rank} (ref {g['ranks'][k - 1]}), state deviation "
              f"{worst[-1]:.3e}, residual deviation {d_res:.3e}", flush=True)
        assert sub.rank == g["ranks"][k - 1], (k, sub.rank, g["ranks"][k - 1])
        np.testing.assert_allclose(res, g["res"][:k], rtol=max(1e-10, tol_per_iteration[k - 1]))
        assert worst[-1] <= tol_per_iteration[k - 1], (k, worst[-1])
        del ends, st, sub
        torch.cuda.empty_cache()
    print(f"{name}: per-iteration max relative deviation vs the reference run: {worst}")


def test_c3_window_matches_reference_run():
    check_window("c3", bounds("c3"))


def test_c3_window_tsqr_two_row_shards_matches_reference_run():
    """The c3 window with the row-sharded (TSQR) factorisation and row-sharded serial
    correction over 2 shards in one process: ranks equal to the reference run, states
    within the same bound as the replicated path."""
    from paper_1510_02237_b200 import _lib

    ctx = _lib.Context.get(0)
    ctx.set_row_shards(2)
    ctx.set_tsqr(True)
    try:
        check_window("c3", bounds("c3"))
    finally:
        ctx.set_tsqr(False)
        ctx.set_row_shards(1)


def test_c4_window_matches_reference_run():
    """c4 (1024^2, P=256) against the reference's run, every iteration the fixture holds.
    The rank gap is tight here (kept min |R_jj|/|R_11| 1.36e-10 against dropped max
    9.45e-11 at iteration 1, cond(R11) ~ 7e9), so two QR algorithms legitimately differ at
    eps * cond ~ 1e-6; the bound is 10 x the reference's own numba-vs-numpy floor."""
    check_window("c4", bounds("c4"))


def test_c3_original_parareal_window_matches_reference_run():
    """c3 with the ORIGINAL Parareal sweep (parareal.py:68-97, no subspace) against the
    reference's own run (tests/golden/make_parareal_window_golden.py).  No ill-conditioned
    factorisation is involved, so the north star's 1e-10 per slice and iteration applies as is."""
    from paper_1510_02237_b200.parareal import parareal_sweep

    path = os.path.join(GOLDEN, "c3_parareal_reference.npz")
    if not os.path.exists(path):
        pytest.skip("c3_parareal_reference.npz not generated")
    g = np.load(path)
    wl, fine, coarse = props("c3")
    q0 = torch.as_tensor(harness.initial_state("c3")).cuda()
    idx = torch.as_tensor(g["idx"]).cuda()
    worst = []
    for k in range(1, len(g["res"]) + 1):
        ends, res = parareal_sweep(q0, fine, coarse, wl.n_p, k, return_device=True)
        st = (torch.stack(list(ends)) if isinstance(ends, (list, tuple)) else ends).reshape(wl.n_p, -1)
        norms = torch.linalg.norm(st, dim=1).cpu().numpy()
        samp = st[:, idx].cpu().numpy()
        worst.append(_stat(norms, samp, g["norms"][k - 1], g["samples"][k - 1]))
        np.testing.assert_allclose(res, g["res"][:k], rtol=1e-10)
        assert worst[-1] <= 1e-10, (k, worst[-1])
    print(f"c3 original Parareal: per-iteration max relative deviation vs the reference run: {worst}")
