"""Device Parareal / KSE sweeps and subspace vs oracles and reference golden data (B200 only).

Parity rule: per config and iteration, max relative L2
per slice <= max(1e-10, 10 x the reference's own noise floor); c1's floor
is 1.6e-15, so 1e-10 is the bar there.
"""
import math

import numpy as np
import pytest

from conftest import floor_bound, golden
from oracle import oracle as orc
from paper_1510_02237_b200 import harness

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_02237_b200 import _lib

    return _lib.Context.get(0)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def mats(a_fine, a_coarse):
    from paper_1510_02237_b200.integrators import MatrixPropagator

    return MatrixPropagator(a_fine), MatrixPropagator(a_coarse)


# ----------------------------------------------------------------- dense seam
def test_dahlquist_golden_value():
    from paper_1510_02237_b200.parareal import parareal_sweep

    dt = 0.5
    fine, coarse = mats(np.array([[math.exp(-dt)]]), np.array([[1.0 - dt]]))
    ends, res = parareal_sweep(np.array([1.0]), fine, coarse, n_c=2, n_it=1)
    assert ends[0][0] == pytest.approx(math.exp(-0.5), rel=1e-12)
    assert ends[1][0] == pytest.approx(0.35653, abs=5e-6)
    ends, _ = parareal_sweep(np.array([1.0]), fine, coarse, n_c=2, n_it=2)
    assert ends[1][0] == pytest.approx(math.exp(-1.0), rel=1e-12)


def test_exactness_after_n_c_iterations_both_modes(rng):
    from paper_1510_02237_b200.parareal import kse_sweep, parareal_sweep

    d, n_c = 10, 4
    a_fine, a_coarse = orc.random_stable_pair(rng, d)
    fine, coarse = mats(a_fine, a_coarse)
    q0 = rng.standard_normal(d)
    seq = [q0]
    for _ in range(n_c):
        seq.append(a_fine @ seq[-1])
    ends, _ = parareal_sweep(q0, fine, coarse, n_c, n_it=n_c)
    for got, want in zip(ends, seq[1:]):
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    ends, _, _ = kse_sweep(q0, fine, coarse, n_c, n_it=n_c)
    for got, want in zip(ends, seq[1:]):
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_original_matches_dense_oracle(rng):
    from paper_1510_02237_b200.parareal import parareal_sweep

    d, n_c, n_it = 7, 3, 2
    a_fine, a_coarse = orc.random_stable_pair(rng, d)
    fine, coarse = mats(a_fine, a_coarse)
    q0 = rng.standard_normal(d)
    ends, res = parareal_sweep(q0, fine, coarse, n_c, n_it)
    o_ends, o_res = orc.dense_parareal_window(q0, a_fine, a_coarse, n_c, n_it)
    for got, want in zip(ends, o_ends):
        assert np.linalg.norm(got - want) <= 1e-13 * max(1.0, np.linalg.norm(want))
    np.testing.assert_allclose(res, o_res, rtol=1e-10)


def test_kse_matches_dense_oracle_random(rng):
    from paper_1510_02237_b200.parareal import kse_sweep

    for _ in range(10):
        d = int(rng.integers(4, 24))
        n_c = int(rng.integers(2, 5))
        n_it = int(rng.integers(1, 4))
        a_fine, a_coarse = orc.random_stable_pair(rng, d)
        fine, coarse = mats(a_fine, a_coarse)
        q0 = rng.standard_normal(d)
        ends, _, _ = kse_sweep(q0, fine, coarse, n_c, n_it)
        o_ends, _ = orc.dense_kse_window(q0, a_fine, a_coarse, n_c, n_it)
        for got, want in zip(ends, o_ends):
            assert np.linalg.norm(got - want) <= 1e-12 * max(1.0, np.linalg.norm(want))


def test_kse_converges_once_dimension_saturates(rng):
    from paper_1510_02237_b200.parareal import kse_sweep

    d, r = 8, 2
    w, _ = np.linalg.qr(rng.standard_normal((d, r)))
    b = np.array([[0.0, 1.0], [-1.0, -0.3]])
    a_fine = w @ (np.eye(r) + 0.3 * b + 0.045 * b @ b) @ w.T
    a_coarse = w @ (np.eye(r) + 0.3 * b) @ w.T
    fine, coarse = mats(a_fine, a_coarse)
    q0 = w @ np.array([1.0, -0.7])
    ends, res, sub = kse_sweep(q0, fine, coarse, n_c=3, n_it=3)
    assert sub.rank == r
    assert res[0] > 1e-6
    assert res[1] <= 1e-12


def test_tolerance_early_exit(rng):
    from paper_1510_02237_b200.parareal import parareal_sweep

    a_fine, _ = orc.random_stable_pair(rng, 6)
    fine, coarse = mats(a_fine, a_fine)
    _, res = parareal_sweep(rng.standard_normal(6), fine, coarse, n_c=4, n_it=10, tol=1e-10)
    assert len(res) < 10


def test_plain_callables_rejected():
    from paper_1510_02237_b200.parareal import kse_sweep

    with pytest.raises(TypeError):
        kse_sweep(np.ones(3), lambda q: q, lambda q: q, 2, 1)


# ----------------------------------------------------------------- subspace API
def test_subspace_reference_contract(rng):
    from paper_1510_02237_b200.subspace import Subspace, kse_coarse

    d = 12
    a_fine, a_coarse = orc.random_stable_pair(rng, d)
    states = [rng.standard_normal(d) for _ in range(4)]
    sub = Subspace(d).update(states, [a_fine @ s for s in states])
    assert sub.rank == 4
    np.testing.assert_allclose(sub.q.T @ sub.q, np.eye(4), atol=1e-12)
    gs = orc.gram_schmidt_basis(states)
    np.testing.assert_allclose(sub.q @ sub.q.T, gs @ gs.T, atol=1e-10)
    direct = a_fine @ sub.q
    assert np.linalg.norm(sub.fq - direct) <= 1e-10 * np.linalg.norm(direct)
    q = rng.standard_normal(d)
    once = sub.project(q)
    np.testing.assert_allclose(sub.project(once), once, atol=1e-12)
    s_mat = np.column_stack(states)
    coef = np.linalg.solve(s_mat.T @ s_mat, s_mat.T @ q)
    np.testing.assert_allclose(once, s_mat @ coef, atol=1e-11)
    from paper_1510_02237_b200.integrators import MatrixPropagator

    coarse = MatrixPropagator(a_coarse)
    pq = sub.project(q)
    want = a_coarse @ (q - pq) + a_fine @ pq
    got = kse_coarse(sub, coarse, q)
    assert np.linalg.norm(got - want) <= 1e-11 * np.linalg.norm(want)
    # duplicates collapse, incremental updates accumulate
    v = rng.standard_normal(d)
    assert Subspace(d).update([v, v.copy()], [v, v]).rank == 1
    sub2 = sub.update([rng.standard_normal(d) for _ in range(3)], [rng.standard_normal(d) for _ in range(3)])
    assert sub2.rank == 7 and sub2.snapshots.shape == (d, 7)
    np.testing.assert_array_equal(sub2.snapshots[:, :4], np.column_stack(states))
    with pytest.raises(ValueError, match="states"):
        Subspace(5).update([rng.standard_normal(5)], [])
    with pytest.raises(ValueError, match="dimension"):
        Subspace(5).update([rng.standard_normal(6)], [rng.standard_normal(6)])


def test_subspace_full_rank_and_empty(rng):
    from paper_1510_02237_b200.integrators import MatrixPropagator
    from paper_1510_02237_b200.subspace import Subspace, kse_coarse

    d = 6
    a_fine, a_coarse = orc.random_stable_pair(rng, d)
    states = [rng.standard_normal(d) for _ in range(d)]
    sub = Subspace(d).update(states, [a_fine @ s for s in states])
    assert sub.rank == d
    q = rng.standard_normal(d)
    got = kse_coarse(sub, MatrixPropagator(a_coarse), q)
    assert np.linalg.norm(got - a_fine @ q) <= 1e-9 * np.linalg.norm(a_fine @ q)
    empty = Subspace(7)
    np.testing.assert_allclose(empty.fine_on_projection(rng.standard_normal(7)), 0.0)


# ----------------------------------------------------------------- PDE windows vs reference
def c1_props():
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    wl = harness.WORKLOADS["c1"]
    g = build_grid(wl.n, wl.n)
    vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
    fine = make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5)
    coarse = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 4.0, 16)
    return wl, SlicePropagator(fine, wl.slice_span), SlicePropagator(coarse, wl.slice_span)


def test_c1_kse_history_matches_reference():
    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    for k in range(1, wl.n_it + 1):
        ends, res, sub = kse_sweep(g["q0"], fine, coarse, wl.n_p, k)
        assert sub.rank == g["kse_ranks"][k - 1]
        worst = max(rel(ends[i], g["kse_hist"][k - 1][i]) for i in range(wl.n_p))
        assert worst <= 1e-10, (k, worst)
        np.testing.assert_allclose(res, g["kse_res"][:k], rtol=1e-10)


def test_c1_kse_lean_mode_matches_reference(monkeypatch):
    """Lean sweep (no separate snapshot copy: the c4-on-one-GPU memory mode) gives the same
    window; the snapshot/image views then refuse instead of returning stale data."""
    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    monkeypatch.setenv("PW_SWEEP_LEAN", "1")
    ends, res, sub = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    assert sub.rank == g["kse_ranks"][-1]
    worst = max(rel(ends[i], g["kse_hist"][-1][i]) for i in range(wl.n_p))
    assert worst <= 1e-10, worst
    np.testing.assert_allclose(res, g["kse_res"], rtol=1e-10)
    with pytest.raises(RuntimeError):
        sub.snapshots
    assert sub.q.shape == (g["q0"].size, sub.rank)


@pytest.mark.parametrize("fold,from_r,implicit", [("0", "0", "1"), ("0", "1", "1"), ("1", "0", "1"),
                                                   ("1", "1", "0"), ("0", "0", "0")])
def test_c1_kse_regrouped_correction_forms_match_reference(monkeypatch, fold, from_r, implicit):
    """The serial correction's algebraic forms on one GPU: the folded correction
    D (alpha(qn_i) - alpha(qk_i)) (PW_FOLD_CORRECTION), the snapshot projections read off the
    pivoted factor (PW_ALPHA_FROM_R) and the implicit / explicit Q (PW_IMPLICIT_Q), in the
    combinations other than the default -- each against the reference's golden c1 history."""
    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    monkeypatch.setenv("PW_FOLD_CORRECTION", fold)
    monkeypatch.setenv("PW_ALPHA_FROM_R", from_r)
    monkeypatch.setenv("PW_IMPLICIT_Q", implicit)
    ends, res, sub = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    assert sub.rank == g["kse_ranks"][-1]
    worst = max(rel(ends[i], g["kse_hist"][-1][i]) for i in range(wl.n_p))
    assert worst <= 1e-10, worst
    np.testing.assert_allclose(res, g["kse_res"], rtol=1e-10)


@pytest.mark.parametrize("nsh", [2, 3, 5])
def test_c1_kse_row_sharded_serial_correction(dev, nsh):
    """The multi-GPU serial step (row shards of D and Q, partial alphas summed, rows
    gathered) run as nsh shards in one process: same window as the
    single-shard loop up to the order of the alpha partial sums."""
    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    ends1, res1, sub1 = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    dev.set_row_shards(nsh)
    try:
        ends, res, sub = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    finally:
        dev.set_row_shards(1)
    assert sub.rank == sub1.rank == g["kse_ranks"][-1]
    assert max(rel(ends[i], ends1[i]) for i in range(wl.n_p)) <= 1e-12
    assert max(rel(ends[i], g["kse_hist"][-1][i]) for i in range(wl.n_p)) <= 1e-10
    np.testing.assert_allclose(res, g["kse_res"], rtol=1e-10)


@pytest.mark.parametrize("nsh", [2, 3])
def test_c1_kse_tsqr_row_sharded_factorisation(dev, nsh):
    """Row-sharded subspace factorisation (distributed TSQR) with nsh shards in
    one process: every shard factors its rows, the stacked R factors are factored once more.
    Same ranks as the reference and the same window within the parity bound."""
    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    ends1, res1, sub1 = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    dev.set_row_shards(nsh)
    dev.set_tsqr(True)
    try:
        for k in range(1, wl.n_it + 1):
            ends, res, sub = kse_sweep(g["q0"], fine, coarse, wl.n_p, k)
            assert sub.rank == g["kse_ranks"][k - 1]
            worst = max(rel(ends[i], g["kse_hist"][k - 1][i]) for i in range(wl.n_p))
            assert worst <= 1e-10, (k, worst)
            np.testing.assert_allclose(res, g["kse_res"][:k], rtol=1e-10)
        # the span of Q is the replicated one's (Q Q^T equal), columns may differ in sign
        qa, qb = sub.q, sub1.q
        proj = qa @ (qa.T @ qb)
        assert np.linalg.norm(proj - qb) <= 1e-10 * np.linalg.norm(qb)
    finally:
        dev.set_tsqr(False)
        dev.set_row_shards(1)


def test_c1_original_matches_reference():
    from paper_1510_02237_b200.parareal import parareal_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    ends, res = parareal_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    np.testing.assert_allclose(res, g["orig_res"], rtol=1e-12)
    for i in range(wl.n_p):
        assert rel(ends[i], g["orig_final"][i]) <= 1e-12


def test_c1_kse_strict_mode_matches_reference(dev):
    """Every kernel in reference operation order (strict): the c1 window vs the reference run."""
    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    dev.set_strict(True)
    try:
        ends, res, sub = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    finally:
        dev.set_strict(False)
    assert sub.rank == g["kse_ranks"][-1]
    worst = max(rel(ends[i], g["kse_hist"][-1][i]) for i in range(wl.n_p))
    assert worst <= 1e-12, worst
    np.testing.assert_allclose(res, g["kse_res"], rtol=1e-12)


def test_edge_cases_zero_state_single_slice_and_tol():
    """Zero initial state (empty subspace: rank 0), n_c = 1, and a PDE tol early exit."""
    from paper_1510_02237_b200.parareal import kse_sweep, parareal_sweep

    wl, fine, coarse = c1_props()
    d = 3 * wl.n * wl.n
    ends, res, sub = kse_sweep(np.zeros(d), fine, coarse, 4, 2)
    assert sub.rank == 0 and res == [0.0, 0.0]
    assert all(np.count_nonzero(e) == 0 for e in ends)
    q0 = harness.initial_state("c1")
    ends1, res1, _ = kse_sweep(q0, fine, coarse, 1, 2)
    np.testing.assert_allclose(ends1[0], fine(q0), rtol=0, atol=1e-14)   # one slice: exact after 1 iteration
    assert res1[1] == 0.0
    _, res_t = parareal_sweep(q0, fine, coarse, wl.n_p, 12, tol=1e-6)
    assert len(res_t) <= wl.n_p + 1 and res_t[-1] <= 1e-6     # exact after n_c iterations
    with pytest.raises(ValueError):
        kse_sweep(q0, fine, coarse, 0, 1)
    with pytest.raises(ValueError):
        kse_sweep(q0[:-3], fine, coarse, 2, 1)


def test_pde8_production_window_matches_reference():
    """nx=8 solid-body production window (reference tests/test_parareal.py:245-265 seam)."""
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, SolidBodyRotation, build_grid
    from paper_1510_02237_b200.parareal import KSE, PitConfig, kse_sweep
    from paper_1510_02237_b200.physics import ModelSpec

    g = golden("small_kse.npz")
    grid = build_grid(8, 8)
    sb = SolidBodyRotation(np.pi)
    fine = make_propagator(RK3, ModelSpec(ACOUSTIC, sb, 6, 30.0, 0.005, 1.0), grid, 0.2)
    coarse = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, sb, 1, 30.0, 0.1, 1.0), grid, 2.0, 4)
    cfg = PitConfig(mode=KSE, fine=fine, coarse=coarse, n_p=3, n_it=2)
    fv, cv = cfg.vector_propagators()
    ends, res, sub = kse_sweep(g["pde8_q0"], fv, cv, 3, 2)
    assert sub.rank == int(g["pde8_rank"])
    for got, want in zip(ends, g["pde8_ends"]):
        assert np.linalg.norm(got - want) <= 1e-11 * max(1.0, np.linalg.norm(want))
    np.testing.assert_allclose(res, g["pde8_res"], rtol=1e-9)


def test_run_windowed_converged_matches_sequential():
    """n_it = n_c: every window exact, chained windows reproduce the fine run (test_parareal.py:186-199)."""
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, make_propagator, propagate
    from paper_1510_02237_b200.mesh import ACOUSTIC, SolidBodyRotation, State, build_grid, init_cosine_bump
    from paper_1510_02237_b200.parareal import KSE, PitConfig, run_windowed
    from paper_1510_02237_b200.physics import ModelSpec

    grid = build_grid(16, 16)
    sb = SolidBodyRotation(np.pi)
    fine = make_propagator(RK3, ModelSpec(ACOUSTIC, sb, 6, 30.0, 0.005, 1.0), grid, 0.2)
    coarse = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, sb, 1, 30.0, 0.1, 1.0), grid, 2.0, 4)
    cfg = PitConfig(mode=KSE, fine=fine, coarse=coarse, n_p=4, n_it=4)
    bump = init_cosine_bump(grid, 0.5, 0.65)
    q0 = State.acoustic(grid, bump, np.zeros_like(bump), np.zeros_like(bump))
    t_end = 2 * cfg.n_p * cfg.coarse.dt
    rep = run_windowed(cfg, q0, t_end)
    seq = propagate(fine, q0, 0.0, t_end)
    assert rel(rep.final_state.fields, seq.fields) <= 1e-10
    assert len(rep.window_endpoints) == 2 and rep.blowup_time is None
    assert rep.timings.fine > 0 and rep.timings.coarse > 0


def test_kse_residual_and_ranks_against_oracle_c1_shape_p16():
    """A 64^2, P=16, K=3 window (deeper than the golden case) against the oracle."""
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.parareal import kse_sweep
    from paper_1510_02237_b200.physics import ModelSpec

    n, p, k, span = 64, 16, 3, 1.0 / 16
    grid = build_grid(n, n)
    vel = ConstantVelocity(0.1, 0.0)
    fine = SlicePropagator(make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), grid, 0.5), span)
    coarse = SlicePropagator(make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), grid, 4.0, 16), span)
    q0 = harness.initial_state("c3", n=n)
    ends, res, sub = kse_sweep(q0, fine, coarse, p, k)
    of = orc.SlicePropagator(orc.RK3, fine.nsteps, nx=n, ny=n, cs=1.0, order=6, nu=0.005, cfl=0.5,
                             velocity=("constant", 0.1, 0.0))
    oc = orc.SlicePropagator(orc.SPLIT_FE_FB, coarse.nsteps, nx=n, ny=n, cs=1.0, order=1, nu=0.1,
                             cfl=4.0, n_sound=16, velocity=("constant", 0.1, 0.0))
    ranks = []
    o_ends, o_res, o_sub = orc.kse_sweep(q0, of, oc, p, k, ranks=ranks)
    assert sub.ranks_history == ranks
    worst = max(rel(a, b) for a, b in zip(ends, o_ends))
    bound = floor_bound("c1_shape_p16", k)
    print(f"c1 shape P=16: max rel L2 per slice vs oracle {worst:.3e} (bound {bound:.1e})")
    assert worst <= bound, worst
    np.testing.assert_allclose(res, o_res, rtol=floor_bound("c1_shape_p16", k, "residual"))


@pytest.mark.parametrize("d,ld,r,g_null", [(786432, 786432, 310, False), (200000, 200000, 1024, False),
                                          (4096, 5000, 600, True), (1001, 1001, 37, False),
                                          (100000, 100002, 0, False)])
def test_serial_step_kernel_against_torch(dev, d, ld, r, g_null):
    """The fused serial-step pass (TMA ring; LSU kernel for odd d / misaligned blocks) on
    caller buffers: y = g + c + D alpha, alpha' = Q^T y, against torch fp64 GEMV."""
    from paper_1510_02237_b200 import _lib

    gen = torch.Generator(device="cuda").manual_seed(d + r)
    rr = max(r, 1)
    Dm = torch.randn(rr, ld, device="cuda", dtype=torch.float64, generator=gen)  # column k = row k
    Qm = torch.randn(rr, ld, device="cuda", dtype=torch.float64, generator=gen)
    g = torch.randn(d, device="cuda", dtype=torch.float64, generator=gen)
    c = torch.randn(d, device="cuda", dtype=torch.float64, generator=gen)
    a = torch.randn(rr, device="cuda", dtype=torch.float64, generator=gen)
    y = torch.empty(d, device="cuda", dtype=torch.float64)
    an = torch.zeros(rr, device="cuda", dtype=torch.float64)
    _lib.check(dev.lib.pw_serial_step(dev.handle, None if g_null else _lib.ptr(g), _lib.ptr(Dm), r,
                                      _lib.ptr(c), _lib.ptr(a), _lib.ptr(Qm), r, d, ld, _lib.ptr(y),
                                      _lib.ptr(an)))
    want_y = (c if g_null else g + c) + (Dm[:r, :d].T @ a[:r] if r else 0.0)
    assert torch.linalg.norm(y - want_y) <= 1e-13 * torch.linalg.norm(want_y)
    if r:
        want_a = Qm[:r, :d] @ want_y
        assert torch.linalg.norm(an[:r] - want_a) <= 1e-12 * torch.linalg.norm(want_a)


def test_sharded_fine_hook_single_rank_group():
    """The multi-GPU fine hook (pw_ctx_set_fine_hook + dist.ShardedFine) on a 1-rank NCCL group."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    wl, fine, coarse = c1_props()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ends_g, res_g, _ = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it, group=dist.group.WORLD)
        import bench  # the collective self-test bench.py runs before multi-GPU windows

        assert bench.comm_selftest(dist)
    finally:
        dist.destroy_process_group()
    ends, res, _ = kse_sweep(g["q0"], fine, coarse, wl.n_p, wl.n_it)
    np.testing.assert_array_equal(np.array(ends_g), np.array(ends))
    assert res_g == res


@pytest.mark.parametrize("tsqr_shards", [0, 2])
def test_c5_shaped_window_against_oracle(dev, tsqr_shards):
    """c5 physics and initial-state generator (all three fields random modes, |k| <= 32) on a
    128^2 grid, P=16, K=3 (the full c5 needs 8 GPUs): ranks and states against the oracle,
    replicated and with the row-sharded TSQR factorisation (2 in-process shards)."""
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.parareal import kse_sweep
    from paper_1510_02237_b200.physics import ModelSpec

    n, p, k, span = 128, 16, 3, 1.0 / 16
    grid = build_grid(n, n)
    vel = ConstantVelocity(0.1, 0.0)
    fine = SlicePropagator(make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), grid, 0.5), span)
    coarse = SlicePropagator(make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), grid, 4.0, 16), span)
    q0 = harness.initial_state("c5", n=n)
    if tsqr_shards:
        dev.set_row_shards(tsqr_shards)
        dev.set_tsqr(True)
    try:
        ends, res, sub = kse_sweep(q0, fine, coarse, p, k)
    finally:
        dev.set_tsqr(False)
        dev.set_row_shards(1)
    of = orc.SlicePropagator(orc.RK3, fine.nsteps, nx=n, ny=n, cs=1.0, order=6, nu=0.005, cfl=0.5,
                             velocity=("constant", 0.1, 0.0))
    oc = orc.SlicePropagator(orc.SPLIT_FE_FB, coarse.nsteps, nx=n, ny=n, cs=1.0, order=1, nu=0.1,
                             cfl=4.0, n_sound=16, velocity=("constant", 0.1, 0.0))
    ranks = []
    o_ends, o_res, _ = orc.kse_sweep(q0, of, oc, p, k, ranks=ranks)
    assert sub.ranks_history == ranks
    worst = max(rel(a, b) for a, b in zip(ends, o_ends))
    bound = floor_bound("c5_shape_128", k)
    print(f"c5 shape 128^2 (tsqr shards {tsqr_shards}): max rel L2 per slice vs oracle {worst:.3e} "
          f"(bound {bound:.1e})")
    assert worst <= bound, worst
    np.testing.assert_allclose(res, o_res, rtol=floor_bound("c5_shape_128", k, "residual"))
