"""Device kernels vs the oracle and the reference's golden outputs (B200 only).

Tolerances: bitwise where the device runs the reference operation order
(strict RK3, split FE-FB coarse); <= 1e-12 relative L2 for the folded fused
RK3 kernel, whose arithmetic differs from the reference only by rounding.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as orc
from paper_1510_02237_b200 import harness

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_02237_b200 import _lib

    ctx = _lib.Context.get(0)
    ctx.set_strict(False)
    yield ctx
    ctx.set_strict(False)


def make_specs(n, *, U=0.1, V=0.0, fine_order=6, nu_f=0.005, cs=1.0, fine_cfl=0.5, coarse_cfl=4.0,
               n_sound=16, velocity=None):
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    g = build_grid(n, n)
    vel = velocity if velocity is not None else ConstantVelocity(U, V)
    fm = ModelSpec(ACOUSTIC, vel, fine_order, cs, nu_f, 1.0 if nu_f > 0 else None)
    cm = ModelSpec(ACOUSTIC, vel, 1, cs, 0.1, 1.0)
    return make_propagator(RK3, fm, g, fine_cfl), make_propagator(SPLIT_FE_FB, cm, g, coarse_cfl, n_sound)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_strict_fine_is_bitwise_with_reference(dev):
    from paper_1510_02237_b200.integrators import SlicePropagator

    g = golden("prop.npz")
    fspec, _ = make_specs(64)
    dev.set_strict(True)
    try:
        prop = SlicePropagator(fspec, nsteps=16)
        got = prop.batch(g["q0"])
    finally:
        dev.set_strict(False)
    np.testing.assert_array_equal(got, g["fine16"])


def test_coarse_is_bitwise_with_reference(dev):
    from paper_1510_02237_b200.integrators import SlicePropagator

    g = golden("prop.npz")
    _, cspec = make_specs(64)
    got = SlicePropagator(cspec, nsteps=2).batch(g["q0"])
    np.testing.assert_array_equal(got, g["coarse2"])


def test_solid_body_fine_and_coarse_bitwise(dev):
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, SolidBodyRotation, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    g = golden("prop.npz")
    grid = build_grid(32, 32)
    sb = SolidBodyRotation(np.pi)
    fine = make_propagator(RK3, ModelSpec(ACOUSTIC, sb, 5, 30.0, 0.005, 1.0), grid, 0.2)
    coarse = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, sb, 1, 30.0, 0.1, 1.0), grid, 4.0, 4)
    np.testing.assert_array_equal(SlicePropagator(fine, nsteps=20)(g["sb_q0"]), g["sb_fine20"])
    np.testing.assert_array_equal(SlicePropagator(coarse, nsteps=3)(g["sb_q0"]), g["sb_coarse3"])


@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("U,V", [(0.1, 0.0), (-0.3, 0.2)])
def test_fused_fine_matches_oracle(dev, order, U, V):
    from paper_1510_02237_b200.integrators import SlicePropagator

    n = 64
    fspec, _ = make_specs(n, U=U, V=V, fine_order=order)
    q0 = harness.fine_batch_states(n=n, batch=3, seed=5)
    prop = SlicePropagator(fspec, nsteps=7)
    got = prop.batch(q0)
    o = orc.SlicePropagator(orc.RK3, 7, nx=n, ny=n, cs=1.0, order=order, nu=0.005, cfl=0.5,
                            velocity=("constant", U, V))
    want = o.batch(q0)
    for b in range(3):
        assert rel(got[b], want[b]) <= 1e-12


@pytest.mark.parametrize("n", [8, 16, 32, 96, 128, 1024])
def test_fused_fine_small_and_odd_tilings(dev, n):
    from paper_1510_02237_b200.integrators import SlicePropagator

    fspec, _ = make_specs(n, U=0.1, V=0.05)
    q0 = harness.fine_batch_states(n=n, batch=2, seed=9)
    got = SlicePropagator(fspec, nsteps=4).batch(q0)
    want = orc.SlicePropagator(orc.RK3, 4, nx=n, ny=n, cs=1.0, order=6, nu=0.005, cfl=0.5,
                               velocity=("constant", 0.1, 0.05)).batch(q0)
    for b in range(2):
        assert rel(got[b], want[b]) <= 1e-12


def test_fused_fine_c2_shape_against_oracle(dev):
    """c2 grid (256^2) on a 4-state sample, 20 steps: fused kernel vs oracle."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    n = 256
    fspec, _ = make_specs(n)
    q0 = harness.fine_batch_states(n=n, batch=4, seed=2001)
    got = SlicePropagator(fspec, nsteps=20).batch(q0)
    want = orc.SlicePropagator(orc.RK3, 20, nx=n, ny=n, cs=1.0, order=6, nu=0.005, cfl=0.5,
                               velocity=("constant", 0.1, 0.0)).batch(q0)
    for b in range(4):
        assert rel(got[b], want[b]) <= 1e-12


def test_fine_linearity_full_c2_batch(dev):
    """Size-independent property at the full c2 batch (64 x 256^2): F(a x + b y) = a F(x) + b F(y)."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    fspec, _ = make_specs(256)
    prop = SlicePropagator(fspec, nsteps=10)
    x = torch.as_tensor(harness.fine_batch_states(n=256, batch=64, seed=2001)).cuda()
    y = torch.roll(x, shifts=1, dims=0)
    a, b = 0.3, -1.7
    lhs = prop.apply(a * x + b * y)
    rhs = a * prop.apply(x) + b * prop.apply(y)
    err = (torch.linalg.vector_norm(lhs - rhs, dim=1) / torch.linalg.vector_norm(rhs, dim=1)).max().item()
    assert err <= 1e-13
    assert torch.isfinite(lhs).all()


def test_in_place_apply_and_zero_steps(dev):
    from paper_1510_02237_b200.integrators import SlicePropagator

    fspec, cspec = make_specs(32)
    q0 = torch.as_tensor(harness.fine_batch_states(n=32, batch=2, seed=3)).cuda()
    for spec in (fspec, cspec):
        prop = SlicePropagator(spec, nsteps=3)
        ref = prop.apply(q0.clone())
        x = q0.clone()
        prop.apply(x, out=x)
        assert torch.equal(x, ref)
    z = SlicePropagator(fspec, nsteps=0).apply(q0)
    assert torch.equal(z, q0)


def test_propagate_api_and_composition_bitwise(dev):
    from paper_1510_02237_b200.integrators import propagate
    from paper_1510_02237_b200.mesh import ACOUSTIC, State

    fspec, _ = make_specs(32)
    st = State.unflatten(fspec.grid, harness.fine_batch_states(n=32, batch=1, seed=4)[0], ACOUSTIC)
    h = fspec.dt
    full = propagate(fspec, st, 0.0, 8 * h)
    half = propagate(fspec, propagate(fspec, st, 0.0, 4 * h), 4 * h, 8 * h)
    np.testing.assert_array_equal(full.fields, half.fields)
    assert propagate(fspec, st, 0.5, 0.5) is st
    with pytest.raises(ValueError, match="integer"):
        propagate(fspec, st, 0.0, 2.5 * h)


@pytest.mark.parametrize("n,batch", [(256, 1), (256, 2), (512, 1), (512, 2), (1024, 1), (96, 1)])
def test_tiled_coarse_bitwise_with_global_variant(dev, n, batch):
    """Temporal-blocked FE-FB (single state: tall tiles, 3 substeps per barrier; batches:
    32^2 tiles, 2 substeps) == per-cell global variant (strict mode), bitwise."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    _, cspec = make_specs(n)
    q0 = torch.as_tensor(harness.fine_batch_states(n=n, batch=batch, seed=13)).cuda()
    tiled = SlicePropagator(cspec, nsteps=2).apply(q0)
    dev.set_strict(True)
    try:
        ref = SlicePropagator(cspec, nsteps=2).apply(q0)
    finally:
        dev.set_strict(False)
    assert torch.equal(tiled, ref)


def test_blowup_is_not_an_error(dev):
    """Unstable coarse steps overflow quietly (integrators.py:141-145)."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    _, cspec = make_specs(32, coarse_cfl=40.0, n_sound=1)
    q0 = harness.fine_batch_states(n=32, batch=1, seed=8)
    out = SlicePropagator(cspec, nsteps=400)(q0[0])
    assert not np.isfinite(out).all()


def test_fine_on_the_c5_grid_against_oracle(dev):
    """Largest BASELINE grid (c5: 2048^2, ~100 MB per state): one seeded c5 state, 2 RK3
    steps, fused kernel vs the oracle (<= 1e-12 relative)."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    n = 2048
    fspec, _ = make_specs(n)
    q0 = harness.initial_state("c5")[None, :]
    got = SlicePropagator(fspec, nsteps=2).batch(q0)
    want = orc.SlicePropagator(orc.RK3, 2, nx=n, ny=n, cs=1.0, order=6, nu=0.005, cfl=0.5,
                               velocity=("constant", 0.1, 0.0)).batch(q0)
    assert rel(got[0], want[0]) <= 1e-12
