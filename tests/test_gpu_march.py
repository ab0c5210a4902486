"""Row-marching fused RK3 kernels (K1: csrc/march_tma.cu; previous generation
csrc/fine_march.cu) vs the oracle (B200 only).

The marching kernels serve V = 0 on grids with nx in {128, 256, 384, 512}.
Tolerance: <= 1e-12 relative L2 per state, as for the tile kernel (its
arithmetic differs from the reference only by rounding).  Cases cover every
flux order, non-square grids, ny not a multiple of the segment count
(ragged segments), the smallest supported ny, strided batches and the full
c2 batch (linearity, and agreement with the tile kernel).
"""

import numpy as np
import pytest

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

def fine_spec(nx, ny, order=6, U=0.1, nu=0.005):
    from paper_1510_02237_b200.integrators import RK3, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    g = build_grid(nx, ny)
    return make_propagator(RK3, ModelSpec(ACOUSTIC, ConstantVelocity(U, 0.0), order, 1.0, nu, 1.0), g, 0.5)

def oracle_batch(q0, nsteps, nx, ny, order=6, U=0.1, nu=0.005):
    return orc.SlicePropagator(orc.RK3, nsteps, nx=nx, ny=ny, cs=1.0, order=order, nu=nu, cfl=0.5,
                               velocity=("constant", U, 0.0)).batch(q0)

def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)

def random_states(nx, ny, batch, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((batch, 3 * nx * ny))

@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 6])
def test_march_orders_match_oracle(dev, order):
    from paper_1510_02237_b200.integrators import SlicePropagator

    nx, ny = 128, 64
    q0 = random_states(nx, ny, 3, 11 + order)
    got = SlicePropagator(fine_spec(nx, ny, order=order), nsteps=5).batch(q0)
    want = oracle_batch(q0, 5, nx, ny, order=order)
    for b in range(3):
        assert rel(got[b], want[b]) <= 1e-12

@pytest.mark.parametrize("nx,ny", [(128, 32), (128, 200), (256, 96), (384, 48), (512, 64), (256, 256),
                                   (1024, 48), (2048, 32)])
def test_march_grids_match_oracle(dev, nx, ny, monkeypatch):
    from paper_1510_02237_b200.integrators import SlicePropagator

    monkeypatch.setenv("PW_MARCH_CLUSTER", "1")  # 1024 / 2048: the cluster variant (opt-in)
    q0 = random_states(nx, ny, 2, nx + ny)
    got = SlicePropagator(fine_spec(nx, ny), nsteps=3).batch(q0)
    want = oracle_batch(q0, 3, nx, ny)
    for b in range(2):
        assert rel(got[b], want[b]) <= 1e-12

@pytest.mark.parametrize("nseg", ["1", "3", "7"])
def test_march_segment_counts(dev, nseg, monkeypatch):
    """Ragged y-segments (ny not divisible by the segment count) give the same states."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    nx, ny = 256, 100
    q0 = random_states(nx, ny, 2, 5)
    monkeypatch.setenv("PW_MARCH_NSEG", nseg)
    got = SlicePropagator(fine_spec(nx, ny), nsteps=2).batch(q0)
    want = oracle_batch(q0, 2, nx, ny)
    for b in range(2):
        assert rel(got[b], want[b]) <= 1e-12

def test_march_agrees_with_tile_kernel_on_c2_batch(dev, monkeypatch):
    """Full c2 batch (64 x 256^2), 4 steps: marching vs tile kernel; then linearity."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    n = 256
    spec = fine_spec(n, n)
    x = torch.as_tensor(harness.fine_batch_states(n=n, batch=64, seed=2001)).cuda()
    prop = SlicePropagator(spec, nsteps=4)
    ym = prop.apply(x)
    monkeypatch.setenv("PW_MARCH", "0")
    yt = prop.apply(x)
    monkeypatch.setenv("PW_MARCH", "1")
    err = ((ym - yt).norm(dim=1) / yt.norm(dim=1)).max().item()
    assert err <= 1e-13, err
    y2 = torch.roll(x, 1, dims=0)
    lhs = prop.apply(2.0 * x - 0.5 * y2)
    rhs = 2.0 * ym - 0.5 * torch.roll(ym, 1, dims=0)
    lin = ((lhs - rhs).norm(dim=1) / rhs.norm(dim=1)).max().item()
    assert lin <= 1e-13, lin

def test_march_strided_batch_and_blowup(dev):
    """ld > d (columns of a larger matrix, ld even) and non-finite inputs propagate quietly."""
    from paper_1510_02237_b200 import _lib
    from paper_1510_02237_b200.integrators import SlicePropagator

    nx, ny = 128, 64
    d = 3 * nx * ny
    ld = d + 16
    q0 = random_states(nx, ny, 3, 3)
    prop = SlicePropagator(fine_spec(nx, ny), nsteps=2)
    want = oracle_batch(q0, 2, nx, ny)
    big = torch.zeros(3, ld, dtype=torch.float64, device="cuda")
    big[:, :d] = torch.as_tensor(q0).cuda()
    out = torch.full_like(big, 7.0)
    prop.ctx.bind_stream()
    _lib.check(prop.ctx.lib.pw_prop_apply(prop.handle, _lib.ptr(big), _lib.ptr(out), 3, ld))
    got = out.cpu().numpy()
    for b in range(3):
        assert rel(got[b, :d], want[b]) <= 1e-12
        assert (got[b, d:] == 7.0).all()  # padding untouched
    bad = q0.copy()
    bad[0, 5] = np.inf
    r = prop.batch(bad)
    assert not np.isfinite(r[0]).all()
    assert rel(r[1], want[1]) <= 1e-12


@pytest.mark.parametrize("nx,ny,batch,nsteps,nseg", [
    (256, 256, 64, 10, 0),   # c2 shape, persistent heuristic (5 segments)
    (256, 256, 64, 7, 4),    # odd step count, the plain kernel's segments
    (512, 96, 6, 4, 3),
    (128, 64, 5, 3, 1),      # one segment: each item waits on itself only
    (384, 48, 3, 2, 2),
])
def test_persistent_march_matches_per_step_launches(dev, monkeypatch, nx, ny, batch, nsteps, nseg):
    """Previous-generation kernels (PW_MARCH_V2=0): the cp.async persistent march
    (PW_MARCH_PERSIST=1) against its per-step launches.  Each row is computed by the same
    arithmetic whatever CTA computes it, so the result is bitwise equal."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    monkeypatch.setenv("PW_MARCH_V2", "0")
    prop = SlicePropagator(fine_spec(nx, ny), nsteps=nsteps)
    x = torch.as_tensor(random_states(nx, ny, batch, 31 + nx)).cuda()
    monkeypatch.setenv("PW_MARCH_PERSIST", "0")  # the per-step launches (the default at 128/256 is persistent)
    want = prop.apply(x)
    monkeypatch.setenv("PW_MARCH_PERSIST", "1")
    if nseg:
        monkeypatch.setenv("PW_MARCH_NSEG", str(nseg))
    got = prop.apply(x)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("nx,ny,batch,nsteps,nseg", [
    (256, 256, 64, 10, 0),   # c2 shape, default segments
    (256, 256, 64, 7, 4),
    (512, 96, 6, 4, 3),
    (128, 64, 5, 3, 1),      # one segment: each item waits on itself only
    (384, 48, 3, 2, 2),
    (256, 100, 4, 5, 6),     # ragged segments (16-row minimum)
])
def test_tma_march_all_steps_vs_one_step_launches(dev, monkeypatch, nx, ny, batch, nsteps, nseg):
    """K1 (march_tma.cu) runs all steps of a propagation in one persistent launch.  Against
    nsteps launches of one step each: the same rows from the same arithmetic, so the
    result is bitwise equal -- and against the previous-generation per-step kernel
    (PW_MARCH_V2=0, different operation order) to rounding."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    spec = fine_spec(nx, ny)
    x = torch.as_tensor(random_states(nx, ny, batch, 77 + nx + ny)).cuda()
    if nseg:
        monkeypatch.setenv("PW_MARCH_NSEG", str(nseg))
    got = SlicePropagator(spec, nsteps=nsteps).apply(x)
    one = SlicePropagator(spec, nsteps=1)
    want = x
    for _ in range(nsteps):
        want = one.apply(want)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    monkeypatch.setenv("PW_MARCH_V2", "0")
    monkeypatch.setenv("PW_MARCH_PERSIST", "0")
    monkeypatch.delenv("PW_MARCH_NSEG", raising=False)
    old = SlicePropagator(spec, nsteps=nsteps).apply(x)
    err = ((got - old).norm(dim=1) / old.norm(dim=1)).max().item()
    assert err <= 1e-13, err


@pytest.mark.parametrize("nx,ny,batch,nsteps", [
    (1024, 48, 2, 3),     # cluster pairs (2 x 512 columns)
    (1024, 100, 3, 4),    # ragged segments
    (2048, 32, 1, 2),     # clusters of 4
    (1024, 256, 4, 5),
])
def test_tma_march_clusters_match_oracle_and_tile_kernel(dev, monkeypatch, nx, ny, batch, nsteps):
    """K1 on 1024- and 2048-wide rows: thread-block clusters of 512-column CTAs (q halos by
    TMA, s1 / s2 halos over DSMEM, a cluster barrier per tick).  Against the oracle
    (<= 1e-12), against one-step launches (bitwise: same rows, same arithmetic) and against
    the tile kernel (PW_MARCH_CLUSTER2=0; different operation order, <= 1e-13)."""
    from paper_1510_02237_b200.integrators import SlicePropagator

    spec = fine_spec(nx, ny)
    q0 = random_states(nx, ny, batch, nx + 3 * ny)
    got = SlicePropagator(spec, nsteps=nsteps).batch(q0)
    want = oracle_batch(q0, nsteps, nx, ny)
    for b in range(batch):
        assert rel(got[b], want[b]) <= 1e-12
    x = torch.as_tensor(q0).cuda()
    full = SlicePropagator(spec, nsteps=nsteps).apply(x)
    one = SlicePropagator(spec, nsteps=1)
    step = x
    for _ in range(nsteps):
        step = one.apply(step)
    torch.cuda.synchronize()
    assert torch.equal(full, step)
    monkeypatch.setenv("PW_MARCH_CLUSTER2", "0")
    tile = SlicePropagator(spec, nsteps=nsteps).apply(x)
    err = ((full - tile).norm(dim=1) / tile.norm(dim=1)).max().item()
    assert err <= 1e-13, err
