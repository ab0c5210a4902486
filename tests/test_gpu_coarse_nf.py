"""Neighbour-flag coarse propagator G (csrc/exact.cu fefb_nf_kernel; B200 only).

The serial sweep's G (one state: split FE-FB, integrators.py:103-106 with fb_substeps,
numba_backend.py:131-146) runs as one persistent launch in which tiles wait only on their
8 neighbours' phase counters (no grid barriers).  Same expressions as the reference in
the reference's operation order (-fmad=false), so every case is BITWISE equal to the
per-cell strict kernel -- for each substep blocking (PW_COARSE_NF = 2, 3, 4 substeps per
phase), square and non-square grids, ragged tile heights, tiles per CTA > 1 (1024^2,
2048^2), an odd block count (copy-back phase), several steps per call, flux orders 1
and 3 (the generic-order instantiation), no damping, and upwind with U < 0 -- and the
row-sharded form (pw_prop_apply_rowshard) against the replicated G.
"""
import numpy as np
import pytest

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


def coarse(nx, ny, *, order=1, U=0.1, nu=0.1, n_sound=16, cfl=4.0):
    from paper_1510_02237_b200.integrators import SPLIT_FE_FB, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    m = ModelSpec(ACOUSTIC, ConstantVelocity(U, 0.0), order, 1.0, nu, 1.0 if nu > 0 else None)
    return make_propagator(SPLIT_FE_FB, m, build_grid(nx, ny), cfl, n_sound)


def states(nx, ny, seed):
    rng = np.random.default_rng(seed)
    return torch.as_tensor(rng.standard_normal((1, 3 * nx * ny))).cuda()


def run_both(dev, spec, x, nsteps):
    from paper_1510_02237_b200.integrators import SlicePropagator

    got = SlicePropagator(spec, nsteps=nsteps).apply(x)
    dev.set_strict(True)
    try:
        want = SlicePropagator(spec, nsteps=nsteps).apply(x)
    finally:
        dev.set_strict(False)
    torch.cuda.synchronize()
    return got, want


@pytest.mark.parametrize("variant", ["2", "3", "4", "5", "6", "7", "8", "9", "10", "11", "12", "13", "17"])
@pytest.mark.parametrize("nx,ny", [(512, 512), (256, 256), (512, 320), (1024, 1024), (128, 128), (256, 96)])
def test_nf_coarse_bitwise(dev, monkeypatch, variant, nx, ny):
    monkeypatch.setenv("PW_COARSE_NF", variant)
    got, want = run_both(dev, coarse(nx, ny), states(nx, ny, nx + ny), 2)
    assert torch.equal(got, want)


@pytest.mark.parametrize("variant", ["3", "6", "10", "11", "12", "13", "17"])
@pytest.mark.parametrize("case", ["odd_blocks", "order3", "no_damping", "upwind_negative", "c5_grid"])
def test_nf_coarse_cases_bitwise(dev, monkeypatch, variant, case):
    monkeypatch.setenv("PW_COARSE_NF", variant)
    kw, nx, ny, nsteps = {}, 512, 512, 3
    if case == "odd_blocks":
        kw = {"n_sound": 7}  # 7 substeps: blocks 3, 3, 1 -> odd count, copy-back phase
    elif case == "order3":
        kw = {"order": 3}
    elif case == "no_damping":
        kw = {"nu": 0.0}
    elif case == "upwind_negative":
        kw = {"U": -0.1}
    elif case == "c5_grid":
        nx = ny = 2048
        nsteps = 1
    x = torch.as_tensor(harness.initial_state("c5" if case == "c5_grid" else "c3", n=nx)[None, :]).cuda() \
        if nx == ny else states(nx, ny, 3)
    got, want = run_both(dev, coarse(nx, ny, **kw), x, nsteps)
    assert torch.equal(got, want)


@pytest.mark.parametrize("nx,ny,nshard", [(512, 512, 2), (512, 512, 4), (1024, 1024, 4), (256, 240, 3),
                                          (512, 512, 8)])
def test_rowsharded_coarse_bitwise_with_replicated(dev, nx, ny, nshard):
    """Row-sharded G (pw_prop_apply_rowshard): the state's rows in nshard row
    shards with their own state / work / flag buffers; tiles on a shard edge read their halo
    rows from the neighbouring shard and wait on its flags.  Every shard's tiles run in one
    launch on this one GPU (a multi-GPU run would launch each shard's tiles on its own device
    with peer pointers).  Bitwise equal to the replicated G, two FE-FB steps."""
    import ctypes

    from paper_1510_02237_b200 import _lib
    from paper_1510_02237_b200.integrators import SlicePropagator

    prop = SlicePropagator(coarse(nx, ny), nsteps=2)
    x = states(nx, ny, 7 + nshard)
    want = prop.apply(x)
    R = ny // nshard
    full = x.view(3, ny, nx)
    st = [full[:, s * R:(s + 1) * R, :].contiguous().reshape(-1) for s in range(nshard)]
    wd = ctypes.c_longlong(0)
    nflag = prop.ctx.lib.pw_rowshard_sizes(prop.handle, nshard, ctypes.byref(wd))
    assert nflag > 0 and wd.value == 6 * R * nx
    work = [torch.empty(wd.value, dtype=torch.float64, device="cuda") for _ in range(nshard)]
    flags = [torch.zeros(nflag, dtype=torch.int32, device="cuda") for _ in range(nshard)]
    arr = lambda ts: (_lib.c_vp * nshard)(*[_lib.c_vp(t.data_ptr()) for t in ts])  # noqa: E731
    prop.ctx.bind_stream()
    _lib.check(prop.ctx.lib.pw_prop_apply_rowshard(prop.handle, nshard, arr(st), arr(work), arr(flags)))
    torch.cuda.synchronize()
    got = torch.cat([b.view(3, R, nx) for b in st], dim=1).reshape(1, -1)
    assert torch.equal(got, want)
