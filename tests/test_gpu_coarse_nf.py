"""Neighbour-flag coarse propagator G (csrc/exact.cu fefb_nf_kernel; B200 only).

The serial sweep's G (one state: split FE-FB, integrators.py:103-106 with fb_substeps,
numba_backend.py:131-146) runs as one persistent launch in which tiles wait only on their
8 neighbours' phase counters (no grid barriers).  Same expressions as the reference in
the reference's operation order (-fmad=false), so every case is BITWISE equal to the
per-cell strict kernel -- for each substep blocking (PW_COARSE_NF = 2, 3, 4 substeps per
phase), square and non-square grids, ragged tile heights, tiles per CTA > 1 (1024^2,
2048^2), an odd block count (copy-back phase), several steps per call, flux orders 1
and 3 (the generic-order instantiation), no damping, and upwind with U < 0.
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


@pytest.mark.parametrize("variant", ["2", "3", "4", "5"])
@pytest.mark.parametrize("nx,ny", [(512, 512), (256, 256), (512, 320), (1024, 1024), (128, 128), (256, 96)])
def test_nf_coarse_bitwise(dev, monkeypatch, variant, nx, ny):
    monkeypatch.setenv("PW_COARSE_NF", variant)
    got, want = run_both(dev, coarse(nx, ny), states(nx, ny, nx + ny), 2)
    assert torch.equal(got, want)


@pytest.mark.parametrize("case", ["odd_blocks", "order3", "no_damping", "upwind_negative", "c5_grid"])
def test_nf_coarse_cases_bitwise(dev, case):
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
