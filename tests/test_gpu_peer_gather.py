"""Slice all-gather fused into the fine kernel: pw_prop_apply_to_peers and
dist.FusedShardedFine (B200 only).

The peer copies hold the registers the local store writes, and the epilogue does
not touch the arithmetic, so everything here is compared bit for bit with
pw_prop_apply.  Row-marching grids (nx 128/256/384/512) take the fused epilogue;
the others (the tile kernel at 1024, the reference-order kernels) copy the result
to the peers afterwards.  The two-process test maps each rank's gather buffer in
the other process with CUDA IPC (both ranks on GPU 0; their kernels only store,
they never wait on each other) and checks that every rank ends with all slices.
"""
import os
import socket

import numpy as np
import pytest

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


def fine_prop(nx, ny, nsteps, scheme="rk3"):
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.physics import ModelSpec

    g = build_grid(nx, ny)
    vel = ConstantVelocity(0.1, 0.0)
    if scheme == "rk3":
        spec = make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5)
    else:
        spec = make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 2.0, 8)
    return SlicePropagator(spec, nsteps=nsteps)


def states(nx, ny, batch, seed):
    rng = np.random.default_rng(seed)
    return torch.as_tensor(rng.standard_normal((batch, 3 * nx * ny))).cuda()


@pytest.mark.parametrize("nx,ny,nsteps,scheme", [
    (256, 64, 3, "rk3"),    # marching kernel, fused epilogue, odd step count
    (512, 48, 2, "rk3"),    # marching kernel, even step count (ping-pong)
    (128, 40, 1, "rk3"),
    (384, 32, 2, "rk3"),
    (1024, 32, 2, "rk3"),   # tile kernel: copied to the peers afterwards
    (64, 64, 2, "rk3"),     # below the marching widths
    (64, 64, 1, "fefb"),    # reference-order coarse kernels
])
def test_apply_to_peers_matches_apply(dev, nx, ny, nsteps, scheme):
    prop = fine_prop(nx, ny, nsteps, scheme)
    x = states(nx, ny, 5, 7 + nx)
    want = prop.apply(x)
    out = torch.empty_like(x)
    peers = [torch.full_like(x, float("nan")) for _ in range(3)]
    prop.apply_to_peers(x, out, [p.data_ptr() for p in peers])
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    for p in peers:
        assert torch.equal(p, want)


def test_apply_to_peers_into_blocks_of_a_gather_buffer(dev):
    """The FusedShardedFine layout: each rank's slices land at rows [lo, hi) of every
    rank's (n, d) buffer; rows outside the block stay untouched."""
    nx, ny, n, lo, hi = 256, 48, 7, 2, 5
    prop = fine_prop(nx, ny, 2)
    x = states(nx, ny, n, 3)
    d = x.shape[1]
    want = prop.apply(x[lo:hi].contiguous())
    bufs = [torch.full((n, d), -1.0, dtype=torch.float64, device="cuda") for _ in range(4)]
    prop.apply_to_peers(x[lo:hi], bufs[0][lo:hi], [b.data_ptr() + lo * d * 8 for b in bufs[1:]])
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b[lo:hi], want)
        assert bool((b[:lo] == -1.0).all()) and bool((b[hi:] == -1.0).all())


def test_apply_to_peers_limits(dev):
    prop = fine_prop(128, 32, 1)
    x = states(128, 32, 1, 1)
    out = torch.empty_like(x)
    with pytest.raises(ValueError):
        prop.apply_to_peers(x, out, [out.data_ptr()] * 8)  # at most 7 peers
    with pytest.raises(ValueError):
        prop.apply_to_peers(x, out, [0])                    # NULL peer buffer


def test_ipc_alloc_free_roundtrip(dev):
    import ctypes

    from paper_1510_02237_b200 import _lib

    ptr, handle = _lib.c_vp(), ctypes.create_string_buffer(64)
    _lib.check(dev.lib.pw_ipc_alloc(dev.handle, 1 << 20, ctypes.byref(ptr), handle))
    assert ptr.value and any(handle.raw)
    _lib.check(dev.lib.pw_ipc_free(dev.handle, ptr))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1510_02237_b200 import _lib
        from paper_1510_02237_b200.dist import FusedShardedFine

        _lib.Context.get(0).set_strict(False)
        ok = []
        for nx, ny, n in ((256, 64, 5), (1024, 32, 3)):  # fused epilogue; copy fallback
            prop = fine_prop(nx, ny, 3)
            fused = FusedShardedFine(prop)
            for seed in (1, 2, 3, 4):  # alternate halves of the gather buffer; calls 3 and 4 reuse them
                x = states(nx, ny, n, seed)
                got = fused(x)
                want = prop.apply(x)
                torch.cuda.synchronize()
                ok.append(bool(torch.equal(got, want)))
            fused.close()
        out_q.put((rank, ok))
    except Exception as exc:  # reported by the parent
        out_q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_sharded_fine_across_processes(dev, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(r[0] for r in results) == list(range(world))
    for rank, ok in results:
        assert isinstance(ok, list) and all(ok), (rank, ok)
