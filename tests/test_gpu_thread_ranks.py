"""The multi-rank (pw_ctx_set_comm) code paths of pw_sweep, run as host-thread ranks.

Each rank is a Python thread with its own library context, stream and
propagators on cuda:0.  Its comm hooks exchange device vectors through host
barriers, summing allreduce partials in rank order.  No kernel waits on another
rank's kernels: every exchange happens on the host between kernel launches.  So
this checks the arithmetic and the collective protocol of the row-sharded serial
correction and of the TSQR factorisation with world > 1. The
in-process row shards of test_gpu_sweeps.py take a different branch and cannot
check these. It is a correctness test and says nothing about multi-GPU speed.
"""
import threading

import numpy as np
import pytest

from conftest import golden
from paper_1510_02237_b200 import harness

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


class ThreadComm:
    """allreduce / all-gather hooks for `world` thread ranks (pw_allreduce_hook semantics)."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world, timeout=120)
        self.slots = [None] * world
        self.errors = []

    def hooks(self, rank, device):
        from paper_1510_02237_b200 import _lib
        from paper_1510_02237_b200.dist import device_vector, row_block

        def allreduce(user, p, count):
            try:
                v = device_vector(p, count, device)
                self.slots[rank] = v.clone()
                torch.cuda.current_stream(device).synchronize()
                self.bar.wait()
                tot = self.slots[0].clone()
                for r in range(1, self.world):  # rank order: identical sums on every rank
                    tot += self.slots[r]
                torch.cuda.current_stream(device).synchronize()
                self.bar.wait()
                v.copy_(tot)
                return 0
            except Exception as exc:  # noqa: BLE001 - reported by the test
                self.errors.append(exc)
                return 1

        def allgather(user, p, block, total):
            try:
                v = device_vector(p, total, device)
                lo, hi = row_block(total, block, rank)
                self.slots[rank] = v[lo:hi].clone()
                torch.cuda.current_stream(device).synchronize()
                self.bar.wait()
                for r in range(self.world):
                    rlo, rhi = row_block(total, block, r)
                    if rhi > rlo:
                        v[rlo:rhi].copy_(self.slots[r])
                torch.cuda.current_stream(device).synchronize()
                self.bar.wait()
                return 0
            except Exception as exc:  # noqa: BLE001
                self.errors.append(exc)
                return 1

        return _lib.ALLREDUCE_HOOK(allreduce), _lib.ALLGATHER_HOOK(allgather)

    def fine_rows_hook(self, rank, device, fine):
        """pw_fine_rows_hook: each rank propagates its block of slices; every rank then
        takes its rows of all slices (the all-to-all of dist.ShardedFine.rows)."""
        from paper_1510_02237_b200 import _lib
        from paper_1510_02237_b200.dist import device_vector, shard_range

        def hook(user, qk_ptr, pred_ptr, n_c, d, lo, rows):
            try:
                qk = device_vector(qk_ptr, n_c * d, device).view(n_c, d)
                pred = device_vector(pred_ptr, n_c * rows, device).view(n_c, rows)
                slo, shi = shard_range(n_c, rank, self.world)
                self.slots[rank] = fine.apply(qk[slo:shi].contiguous()) if shi > slo else None
                torch.cuda.current_stream(device).synchronize()
                self.bar.wait()
                for r in range(self.world):
                    rlo, rhi = shard_range(n_c, r, self.world)
                    if rhi > rlo:
                        pred[rlo:rhi].copy_(self.slots[r][:, lo:lo + rows])
                torch.cuda.current_stream(device).synchronize()
                self.bar.wait()
                return 0
            except Exception as exc:  # noqa: BLE001
                self.errors.append(exc)
                return 1

        return _lib.FINE_ROWS_HOOK(hook)


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


_build_lock = threading.Lock()


def rank_main(rank, world, comm, tsqr, q0, results, rows_hook=False):
    from paper_1510_02237_b200 import _lib
    from paper_1510_02237_b200.parareal import kse_sweep

    device = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device)
    try:
        with torch.cuda.stream(stream):
            ctx = _lib.Context(0)  # this rank's own context on this thread's stream
            with _build_lock:      # propagators of this context (Context.get returns it meanwhile)
                saved = _lib.Context._instances.get(0)
                _lib.Context._instances[0] = ctx
                try:
                    wl, fine, coarse = c1_props()
                finally:
                    if saved is None:
                        _lib.Context._instances.pop(0, None)
                    else:
                        _lib.Context._instances[0] = saved
            ar, ag = comm.hooks(rank, device)
            _lib.check(ctx.lib.pw_ctx_set_comm(ctx.handle, rank, world, ar, ag, None))
            fh = comm.fine_rows_hook(rank, device, fine) if rows_hook else _lib.FINE_ROWS_HOOK()
            _lib.check(ctx.lib.pw_ctx_set_fine_rows_hook(ctx.handle, fh, None))
            ctx.set_tsqr(tsqr)
            out = []
            for k in range(1, wl.n_it + 1):
                ends, res, sub = kse_sweep(q0, fine, coarse, wl.n_p, k)
                out.append((np.array(ends), list(res), sub.rank))
            results[rank] = out
            ctx.lib.pw_ctx_set_comm(ctx.handle, 0, 1, _lib.ALLREDUCE_HOOK(), _lib.ALLGATHER_HOOK(), None)
            del fine, coarse, sub
    except Exception as exc:  # noqa: BLE001
        results[rank] = exc
        comm.bar.abort()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("tsqr,rows_hook", [(False, False), (True, False), (True, True)])
def test_thread_ranks_c1_window_matches_reference(world, tsqr, rows_hook):
    """tsqr: row-sharded factorisation with a row-local basis and row-local fine/coarse
    images; rows_hook: the fine images arrive through the all-to-all hook (each rank
    propagates only its slices) instead of every rank propagating all of them."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_02237_b200.parareal import kse_sweep

    g = golden("c1_kse.npz")
    # the single-process windows (1 GPU, no sharding) for the 1-vs-N equivalence check
    wl, fine1, coarse1 = c1_props()
    single = [np.array(kse_sweep(g["q0"], fine1, coarse1, wl.n_p, k)[0]) for k in range(1, wl.n_it + 1)]
    comm = ThreadComm(world)
    results = [None] * world
    threads = [threading.Thread(target=rank_main, args=(r, world, comm, tsqr, g["q0"], results, rows_hook))
               for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    for r in range(world):  # a rank's own exception first (the other then sees a broken barrier)
        assert not isinstance(results[r], Exception), (r, results, comm.errors)
        assert results[r] is not None
    assert not comm.errors, comm.errors
    n_it = len(results[0])
    for k in range(n_it):
        ends0 = results[0][k][0]
        for r in range(world):
            ends, res, rank = results[r][k]
            assert rank == g["kse_ranks"][k]
            # every rank holds the same iterates (rows gathered, identical rank-order sums)
            np.testing.assert_array_equal(ends, ends0)
            worst = max(np.linalg.norm(ends[i] - g["kse_hist"][k][i]) / np.linalg.norm(g["kse_hist"][k][i])
                        for i in range(ends.shape[0]))
            assert worst <= 1e-10, (r, k, worst)
            np.testing.assert_allclose(res, g["kse_res"][:k + 1], rtol=1e-10)
            # 1-vs-N: only the order of the alpha partial sums differs without
            # TSQR; TSQR is a different (equally valid) factorisation of the same snapshots
            dev1 = max(np.linalg.norm(ends[i] - single[k][i]) / np.linalg.norm(single[k][i])
                       for i in range(ends.shape[0]))
            assert dev1 <= (1e-12 if not tsqr else 1e-10), (r, k, dev1)


def c3_rank_main(rank, world, comm, q0, results):
    """One thread rank of the c3 window with TSQR, the row-local basis and the all-to-all
    fine hook; per iteration: ranks, residuals, per-slice norms and the sampled entries."""
    import os

    from conftest import GOLDEN
    from paper_1510_02237_b200 import _lib
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
    from paper_1510_02237_b200.parareal import kse_sweep
    from paper_1510_02237_b200.physics import ModelSpec

    device = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device)
    try:
        with torch.cuda.stream(stream):
            ctx = _lib.Context(0)
            with _build_lock:
                saved = _lib.Context._instances.get(0)
                _lib.Context._instances[0] = ctx
                try:
                    wl = harness.WORKLOADS["c3"]
                    g = build_grid(wl.n, wl.n)
                    vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
                    fine = SlicePropagator(make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g,
                                                          0.5), wl.slice_span)
                    coarse = SlicePropagator(make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0),
                                                            g, 4.0, 16), wl.slice_span)
                finally:
                    if saved is None:
                        _lib.Context._instances.pop(0, None)
                    else:
                        _lib.Context._instances[0] = saved
            ar, ag = comm.hooks(rank, device)
            _lib.check(ctx.lib.pw_ctx_set_comm(ctx.handle, rank, world, ar, ag, None))
            fh = comm.fine_rows_hook(rank, device, fine)
            _lib.check(ctx.lib.pw_ctx_set_fine_rows_hook(ctx.handle, fh, None))
            ctx.set_tsqr(True)
            ref = np.load(os.path.join(GOLDEN, "c3_reference.npz"))
            idx = torch.as_tensor(ref["idx"]).cuda()
            q = torch.as_tensor(q0).cuda()
            out = []
            for k in range(1, len(ref["res"]) + 1):
                ends, res, sub = kse_sweep(q, fine, coarse, wl.n_p, k, return_device=True)
                st = ends.reshape(wl.n_p, -1)
                out.append((sub.rank, list(res), torch.linalg.norm(st, dim=1).cpu().numpy(),
                            st[:, idx].cpu().numpy()))
                del ends, st, sub
            results[rank] = out
            ctx.lib.pw_ctx_set_comm(ctx.handle, 0, 1, _lib.ALLREDUCE_HOOK(), _lib.ALLGATHER_HOOK(), None)
            del fine, coarse
    except Exception as exc:  # noqa: BLE001
        results[rank] = exc
        comm.bar.abort()


def test_thread_ranks_c3_window_tsqr_matches_reference_run():
    """c3 (512^2, P=64, K=5) over 2 thread ranks with the multi-rank TSQR sweep (row-local
    basis and fine/coarse images, all-to-all fine hook): the reference run's ranks, and
    states within the c3 parity bound (as test_gpu_windows_ref.py)."""
    import os

    from conftest import GOLDEN

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    path = os.path.join(GOLDEN, "c3_reference.npz")
    if not os.path.exists(path):
        pytest.skip("c3_reference.npz not generated")
    ref = np.load(path)
    floor = [2.8e-9, 1.1e-8, 9.0e-9, 3.6e-8, 2.1e-7]  # test_gpu_windows_ref.C3_FLOOR
    world = 2
    comm = ThreadComm(world)
    results = [None] * world
    q0 = harness.initial_state("c3")
    threads = [threading.Thread(target=c3_rank_main, args=(r, world, comm, q0, results)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=900)
    for r in range(world):  # a rank's own exception first (the other then sees a broken barrier)
        assert not isinstance(results[r], Exception), (r, results, comm.errors)
    assert not comm.errors, comm.errors
    for k, (rank_k, res, norms, samp) in enumerate(results[0]):
        tol = max(1e-10, 10 * floor[k])
        assert rank_k == ref["ranks"][k], (k, rank_k, ref["ranks"][k])
        assert results[1][k][0] == rank_k
        np.testing.assert_allclose(res, ref["res"][:k + 1], rtol=tol)
        d_norm = np.max(np.abs(norms - ref["norms"][k]) / ref["norms"][k])
        d_samp = np.max(np.linalg.norm(samp - ref["samples"][k], axis=1) / np.linalg.norm(ref["samples"][k], axis=1))
        print(f"c3 thread ranks, iteration {k + 1}: rank {rank_k}, deviation {max(d_norm, d_samp):.3e}")
        assert max(d_norm, d_samp) <= tol
