"""Multi-process (world_size 2, gloo, CPU) tests of the slice-sharded fine predictor.

The device sweep installs paper_1510_02237_b200.dist.ShardedFine as its fine
hook when given a process group; here the same sharding/all-gather logic is
driven by the CPU oracle's fine propagator inside the oracle's KSE sweep,
and must reproduce the single-process window bitwise on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1510_02237_b200.dist import shard_range


def test_shard_range_partitions():
    for n in (1, 7, 8, 64, 256):
        for world in (1, 2, 3, 4, 8):
            blocks = [shard_range(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in blocks]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_1510_02237_b200 import harness
        from paper_1510_02237_b200.dist import ShardedFine

        n, p, k, span = 32, 6, 2, 1.0 / 16
        fine = orc.SlicePropagator(orc.RK3, 4, nx=n, ny=n, cs=1.0, order=6, nu=0.005, cfl=0.5,
                                   velocity=("constant", 0.1, 0.0))
        coarse = orc.SlicePropagator(orc.SPLIT_FE_FB, 1, nx=n, ny=n, cs=1.0, order=1, nu=0.1,
                                     cfl=2.0, n_sound=8, velocity=("constant", 0.1, 0.0))
        q0 = harness.initial_state("c3", n=n)
        sharded = ShardedFine(lambda x: torch.as_tensor(fine.batch(x.numpy())))
        sweep = orc.kse_sweep if mode == "kse" else orc.parareal_sweep
        res_sh = sweep(q0, sharded, coarse, p, k)
        res_1 = sweep(q0, fine, coarse, p, k)
        ends_sh, ends_1 = np.array(res_sh[0]), np.array(res_1[0])
        out_q.put((rank, bool(np.array_equal(ends_sh, ends_1)), list(res_sh[1]) == list(res_1[1])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["kse", "original"])
def test_sharded_fine_matches_single_process_world2(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert sorted(r[0] for r in results) == [0, 1]
    assert all(r[1] for r in results), results   # bitwise-equal endpoints on both ranks
    assert all(r[2] for r in results), results   # identical residual histories


def _row_worker(rank, world, port, out_q):
    """Row-sharded serial correction arithmetic (the per-step work of pw_sweep with
    pw_ctx_set_comm): each rank combines its row block of D and Q, the partial alphas
    are allreduced and the rows of qn_{i+1} all-gathered -- over gloo on CPU tensors,
    against the unsharded recursion."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_02237_b200.dist import gather_rows, row_block

        g = torch.Generator().manual_seed(5)
        d, r, steps = 1001, 7, 5  # odd d: the last block is short
        D = torch.randn(d, r, generator=g, dtype=torch.float64)
        Q = torch.linalg.qr(torch.randn(d, r, generator=g, dtype=torch.float64))[0]
        G = torch.randn(d, d, generator=g, dtype=torch.float64) / d ** 0.5
        c = torch.randn(steps, d, generator=g, dtype=torch.float64)
        q0 = torch.randn(d, generator=g, dtype=torch.float64)
        # unsharded: q_{i+1} = G q_i + c_i + D alpha_i,  alpha_i = Q^T q_i
        q, a = q0.clone(), Q.T @ q0
        for i in range(steps):
            q = G @ q + c[i] + D @ a
            a = Q.T @ q
        block = ((d + world - 1) // world + 1) // 2 * 2
        lo, hi = row_block(d, block, rank)
        qs, as_ = q0.clone(), Q.T @ q0
        for i in range(steps):
            gq = G @ qs                                   # replicated coarse step
            y = torch.zeros(d, dtype=torch.float64)
            y[lo:hi] = gq[lo:hi] + c[i, lo:hi] + D[lo:hi] @ as_
            part = Q[lo:hi].T @ y[lo:hi]
            dist.all_reduce(part)                         # partial alphas -> alpha_{i+1}
            gather_rows(y, block)                         # rows of qn_{i+1} -> every rank
            qs, as_ = y, part
        out_q.put((rank, float((qs - q).norm() / q.norm()), float((as_ - a).norm() / a.norm())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_serial_correction_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert len(results) == world
    for _, dq, da in results:
        assert dq <= 1e-13 and da <= 1e-13


def _tsqr_worker(rank, world, port, out_q):
    """Row-sharded TSQR (dist.tsqr, the decomposition of the device factor_tsqr) over gloo
    against the unsharded factorisation of the whole snapshot matrix."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import scipy.linalg as sla

        from paper_1510_02237_b200.dist import row_block, tsqr

        g = torch.Generator().manual_seed(11)
        d, m = 997, 24
        # Parareal-like snapshots: a few near-duplicate and dependent columns
        a = torch.randn(d, m, generator=g, dtype=torch.float64)
        a[:, 5] = a[:, 1] + 1e-12 * a[:, 7]
        a[:, 9] = 2.0 * a[:, 3] - a[:, 4]
        a[:, 17] = a[:, 2]
        block = ((d + world - 1) // world + 1) // 2 * 2
        lo, hi = row_block(d, block, rank)
        r, q_rows = tsqr(a[lo:hi].contiguous())
        # this rank's rows of Q, gathered: Q spans what A's QR spans, Q^T Q = I, A = Q R
        full_q = torch.zeros(d, m, dtype=torch.float64)
        full_q[lo:hi] = q_rows
        dist.all_reduce(full_q)
        recon = float((full_q @ r - a).norm() / a.norm())
        ortho = float((full_q.T @ full_q - torch.eye(m, dtype=torch.float64)).norm())
        # R is A's R up to row signs (not unique past a dependent column): R^T R = A^T A
        gram = a.T @ a
        rdiff = float((r.T @ r - gram).norm() / gram.norm())
        # the reference's rank rule on pivoted QR (subspace.py): R of TSQR vs A itself
        _, rr, piv = sla.qr(r.numpy(), pivoting=True, mode="economic")
        _, ra, piva = sla.qr(a.numpy(), pivoting=True, mode="economic")
        tol = 1e-10
        rank_t = int(np.sum(np.abs(np.diag(rr)) > tol * abs(rr[0, 0])))
        rank_a = int(np.sum(np.abs(np.diag(ra)) > tol * abs(ra[0, 0])))
        # kept columns: ties between duplicate columns may pick either copy, so compare the
        # spans of the kept columns of A
        qa_t = np.linalg.qr(a.numpy()[:, piv[:rank_t]])[0]
        qa_a = np.linalg.qr(a.numpy()[:, piva[:rank_a]])[0]
        same_span = bool(np.linalg.norm(qa_t @ (qa_t.T @ qa_a) - qa_a) <= 1e-10 * np.sqrt(rank_a))
        out_q.put((rank, recon, ortho, rdiff, rank_t, rank_a, same_span))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tsqr_matches_unsharded_factorisation(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tsqr_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert len(results) == world
    for _, recon, ortho, rdiff, rank_t, rank_a, same_span in results:
        assert recon <= 1e-14 and ortho <= 1e-13 and rdiff <= 1e-13
        assert rank_t == rank_a == 21   # 3 dependent columns dropped by the rank rule
        assert same_span


def _rows_worker(rank, world, port, out_q):
    """dist.ShardedFine.rows: slice-sharded propagation + all-to-all of row blocks (the
    fine rows hook of row-local sweeps) against the rows of the unsharded images."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_02237_b200.dist import ShardedFine, row_block

        g = torch.Generator().manual_seed(3)
        n, d = 7, 203  # slices not divisible by the world, odd d: short last row block
        a = torch.randn(d, d, generator=g, dtype=torch.float64)
        qk = torch.randn(n, d, generator=g, dtype=torch.float64)
        full = qk @ a.T
        sharded = ShardedFine(lambda x: x @ a.T)
        block = ((d + world - 1) // world + 1) // 2 * 2
        lo, hi = row_block(d, block, rank)
        got = sharded.rows(qk, lo, hi)
        out_q.put((rank, tuple(got.shape) == (n, hi - lo), float((got - full[:, lo:hi]).abs().max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fine_rows_all_to_all(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert len(results) == world
    for _, shape_ok, err in results:
        assert shape_ok and err <= 1e-12


def _host_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_02237_b200.dist import same_host

        out_q.put((rank, same_host()))
    finally:
        dist.destroy_process_group()


def test_same_host_world2():
    """The fused (peer-store) all-gather is chosen only when every rank shares the host."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert sorted(results) == [(0, True), (1, True)]
