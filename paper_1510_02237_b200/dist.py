"""Multi-GPU plumbing for the Parareal window (host side, torch.distributed).

Slice sharding of the fine predictor: the P fine propagations of one
iteration are independent (the reference's ``_fine_all`` thread pool,
parareal.py:62-65).  Rank r propagates the contiguous block of slices
``shard_range(P, r, N)`` on its own GPU, and one all-gather (NCCL over
NVLink, or gloo on CPU in the tests) gives every rank all P fine images.
The rest of the window -- subspace refactorisation and serial correction
sweep -- runs replicated on every rank with identical inputs and
deterministic kernels, so all ranks hold bitwise-identical iterates.

Row-sharded pieces of SURVEY.md 8(e), through the C-ABI comm hooks
(pw_ctx_set_comm, RowShardComm below): the serial correction streams each
rank's row block of D and Q with one allreduce of r inner products and one
all-gather of qn rows per step, and (pw_ctx_set_tsqr) the subspace is factored
by TSQR: local Householder QR of each rank's rows, one all-gather of the m x m
R factors, their QR replicated.  ``tsqr`` below is that decomposition on torch
tensors (the gloo tests check it against the unsharded QR).

``FusedShardedFine`` is the NVLink form of the slice all-gather: the last RK3
step's kernel stores every output row into all ranks' gather buffers (peer
memory mapped by CUDA IPC, ``PeerGather``), so the exchange overlaps the step's
compute and no NCCL call sits on the data path.  ``kse_sweep(..., group=)`` uses
it under the NCCL backend when PW_FUSED_GATHER=1 (opt-in until an 8-GPU run has
measured it; the default is the NCCL all-gather).
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as tdist


def shard_range(n: int, rank: int, world: int):
    """Contiguous [lo, hi) block of n items for `rank` of `world` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class ShardedFine:
    """Fine predictor over a batch of slices, sharded over a process group.

    ``apply_fn(states)`` maps a (b, d) tensor of slice states to their fine
    images (same device).  ``__call__(qk)`` takes all n (n, d) states on
    every rank and returns all n images on every rank.
    """

    def __init__(self, apply_fn, group=None):
        self.apply_fn = apply_fn
        self.group = group

    @property
    def world(self):
        return tdist.get_world_size(self.group) if tdist.is_initialized() else 1

    @property
    def rank(self):
        return tdist.get_rank(self.group) if tdist.is_initialized() else 0

    def __call__(self, qk: torch.Tensor) -> torch.Tensor:
        world, rank = self.world, self.rank
        n = qk.shape[0]
        if world == 1:
            return self.apply_fn(qk)
        lo, hi = shard_range(n, rank, world)
        width = (n + world - 1) // world  # all_gather needs equal blocks: pad
        local = torch.zeros((width, qk.shape[1]), dtype=qk.dtype, device=qk.device)
        if hi > lo:
            local[: hi - lo] = self.apply_fn(qk[lo:hi].contiguous())
        blocks = [torch.empty_like(local) for _ in range(world)]
        tdist.all_gather(blocks, local, group=self.group)
        out = torch.empty_like(qk)
        for r in range(world):
            rlo, rhi = shard_range(n, r, world)
            if rhi > rlo:
                out[rlo:rhi] = blocks[r][: rhi - rlo]
        return out

    def rows(self, qk: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
        """Rows [lo, hi) of all n fine images (n, hi - lo) on this rank: the all-to-all of
        SURVEY 8(e).  Each rank propagates its block of slices and sends every rank g the
        rows of g's block (row blocks of ``row_block`` with the sweep's even block size)."""
        world, rank = self.world, self.rank
        n, d = qk.shape
        if world == 1:
            return self.apply_fn(qk)[:, lo:hi].contiguous()
        slo, shi = shard_range(n, rank, world)
        width = (n + world - 1) // world
        blk = ((d + world - 1) // world + 1) // 2 * 2
        send = torch.zeros((world, width, blk), dtype=qk.dtype, device=qk.device)
        if shi > slo:
            mine = self.apply_fn(qk[slo:shi].contiguous())
            for g in range(world):
                glo, ghi = row_block(d, blk, g)
                if ghi > glo:
                    send[g, : shi - slo, : ghi - glo] = mine[:, glo:ghi]
        recv = torch.empty_like(send)
        tdist.all_to_all_single(recv, send, group=self.group)
        out = torch.empty((n, hi - lo), dtype=qk.dtype, device=qk.device)
        for src in range(world):
            s_lo, s_hi = shard_range(n, src, world)
            if s_hi > s_lo:
                out[s_lo:s_hi] = recv[src, : s_hi - s_lo, : hi - lo]
        return out

    # the oracle sweeps (tests) call fine.batch(states) on numpy arrays
    def batch(self, states):
        t = torch.as_tensor(states)
        return self(t).cpu().numpy()


def same_host(group=None) -> bool:
    """True when every rank of `group` runs on this host (CUDA IPC / NVLink peers)."""
    import socket

    names = [None] * tdist.get_world_size(group)
    tdist.all_gather_object(names, socket.gethostname(), group=group)
    return len(set(names)) == 1


class PeerGather:
    """Every rank's gather buffer of `numel` doubles, mapped on every rank.

    Collective over `group`.  Rank r allocates its buffer with pw_ipc_alloc and
    all-gathers (pid, address, IPC handle).  Buffers of other processes are mapped
    with pw_ipc_open (NVLink peer memory on an NVSwitch node; CUDA IPC also maps
    another process's buffer on the same GPU, which the tests use).  Buffers of the
    same process (thread ranks) are used directly.
    """

    def __init__(self, ctx, numel: int, group=None):
        from . import _lib

        self.ctx, self.group, self.numel = ctx, group, int(numel)
        lib = ctx.lib
        ptr, handle = _lib.c_vp(), ctypes.create_string_buffer(64)
        _lib.check(lib.pw_ipc_alloc(ctx.handle, self.numel * 8, ctypes.byref(ptr), handle))
        self.ptr = int(ptr.value)
        self.local = device_vector(self.ptr, self.numel, torch.device("cuda", ctx.device))
        world, rank = tdist.get_world_size(group), tdist.get_rank(group)
        info = [None] * world
        tdist.all_gather_object(info, (os.getpid(), self.ptr, handle.raw), group=group)
        self.peer_ptrs, self._mapped = [], []
        for r, (pid, addr, h) in enumerate(info):
            if r == rank:
                continue
            if pid == os.getpid():
                self.peer_ptrs.append(int(addr))
            else:
                q = _lib.c_vp()
                _lib.check(lib.pw_ipc_open(ctx.handle, h, ctypes.byref(q)))
                self.peer_ptrs.append(int(q.value))
                self._mapped.append(int(q.value))

    def close(self):
        """Collective: unmap the peers' buffers, then free this rank's once nobody maps it."""
        from . import _lib

        if self.ptr is None:
            return
        lib = self.ctx.lib
        tdist.barrier(group=self.group)
        for q in self._mapped:
            _lib.check(lib.pw_ipc_close(self.ctx.handle, _lib.c_vp(q)))
        tdist.barrier(group=self.group)
        _lib.check(lib.pw_ipc_free(self.ctx.handle, _lib.c_vp(self.ptr)))
        self.ptr, self.peer_ptrs, self._mapped, self.local = None, [], [], None


class FusedShardedFine:
    """ShardedFine with the all-gather fused into the fine kernel.

    Rank r propagates its block of slices with ``prop.apply_to_peers``
    (pw_prop_apply_to_peers).  The last RK3 step of the row-marching kernel stores
    each output row into this rank's gather buffer and into every peer's, over
    NVLink, while the other rows are still being computed.  There is no NCCL call
    on the data path.

    The gather buffer has two halves used by alternate calls, so ONE barrier per call
    (after the stores: every rank's rows have landed everywhere) also orders the reuse:
    a rank storing into half h at call k is past call k-1's barrier, which every peer
    joined only after its stream had consumed half h at call k-2.  Under NCCL that
    barrier is stream-ordered (a one-element all-reduce enqueued behind the kernel; the
    host does not block); under gloo (CPU rendezvous, the one-GPU tests) it is a host
    synchronise + barrier.
    """

    def __init__(self, prop, group=None):
        self.prop = prop
        self.group = group
        self._buf = None
        self._cap = 0
        self._calls = 0
        self._token = None

    @property
    def world(self):
        return tdist.get_world_size(self.group) if tdist.is_initialized() else 1

    @property
    def rank(self):
        return tdist.get_rank(self.group) if tdist.is_initialized() else 0

    def _buffer(self, numel):
        if self._buf is None or self._cap < numel:
            if self._buf is not None:
                self._buf.close()
            self._buf = PeerGather(self.prop.ctx, 2 * numel, self.group)  # collective (host rendezvous)
            self._cap, self._calls = numel, 0
        return self._buf

    def close(self):
        if self._buf is not None:
            self._buf.close()
            self._buf = None

    def _barrier(self, stream):
        """Every rank's stores of this call are complete and visible on every rank."""
        if tdist.get_backend(self.group) == "nccl":
            if self._token is None:
                self._token = torch.zeros(1, dtype=torch.float32, device=stream.device)
            tdist.all_reduce(self._token, group=self.group)  # ordered on the current stream
        else:
            stream.synchronize()
            tdist.barrier(group=self.group)

    def __call__(self, qk: torch.Tensor) -> torch.Tensor:
        world, rank = self.world, self.rank
        n, d = qk.shape
        if world == 1:
            return self.prop.apply(qk)
        buf = self._buffer(n * d)
        base = (self._calls & 1) * self._cap
        self._calls += 1
        lo, hi = shard_range(n, rank, world)
        stream = torch.cuda.current_stream(qk.device)
        if hi > lo:
            out = buf.local[base + lo * d:base + hi * d].view(hi - lo, d)
            self.prop.apply_to_peers(qk[lo:hi], out, [p + (base + lo * d) * 8 for p in buf.peer_ptrs])
        self._barrier(stream)
        return buf.local[base:base + n * d].view(n, d).clone()

    def batch(self, states):
        t = torch.as_tensor(states)
        return self(t).cpu().numpy()


class _DevVector:
    """A raw device pointer seen by torch without a copy (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_vector(ptr: int, n: int, device) -> torch.Tensor:
    return torch.as_tensor(_DevVector(ptr, n), device=device)


class NcclComm:
    """The library's own NCCL communicator for the row-sharded sweep (pw_ctx_set_nccl).

    Collective over `group`: rank 0 creates the 128-byte ncclUniqueId (pw_nccl_unique_id),
    torch.distributed broadcasts it once, and every rank initialises the context's
    communicator.  From then on the serial correction's allreduce of r doubles and
    all-gather of qn's row blocks, and the TSQR all-gather, are NCCL calls the library
    enqueues on its stream -- no Python callback per serial step.
    """

    def __init__(self, ctx, group=None):
        from . import _lib

        self.ctx = ctx
        rank, world = tdist.get_rank(group), tdist.get_world_size(group)
        idbuf = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.check(ctx.lib.pw_nccl_unique_id(idbuf))
        obj = [idbuf.raw]
        tdist.broadcast_object_list(obj, src=tdist.get_global_rank(group, 0) if group is not None else 0,
                                    group=group)
        _lib.check(ctx.lib.pw_ctx_set_nccl(ctx.handle, obj[0], rank, world))
        self.rank, self.world = rank, world

    def allreduce(self, t: torch.Tensor) -> None:
        from . import _lib

        _lib.check(self.ctx.lib.pw_comm_allreduce(self.ctx.handle, _lib.ptr(t), t.numel()))

    def allgather(self, t: torch.Tensor, block: int) -> None:
        from . import _lib

        _lib.check(self.ctx.lib.pw_comm_allgather(self.ctx.handle, _lib.ptr(t), int(block), t.numel()))


class RowShardComm:
    """Collectives of the row-sharded serial correction (include/pitwave_b200.h,
    pw_ctx_set_comm): an in-place allreduce of the partial alpha (r doubles) and an
    all-gather of the ranks' row blocks of qn_{i+1}, over a torch.distributed group."""

    def __init__(self, group, device):
        self.group = group
        self.device = device
        self.world = tdist.get_world_size(group)
        self.rank = tdist.get_rank(group)
        self.last_error = None

    def allreduce(self, ptr: int, count: int) -> None:
        tdist.all_reduce(device_vector(ptr, count, self.device), group=self.group)

    def allgather(self, ptr: int, block: int, total: int) -> None:
        gather_rows(device_vector(ptr, total, self.device), block, self.group)


def tsqr(local: torch.Tensor, group=None):
    """Row-sharded QR of A = [A_0; A_1; ...] (A_g = ``local`` on rank g, rows_g >= m).

    The decomposition of the device path (csrc/api.cu factor_tsqr / form_q_tsqr):
    A_g = Q_g R_g locally (Householder), the R_g are all-gathered and stacked,
    [R_0; R_1; ...] = Q_R R.  Returns (R, this rank's rows of Q = Q_g Q_R[g m:(g+1) m]).
    R is the R of A up to row signs; pivoted QR of R gives dgeqp3's pivots on A.
    """
    m = local.shape[1]
    if local.shape[0] < m:
        raise ValueError("TSQR needs at least as many rows per rank as columns")
    q_loc, r_loc = torch.linalg.qr(local)
    world = tdist.get_world_size(group) if tdist.is_initialized() else 1
    rank = tdist.get_rank(group) if tdist.is_initialized() else 0
    if world == 1:
        return r_loc, q_loc
    parts = [torch.empty_like(r_loc) for _ in range(world)]
    tdist.all_gather(parts, r_loc.contiguous(), group=group)
    q_r, r = torch.linalg.qr(torch.cat(parts))
    return r, q_loc @ q_r[rank * m:(rank + 1) * m]


def row_block(total: int, block: int, rank: int):
    """[lo, hi) of `rank`'s rows for blocks of `block` rows (the last may be short or empty)."""
    lo = min(total, rank * block)
    return lo, min(total, lo + block)


def gather_rows(full: torch.Tensor, block: int, group=None) -> None:
    """In-place all-gather of a (total,) vector whose block `rank` is valid on each rank."""
    world, rank = tdist.get_world_size(group), tdist.get_rank(group)
    total = full.shape[0]
    lo, hi = row_block(total, block, rank)
    mine = torch.zeros(block, dtype=full.dtype, device=full.device)
    mine[: hi - lo] = full[lo:hi]
    out = torch.empty(world * block, dtype=full.dtype, device=full.device)
    if out.device.type == "cuda":
        tdist.all_gather_into_tensor(out, mine, group=group)
    else:  # gloo: list form
        parts = list(out.split(block))
        tdist.all_gather(parts, mine, group=group)
        out = torch.cat(parts)
    full.copy_(out[:total])
