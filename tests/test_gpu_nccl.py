"""The library's own NCCL transport (csrc/comm.cu, pw_ctx_set_nccl; B200 only).

Only one GPU is available to this build, and NCCL refuses two ranks on one device, so the
transport runs at world 1 here: the unique id round trip through torch.distributed, the
communicator on the context's device, the in-place allreduce (identity at world 1), the
padded all-gather (identity when the one block covers the vector; an uncovered vector is
refused), and a KSE window over an NCCL process group of one rank, whose result must equal
the same window without a group.  The sharded arithmetic the transport carries at world > 1
is the hook path's (thread ranks on one GPU, gloo on CPU: tests/test_gpu_thread_ranks.py,
tests/test_dist_gloo.py), which calls the same two entry points of comm.cu.
"""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(port, out_q):
    import numpy as np
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1510_02237_b200 import _lib, harness
        from paper_1510_02237_b200.dist import NcclComm
        from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, SlicePropagator, make_propagator
        from paper_1510_02237_b200.mesh import ACOUSTIC, ConstantVelocity, build_grid
        from paper_1510_02237_b200.parareal import kse_sweep
        from paper_1510_02237_b200.physics import ModelSpec

        ctx = _lib.Context.get(0)
        ctx.set_strict(False)
        ctx.bind_stream()
        comm = NcclComm(ctx)
        res = {}
        x = torch.arange(1000, dtype=torch.float64, device="cuda")
        y = x.clone()
        comm.allreduce(y)
        comm.allgather(y, 1000)
        torch.cuda.synchronize()
        res["identity"] = bool(torch.equal(x, y))
        try:
            comm.allgather(y, 999)  # one block of 999 cannot cover 1000 rows
            res["refuses_uncovered"] = False
        except Exception:
            res["refuses_uncovered"] = True
        # a KSE window over the one-rank NCCL group equals the window without a group
        n = 64
        g = build_grid(n, n)
        vel = ConstantVelocity(harness.VEL_U, harness.VEL_V)
        fine = SlicePropagator(make_propagator(RK3, ModelSpec(ACOUSTIC, vel, 6, 1.0, 0.005, 1.0), g, 0.5), 1.0 / 8)
        coarse = SlicePropagator(make_propagator(SPLIT_FE_FB, ModelSpec(ACOUSTIC, vel, 1, 1.0, 0.1, 1.0), g, 4.0, 16),
                                 1.0 / 8)
        q0 = harness.initial_state("c1", n=n)
        e1, r1, s1 = kse_sweep(q0, fine, coarse, 8, 3)
        e2, r2, s2 = kse_sweep(q0, fine, coarse, 8, 3, group=dist.group.WORLD)
        res["window"] = bool(s1.rank == s2.rank and np.array_equal(np.asarray(r1), np.asarray(r2)) and
                             all(np.array_equal(a, b) for a, b in zip(e1, e2)))
        out_q.put(res)
    except Exception as exc:  # reported by the parent
        out_q.put(repr(exc))
    finally:
        dist.destroy_process_group()


def test_native_nccl_transport_world_one():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert isinstance(res, dict), res
    assert all(res.values()), res
