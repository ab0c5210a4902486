"""ctypes binding of libpitwave_b200.so (the C ABI in include/pitwave_b200.h).

The library is the only compute path of this package: there is no CPU
fallback.  Loading fails loudly when the .so is missing (run
``python -c "import __graft_entry__ as g; g.build()"``) or when no sm_100
device is present.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpitwave_b200.so")

PW_OK = 0
SCHEME_RK3 = 0
SCHEME_SPLIT_FE_FB = 1
SCHEME_RK3_SCALAR = 2
SCHEME_SPLIT_RK3_FB = 3
MODE_ORIGINAL = 0
MODE_KSE = 1

c_dp = ctypes.POINTER(ctypes.c_double)
c_ip = ctypes.POINTER(ctypes.c_int)
c_vp = ctypes.c_void_p
FINE_HOOK = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_longlong)
FINE_ROWS_HOOK = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_longlong,
                                  ctypes.c_longlong, ctypes.c_longlong)
ALLREDUCE_HOOK = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_vp, ctypes.c_longlong)
ALLGATHER_HOOK = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_vp, ctypes.c_longlong, ctypes.c_longlong)


class PdeDesc(ctypes.Structure):
    _fields_ = [
        ("scheme", ctypes.c_int),
        ("nx", ctypes.c_int), ("ny", ctypes.c_int),
        ("dx", ctypes.c_double), ("dy", ctypes.c_double),
        ("cs", ctypes.c_double),
        ("order", ctypes.c_int),
        ("a1", ctypes.c_double), ("a2", ctypes.c_double),
        ("h", ctypes.c_double),
        ("n_sound", ctypes.c_int),
        ("nsteps", ctypes.c_int),
        ("const_velocity", ctypes.c_int),
        ("vel_u", ctypes.c_double), ("vel_v", ctypes.c_double),
        ("uf", c_dp), ("vf", c_dp),
        ("nu_damp", ctypes.c_double),
    ]


# (name, restype, argtypes) -- every symbol include/pitwave_b200.h declares
SIGNATURES = [
    ("pw_last_error", ctypes.c_char_p, []),
    ("pw_version", ctypes.c_int, []),
    ("pw_ctx_create", ctypes.c_int, [ctypes.c_int, c_vp, ctypes.POINTER(c_vp)]),
    ("pw_ctx_destroy", ctypes.c_int, [c_vp]),
    ("pw_ctx_set_stream", ctypes.c_int, [c_vp, c_vp]),
    ("pw_ctx_synchronize", ctypes.c_int, [c_vp]),
    ("pw_ctx_set_strict", ctypes.c_int, [c_vp, ctypes.c_int]),
    ("pw_ctx_launch_count", ctypes.c_longlong, [c_vp]),
    ("pw_prop_create_pde", ctypes.c_int, [c_vp, ctypes.POINTER(PdeDesc), ctypes.POINTER(c_vp)]),
    ("pw_prop_create_dense", ctypes.c_int, [c_vp, c_vp, ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("pw_prop_destroy", ctypes.c_int, [c_vp]),
    ("pw_prop_dim", ctypes.c_longlong, [c_vp]),
    ("pw_prop_apply", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_longlong]),
    ("pw_prop_apply_to_peers", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_longlong,
                                              ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("pw_ipc_alloc", ctypes.c_int, [c_vp, ctypes.c_longlong, ctypes.POINTER(c_vp), ctypes.c_char_p]),
    ("pw_ipc_free", ctypes.c_int, [c_vp, c_vp]),
    ("pw_ipc_open", ctypes.c_int, [c_vp, ctypes.c_char_p, ctypes.POINTER(c_vp)]),
    ("pw_ipc_close", ctypes.c_int, [c_vp, c_vp]),
    ("pw_basis_create", ctypes.c_int, [c_vp, ctypes.c_longlong, ctypes.c_double, ctypes.c_int,
                                       ctypes.POINTER(c_vp)]),
    ("pw_basis_destroy", ctypes.c_int, [c_vp]),
    ("pw_basis_update", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int]),
    ("pw_basis_rank", ctypes.c_int, [c_vp]),
    ("pw_basis_ncols", ctypes.c_int, [c_vp]),
    ("pw_basis_views", ctypes.c_int, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                      ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    ("pw_basis_diag", ctypes.c_int, [c_vp, c_dp, c_ip]),
    ("pw_basis_project", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_longlong]),
    ("pw_basis_fine_on_projection", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int,
                                                   ctypes.c_longlong]),
    ("pw_kse_coarse", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_longlong]),
    ("pw_sweep", ctypes.c_int, [c_vp, ctypes.c_int, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int,
                                ctypes.c_double, ctypes.c_double, c_vp, c_dp, c_ip, c_dp, c_ip,
                                ctypes.POINTER(c_vp)]),
    ("pw_ctx_set_fine_hook", ctypes.c_int, [c_vp, FINE_HOOK, c_vp]),
    ("pw_ctx_set_fine_rows_hook", ctypes.c_int, [c_vp, FINE_ROWS_HOOK, c_vp]),
    ("pw_ctx_set_comm", ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ALLREDUCE_HOOK, ALLGATHER_HOOK,
                                       c_vp]),
    ("pw_ctx_set_row_shards", ctypes.c_int, [c_vp, ctypes.c_int]),
    ("pw_prop_apply_rowshard", ctypes.c_int, [c_vp, ctypes.c_int, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                              ctypes.POINTER(c_vp)]),
    ("pw_rowshard_sizes", ctypes.c_longlong, [c_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]),
    ("pw_nccl_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("pw_ctx_set_nccl", ctypes.c_int, [c_vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]),
    ("pw_comm_allreduce", ctypes.c_int, [c_vp, c_vp, ctypes.c_longlong]),
    ("pw_comm_allgather", ctypes.c_int, [c_vp, c_vp, ctypes.c_longlong, ctypes.c_longlong]),
    ("pw_ctx_set_tsqr", ctypes.c_int, [c_vp, ctypes.c_int]),
    ("pw_copy", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_longlong]),
    ("pw_residual", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_longlong, c_dp]),
    ("pw_dgemm", ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong,
                                ctypes.c_double, c_vp, ctypes.c_longlong, c_vp, ctypes.c_longlong, ctypes.c_double,
                                c_vp, ctypes.c_longlong]),
    ("pw_geqrf", ctypes.c_int, [c_vp, ctypes.c_longlong, ctypes.c_int, c_vp, ctypes.c_longlong, c_vp]),
    ("pw_window_diag", ctypes.c_int, [c_vp, c_vp, ctypes.c_longlong, ctypes.c_double, c_vp, ctypes.c_int, c_dp]),
    ("pw_probe_fp64_peak", ctypes.c_int, [c_vp, ctypes.c_int, c_dp]),
    ("pw_mem_stats", ctypes.c_int, [c_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong),
                                    ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]),
    ("pw_serial_step", ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp, c_vp, ctypes.c_int,
                                      ctypes.c_longlong, ctypes.c_longlong, c_vp, c_vp]),
]

_lib = None
_lock = threading.Lock()


class PitwaveError(RuntimeError):
    """A failed library call; .code is the PW_ERR_* status."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def load_library():
    """Load the .so and declare every exported symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: the sm_100a CUDA library is the only compute path "
                    "of paper_1510_02237_b200 (no CPU fallback). Build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'`.")
            lib = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc):
    if rc != PW_OK:
        msg = load_library().pw_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise PitwaveError(rc, msg)


class Context:
    """One library context per CUDA device, bound to torch's current stream."""

    _instances: dict = {}

    def __init__(self, device: int):
        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1510_02237_b200 needs a CUDA (B200, sm_100) device; none is visible")
        self.device = device
        self.lib = lib
        h = c_vp()
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream(device).cuda_stream
            check(lib.pw_ctx_create(device, c_vp(stream), ctypes.byref(h)))
        self.handle = h
        self._stream = stream

    @classmethod
    def get(cls, device=None) -> "Context":
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        ctx = cls._instances.get(device)
        if ctx is None:
            ctx = cls(device)
            cls._instances[device] = ctx
        ctx.bind_stream()
        return ctx

    def bind_stream(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            check(self.lib.pw_ctx_set_stream(self.handle, c_vp(s)))
            self._stream = s

    def set_strict(self, strict: bool):
        check(self.lib.pw_ctx_set_strict(self.handle, int(bool(strict))))

    def launch_count(self) -> int:
        return int(self.lib.pw_ctx_launch_count(self.handle))

    def synchronize(self):
        check(self.lib.pw_ctx_synchronize(self.handle))

    def set_row_shards(self, n: int):
        """Run the serial correction as n row shards in this process (tests of the
        multi-GPU arithmetic); 1 restores the single-shard loop."""
        check(self.lib.pw_ctx_set_row_shards(self.handle, int(n)))

    def set_tsqr(self, on: bool):
        """Factor the subspace by row-sharded TSQR in sharded sweeps."""
        check(self.lib.pw_ctx_set_tsqr(self.handle, int(bool(on))))

    def fp64_peak_tflops(self, iters: int = 4096) -> float:
        """DFMA-throughput probe (TFLOP/s, FMA = 2 flop): the fp64 roofline denominator."""
        out = ctypes.c_double()
        check(self.lib.pw_probe_fp64_peak(self.handle, int(iters), ctypes.byref(out)))
        return float(out.value)


    def mem_stats(self, reset: bool = False) -> dict:
        """Library pool high-water marks and the device's in-use bytes (cudaMemGetInfo)."""
        used, reserved, now = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_longlong()
        check(self.lib.pw_mem_stats(self.handle, int(bool(reset)), ctypes.byref(used), ctypes.byref(reserved),
                                    ctypes.byref(now)))
        return {"pool_used_high": used.value, "pool_reserved_high": reserved.value, "device_used_now": now.value}


def ptr(t: torch.Tensor):
    return c_vp(t.data_ptr())
