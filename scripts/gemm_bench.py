"""DMMA GEMM (pw_dgemm) vs cuBLAS (PW_CUBLAS=1) on the subspace's product shapes.

    python scripts/gemm_bench.py

Shapes (m, n, k, trans_a): the c4 / c3 window products of the refactorisation --
applyQ1T's V^T N (k = d reduction) and V (T^T V^T N) (tall), Q = Q1 [Q2; 0] (tall,
k = m), Y = M X (tall) -- timed with CUDA events, TFLOP/s against the fp64 peak.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1510_02237_b200 import _lib  # noqa: E402

SHAPES = [
    ("c4 V^T N   (k=d)", 768, 256, 3145728, True),
    ("c4 V X2    (tall)", 3145728, 256, 768, False),
    ("c4 Q=Q1Q2  (tall)", 3145728, 578, 1024, False),
    ("c3 V^T N   (k=d)", 256, 64, 786432, True),
    ("c3 Q=Q1Q2  (tall)", 786432, 310, 320, False),
    ("c3 Q^T qk  (k=d)", 310, 64, 786432, True),
    ("tsqr trail (tall, k=32)", 3145728, 224, 32, False),
]


def run(ctx, m, n, k, ta, reps=5):
    a = torch.randn((k * m), device="cuda", dtype=torch.float64)
    b = torch.randn((k * n), device="cuda", dtype=torch.float64)
    c = torch.zeros((m * n), device="cuda", dtype=torch.float64)
    lda = k if ta else m

    def once():
        _lib.check(ctx.lib.pw_dgemm(ctx.handle, int(ta), m, n, k, 1.0, ctypes.c_void_p(a.data_ptr()), lda,
                                    ctypes.c_void_p(b.data_ptr()), k, 0.0, ctypes.c_void_p(c.data_ptr()), m))

    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out = c.clone()
    del a, b, c
    return ms, out


def main():
    ctx = _lib.Context.get(0)
    ctx.bind_stream()
    for name, m, n, k, ta in SHAPES:
        flop = 2.0 * m * n * k
        os.environ["PW_CUBLAS"] = "0"
        ms, own = run(ctx, m, n, k, ta)
        os.environ["PW_CUBLAS"] = "1"
        ms_b, ref = run(ctx, m, n, k, ta)
        os.environ["PW_CUBLAS"] = "0"
        print(f"{name:26s} {m}x{n}x{k}: own {ms:8.3f} ms {flop / ms / 1e9:6.1f} TF | cuBLAS {ms_b:8.3f} ms "
              f"{flop / ms_b / 1e9:6.1f} TF", flush=True)


if __name__ == "__main__":
    main()
