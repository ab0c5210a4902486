"""pw_geqrf (TSQR + reconstruction) on the subspace panel shapes, CUDA-event timed.
cuSOLVER Xgeqrf reference times on B200 (profiles/r01/NOTES.md, scripts/ubench_geqrf.cu):
786432 x 32/64/128/256: 3.6 / 7.5 / 16.3 / 35.1 ms; 3145728 x 32/64/128/256: 11.8 / 25.0 / 55.2 / 121.7 ms."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1510_02237_b200 import _lib  # noqa: E402


def main():
    ctx = _lib.Context.get(0)
    ctx.bind_stream()
    shapes = [(786432, 32), (786432, 64), (786432, 128), (786432, 256), (3145728, 32),
              (3145728, 64), (3145728, 128), (3145728, 256)]
    if len(sys.argv) == 3:
        shapes = [(int(sys.argv[1]), int(sys.argv[2]))]
    for rows, cols in shapes:
        a0 = torch.randn(rows * cols, dtype=torch.float64, device="cuda")
        a = a0.clone()
        tau = torch.empty(cols, dtype=torch.float64, device="cuda")

        def once():
            a.copy_(a0)
            _lib.check(ctx.lib.pw_geqrf(ctx.handle, rows, cols, ctypes.c_void_p(a.data_ptr()), rows,
                                        ctypes.c_void_p(tau.data_ptr())))

        once()
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        reps = int(os.environ.get("QR_REPS", "3"))
        tot = 0.0
        for _ in range(reps):
            e0.record()
            a.copy_(a0)
            e1.record()
            _lib.check(ctx.lib.pw_geqrf(ctx.handle, rows, cols, ctypes.c_void_p(a.data_ptr()), rows,
                                        ctypes.c_void_p(tau.data_ptr())))
            e2.record()
            torch.cuda.synchronize()
            tot += e1.elapsed_time(e2)
        ms = tot / reps
        print(f"geqrf {rows} x {cols}: {ms:8.3f} ms  ({8.0 * rows * cols / ms / 1e6:7.1f} GB/s per pass)", flush=True)
        del a, a0


if __name__ == "__main__":
    main()
