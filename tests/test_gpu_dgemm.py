"""The library's fp64 DMMA GEMM (csrc/dgemm.cu, pw_dgemm) against torch fp64 matmul.

Covers both operand forms the subspace uses (op(A) = A: the tall d x r products;
op(A) = A^T: the k = d reductions, which split the k range over grid.z), ragged and
odd sizes, odd leading dimensions and misaligned views (the 8-byte copy path),
beta in {0, 1, other} (beta = 0 must not read C: C starts as NaN there), k = 0,
and the column-gather / upper-triangular-B options behind Y = M[:, piv] R11^-1.
fp64 tensor cores round each k4 partial product once more than a serial dot
product, so the bound is relative to |op(A)| |B| (1e-14 per unit of k^(1/2))."""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_1510_02237_b200 import _lib

    return _lib.Context.get(0)


def call(dev, ta, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc):
    from paper_1510_02237_b200 import _lib

    _lib.check(dev.lib.pw_dgemm(dev.handle, int(ta), m, n, k, alpha, ctypes.c_void_p(A.data_ptr()), lda,
                                ctypes.c_void_p(B.data_ptr()), ldb, beta, ctypes.c_void_p(C.data_ptr()), ldc))
    torch.cuda.synchronize()


def col_major(rows, cols, ld, gen, off=0):
    """(storage, view): a column-major rows x cols matrix with leading dimension ld at
    element offset `off` of its storage."""
    buf = torch.randn(off + ld * cols, device="cuda", dtype=torch.float64, generator=gen)
    view = buf[off:off + ld * cols].view(cols, ld)[:, :rows].t()  # view[i, j] = buf[off + i + j*ld]
    return buf[off:], view


@pytest.mark.parametrize("ta,m,n,k,lda_pad,ldb_pad,ldc_pad,off,beta", [
    (False, 256, 64, 64, 0, 0, 0, 0, 0.0),
    (False, 1000, 37, 129, 3, 1, 5, 0, 1.0),       # ragged, odd lds: 8-byte copies
    (False, 786432, 64, 320, 0, 0, 0, 0, 0.0),     # c3-shaped tall product
    (False, 5000, 600, 17, 0, 2, 0, 1, -0.5),      # misaligned view, odd k
    (True, 64, 64, 786432, 0, 0, 0, 0, 0.0),       # c3 reduction (split k)
    (True, 320, 64, 100001, 1, 1, 3, 0, 1.0),      # odd reduction length
    (True, 7, 5, 3, 0, 0, 0, 1, 2.0),              # tiny
    (True, 768, 256, 200000, 0, 0, 0, 0, 0.0),
    (False, 33, 1, 1, 0, 0, 0, 0, 0.0),
])
def test_dgemm_matches_torch(dev, ta, m, n, k, lda_pad, ldb_pad, ldc_pad, off, beta):
    gen = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    ar, ac = (k, m) if ta else (m, k)
    a_buf, A = col_major(ar, ac, ar + lda_pad, gen, off)
    b_buf, B = col_major(k, n, k + ldb_pad, gen, off)
    c_buf, C = col_major(m, n, m + ldc_pad, gen, 0)
    if beta == 0.0:
        C.fill_(float("nan"))  # must not be read
    C0 = C.clone()
    alpha = 0.75
    call(dev, ta, m, n, k, alpha, a_buf, ar + lda_pad, b_buf, k + ldb_pad, beta, c_buf, m + ldc_pad)
    opA = A.t() if ta else A
    want = alpha * (opA @ B) + (beta * C0 if beta != 0.0 else 0.0)
    scale = alpha * (opA.abs() @ B.abs()) + abs(beta) * (C0.abs() if beta != 0.0 else 0.0)
    err = ((C - want).abs() / scale.clamp_min(1e-300)).max().item()
    assert err <= 1e-14 * max(1.0, np.sqrt(k) / 8), err


def test_dgemm_k0_and_empty(dev):
    gen = torch.Generator(device="cuda").manual_seed(3)
    c_buf, C = col_major(40, 6, 40, gen)
    c0 = C.clone()
    call(dev, False, 40, 6, 0, 1.0, c_buf, 40, c_buf, 1, 1.0, c_buf, 40)   # k = 0, beta 1: unchanged
    assert torch.equal(C, c0)
    call(dev, False, 40, 6, 0, 1.0, c_buf, 40, c_buf, 1, 0.0, c_buf, 40)   # k = 0, beta 0: zeroed
    assert torch.count_nonzero(C) == 0
    call(dev, True, 0, 6, 5, 1.0, c_buf, 5, c_buf, 5, 0.0, c_buf, 1)       # m = 0: no-op


def test_dgemm_deterministic(dev):
    """The split-k reduction sums partial tiles in a fixed order: bitwise repeatable."""
    gen = torch.Generator(device="cuda").manual_seed(11)
    a_buf, _ = col_major(300000, 96, 300000, gen)
    b_buf, _ = col_major(300000, 48, 300000, gen)
    outs = []
    for _ in range(3):
        c = torch.empty(96 * 48, device="cuda", dtype=torch.float64)
        call(dev, True, 96, 48, 300000, 1.0, a_buf, 300000, b_buf, 300000, 0.0, c, 96)
        outs.append(c)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
