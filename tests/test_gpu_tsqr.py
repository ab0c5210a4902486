"""The library's tall-skinny Householder QR (csrc/tsqr.cu, pw_geqrf) against LAPACK
dgeqrf (scipy.linalg.lapack, the library under the reference's scipy qr,
subspace.py:66-68).

Checked on the geqrf output format itself: the reflectors rebuild an orthogonal Q
(||Q^T Q - I|| ~ eps), Q R reproduces A to backward-error level (~eps ||A||), and for
well-conditioned panels R and tau equal LAPACK's to ~1e-13 (same sign convention:
R_jj = -sign(alpha_j) ||x_j||).  Shapes: one leaf, ragged leaves, several tree
levels, sub-panel blocking (cols > 32, not a multiple of 32), cols > rows, zero and
near-dependent columns (the Parareal snapshots are nearly dependent)."""
import ctypes

import numpy as np
import pytest
import torch
from scipy.linalg import lapack

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_1510_02237_b200 import _lib

    return _lib.Context.get(0)


def geqrf(dev, A, lda_pad=0):
    from paper_1510_02237_b200 import _lib

    rows, cols = A.shape
    lda = rows + lda_pad
    buf = torch.zeros(lda * max(cols, 1), dtype=torch.float64, device="cuda")
    buf.view(max(cols, 1), lda)[:cols, :rows] = torch.as_tensor(A.T.copy()).cuda()
    tau = torch.zeros(max(1, min(rows, cols)), dtype=torch.float64, device="cuda")
    _lib.check(dev.lib.pw_geqrf(dev.handle, rows, cols, ctypes.c_void_p(buf.data_ptr()), lda,
                                ctypes.c_void_p(tau.data_ptr())))
    torch.cuda.synchronize()
    out = buf.view(max(cols, 1), lda)[:cols, :rows].cpu().numpy().T.copy()
    return out, tau.cpu().numpy()[:min(rows, cols)]


def q_from(qr, tau):
    rows, cols = qr.shape
    k = len(tau)
    Q = np.eye(rows, k)
    for j in reversed(range(k)):
        v = np.zeros(rows)
        v[j] = 1.0
        v[j + 1:] = qr[j + 1:, j]
        Q -= tau[j] * np.outer(v, v @ Q)
    return Q


@pytest.mark.parametrize("rows,cols,lda_pad,kind", [
    (128, 8, 0, "rand"), (1000, 32, 3, "rand"), (5000, 45, 0, "rand"), (200000, 64, 0, "rand"),
    (70000, 96, 1, "graded"), (33, 40, 0, "rand"), (300, 16, 0, "dependent"), (4097, 32, 0, "zero_col"),
    (786432, 64, 0, "graded"),
])
def test_geqrf_matches_lapack(dev, rows, cols, lda_pad, kind):
    rng = np.random.default_rng(rows + cols)
    A = rng.standard_normal((rows, cols))
    if kind == "graded":      # column scales down to 1e-12 (the snapshot spectra)
        A = A @ np.diag(np.logspace(0, -12, cols))
    elif kind == "dependent":  # near-duplicate columns
        A[:, 5] = A[:, 3] + 1e-11 * A[:, 5]
        A[:, 9] = A[:, 2]
    elif kind == "zero_col":
        A[:, 7] = 0.0
    qr, tau = geqrf(dev, A, lda_pad)
    k = min(rows, cols)
    R = np.triu(qr[:k, :])
    Q = q_from(qr, tau)
    assert np.abs(Q.T @ Q - np.eye(k)).max() <= 1e-13
    assert np.abs(Q @ R - A).max() <= 1e-13 * np.abs(A).max()
    if kind == "rand" and rows * cols <= 2e7:
        ql, taul, _, info = lapack.dgeqrf(A)
        assert info == 0
        Rl = np.triu(ql[:k, :])
        # equal up to the reflector of a length-1 column (rows <= cols: LAPACK takes H = I
        # there, the reconstruction H = -1), i.e. up to row signs of R
        sg = np.sign(np.diag(R)) * np.sign(np.diag(Rl))
        assert np.abs(sg[:, None] * R - Rl).max() <= 1e-12 * np.abs(Rl).max()
        same = sg > 0
        np.testing.assert_allclose(tau[same], taul[:k][same], rtol=0, atol=1e-12)


@pytest.mark.parametrize("d,m,dup", [(4096, 40, 0), (5000, 96, 7), (700, 300, 25), (64, 64, 3), (33, 50, 0)])
def test_pivoted_qr_one_barrier_kernel_is_bitwise_equal_to_the_two_barrier_kernel(dev, monkeypatch, d, m, dup):
    """The small pivoted QR of R1 (pqr1_kernel: every block forms the pivot column's reflector,
    one grid barrier per column) against the two-barrier kernel (PW_PQR=2): same pivots, same
    rank, bitwise equal Q and images -- including near-duplicate snapshots (rank decisions) and
    more snapshots than rows."""
    from paper_1510_02237_b200.subspace import Subspace

    rng = np.random.default_rng(d + m)
    cols = [rng.standard_normal(d) for _ in range(m - dup)]
    for k in range(dup):  # near-duplicates: a kept column plus a perturbation at the rank tolerance
        cols.append(cols[k] * (1.0 + 1e-3 * k) + 1e-11 * rng.standard_normal(d))
    imgs = [np.roll(c, 1) * 0.5 for c in cols]
    out = {}
    for variant in ("2", "1"):
        monkeypatch.setenv("PW_PQR", variant)
        sub = Subspace(d).update(cols[: m // 2], imgs[: m // 2]).update(cols[m // 2:], imgs[m // 2:])
        out[variant] = (sub.rank, sub.q.copy(), sub.fq.copy())
    assert out["1"][0] == out["2"][0]
    assert out["1"][0] <= min(d, m)
    np.testing.assert_array_equal(out["1"][1], out["2"][1])
    np.testing.assert_array_equal(out["1"][2], out["2"][2])


@pytest.mark.parametrize("rows,cols,lda_pad", [(1000, 32, 3), (5000, 45, 0), (200000, 64, 0), (70001, 96, 1), (33, 40, 0)])
def test_geqrf_leaf_expand_and_trailing_update_variants(dev, monkeypatch, rows, cols, lda_pad):
    """The panel QR's two streaming kernels against the kernels they replaced: the row-per-thread
    leaf pass of the explicit Q (tsqr_expand_leaf_rows_kernel) accumulates in the staged kernel's
    order, so geqrf's output is bitwise equal (PW_TSQR_EXPAND=1); the rank-32 trailing update
    (rank_tb_update_kernel) sums its 32 products in another order than the GEMM tiles
    (PW_TSQR_TRAIL_GEMM=1), so that pair agrees to rounding."""
    rng = np.random.default_rng(3 * rows + cols)
    A = rng.standard_normal((rows, cols)) @ np.diag(np.logspace(0, -9, cols))
    qr0, tau0 = geqrf(dev, A, lda_pad)
    monkeypatch.setenv("PW_TSQR_EXPAND", "1")
    qr1, tau1 = geqrf(dev, A, lda_pad)
    np.testing.assert_array_equal(qr0, qr1)
    np.testing.assert_array_equal(tau0, tau1)
    monkeypatch.delenv("PW_TSQR_EXPAND")
    monkeypatch.setenv("PW_TSQR_TRAIL_GEMM", "1")
    qr2, tau2 = geqrf(dev, A, lda_pad)
    k = min(rows, cols)
    scale = np.abs(np.triu(qr0[:k, :])).max(axis=0)  # per column: R's largest entry
    assert (np.abs(np.triu(qr2[:k, :]) - np.triu(qr0[:k, :])).max(axis=0) <= 1e-12 * scale + 1e-300).all()
    np.testing.assert_allclose(tau2, tau0, rtol=0, atol=1e-12)
