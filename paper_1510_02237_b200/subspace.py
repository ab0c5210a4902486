"""Device-resident Krylov subspace (reference subspace.py:31-111).

``Subspace`` keeps the reference's contract -- ``update`` returns a new
object holding every snapshot/image pair, re-runs a column-pivoted QR over
all snapshots, truncates at ``rank_tol * |R_11|`` and rebuilds
``FQ = images * scatter(R11^-1)`` -- but all of it runs on the B200:
cuSOLVER Householder QR of the d x m block, the sm_100a pivoted QR of its
m x m factor (csrc/linalg.cu), DGEMMs for Q and FQ.  ``q``, ``fq``,
``snapshots`` and ``images`` are host copies made on access, as the
reference tests inspect them as numpy arrays.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

DEFAULT_RANK_TOL = 1e-10


class Subspace:
    """Orthonormal basis q (d x r) plus fine images fq of its columns."""

    def __init__(self, dim: int, rank_tol: float = DEFAULT_RANK_TOL, *, _handle=None, _ctx=None,
                 _keep=None):
        self.dim = int(dim)
        self.rank_tol = float(rank_tol)
        self._ctx = _ctx
        self._handle = _handle
        self._keep = _keep  # objects the handle depends on (coarse propagator of a sweep basis)
        self._pending = []  # (states, images) host/device columns not yet uploaded

    # ------------------------------------------------------------ plumbing
    def _context(self):
        if self._ctx is None:
            self._ctx = _lib.Context.get()
        return self._ctx

    @property
    def rank(self) -> int:
        if self._handle is None:
            return 0
        return int(self._ctx.lib.pw_basis_rank(self._handle))

    @property
    def ncols(self) -> int:
        if self._handle is None:
            return 0
        return int(self._ctx.lib.pw_basis_ncols(self._handle))

    def _views(self):
        q, fq, s, im = (_lib.c_vp() for _ in range(4))
        _lib.check(self._ctx.lib.pw_basis_views(self._handle, ctypes.byref(q), ctypes.byref(fq),
                                                ctypes.byref(s), ctypes.byref(im)))
        return q.value, fq.value, s.value, im.value

    def _host_cols(self, ptr, ncols):
        if ncols == 0 or not ptr:
            return np.empty((self.dim, 0))
        out = np.empty((ncols, self.dim))
        # device column-major (d x ncols) == host row-major (ncols x d)
        _lib.check(self._ctx.lib.pw_copy(self._ctx.handle, _lib.c_vp(out.ctypes.data),
                                         _lib.c_vp(ptr), out.nbytes))
        return out.T.copy()

    @property
    def q(self):
        if self._handle is None:
            return np.empty((self.dim, 0))
        return self._host_cols(self._views()[0], self.rank)

    @property
    def fq(self):
        if self._handle is None:
            return np.empty((self.dim, 0))
        return self._host_cols(self._views()[1], self.rank)

    @property
    def snapshots(self):
        if self._handle is None:
            return np.empty((self.dim, 0))
        ptr = self._views()[2]
        if not ptr and self.ncols:
            raise RuntimeError("snapshots were not retained: this subspace came from a lean sweep "
                               "(device memory too small for a separate snapshot copy)")
        return self._host_cols(ptr, self.ncols)

    @property
    def images(self):
        if self._handle is None:
            return np.empty((self.dim, 0))
        ptr = self._views()[3]
        if not ptr and self.ncols:
            raise RuntimeError("images were not retained: this subspace came from a lean sweep")
        return self._host_cols(ptr, self.ncols)

    def diag_ratios(self):
        """|R_jj| / |R_11| of the last refactorisation (rank diagnostics)."""
        if self._handle is None or self.ncols == 0:
            return np.empty(0)
        out = np.empty(min(self.ncols, self.dim))
        piv = np.empty(self.ncols, dtype=np.int32)
        _lib.check(self._ctx.lib.pw_basis_diag(self._handle, out.ctypes.data_as(_lib.c_dp),
                                               piv.ctypes.data_as(_lib.c_ip)))
        return out

    # ------------------------------------------------------------ reference API
    def update(self, new_states, new_images) -> "Subspace":
        """Return a new subspace including the given snapshot/image pairs (subspace.py:46-80)."""
        if len(new_states) != len(new_images):
            raise ValueError(f"got {len(new_states)} states but {len(new_images)} images")
        for vec in (*new_states, *new_images):
            if tuple(np.shape(vec)) != (self.dim,):
                raise ValueError(f"snapshot shape {tuple(np.shape(vec))} does not match dimension {self.dim}")
        ctx = self._context()
        dev = torch.device("cuda", ctx.device)
        m_old = self.ncols
        cols_s = [torch.as_tensor(np.asarray(c, dtype=np.float64)) if not isinstance(c, torch.Tensor) else c
                  for c in new_states]
        cols_i = [torch.as_tensor(np.asarray(c, dtype=np.float64)) if not isinstance(c, torch.Tensor) else c
                  for c in new_images]
        p = len(cols_s)
        s_all = torch.empty((m_old + p, self.dim), dtype=torch.float64, device=dev)
        i_all = torch.empty((m_old + p, self.dim), dtype=torch.float64, device=dev)
        if m_old:  # device-to-device copy of the retained columns
            _, _, sp, ip = self._views()
            nb = m_old * self.dim * 8
            _lib.check(ctx.lib.pw_copy(ctx.handle, _lib.ptr(s_all), _lib.c_vp(sp), nb))
            _lib.check(ctx.lib.pw_copy(ctx.handle, _lib.ptr(i_all), _lib.c_vp(ip), nb))
        for k in range(p):
            s_all[m_old + k] = cols_s[k].to(dev, torch.float64)
            i_all[m_old + k] = cols_i[k].to(dev, torch.float64)
        h = _lib.c_vp()
        _lib.check(ctx.lib.pw_basis_create(ctx.handle, self.dim, self.rank_tol, max(m_old + p, 1),
                                           ctypes.byref(h)))
        out = Subspace(self.dim, self.rank_tol, _handle=h, _ctx=ctx)
        ctx.bind_stream()
        _lib.check(ctx.lib.pw_basis_update(h, _lib.ptr(s_all), _lib.ptr(i_all), m_old + p))
        return out

    def _apply(self, fn, vec):
        vec_np = not isinstance(vec, torch.Tensor)
        v = torch.as_tensor(np.asarray(vec, dtype=np.float64)) if vec_np else vec
        if tuple(v.shape) != (self.dim,):
            raise ValueError(f"vector shape {tuple(v.shape)} does not match dimension {self.dim}")
        if self._handle is None or self.rank == 0:
            z = torch.zeros(self.dim, dtype=torch.float64)
            return z.numpy() if vec_np else z.to(v.device)
        ctx = self._ctx
        ctx.bind_stream()
        dv = v.to(torch.device("cuda", ctx.device), torch.float64).contiguous()
        out = torch.empty_like(dv)
        _lib.check(fn(self._handle, _lib.ptr(dv), _lib.ptr(out), 1, self.dim))
        return out.cpu().numpy() if vec_np else out

    def project(self, vec):
        """Euclidean orthogonal projection Q (Q^T v) (subspace.py:82-89)."""
        return self._apply(self._context().lib.pw_basis_project, vec)

    def fine_on_projection(self, vec):
        """FQ (Q^T v) from stored images only (subspace.py:91-98)."""
        return self._apply(self._context().lib.pw_basis_fine_on_projection, vec)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            try:
                self._ctx.lib.pw_basis_destroy(h)
            except Exception:
                pass
            self._handle = None


def update_subspace(sub: Subspace, new_states, new_images) -> Subspace:
    return sub.update(new_states, new_images)


def kse_coarse(sub: Subspace, coarse, vec):
    """K(q) = G((I - P) q) + F~(P q) (subspace.py:105-111); coarse is a DevicePropagator."""
    from .integrators import DevicePropagator

    if not isinstance(coarse, DevicePropagator):
        raise TypeError("kse_coarse needs a device propagator (SlicePropagator / MatrixPropagator); "
                        "arbitrary Python callables have no device implementation")
    vec_np = not isinstance(vec, torch.Tensor)
    if sub._handle is None or sub.rank == 0:
        return coarse(vec)
    ctx = sub._ctx
    ctx.bind_stream()
    v = torch.as_tensor(np.asarray(vec, dtype=np.float64)) if vec_np else vec
    dv = v.to(torch.device("cuda", ctx.device), torch.float64).contiguous()
    out = torch.empty_like(dv)
    _lib.check(ctx.lib.pw_kse_coarse(sub._handle, coarse.handle, _lib.ptr(dv), _lib.ptr(out), 1, sub.dim))
    return out.cpu().numpy() if vec_np else out
