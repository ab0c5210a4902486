"""Fixed-step propagators on the B200 (reference integrators.py).

``PropagatorSpec`` / ``make_propagator`` keep the reference's semantics
(integrators.py:26-76).  Execution goes through device propagator objects
that wrap a C-ABI ``pw_prop``:

* ``SlicePropagator(spec, span)`` -- ``propagate(spec, ., 0, span)`` for a
  whole batch of slices in one call (the reference's per-slice closures of
  PitConfig.vector_propagators, parareal.py:182-194, plus its _fine_all
  thread pool, parareal.py:62-65);
* ``MatrixPropagator(A)`` -- the dense linear map the reference tests use as
  a propagator seam (tests/test_parareal.py:14-15), executed with DGEMM.

Both are callable on a flat host vector (drop-in for the reference
closures) and expose ``apply(x)`` on a (batch, d) CUDA tensor.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .mesh import ACOUSTIC, Grid2D, State, face_normal_velocities
from .physics import ModelSpec, damping_coefficients

RK3 = "rk3"
SPLIT_FE_FB = "split_fe_fb"
SPLIT_RK3_FB = "split_rk3_fb"
SCHEMES = (RK3, SPLIT_FE_FB, SPLIT_RK3_FB)


@dataclass(frozen=True)
class PropagatorSpec:
    """Scheme + model + mesh + Courant number (reference integrators.py:26-61)."""

    scheme: str
    model: ModelSpec
    grid: Grid2D
    cfl: float
    n_sound: int = 1

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"scheme must be one of {SCHEMES}, got {self.scheme!r}")
        if self.cfl <= 0:
            raise ValueError(f"cfl must be positive, got {self.cfl}")
        if self.n_sound < 1:
            raise ValueError(f"n_sound must be at least 1, got {self.n_sound}")
        if self.scheme != RK3 and self.model.kind != ACOUSTIC:
            raise ValueError(f"{self.scheme} is a split acoustic scheme; model is {self.model.kind}")
        if self.reference_speed <= 0:
            raise ValueError("reference wave speed is zero; cannot derive a step size")

    @property
    def reference_speed(self) -> float:
        if self.model.kind == ACOUSTIC:
            return self.model.sound_speed
        return self.model.vel.max_component_speed(self.grid)

    @property
    def dt(self) -> float:
        return self.cfl * min(self.grid.dx, self.grid.dy) / self.reference_speed


def make_propagator(scheme, model, grid, cfl, n_sound=1) -> PropagatorSpec:
    """Fill the damping timescale: h (RK3) or h / n_sound (split), integrators.py:64-76."""
    spec = PropagatorSpec(scheme=scheme, model=model, grid=grid, cfl=cfl, n_sound=n_sound)
    if model.nu_damp > 0:
        tau = spec.dt if scheme == RK3 else spec.dt / n_sound
        spec = PropagatorSpec(scheme=scheme, model=model.with_timescale(tau), grid=grid, cfl=cfl,
                              n_sound=n_sound)
    return spec


def step_count(span: float, h: float) -> int:
    """n = round(span / h) with the reference's 1e-9 integrality check (integrators.py:135-139)."""
    n_real = span / h
    n = round(n_real)
    if n < 1 or abs(n_real - n) > 1e-9 * max(1.0, abs(n_real)):
        raise ValueError(f"interval {span} is not an integer multiple of the step {h} (ratio {n_real})")
    return n


def _as_device_batch(x, dim, device):
    """(tensor (B, d) on device, was_numpy, squeeze)"""
    if isinstance(x, torch.Tensor):
        t = x
        was_np = False
    else:
        t = torch.as_tensor(np.asarray(x, dtype=np.float64))
        was_np = True
    squeeze = t.dim() == 1
    if squeeze:
        t = t.unsqueeze(0)
    if t.dim() != 2 or t.shape[1] != dim:
        raise ValueError(f"state vector shape {tuple(x.shape)} does not match dimension {dim}")
    t = t.to(device=device, dtype=torch.float64).contiguous()
    return t, was_np, squeeze


class DevicePropagator:
    """Linear propagator executed by libpitwave_b200 (base of the two kinds)."""

    dim: int
    handle: ctypes.c_void_p

    def __init__(self, device=None):
        self.ctx = _lib.Context.get(device)
        self.device = torch.device("cuda", self.ctx.device)
        self.handle = None

    def apply(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """out[b] = P(x[b]) for a (B, d) float64 CUDA tensor (enqueued, no sync)."""
        self.ctx.bind_stream()
        if x.dim() != 2 or x.shape[1] != self.dim or x.dtype != torch.float64 or not x.is_cuda:
            raise ValueError("apply expects a (batch, dim) float64 CUDA tensor")
        x = x.contiguous()
        if out is None:
            out = torch.empty_like(x)
        _lib.check(self.ctx.lib.pw_prop_apply(self.handle, _lib.ptr(x), _lib.ptr(out),
                                              x.shape[0], self.dim))
        return out

    def apply_to_peers(self, x: torch.Tensor, out: torch.Tensor, peer_ptrs) -> torch.Tensor:
        """apply(x, out) that also stores the result at each device address in peer_ptrs
        (buffers laid out like `out`, e.g. other ranks' buffers mapped by dist.PeerGather):
        pw_prop_apply_to_peers.  Enqueued, no sync."""
        self.ctx.bind_stream()
        if x.dim() != 2 or x.shape[1] != self.dim or x.dtype != torch.float64 or not x.is_cuda:
            raise ValueError("apply_to_peers expects a (batch, dim) float64 CUDA tensor")
        if out.shape != x.shape or out.stride(1) != 1 or out.stride(0) != self.dim:
            raise ValueError("out must be a contiguous (batch, dim) tensor")
        x = x.contiguous()
        arr = (_lib.c_vp * max(1, len(peer_ptrs)))(*[_lib.c_vp(int(p)) for p in peer_ptrs])
        _lib.check(self.ctx.lib.pw_prop_apply_to_peers(self.handle, _lib.ptr(x), _lib.ptr(out), x.shape[0],
                                                       self.dim, len(peer_ptrs), arr))
        return out

    def batch(self, states):
        """Host (B, d) -> host (B, d)."""
        t, _, _ = _as_device_batch(states, self.dim, self.device)
        return self.apply(t).cpu().numpy()

    def __call__(self, vec):
        t, was_np, squeeze = _as_device_batch(vec, self.dim, self.device)
        out = self.apply(t)
        if squeeze:
            out = out[0]
        return out.cpu().numpy() if was_np else out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                self.ctx.lib.pw_prop_destroy(h)
            except Exception:
                pass
            self.handle = None


class SlicePropagator(DevicePropagator):
    """propagate(spec, ., 0, span) as one batched device call over any number of states."""

    def __init__(self, spec: PropagatorSpec, span: float | None = None, nsteps: int | None = None,
                 h: float | None = None, device=None):
        super().__init__(device)
        self.spec = spec
        self.h = spec.dt if h is None else float(h)
        if nsteps is None:
            nsteps = 0 if (span is None or span == 0) else step_count(span, self.h)
        self.nsteps = int(nsteps)
        g = spec.grid
        self.grid = g
        model = spec.model
        scalar = model.kind != ACOUSTIC
        self.dim = (1 if scalar else 3) * g.nx * g.ny
        a1 = a2 = 0.0
        if scalar:                   # advection_rhs (physics.py:77-80): no acoustics, no damping
            scheme = _lib.SCHEME_RK3_SCALAR
        elif spec.scheme == RK3:
            if model.nu_damp > 0:   # physics._alphas: tau = model.damping_timescale
                a1, a2 = damping_coefficients(model.nu_damp, g.dx, g.dy, model.damping_timescale)
            scheme = _lib.SCHEME_RK3
        elif spec.scheme == SPLIT_FE_FB:   # _fb_integrate: tau = dt / n_sound
            tau = self.h / spec.n_sound
            if model.nu_damp > 0:
                a1, a2 = damping_coefficients(model.nu_damp, g.dx, g.dy, tau)
            scheme = _lib.SCHEME_SPLIT_FE_FB
        else:                        # split_rk3_fb: the device derives each stage's damping
            scheme = _lib.SCHEME_SPLIT_RK3_FB
        ux, vy = face_normal_velocities(model.vel, g)
        self._uf = np.ascontiguousarray(ux, dtype=np.float64)
        self._vf = np.ascontiguousarray(vy, dtype=np.float64)
        desc = _lib.PdeDesc(
            scheme=scheme, nx=g.nx, ny=g.ny, dx=g.dx, dy=g.dy, cs=float(model.sound_speed),
            order=int(model.advective_flux_order), a1=float(a1), a2=float(a2), h=self.h,
            n_sound=int(spec.n_sound), nsteps=self.nsteps, const_velocity=0, vel_u=0.0, vel_v=0.0,
            uf=self._uf.ctypes.data_as(_lib.c_dp), vf=self._vf.ctypes.data_as(_lib.c_dp),
            nu_damp=float(model.nu_damp))
        h = _lib.c_vp()
        _lib.check(self.ctx.lib.pw_prop_create_pde(self.ctx.handle, ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h
        self.a1, self.a2 = a1, a2


class MatrixPropagator(DevicePropagator):
    """q -> A q on the device (the reference tests' dense-matrix seam)."""

    def __init__(self, a, device=None):
        super().__init__(device)
        a_t = torch.as_tensor(np.asarray(a, dtype=np.float64) if not isinstance(a, torch.Tensor) else a)
        if a_t.dim() != 2 or a_t.shape[0] != a_t.shape[1]:
            raise ValueError("MatrixPropagator needs a square matrix")
        self.dim = int(a_t.shape[0])
        # column-major on the device == row-major transpose
        a_cm = a_t.to(self.device, torch.float64).t().contiguous()
        h = _lib.c_vp()
        _lib.check(self.ctx.lib.pw_prop_create_dense(self.ctx.handle, _lib.ptr(a_cm), self.dim,
                                                     ctypes.byref(h)))
        self.ctx.synchronize()
        self.handle = h


def propagate(spec: PropagatorSpec, state: State, t0: float, t1: float) -> State:
    """Advance state from t0 to t1 with the scheme's fixed step, on the device.

    Reference integrators.py:126-146: (t1-t0) must be an integer number of
    steps (1e-9 relative); blow-up overflows quietly to inf/nan.
    """
    if t1 == t0:
        return state
    n = step_count(t1 - t0, spec.dt)
    prop = SlicePropagator(spec, nsteps=n)
    return State.unflatten(state.grid, prop(state.flatten()), state.kind)


def rk3_step(state: State, spec: PropagatorSpec, h: float) -> State:
    """One RK3 step of size h (reference integrators.py:79-85)."""
    if spec.scheme != RK3:
        spec = PropagatorSpec(RK3, spec.model, spec.grid, spec.cfl, spec.n_sound)
    prop = SlicePropagator(spec, nsteps=1, h=h)
    return State.unflatten(state.grid, prop(state.flatten()), state.kind)


def split_rk3_fb_step(state: State, spec: PropagatorSpec, dt: float) -> State:
    """One split RK3-FB step of size dt (reference integrators.py:109-120)."""
    if spec.scheme != SPLIT_RK3_FB:
        spec = PropagatorSpec(SPLIT_RK3_FB, spec.model, spec.grid, spec.cfl, spec.n_sound)
    prop = SlicePropagator(spec, nsteps=1, h=dt)
    return State.unflatten(state.grid, prop(state.flatten()), state.kind)


def split_fe_fb_step(state: State, spec: PropagatorSpec, dt: float) -> State:
    """One split FE-FB step of size dt (reference integrators.py:103-106)."""
    if spec.scheme != SPLIT_FE_FB:
        spec = PropagatorSpec(SPLIT_FE_FB, spec.model, spec.grid, spec.cfl, spec.n_sound)
    prop = SlicePropagator(spec, nsteps=1, h=dt)
    return State.unflatten(state.grid, prop(state.flatten()), state.kind)
