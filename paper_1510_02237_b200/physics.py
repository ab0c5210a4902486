"""Parameters of the linear acoustic-advection model (reference ``pkg/src/pitwave/physics.py``).

The right-hand side itself never runs on the host here: the sm_100a kernels
(csrc/exact.cu, fine_fused.cu, fine_march.cu) evaluate it.  This module only
carries what those kernels are configured from -- the model kind, advecting
velocity, flux order, sound speed and divergence-damping strength -- with the
reference's up-front validation (``physics.py:21-51``), and the damping
coefficients alpha = nu h^2 / tau the launchers pass down (``physics.py:54-64``).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from .mesh import ACOUSTIC, SCALAR

VALID_ORDERS = (1, 2, 3, 4, 5, 6)


def _check_order(order: int) -> int:
    if order not in VALID_ORDERS:
        raise ValueError(f"flux order must be one of {VALID_ORDERS}, got {order}")
    return int(order)


def _damping_problem(kind, nu, tau):
    """Why (kind, nu, tau) is not a valid damping setting, or None."""
    if nu < 0:
        return f"damping strength must be nonnegative, got {nu}"
    needs_tau = nu > 0 and kind == ACOUSTIC
    if needs_tau and not (tau is not None and tau > 0):
        return "damping_timescale must be positive when nu_damp > 0"
    return None


@dataclass(frozen=True)
class ModelSpec:
    """Model kind + advecting velocity + the discretisation knobs of one propagator.

    ``damping_timescale`` is the tau of alpha = nu dx^2 / tau: the fine step for
    RK3, dt / n_sound for the split coarse scheme (set by make_propagator).
    """

    kind: str
    vel: object
    advective_flux_order: int = 6
    sound_speed: float = 30.0
    nu_damp: float = 0.0
    damping_timescale: float | None = None

    def __post_init__(self):
        if self.kind not in (SCALAR, ACOUSTIC):
            raise ValueError(f"model kind must be {SCALAR!r} or {ACOUSTIC!r}, got {self.kind!r}")
        _check_order(self.advective_flux_order)
        if self.kind == ACOUSTIC and not self.sound_speed > 0:
            raise ValueError(f"sound speed must be positive, got {self.sound_speed}")
        problem = _damping_problem(self.kind, self.nu_damp, self.damping_timescale)
        if problem:
            raise ValueError(problem)

    def with_timescale(self, tau: float) -> "ModelSpec":
        return replace(self, damping_timescale=tau)


def damping_coefficients(nu: float, dx: float, dy: float, tau: float):
    """(alpha1, alpha2) for the x and y damping terms; evaluated as (nu dx) dx / tau so
    the bits match the reference's kernels' coefficients."""
    if not tau > 0:
        raise ValueError(f"damping timescale must be positive, got {tau}")
    return tuple(nu * h * h / tau for h in (dx, dy))
