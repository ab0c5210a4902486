"""Model description of the linear acoustic-advection system (reference physics.py).

Only the model *parameters* live here; the right-hand side itself is
evaluated inside the sm_100a kernels (csrc/exact.cu, csrc/fine_fused.cu).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from .mesh import ACOUSTIC, SCALAR

VALID_ORDERS = (1, 2, 3, 4, 5, 6)


def _check_order(order: int) -> int:
    if order not in VALID_ORDERS:
        raise ValueError(f"flux order must be one of {VALID_ORDERS}, got {order}")
    return int(order)


@dataclass(frozen=True)
class ModelSpec:
    """Continuous model + discretisation knobs (reference physics.py:21-51)."""

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
        if self.kind == ACOUSTIC and self.sound_speed <= 0:
            raise ValueError(f"sound speed must be positive, got {self.sound_speed}")
        if self.nu_damp < 0:
            raise ValueError(f"damping strength must be nonnegative, got {self.nu_damp}")
        if self.nu_damp > 0 and self.kind == ACOUSTIC:
            if self.damping_timescale is None or self.damping_timescale <= 0:
                raise ValueError("damping_timescale must be positive when nu_damp > 0")

    def with_timescale(self, tau: float) -> "ModelSpec":
        return replace(self, damping_timescale=tau)


def damping_coefficients(nu: float, dx: float, dy: float, tau: float):
    """(alpha1, alpha2) = nu (dx^2, dy^2) / tau (reference physics.py:54-58)."""
    if tau <= 0:
        raise ValueError(f"damping timescale must be positive, got {tau}")
    return nu * dx * dx / tau, nu * dy * dy / tau
