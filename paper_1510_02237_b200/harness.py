"""BASELINE.json workloads: the config completion of SURVEY.md section 8(d).

The reference cannot express BASELINE.json's configs directly (SURVEY.md
section 0, finding 1): its ``PitConfig`` makes a slice exactly one coarse
step, and the 10x/20x coarse ratios do not divide the 16-fine-step slice.
Both this package and the oracle therefore run the completed parameters
below -- slice = T/P, fine RK3 (CFL 0.5, order 6, nu 0.005), coarse split
FE-FB (CFL 4.0 = 8 fine steps, order 1, n_sound 16, nu 0.1) applied twice
per slice, the measured-stable choice (spectral growth 0.9969 per step).

The seeded initial-state generators are specified in SURVEY.md section 8(d);
all inputs are synthetic (no dataset is involved).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Physics shared by every config (SURVEY.md 8(d) "Common to all configs").
CS = 1.0
VEL_U = 0.1
VEL_V = 0.0
FINE = dict(scheme="rk3", cfl=0.5, order=6, nu=0.005, n_sound=1)
COARSE = dict(scheme="split_fe_fb", cfl=4.0, order=1, nu=0.1, n_sound=16)
RANK_TOL = 1e-10


@dataclass(frozen=True)
class Workload:
    name: str
    n: int                 # grid side (nx = ny = n), periodic unit square
    t_end: float = 1.0
    n_p: int = 1           # slices
    n_it: int = 1          # Parareal iterations
    batch: int = 0         # c2 only: independent fine states
    fine_steps: int = 0    # c2 only: RK3 steps per state
    gpus: tuple = (1,)
    notes: str = ""

    @property
    def d(self) -> int:
        return 3 * self.n * self.n

    @property
    def dx(self) -> float:
        return 1.0 / self.n

    @property
    def h_fine(self) -> float:
        return FINE["cfl"] * self.dx / CS

    @property
    def h_coarse(self) -> float:
        return COARSE["cfl"] * self.dx / CS

    @property
    def slice_span(self) -> float:
        return self.t_end / self.n_p

    @property
    def fine_steps_per_slice(self) -> int:
        return _int_ratio(self.slice_span, self.h_fine)

    @property
    def coarse_steps_per_slice(self) -> int:
        return _int_ratio(self.slice_span, self.h_coarse)


def _int_ratio(span, h):
    r = span / h
    n = round(r)
    if n < 1 or abs(r - n) > 1e-9 * max(1.0, r):
        raise ValueError(f"span {span} is not an integer multiple of step {h}")
    return n


WORKLOADS = {
    "c1": Workload("c1", 64, t_end=1.0, n_p=8, n_it=3,
                   notes="CPU-runnable oracle case; Gaussian p, u=v=0"),
    "c2": Workload("c2", 256, batch=64, fine_steps=200,
                   notes="fine-propagator throughput: 64 random-mode states x 200 RK3 steps"),
    "c3": Workload("c3", 512, t_end=1.0, n_p=64, n_it=5,
                   notes="single-GPU KSE-Parareal"),
    "c4": Workload("c4", 1024, t_end=2.0, n_p=256, n_it=4, gpus=(1, 2, 4, 8),
                   notes="slice-sharded KSE-Parareal"),
    "c5": Workload("c5", 2048, t_end=1.0, n_p=256, n_it=4, gpus=(8,),
                   notes="large-basis stress (T unspecified in BASELINE.json -> 1.0)"),
}


def centers(n):
    x = (np.arange(n) + 0.5) / n
    return np.meshgrid(x, x)  # (X, Y), each (ny, nx)


def gaussian(n, width2):
    xx, yy = centers(n)
    return np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / width2)


def mode_sum(rng, n, kmax, n_modes=16):
    """sum_m |k_m|^-2 cos(2 pi (kx x + ky y) + phi_m), k uniform in the |k|<=kmax disc."""
    ks = []
    while len(ks) < n_modes:
        kx, ky = (int(v) for v in rng.integers(-kmax, kmax + 1, size=2))
        k2 = kx * kx + ky * ky
        if 0 < k2 <= kmax * kmax:
            ks.append((kx, ky))
    phases = rng.uniform(0.0, 2.0 * math.pi, size=n_modes)
    xx, yy = centers(n)
    out = np.zeros((n, n))
    for (kx, ky), ph in zip(ks, phases):
        out += (1.0 / (kx * kx + ky * ky)) * np.cos(2.0 * math.pi * (kx * xx + ky * yy) + ph)
    return out


def initial_state(name: str, n: int | None = None) -> np.ndarray:
    """Flat (3*n*n,) initial state of a Parareal config (c1, c3, c4, c5)."""
    wl = WORKLOADS[name]
    n = wl.n if n is None else n
    if name == "c1":
        p = gaussian(n, 0.01)
        return np.stack([np.zeros((n, n)), np.zeros((n, n)), p]).ravel()
    if name in ("c3", "c4"):
        rng = np.random.default_rng(3001 if name == "c3" else 4001)
        p = gaussian(n, 0.05 ** 2)
        u = mode_sum(rng, n, 8)
        u *= 1e-3 / np.max(np.abs(u))
        v = mode_sum(rng, n, 8)
        v *= 1e-3 / np.max(np.abs(v))
        return np.stack([u, v, p]).ravel()
    if name == "c5":
        rng = np.random.default_rng(5001)
        return np.stack([mode_sum(rng, n, 32) for _ in range(3)]).ravel()
    raise ValueError(f"{name} has no single initial state")


def fine_batch_states(n: int = 256, batch: int = 64, seed: int = 2001) -> np.ndarray:
    """c2 input: (batch, 3*n*n) random-mode states, state-major then u, v, p."""
    rng = np.random.default_rng(seed)
    out = np.empty((batch, 3 * n * n))
    for b in range(batch):
        out[b] = np.stack([mode_sum(rng, n, 8) for _ in range(3)]).ravel()
    return out
