"""Parallel-in-time configuration and the windowed run on the device.

Drop-in for the reference's run-level API (``PitConfig``, ``window_count``,
``parareal_window``, ``kse_parareal_window``, ``RunReport``, ``run_windowed``,
``run_sequential``; reference ``pkg/src/pitwave/parareal.py:141-345``), re-exported
from :mod:`.parareal` under the reference's names.

What differs from a host driver is where the window chain lives:

* the seed of window w+1 is window w's last endpoint *on the device*: a window is
  one ``pw_sweep`` call with device output, and nothing goes host-ward to start
  the next one;
* every window is recorded by the K7 device pass (``diagnostics.window_diag``:
  max norm, energy, finiteness and the probe samples in one read of the
  endpoint), so the blow-up check and the CSV series never wait on a host copy;
* the endpoint states the report keeps (``window_endpoints``, the reference's
  record) come back in one D2H copy per window, as views of one host array.

The structural checks are the reference's (step ratio, window divisibility,
recording cadence), expressed once as an integer-quotient test with the
reference's 1e-9 relative slack.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .diagnostics import ProbeSeries, max_norm, probe_flat_index, sample_probe, total_energy, window_diag
from .integrators import PropagatorSpec, SlicePropagator
from .mesh import ACOUSTIC, State
from .subspace import DEFAULT_RANK_TOL

ORIGINAL = "original"
KSE = "kse"
DEFAULT_PROBE = (0.49, 0.34)


def _whole_quotient(num: float, den: float, complaint) -> int:
    """round(num / den) when that quotient is a positive integer to 1e-9 relative
    (the tolerance of reference ``parareal.py:181-184, 201-206, 331-333``), else
    ``ValueError(complaint(quotient))``."""
    q = num / den
    n = round(q)
    if n >= 1 and abs(q - n) <= 1e-9 * max(1.0, q):
        return int(n)
    raise ValueError(complaint(q))


@dataclass
class Timings:
    """Accumulated time per phase in seconds (reference ``parareal.py:31-47``).

    Filled from CUDA events of the device sweep; as in the reference the K
    projections of the correction sweep are billed to ``coarse``.
    """

    coarse: float = 0.0
    fine: float = 0.0
    qr: float = 0.0

    @property
    def total(self) -> float:
        return self.coarse + self.fine + self.qr

    def fractions(self) -> dict:
        tot = self.total
        return {k: (getattr(self, k) / tot if tot else 0.0) for k in ("coarse", "fine", "qr")}


@dataclass(frozen=True)
class PitConfig:
    """One window = ``n_p`` coarse intervals, one coarse step each (reference ``parareal.py:141-194``)."""

    mode: str
    fine: PropagatorSpec
    coarse: PropagatorSpec
    n_p: int
    n_it: int
    tol: float | None = None
    rank_tol: float = DEFAULT_RANK_TOL
    workers: int = 1

    def __post_init__(self):
        checks = (
            (self.mode in (ORIGINAL, KSE), f"mode must be {ORIGINAL!r} or {KSE!r}, got {self.mode!r}"),
            (min(self.n_p, self.n_it) >= 1, f"n_p and n_it must be at least 1, got {self.n_p}, {self.n_it}"),
            (self.workers >= 1, f"workers must be at least 1, got {self.workers}"),
            (self.fine.grid == self.coarse.grid, "fine and coarse propagators must share the grid"),
            (self.fine.model.kind == self.coarse.model.kind,
             "fine and coarse propagators must share the model kind"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        _ = self.n_fine_per_coarse  # the step ratio must be a whole number

    @property
    def n_fine_per_coarse(self) -> int:
        c, f = self.coarse.dt, self.fine.dt
        return _whole_quotient(c, f, lambda q: "coarse/fine step ratio must be a positive integer: "
                                               f"dt_coarse={c}, dt_fine={f}, ratio={q}")

    def vector_propagators(self):
        """(fine, coarse) device propagators over one coarse interval."""
        span = self.coarse.dt
        return SlicePropagator(self.fine, span), SlicePropagator(self.coarse, span)


def window_count(cfg: PitConfig, t_end: float, t_start: float = 0.0) -> int:
    """Windows M_p covering [t_start, t_end] (reference ``parareal.py:197-210``)."""
    span, dt = t_end - t_start, cfg.coarse.dt
    m_c = _whole_quotient(span, dt, lambda q: f"time span {span} is not an integer number of coarse "
                                              f"intervals (dt={dt}, ratio={q})")
    if m_c % cfg.n_p:
        raise ValueError(f"M_c={m_c} coarse intervals not divisible by N_p={cfg.n_p}")
    return m_c // cfg.n_p


# ---------------------------------------------------------------- one window
def _run_window(cfg: PitConfig, mode: str, seed, props, timings):
    """One parallel step of ``mode`` from ``seed`` (host vector or device tensor): device
    endpoints (n_p, d), residuals and (KSE) the subspace."""
    from .parareal import _sweep

    fine, coarse = props if props is not None else cfg.vector_propagators()
    rank_tol = cfg.rank_tol if mode == KSE else DEFAULT_RANK_TOL
    return _sweep(mode, seed, fine, coarse, cfg.n_p, cfg.n_it, cfg.tol, rank_tol, timings, True)


def _as_states(ends_dev, grid, kind):
    host = ends_dev.cpu().numpy()  # one D2H copy; the states are row views of it
    return [State._from_vec(grid, row) for row in host]


def parareal_window(cfg: PitConfig, q_start: State, t_start: float = 0.0, timings=None, pool=None,
                    props=None):
    """Original Parareal over one window -> (endpoint States, residuals)."""
    ends, res, _ = _run_window(cfg, ORIGINAL, q_start.flatten(), props, timings)
    return _as_states(ends, q_start.grid, q_start.kind), res


def kse_parareal_window(cfg: PitConfig, q_start: State, t_start: float = 0.0, timings=None, pool=None,
                        props=None):
    """KSE-Parareal over one window -> (endpoint States, residuals, Subspace)."""
    ends, res, sub = _run_window(cfg, KSE, q_start.flatten(), props, timings)
    return _as_states(ends, q_start.grid, q_start.kind), res, sub


# ---------------------------------------------------------------- the run record
@dataclass
class RunReport:
    """Per-window record of a run (reference ``parareal.py:237-273``)."""

    window_endpoints: list = field(default_factory=list)
    residuals: list = field(default_factory=list)
    window_indices: list = field(default_factory=list)
    times: list = field(default_factory=list)
    max_norms: list = field(default_factory=list)
    energies: list = field(default_factory=list)
    probe_u: ProbeSeries | None = None
    probe_pi: ProbeSeries | None = None
    timings: Timings = field(default_factory=Timings)
    blowup_time: float | None = None
    final_state: State | None = None

    def _series(self):
        return [s for s in (self.probe_u, self.probe_pi) if s is not None]

    def _push(self, window_index, t, mx, energy, samples, state):
        self.window_indices.append(window_index)
        self.times.append(t)
        self.max_norms.append(mx)
        self.energies.append(energy)
        for series, value in zip(self._series(), samples):
            series.append_value(t, value)
        if state is not None:
            self.final_state = state

    def record(self, window_index: int, t: float, state: State) -> None:
        """Record a host state (reference ``RunReport.record``)."""
        samples = [sample_probe(state, s.x, s.y, s.variable) for s in self._series()]
        self._push(window_index, t, max_norm(state), total_energy(state, state.grid), samples, state)

    def record_device(self, window_index: int, t: float, ctx, vec, grid, kind, state=None) -> bool:
        """Record a device vector through the K7 pass; returns its finiteness."""
        idx = [probe_flat_index(grid, s.x, s.y, s.variable, kind) for s in self._series()]
        d = window_diag(ctx, vec, grid, idx)
        self._push(window_index, t, d.max_norm, d.energy, d.probes, state)
        return d.finite

    def series_rows(self):
        """(window_index, t, max_norm, energy, probe_u, probe_pi) per record."""
        pu = self.probe_u.values if self.probe_u is not None else [0.0] * len(self.times)
        pp = self.probe_pi.values if self.probe_pi is not None else [0.0] * len(self.times)
        return list(zip(self.window_indices, self.times, self.max_norms, self.energies, pu, pp))


def _report_for(kind: str, probe) -> RunReport:
    px, py = probe
    acoustic = kind == ACOUSTIC
    return RunReport(probe_u=ProbeSeries(px, py, "u" if acoustic else "q"),
                     probe_pi=ProbeSeries(px, py, "pi") if acoustic else None)


def _upload(ctx, q: State):
    return torch.as_tensor(q.vec).to(torch.device("cuda", ctx.device), torch.float64).reshape(1, -1)


# ---------------------------------------------------------------- windowed and sequential runs
def run_windowed(cfg: PitConfig, q0: State, t_end: float, t_start: float = 0.0,
                 probe=DEFAULT_PROBE) -> RunReport:
    """Chain parallel steps over [t_start, t_end] (reference ``parareal.py:285-322``).

    Each window starts from the previous window's last corrected endpoint,
    which stays on the device; KSE rebuilds its subspace every window; the run
    stops after the first window whose endpoint is not finite.
    """
    n_windows = window_count(cfg, t_end, t_start)
    span = cfg.n_p * cfg.coarse.dt
    props = cfg.vector_propagators()
    ctx, grid, kind = props[0].ctx, q0.grid, q0.kind
    report = _report_for(kind, probe)
    seed = _upload(ctx, q0)
    report.record_device(0, t_start, ctx, seed, grid, kind, state=q0)
    for w in range(1, n_windows + 1):
        # [:2] drops the window's Subspace at once: kept in a name until the next call returns,
        # it would pin its d x m basis buffers while the next window allocates its own
        ends, residuals = _run_window(cfg, cfg.mode, seed.reshape(-1), props, report.timings)[:2]
        t = t_start + w * span
        states = _as_states(ends, grid, kind)
        report.window_endpoints.append(states)
        report.residuals.append(residuals)
        seed = ends[-1:].clone()
        if not report.record_device(w, t, ctx, seed, grid, kind, state=states[-1]):
            report.blowup_time = t
            break
    return report


def run_sequential(spec: PropagatorSpec, q0: State, t_end: float, record_dt: float,
                   t_start: float = 0.0, probe=DEFAULT_PROBE, phase: str = "fine") -> RunReport:
    """One propagator stepped serially on the window cadence (reference ``parareal.py:325-345``).

    The state stays on the device; each record is a K7 pass, and only the final
    state (or the first non-finite one) comes back to the host.
    """
    n_rec = _whole_quotient(t_end - t_start, record_dt,
                            lambda q: f"(t_end - t_start)={t_end - t_start} is not a multiple of "
                                      f"record_dt={record_dt}")
    prop = SlicePropagator(spec, record_dt)
    ctx, grid, kind = prop.ctx, q0.grid, q0.kind
    report = _report_for(kind, probe)
    cur = _upload(ctx, q0)
    report.record_device(0, t_start, ctx, cur, grid, kind, state=q0)
    spent = 0.0
    for w in range(1, n_rec + 1):
        tic = time.perf_counter()
        cur = prop.apply(cur)
        torch.cuda.synchronize(prop.device)
        spent += time.perf_counter() - tic
        t = t_start + w * record_dt
        finite = report.record_device(w, t, ctx, cur, grid, kind)
        if not finite or w == n_rec:
            report.final_state = State._from_vec(grid, cur.reshape(-1).cpu().numpy())
        if not finite:
            report.blowup_time = t
            break
    setattr(report.timings, phase, getattr(report.timings, phase) + spent)
    return report
