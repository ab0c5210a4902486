"""Runner / perf-model host logic -- no device needed.

Mirrors the reference's tests/test_runner.py (field round trip, filename format,
estimate mode) and checks the perf model against the reference's formulas."""
import math

import numpy as np
import pytest

from paper_1510_02237_b200.config import parse_config
from paper_1510_02237_b200.perfmodel import (SpeedupInputs, speedup_bounds, speedup_cfl_estimate,
                                             speedup_estimate)
from paper_1510_02237_b200.runner import (field_filename, read_field, read_residuals, read_series,
                                          read_timing, run_experiment, write_field, write_residuals,
                                          write_series, write_timing)

ESTIMATE_BASELINE = """
model = acoustic
nx = 40
ny = 40
t_end = 2.0
y0 = 0.65
fine_cfl = 0.2
coarse_cfl = 4.0
n_sound = 4
nu_c = 0.1
n_p = 6
n_it = 2
"""


def test_field_round_trip_bit_exact(tmp_path, rng):
    field = rng.standard_normal((9, 13)) * np.exp(rng.uniform(-30, 30, (9, 13)))
    path = tmp_path / "u_1.000000.csv"
    write_field(path, field)
    np.testing.assert_array_equal(read_field(path), field)


def test_field_header_mismatch_raises(tmp_path):
    path = tmp_path / "u_0.000000.csv"
    path.write_text("nx,3\nny,2\n1,2\n3,4\n")
    with pytest.raises(ValueError):
        read_field(path)


def test_filename_format():
    assert field_filename("pi", 2.0) == "pi_2.000000.csv"
    assert field_filename("q", 1.08) == "q_1.080000.csv"


def test_series_residuals_timing_round_trip(tmp_path, rng):
    from paper_1510_02237_b200.parareal import Timings

    rows = [(k, *rng.standard_normal(5)) for k in range(4)]
    write_series(tmp_path / "s.csv", rows)
    assert read_series(tmp_path / "s.csv") == [tuple(r) for r in rows]
    res = [list(rng.uniform(0, 1, 3)), list(rng.uniform(0, 1, 2))]
    write_residuals(tmp_path / "r.csv", res)
    back = read_residuals(tmp_path / "r.csv")
    assert [(w, k) for w, k, _ in back] == [(1, 1), (1, 2), (1, 3), (2, 1), (2, 2)]
    assert [r for *_, r in back] == res[0] + res[1]
    tm = Timings(coarse=0.5, fine=1.25, qr=0.25)
    write_timing(tmp_path / "t.csv", tm)
    t = read_timing(tmp_path / "t.csv")
    assert t["fine"] == (1.25, 0.625) and t["qr"] == (0.25, 0.125)


def test_estimate_mode(tmp_path):
    """reference tests/test_runner.py:127-134 (no numerics: runs without a device)"""
    cfg = parse_config(ESTIMATE_BASELINE)
    messages = []
    assert run_experiment(cfg, "estimate", out_dir=str(tmp_path), log=messages.append) == 0
    text = (tmp_path / "estimate.csv").read_text().splitlines()
    values = dict(zip(text[0].split(","), text[1].split(",")))
    assert float(values["estimate_cfl"]) == pytest.approx(1.97, abs=0.01)
    assert any("estimated speedup" in m for m in messages)


def test_perfmodel_formulas():
    x = SpeedupInputs(n_p=8, n_it=3, n_c=8, n_f=16, tau_c=0.25, tau_f=1.0, tau_qr=2.0)
    denom = 8 * 0.25 + 3 * (8 * 0.25 + (128 / 8) * 1.0) + 3 * 2.0
    assert speedup_estimate(x) == 128 * 1.0 / denom
    assert speedup_bounds(x) == (8 / 3, 16 * 1.0 / (4 * 0.25), 128 * 1.0 / (3 * 2.0))
    free = SpeedupInputs(n_p=4, n_it=0, n_c=4, n_f=2, tau_c=1.0, tau_f=1.0)
    b = speedup_bounds(free)
    assert math.isinf(b[0]) and math.isinf(b[2])
    assert speedup_cfl_estimate(0.5, 4.0, 1.0, 64, 5) == 1.0 / (6 * (0.5 / 4.0) * 1.0 + 5 / 64)
    assert speedup_cfl_estimate(0.5, 4.0, 1.0, 64, 5, printed_form=True) == 1.0 / (6 * 0.125 + 64 / 5)


@pytest.mark.parametrize("kw", [dict(n_p=0), dict(n_c=0), dict(n_f=0), dict(n_it=-1), dict(tau_c=0.0),
                                dict(tau_f=-1.0), dict(tau_qr=-0.5)])
def test_perfmodel_rejects_bad_inputs(kw):
    args = dict(n_p=2, n_it=1, n_c=2, n_f=2, tau_c=1.0, tau_f=1.0, tau_qr=0.0)
    args.update(kw)
    with pytest.raises(ValueError):
        SpeedupInputs(**args)
    with pytest.raises(ValueError):
        speedup_cfl_estimate(0.0, 1.0, 1.0, 2, 1)


def test_unknown_mode_rejected(tmp_path):
    with pytest.raises(ValueError):
        run_experiment(parse_config(ESTIMATE_BASELINE), "bogus", out_dir=str(tmp_path))
