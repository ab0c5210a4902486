"""The reference's shipped configs (pkg/configs/*.cfg: acoustic baseline, coarse-CFL-2,
low dissipation, the scalar advection-instability case) through this package's runner
on the device, against the reference runner's own output of the same runs
(tests/golden/make_configs_golden.py -> configs_reference.npz): exit codes, the
per-window diagnostics of series.csv and the per-iteration residuals of residuals.csv.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1510_02237_b200.config import parse_config
from paper_1510_02237_b200.runner import read_residuals, read_series, run_experiment

pytestmark = pytest.mark.gpu

PATH = os.path.join(GOLDEN, "configs_reference.npz")
MODES = ("kse", "parareal", "fine-seq", "coarse-seq")
RTOL = 1e-8  # relative, per series value / residual, over up to 200 chained windows


def _cases():
    if not os.path.exists(PATH):
        return []
    g = np.load(PATH)
    names = sorted({k.split("__")[0] for k in g.files})
    return [(n, m) for n in names for m in MODES if f"{n}__{m}__code" in g.files]


@pytest.mark.parametrize("name,mode", _cases() or [pytest.param("none", "none", marks=pytest.mark.skip)])
def test_shipped_config_matches_reference_runner(tmp_path, name, mode):
    g = np.load(PATH)
    cfg = parse_config(str(g[f"{name}__cfg"]))
    key = f"{name}__{mode}"
    code = run_experiment(cfg, mode, out_dir=str(tmp_path), workers=1, log=lambda *_: None)
    assert code == int(g[f"{key}__code"])
    series = np.array(read_series(tmp_path / "series.csv"))
    want = g[f"{key}__series"]
    assert series.shape == want.shape
    np.testing.assert_array_equal(series[:, 0], want[:, 0])
    np.testing.assert_allclose(series[:, 1], want[:, 1], rtol=1e-13)
    finite = np.isfinite(want[:, 2:])
    np.testing.assert_array_equal(np.isfinite(series[:, 2:]), finite)
    np.testing.assert_allclose(series[:, 2:][finite], want[:, 2:][finite], rtol=RTOL, atol=1e-13)
    res = np.array(read_residuals(tmp_path / "residuals.csv")).reshape(-1, 3)
    want_r = g[f"{key}__residuals"]
    assert res.shape == want_r.shape
    np.testing.assert_array_equal(res[:, :2], want_r[:, :2])
    fin = np.isfinite(want_r[:, 2])
    np.testing.assert_allclose(res[fin, 2], want_r[fin, 2], rtol=RTOL, atol=1e-13)
