"""Device runs through the runner against the reference's own
runner output (tests/golden/runner_small.npz from make_runner_golden.py) plus the
reference's runner tests (tests/test_runner.py:59-146) on the device path."""
import numpy as np
import pytest

from conftest import golden
from paper_1510_02237_b200.config import parse_config
from paper_1510_02237_b200.runner import (EXIT_BLOWUP, compare_runs, field_filename, read_field,
                                          read_residuals, read_series, read_timing, run_experiment)

pytestmark = pytest.mark.gpu

SMALL_ACOUSTIC = """
model = acoustic
nx = 16
ny = 16
t_end = {t_end}
y0 = 0.65
fine_cfl = 0.2
coarse_cfl = 2.0
n_sound = 4
nu_c = 0.1
n_p = 4
n_it = 2
"""


def small_cfg(windows=2):
    return parse_config(SMALL_ACOUSTIC.format(t_end=windows * 4 / 240))


def quiet(*_):
    pass


@pytest.mark.parametrize("mode", ["kse", "parareal", "fine-seq"])
def test_csv_outputs_match_reference_runner(tmp_path, mode):
    g = golden("runner_small.npz")
    cfg = parse_config(str(g["config"]))
    assert run_experiment(cfg, mode, out_dir=str(tmp_path), workers=1, log=quiet) == 0
    key = mode.replace("-", "_")
    series = np.array(read_series(tmp_path / "series.csv"))
    want = g[f"{key}_series"]
    assert series.shape == want.shape
    np.testing.assert_array_equal(series[:, 0], want[:, 0])         # window indices
    np.testing.assert_allclose(series[:, 1], want[:, 1], rtol=0, atol=1e-15)  # times
    np.testing.assert_allclose(series[:, 2:], want[:, 2:], rtol=1e-10, atol=1e-14)
    res = np.array(read_residuals(tmp_path / "residuals.csv")).reshape(-1, 3)
    want_r = g[f"{key}_residuals"]
    assert res.shape == want_r.shape
    np.testing.assert_array_equal(res[:, :2], want_r[:, :2])
    np.testing.assert_allclose(res[:, 2], want_r[:, 2], rtol=1e-10, atol=1e-14)
    got = np.stack([read_field(tmp_path / field_filename(v, cfg.t_end)) for v in ("u", "v", "pi")])
    want_f = g[f"{key}_fields"]
    assert np.linalg.norm(got - want_f) <= 1e-10 * np.linalg.norm(want_f)


def test_fine_seq_writes_outputs(tmp_path):
    cfg = small_cfg()
    assert run_experiment(cfg, "fine-seq", out_dir=str(tmp_path), log=quiet) == 0
    series = read_series(tmp_path / "series.csv")
    assert len(series) == 3 and series[0][0] == 0
    assert series[-1][1] == pytest.approx(cfg.t_end)
    for var in ("u", "v", "pi"):
        assert (tmp_path / field_filename(var, cfg.t_end)).exists()
    timing = read_timing(tmp_path / "timing.csv")
    assert timing["fine"][0] > 0 and timing["coarse"][0] == 0.0
    assert (tmp_path / "residuals.csv").read_text().strip() == "window_index,iteration,r_k"


def test_kse_writes_residuals_and_energy_decays(tmp_path):
    cfg = small_cfg()
    assert run_experiment(cfg, "kse", out_dir=str(tmp_path / "k"), log=quiet) == 0
    rows = read_residuals(tmp_path / "k" / "residuals.csv")
    assert len(rows) == 2 * cfg.n_it and all(r >= 0 for *_, r in rows)
    cfg4 = small_cfg(windows=4)
    run_experiment(cfg4, "fine-seq", out_dir=str(tmp_path / "f"), log=quiet)
    energies = [r[3] for r in read_series(tmp_path / "f" / "series.csv")]
    assert energies[-1] < energies[0]


def test_compare_runs_and_converged_kse_exactness(tmp_path):
    text = SMALL_ACOUSTIC.format(t_end=4 / 240) + "tolerance = 0\n"
    cfg = parse_config(text.replace("n_it = 2", "n_it = 4"))
    a, b = tmp_path / "a", tmp_path / "b"
    run_experiment(cfg, "fine-seq", out_dir=str(a), log=quiet)
    run_experiment(cfg, "kse", out_dir=str(b), log=quiet)
    same = compare_runs(str(a), str(a))
    assert len(same) == 1 and same[0][1] == 0.0
    assert compare_runs(str(b), str(a))[0][1] <= 1e-10


def test_blowup_exits_3(tmp_path):
    cfg = parse_config("""
model = acoustic
nx = 16
ny = 16
t_end = 4.0
fine_cfl = 3.0
coarse_cfl = 6.0
n_p = 4
n_it = 1
""")
    messages = []
    assert run_experiment(cfg, "fine-seq", out_dir=str(tmp_path), log=messages.append) == EXIT_BLOWUP
    assert any("blow-up" in m for m in messages)
    assert len(read_series(tmp_path / "series.csv")) >= 1


def test_workers_env_override(tmp_path, monkeypatch):
    monkeypatch.setenv("PIT_WORKERS", "2")
    assert run_experiment(small_cfg(), "parareal", out_dir=str(tmp_path), log=quiet) == 0
