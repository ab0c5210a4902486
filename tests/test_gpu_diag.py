"""K7 window diagnostics on the device (pw_window_diag) against the reference's host
formulas (reference diagnostics.py:20-36 max_norm / total_energy, mesh.py:140-141
all_finite, diagnostics.py:39-50 sample_probe), including the blow-up cases the
reference's run_windowed meets (parareal.py:316-318: inf and NaN entries)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ctx():
    from paper_1510_02237_b200 import _lib

    return _lib.Context.get()


def _ref(fields, grid):
    # the reference's own expressions (diagnostics.py:20-23, 34-36)
    with np.errstate(over="ignore", invalid="ignore"):
        energy = float(np.sum(fields ** 2) * grid.cell_area)
    return float(np.max(np.abs(fields))), energy, bool(np.isfinite(fields).all())


@pytest.mark.parametrize("n", [8, 64, 256, 1024])
def test_window_diag_matches_host(n):
    from paper_1510_02237_b200.diagnostics import probe_flat_index, window_diag
    from paper_1510_02237_b200.mesh import ACOUSTIC, State, build_grid

    g = build_grid(n, n // 2 if n > 8 else n, 1.0, 0.5)
    rng = np.random.default_rng(n)
    st = State(g, rng.standard_normal((3, g.ny, g.nx)))
    idx = [probe_flat_index(g, 0.49, 0.34 * 0.5, v, ACOUSTIC) for v in ("u", "v", "pi")]
    vec = torch.as_tensor(st.vec).cuda()
    d = window_diag(_ctx(), vec, g, idx)
    mx, en, fin = _ref(st.fields, g)
    assert d.max_norm == mx
    assert d.energy == pytest.approx(en, rel=1e-13)
    assert d.finite is True and fin
    assert d.probes == tuple(float(st.vec[i]) for i in idx)


@pytest.mark.parametrize("bad", ["inf", "nan", "both", "overflow"])
def test_window_diag_blowup(bad):
    from paper_1510_02237_b200.diagnostics import window_diag
    from paper_1510_02237_b200.mesh import State, build_grid

    g = build_grid(64, 64)
    x = np.random.default_rng(7).standard_normal((3, 64, 64))
    if bad in ("inf", "both"):
        x[1, 5, 9] = -np.inf
    if bad in ("nan", "both"):
        x[2, 60, 3] = np.nan
    if bad == "overflow":
        x[0, 0, 0] = 1e200  # finite entry whose square overflows
    st = State(g, x)
    d = window_diag(_ctx(), torch.as_tensor(st.vec).cuda(), g)
    mx, en, fin = _ref(st.fields, g)
    assert d.finite == fin
    if np.isnan(mx):
        assert np.isnan(d.max_norm) and np.isnan(d.energy) and np.isnan(en)
    else:
        assert d.max_norm == mx
        assert d.energy == en == np.inf


def test_run_windowed_records_through_the_device():
    """run_windowed's per-window max_norm / energy / probes (device K7) equal the host
    formulas on the endpoints it returns."""
    from paper_1510_02237_b200.config import parse_config
    from paper_1510_02237_b200.diagnostics import max_norm, sample_probe, total_energy
    from paper_1510_02237_b200.parareal import run_windowed

    cfg = parse_config("model = acoustic\nnx = 32\nny = 32\nt_end = {}\nfine_cfl = 0.2\ncoarse_cfl = 2.0\n"
                       "n_sound = 4\nnu_c = 0.1\nn_p = 4\nn_it = 2\n".format(3 * 4 * 2.0 / (30 * 32)))
    rep = run_windowed(cfg.pit_config("kse"), cfg.initial_state(), cfg.t_end, probe=cfg.probe)
    assert len(rep.window_endpoints) == 3 and rep.blowup_time is None
    for w, ends in enumerate(rep.window_endpoints, start=1):
        st = ends[-1]
        assert rep.max_norms[w] == max_norm(st)
        assert rep.energies[w] == pytest.approx(total_energy(st, st.grid), rel=1e-13)
        assert rep.probe_u.values[w] == sample_probe(st, *cfg.probe, "u")
        assert rep.probe_pi.values[w] == sample_probe(st, *cfg.probe, "pi")
    assert np.array_equal(rep.final_state.vec, rep.window_endpoints[-1][-1].vec)
