"""CPU-only tests: C ABI surface, host-side API logic and workload generators."""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pitwave_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(pw_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    from paper_1510_02237_b200 import _lib

    lib = _lib.load_library()
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/pitwave_b200.h but not exported"
    bound = {s[0] for s in _lib.SIGNATURES}
    assert bound == set(declared), set(declared) ^ bound
    assert lib.pw_version() == 100


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1510_02237_b200", "libpitwave_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_device_entry_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1510_02237_b200 import _lib

    with pytest.raises(RuntimeError, match="CUDA"):
        _lib.Context.get(0)


def test_error_reporting_through_abi():
    import ctypes

    from paper_1510_02237_b200 import _lib

    lib = _lib.load_library()
    rc = lib.pw_ctx_create(0, None, None)
    assert rc == -1
    assert b"NULL" in lib.pw_last_error()


# ------------------------------------------------------------------ reference API (host logic)
def test_propagator_spec_and_make_propagator():
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, PropagatorSpec, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, SCALAR, ConstantVelocity, SolidBodyRotation, build_grid
    from paper_1510_02237_b200.parareal import PitConfig
    from paper_1510_02237_b200.physics import ModelSpec

    g = build_grid(8, 8)
    model = ModelSpec(kind=ACOUSTIC, vel=ConstantVelocity(0, 0), sound_speed=2.0, nu_damp=0.1,
                      damping_timescale=1.0)
    fine = make_propagator(RK3, model, g, cfl=0.2)
    assert fine.model.damping_timescale == pytest.approx(fine.dt)
    coarse = make_propagator(SPLIT_FE_FB, model, g, cfl=1.0, n_sound=5)
    assert coarse.model.damping_timescale == pytest.approx(coarse.dt / 5)
    with pytest.raises(ValueError, match="split"):
        PropagatorSpec(SPLIT_FE_FB, ModelSpec(kind=SCALAR, vel=ConstantVelocity(1, 1)), g, 1.0, 2)
    with pytest.raises(ValueError, match="speed"):
        PropagatorSpec(RK3, ModelSpec(kind=SCALAR, vel=ConstantVelocity(0.0, 0.0)), g, 0.5)
    g40 = build_grid(40, 40)
    m40 = ModelSpec(kind=ACOUSTIC, vel=SolidBodyRotation(), sound_speed=30.0)
    cfg = PitConfig("original", make_propagator(RK3, m40, g40, 0.2),
                    make_propagator(SPLIT_FE_FB, m40, g40, 4.0, 4), n_p=6, n_it=2)
    assert cfg.n_fine_per_coarse == 20


def test_window_count_and_validation():
    from paper_1510_02237_b200.integrators import RK3, SPLIT_FE_FB, make_propagator
    from paper_1510_02237_b200.mesh import ACOUSTIC, SolidBodyRotation, build_grid
    from paper_1510_02237_b200.parareal import ORIGINAL, PitConfig, window_count
    from paper_1510_02237_b200.physics import ModelSpec

    g = build_grid(40, 40)
    model = ModelSpec(kind=ACOUSTIC, vel=SolidBodyRotation(np.pi), sound_speed=30.0)
    cfg = PitConfig(ORIGINAL, make_propagator(RK3, model, g, 0.2),
                    make_propagator(SPLIT_FE_FB, model, g, 4.0, 4), n_p=6, n_it=2)
    assert window_count(cfg, 2.0) == 100
    with pytest.raises(ValueError, match="M_c=7.*N_p=6"):
        window_count(cfg, 7 * cfg.coarse.dt)
    with pytest.raises(ValueError, match="integer"):
        PitConfig(ORIGINAL, make_propagator(RK3, model, g, 0.3),
                  make_propagator(SPLIT_FE_FB, model, g, 4.0, 4), n_p=4, n_it=1)


def test_config_parser_matches_reference_grammar():
    from paper_1510_02237_b200.config import ConfigError, parse_config

    base = ("model = acoustic\nnx = 40\nny = 40\nt_end = 2.0\nfine_cfl = 0.2\n"
            "coarse_cfl = 4.0\nn_p = 6\nn_it = 2\n")
    cfg = parse_config(base + "# comment\n\nn_sound = 4  # trailing\n")
    assert cfg.n_windows == 100 and cfg.cs == 30.0 and cfg.coarse_scheme == "split_fe_fb"
    with pytest.raises(ConfigError, match="unknown key 'bogus'"):
        parse_config(base + "bogus = 1\n")
    with pytest.raises(ConfigError, match="duplicate key 'nx'"):
        parse_config(base + "nx = 8\n")
    with pytest.raises(ConfigError, match="missing required keys"):
        parse_config("")
    with pytest.raises(ConfigError, match="flux order"):
        parse_config(base + "fine_order = 7\n")
    with pytest.raises(ConfigError, match="vel_u"):
        parse_config(base + "velocity = constant\n")
    with pytest.raises(ConfigError, match="grid"):
        parse_config(base.replace("nx = 40", "nx = 4"))
    with pytest.raises(ConfigError, match="integer"):
        parse_config(base.replace("fine_cfl = 0.2", "fine_cfl = 0.3"))


def test_reference_shipped_configs_parse():
    """The reference's own .cfg files load unchanged (copied inline: keys only)."""
    from paper_1510_02237_b200.config import parse_config

    text = ("model = acoustic\nnx = 40\nny = 40\nt_end = 2.0\ny0 = 0.65\nfine_cfl = 0.2\n"
            "fine_order = 5\nnu_f = 0.005\ncoarse_scheme = split_fe_fb\ncoarse_cfl = 4.0\n"
            "coarse_order = 1\nn_sound = 4\nnu_c = 0.1\nn_p = 6\nn_it = 2\nprobe_x = 0.49\nprobe_y = 0.34\n")
    cfg = parse_config(text)
    assert cfg.n_windows == 100
    st = cfg.initial_state()
    assert st.fields.shape == (3, 40, 40) and st.u.max() == pytest.approx(1.0, abs=0.05)


def test_mesh_state_layout():
    from paper_1510_02237_b200.mesh import ACOUSTIC, State, build_grid, face_normal_velocities
    from paper_1510_02237_b200.mesh import SolidBodyRotation

    g = build_grid(8, 16)
    st = State(g, np.arange(3 * 16 * 8, dtype=float).reshape(3, 16, 8))
    v = st.flatten()
    assert v[1] == 1.0 and v[8] == 8.0 and v[16 * 8] == 128.0
    assert np.array_equal(State.unflatten(g, v, ACOUSTIC).fields, st.fields)
    ux, vy = face_normal_velocities(SolidBodyRotation(np.pi), g)
    assert ux.shape == (16, 8) and vy[0, 0] == pytest.approx(-np.pi * (0.5 / 8 - 0.5))
    with pytest.raises(ValueError, match="too small"):
        build_grid(4, 16)


# ------------------------------------------------------------------ workloads
def test_workload_completion():
    from paper_1510_02237_b200 import harness

    for name in ("c1", "c3", "c4", "c5"):
        wl = harness.WORKLOADS[name]
        assert wl.fine_steps_per_slice == 16
        assert wl.coarse_steps_per_slice == 2
    assert harness.WORKLOADS["c3"].d == 786432


def test_initial_state_generators_seeded():
    from paper_1510_02237_b200 import harness

    a = harness.fine_batch_states(n=32, batch=2)
    b = harness.fine_batch_states(n=32, batch=2)
    assert np.array_equal(a, b)
    q3 = harness.initial_state("c3", n=64)
    u = q3[: 64 * 64]
    assert np.max(np.abs(u)) == pytest.approx(1e-3)
    assert q3[2 * 64 * 64:].max() <= 1.0


def test_damping_coefficient_known_values():
    """reference tests/test_physics.py:19-35"""
    from paper_1510_02237_b200.physics import damping_coefficients

    assert damping_coefficients(0.0, 0.025, 0.1, 0.3) == (0.0, 0.0)
    a1, a2 = damping_coefficients(0.1, 0.025, 0.025, (1.0 / 300.0) / 4.0)
    assert a1 == pytest.approx(0.075, rel=1e-12) and a2 == pytest.approx(0.075, rel=1e-12)
    a1, _ = damping_coefficients(0.005, 0.025, 0.025, 0.2 * 0.025 / 30.0)
    assert a1 == pytest.approx(0.01875, rel=1e-10)
    with pytest.raises(ValueError, match="timescale"):
        damping_coefficients(0.1, 0.025, 0.025, 0.0)


def test_bench_reference_arm_json_contract():
    """bench.py --impl reference (the CPU arm the driver runs next to ours) prints one JSON
    line with the device arm's metric, unit, config and the cpu_baseline / e2e keys."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "fine RK-3 fp64 cell-updates/s"
    assert d["unit"] == "cell-updates/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"].startswith("c2: 64 states x 256^2")
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
