"""Runner fixtures from the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_runner_golden.py

Runs the reference's ``run_experiment`` (src/runner.py:117-146) on the small
acoustic config of its own runner tests (tests/test_runner.py:9-21, two windows) in
modes kse, parareal and fine-seq, and stores the parsed series.csv / residuals.csv
rows and the end-time field files in runner_small.npz.  The device runner's CSVs
are compared against these values (timing.csv is wall-clock and is not compared).
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from pitwave.config import parse_config  # noqa: E402
from pitwave.kernels import BACKEND_NAME  # noqa: E402
from pitwave.runner import field_filename, read_field, read_series, run_experiment  # noqa: E402

assert BACKEND_NAME == "numba"

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


def main():
    text = SMALL_ACOUSTIC.format(t_end=2 * 4 / 240)
    cfg = parse_config(text)
    out = {"config": np.array(text)}
    for mode in ("kse", "parareal", "fine-seq"):
        with tempfile.TemporaryDirectory() as d:
            assert run_experiment(cfg, mode, out_dir=d, workers=1, log=lambda *_: None) == 0
            key = mode.replace("-", "_")
            out[f"{key}_series"] = np.array(read_series(os.path.join(d, "series.csv")))
            with open(os.path.join(d, "residuals.csv")) as fh:
                rows = [ln.strip().split(",") for ln in fh.readlines()[1:] if ln.strip()]
            out[f"{key}_residuals"] = np.array([[float(x) for x in r] for r in rows]).reshape(-1, 3)
            out[f"{key}_fields"] = np.stack([read_field(os.path.join(d, field_filename(v, cfg.t_end)))
                                             for v in ("u", "v", "pi")])
    np.savez_compressed(os.path.join(HERE, "runner_small.npz"), **out)
    print("wrote runner_small.npz", sorted(out))


if __name__ == "__main__":
    main()
