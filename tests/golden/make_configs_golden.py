"""The reference package's shipped configs (pkg/configs/*.cfg) through the REFERENCE runner
(this container only):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_configs_golden.py

For every config and mode (kse, parareal, fine-seq, coarse-seq) it stores the exit code
and the parsed series.csv / residuals.csv rows in configs_reference.npz, together with
the config text (the GPU box has no /root/reference).  tests/test_gpu_configs.py runs
the same configs through this package's runner on the device.
"""
from __future__ import annotations

import glob
import os
import sys
import tempfile
import time

import numpy as np

from pitwave.config import parse_config
from pitwave.kernels import BACKEND_NAME
from pitwave.runner import read_series, run_experiment

assert BACKEND_NAME == "numba"
HERE = os.path.dirname(os.path.abspath(__file__))
CFG_DIR = "/root/reference/pkg/configs"
MODES = ("kse", "parareal", "fine-seq", "coarse-seq")


def main(names=None):
    out = {}
    for path in sorted(glob.glob(os.path.join(CFG_DIR, "*.cfg"))):
        name = os.path.splitext(os.path.basename(path))[0]
        if names and name not in names:
            continue
        with open(path) as fh:
            text = fh.read()
        cfg = parse_config(text)
        out[f"{name}__cfg"] = np.array(text)
        for mode in MODES:
            t0 = time.time()
            with tempfile.TemporaryDirectory() as d:
                code = run_experiment(cfg, mode, out_dir=d, workers=4, log=lambda *_: None)
                key = f"{name}__{mode}"
                out[f"{key}__code"] = np.array(code)
                out[f"{key}__series"] = np.array(read_series(os.path.join(d, "series.csv")))
                with open(os.path.join(d, "residuals.csv")) as fh:
                    rows = [ln.strip().split(",") for ln in fh.readlines()[1:] if ln.strip()]
                out[f"{key}__residuals"] = np.array([[float(x) for x in r] for r in rows]).reshape(-1, 3)
            print(f"{name} {mode}: exit {code}, {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(os.path.join(HERE, "configs_reference.npz"), **out)
    print("wrote configs_reference.npz")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
