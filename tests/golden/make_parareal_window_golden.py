"""c3 ORIGINAL-Parareal window fixture from the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_parareal_window_golden.py [config] [n_it]

Runs the reference's parareal_sweep (parareal.py:68-97, no Krylov subspace) on a BASELINE
config (default c3: 512^2, P=64, K=5) with a thread pool for the fine sweep and stores, like
make_window_golden.py, the residual history, the per-slice L2 norms of qn[1:] after every
iteration and 512 fixed-seed sampled entries per slice (<config>_parareal_reference.npz).
Plain Parareal has no ill-conditioned factorisation, so the device must match at 1e-10.
"""
from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, HERE)

import pitwave.parareal as ref_par  # noqa: E402

from make_golden import slice_closures  # noqa: E402
from paper_1510_02237_b200 import harness  # noqa: E402  (seeded generators only)

N_SAMPLE = 512


def main(name="c3", n_it=None):
    wl = harness.WORKLOADS[name]
    n_it = wl.n_it if n_it is None else n_it
    fine, coarse = slice_closures(wl)
    q0 = harness.initial_state(name)
    idx = np.sort(np.random.default_rng(4242).choice(q0.size, N_SAMPLE, replace=False))
    norms, samples = [], []
    orig_res = ref_par.iteration_residual

    def spy_res(prev, nxt):
        st = np.stack([np.asarray(v) for v in nxt])
        norms.append(np.linalg.norm(st, axis=1))
        samples.append(st[:, idx])
        r = orig_res(prev, nxt)
        print(f"  iteration {len(norms)}: residual {r:.6e} ({time.time() - t0:.0f} s)", flush=True)
        return r

    ref_par.iteration_residual = spy_res
    t0 = time.time()
    try:
        with ThreadPoolExecutor(os.cpu_count()) as pool:
            ends, res = ref_par.parareal_sweep(q0, fine, coarse, wl.n_p, n_it, pool=pool)
    finally:
        ref_par.iteration_residual = orig_res
    np.savez_compressed(os.path.join(HERE, f"{name}_parareal_reference.npz"), res=np.array(res),
                        norms=np.array(norms), samples=np.array(samples), idx=idx,
                        seconds=time.time() - t0, threads=os.cpu_count())
    print(f"done in {time.time() - t0:.0f} s: residuals {res}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c3", int(sys.argv[2]) if len(sys.argv) > 2 else None)
