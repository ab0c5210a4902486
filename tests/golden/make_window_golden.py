"""c3 / c4 KSE-window fixtures from the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_window_golden.py [n_it] [config]

Runs the reference's kse_sweep on a BASELINE config (default c4 = harness.WORKLOADS["c4"],
1024^2, P=256; or c3) for n_it iterations (default 1; at c4 each further iteration
costs the reference a single-threaded pivoted QR of 3.1M x 256k) with a thread pool for
the fine sweep, and stores what a multi-GB window can be pinned by in a small file
(<config>_reference.npz): the residual history, the ranks, the per-slice L2 norms of
qn[1:] after every iteration and 512 fixed-seed sampled entries per slice.  The states
themselves (6 GB per iteration at c4) are not stored.

PW_GOLDEN_SPILL=<dir> keeps the subspace's d x m matrices in file-backed memmaps
(see _SpillNumpy), which is how the K=2 c4 fixtures were made in a 62 GB container.
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

from pitwave import subspace as ref_sub  # noqa: E402
from pitwave.parareal import kse_sweep  # noqa: E402

from make_golden import slice_closures  # noqa: E402
from paper_1510_02237_b200 import harness  # noqa: E402  (seeded generators only)

N_SAMPLE = 512


class _SpillNumpy:
    """numpy as the reference's subspace module sees it, except that the two d x m
    allocations of Subspace.update (column_stack of the snapshots / images and the
    F-order scratch copy handed to LAPACK) are file-backed memmaps under ``root``.
    Same values, same LAPACK calls; only the pages live on disk, so a c4 window with
    K=2 (~100 GB of working set) runs in a 62 GB container.  PW_GOLDEN_SPILL=<dir>.
    """

    def __init__(self, root):
        self._root = root
        self._n = 0
        os.makedirs(root, exist_ok=True)

    def _alloc(self, shape, order):
        self._n += 1
        path = os.path.join(self._root, f"spill_{self._n}.bin")
        a = np.lib.format.open_memmap(path, mode="w+", dtype=np.float64, shape=shape,
                                      fortran_order=(order == "F"))
        os.unlink(path)  # pages stay mapped; the file disappears with the array
        return a

    def column_stack(self, cols):
        cols = [np.asarray(c) for c in cols]
        m = sum(1 if c.ndim == 1 else c.shape[1] for c in cols)
        out = self._alloc((cols[0].shape[0], m), "C")
        j = 0
        for c in cols:
            if c.ndim == 1:
                out[:, j] = c
                j += 1
            elif c.shape[1]:
                out[:, j:j + c.shape[1]] = c
                j += c.shape[1]
        return out

    def asfortranarray(self, a):
        out = self._alloc(a.shape, "F")
        out[...] = a
        return out

    def __getattr__(self, name):
        return getattr(np, name)


def main(n_it=1, name="c4", suffix=""):
    wl = harness.WORKLOADS[name]
    fine, coarse = slice_closures(wl)
    q0 = harness.initial_state(name)
    d = q0.size
    idx = np.sort(np.random.default_rng(4242).choice(d, N_SAMPLE, replace=False))
    norms, samples, ranks = [], [], []
    orig_update = ref_sub.Subspace.update

    def spy_update(self, states, images):
        new = orig_update(self, states, images)
        ranks.append(new.rank)
        print(f"  update: rank {new.rank} ({time.time() - t0:.0f} s)", flush=True)
        return new

    import pitwave.parareal as ref_par
    orig_res = ref_par.iteration_residual

    def spy_res(prev, nxt):
        st = np.stack([np.asarray(v) for v in nxt])
        norms.append(np.linalg.norm(st, axis=1))
        samples.append(st[:, idx])
        r = orig_res(prev, nxt)
        print(f"  iteration {len(norms)}: residual {r:.6e} ({time.time() - t0:.0f} s)", flush=True)
        return r

    spill = os.environ.get("PW_GOLDEN_SPILL")
    if spill:
        ref_sub.np = _SpillNumpy(spill)
    ref_sub.Subspace.update = spy_update
    ref_par.iteration_residual = spy_res
    t0 = time.time()
    try:
        with ThreadPoolExecutor(os.cpu_count()) as pool:
            ends, res, sub = kse_sweep(q0, fine, coarse, wl.n_p, n_it, pool=pool)
    finally:
        ref_sub.Subspace.update = orig_update
        ref_par.iteration_residual = orig_res
        ref_sub.np = np
    np.savez_compressed(os.path.join(HERE, f"{name}_reference{suffix}.npz"), res=np.array(res), ranks=np.array(ranks),
                        norms=np.array(norms), samples=np.array(samples), idx=idx,
                        seconds=time.time() - t0, threads=os.cpu_count())
    print(f"done in {time.time() - t0:.0f} s: residuals {res}, ranks {ranks}")


if __name__ == "__main__":
    # a third argument names a variant file, e.g. "_numpy" for a PITWAVE_KERNELS=numpy run
    # (the reference's own backend-to-backend noise floor)
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1, sys.argv[2] if len(sys.argv) > 2 else "c4",
         sys.argv[3] if len(sys.argv) > 3 else "")
