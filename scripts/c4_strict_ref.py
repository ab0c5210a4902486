"""c4 iteration-1 deviation from the reference run, fast vs strict kernels."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1510_02237_b200 import _lib, harness  # noqa: E402
from paper_1510_02237_b200.parareal import kse_sweep  # noqa: E402
from test_gpu_windows_ref import props  # noqa: E402

g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "c4_reference.npz"))
wl, fine, coarse = props("c4")
q0 = torch.as_tensor(harness.initial_state("c4")).cuda()
idx = torch.as_tensor(g["idx"]).cuda()
ctx = _lib.Context.get(0)
for strict in (False, True):
    ctx.set_strict(strict)
    ends, res, sub = kse_sweep(q0, fine, coarse, wl.n_p, 1, return_device=True)
    st = ends.reshape(wl.n_p, -1)
    samp = st[:, idx].cpu().numpy()
    dev = np.linalg.norm(samp - g["samples"][0], axis=1) / np.linalg.norm(g["samples"][0], axis=1)
    rat = np.sort(sub.diag_ratios())[::-1]
    print(f"strict={strict}: rank {sub.rank}, max dev {dev.max():.3e}, median {np.median(dev):.3e}, "
          f"residual {res[0]!r} (ref {g['res'][0]!r}); ratios around the cut: {rat[sub.rank-3:sub.rank+3]}",
          flush=True)
    del ends, st, sub
    torch.cuda.empty_cache()
ctx.set_strict(False)
