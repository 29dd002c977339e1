"""Dump the leaf-level norm grid of the config-2 matrix (Morton order, -1 =
null) to gpurun_out/cfg2_leafnorms.npy, plus the sweep bounds of the current
kernels for the 32/64/128-tau grids (for offline analysis of the tau-sweep's
piece structure and as a regression reference for new sweep kernels).
    python tools/dump_norms.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

out = Path("gpurun_out")
out.mkdir(exist_ok=True)
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, 64, 3.0, 0.1, 2005, 10680, 1e-10)
lev = A.level_norms(9)
np.save(out / "cfg2_leafnorms.npy", lev)
for nt in (32, 64, 128):
    taus = log_grid(nt)
    np.save(out / f"cfg2_bounds_{nt}.npy", nat.cse(ctx, A, A, taus))
print("ok", lev.shape, (lev >= 0).sum())
