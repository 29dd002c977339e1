"""Breakpoint statistics of the tau-sweep on cfg2 (host, numpy): per node of
levels d-1, d-2 and d-3 (the tile root), the [lo-1, hi) range width over k and
(level d-1) the number of distinct leaf breakpoints -- the evaluation counts of
range evaluation (v8) and of breakpoint evaluation (v9).  Leaf norms from the
product's host generator (spg_synth_cluster_host), summed in numpy order (the
counts do not depend on the last bit).
    python tools/sweep_stats.py        (~8 GB of host memory, a few minutes)"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import CONFIGS, log_grid  # noqa: E402

w = CONFIGS["cfg2"]
r, c, p = nat.synth_cluster_host(w.n, w.leaf, w.ell, w.density, w.site_seed, w.value_seed, w.drop)
nb = -(-w.n // w.leaf)
N = np.zeros((nb, nb))
N[r, c] = np.sqrt((np.asarray(p).reshape(len(r), -1) ** 2).sum(1))
del p


def level_stats(K, shape, nt):
    hi = K.max(-1)
    lo = np.where(K > 0, K, 10 ** 6).min(-1)
    return np.bincount(np.where(hi > 0, hi - lo + 1, 0).ravel(), minlength=nt + 2)


for nt, lo_tau in ((32, 1e-12), (64, 1e-12), (128, 1e-14)):
    asc = np.sort(log_grid(nt, 1e-2, lo_tau))
    w1 = w2 = w3 = d1 = 0
    for i0 in range(0, nb, 64):
        P = N[i0:i0 + 64, :, None] * N[None, :, :]          # (i, k, j) leaf products
        k0 = nt - np.searchsorted(asc, P, side="right")       # #{k : p < tau_k}
        k0[P == 0] = 0
        K1 = k0.reshape(32, 2, nb // 2, 2, nb // 2, 2).transpose(0, 2, 4, 1, 3, 5).reshape(32, nb // 2, nb // 2, 8)
        w1 = w1 + level_stats(K1, None, nt)
        s = np.sort(K1, -1)
        dist = ((np.diff(s, axis=-1) != 0) & (s[..., 1:] > 0)).sum(-1) + (s[..., 0] > 0)
        d1 = d1 + np.bincount(dist.ravel(), minlength=9)
        K2 = k0.reshape(16, 4, nb // 4, 4, nb // 4, 4).transpose(0, 2, 4, 1, 3, 5).reshape(16, nb // 4, nb // 4, 64)
        w2 = w2 + level_stats(K2, None, nt)
        K3 = k0.reshape(8, 8, nb // 8, 8, nb // 8, 8).transpose(0, 2, 4, 1, 3, 5).reshape(8, nb // 8, nb // 8, 512)
        w3 = w3 + level_stats(K3, None, nt)
    mean = lambda h: float((np.arange(len(h)) * h).sum() / h.sum())  # noqa: E731
    print(f"n_taus {nt}: level d-1 range {mean(w1):.2f}, distinct breakpoints {mean(d1):.2f}; "
          f"level d-2 range {mean(w2):.2f}; tile root range {mean(w3):.2f}", flush=True)
