"""Helper for test_gpu_parity.test_sweep_paths_in_subprocesses: the sweep
kernel path is chosen once per process (SPG_CSE* environment switches), so
each path runs in its own process.  Prints the bound bits of a few cases."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402


def cases():
    """(name, n, L, dense A, dense B, taus) -- shared with the parent test."""
    out = []
    for seed, (n, L, nt) in enumerate([(512, 8, 32), (512, 8, 128), (700, 16, 64), (1024, 16, 32)]):
        rng = np.random.default_rng(4000 + seed)
        nb = -(-n // L)
        sc = np.repeat(np.repeat(10.0 ** rng.uniform(-8, 0, (nb, nb)), L, 0), L, 1)[:n, :n]
        da = rng.uniform(-1, 1, (n, n)) * sc
        db = rng.uniform(-1, 1, (n, n)) * sc.T
        da[:, n // 5: n // 4] = 0.0  # null blocks
        out.append((f"n{n}_L{L}_t{nt}", n, L, da, db, log_grid(nt, 1.0, 1e-14)))
    return out


if __name__ == "__main__":
    ctx = nat.Context(0)
    for name, n, L, da, db, taus in cases():
        A = nat.upload(ctx, n, L, *nat.dense_to_leaves(da, L))
        B = nat.upload(ctx, n, L, *nat.dense_to_leaves(db, L))
        print(name, nat.cse(ctx, A, B, taus).view(np.uint64).tobytes().hex())
