"""Helper for test_gpu_parity.test_gemm_paths_in_subprocesses: the leaf-GEMM
variant is fixed per process (SPG_GEMM32 etc.), so each runs in a child.
Prints a digest of C~ (block coordinates, payload bits, norms) per case."""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2005_10680_b200 import _native as nat  # noqa: E402


def digest(C):
    r, c, p, nrm = C.download()
    h = hashlib.sha256()
    for x in (r, c, p, nrm):
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


if __name__ == "__main__":
    ctx = nat.Context(0)
    for n, L, tau in [(4096, 32, 1e-9), (4096, 32, 0.0), (2080, 32, 1e-7),
                      (8192, 128, 1e-9), (4224, 128, 0.0), (4096, 64, 1e-8), (1000, 8, 1e-6),
                      (40, 8, 1e-6)]:
        A = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 11, 1e-10)
        B = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 12, 1e-10)
        C, st = nat.spamm(ctx, A, B, tau)
        print(f"n{n}_L{L}_tau{tau}", digest(C), st["survivors"])
