"""Truncation timing on the config-2 matrix for a range of delta / ||A||_F
(python tools/truncate_probe.py)."""
import sys, time
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2005_10680_b200 import _native as nat
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, 64, 3.0, 0.1, 2005, 10680, 1e-10)
fro = A.frobenius_norm
for rel in (1e-8, 1e-6, 1e-4, 1e-2, 0.3):
    for rep in range(2):
        ctx.synchronize(); t0 = time.perf_counter()
        Y, bound, count = nat.truncate(ctx, A, rel * fro)
        ctx.synchronize(); dt = time.perf_counter() - t0
    print(rel, "removed", count, "of", A.nnz_blocks, "ms", round(1e3 * dt, 2), flush=True)
