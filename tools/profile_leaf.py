"""One controlled product of the config-5 matrix (3-D cluster, N=32768) at
leaf size L, for ncu captures of the leaf GEMM: python tools/profile_leaf.py L [delta]"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, L, 3.0, 0.1, 2005, 10680, 1e-10)
for _ in range(2):
    C, st, _ = nat.spamm_with_error_control(ctx, A, A, delta, log_grid(128, 1e-2, 1e-14))
    del C
sp = st["spamm"]
print(L, delta, round(sp["flops"] / sp["ms_gemm"] / 1e9, 2), "TFLOP/s",
      round(1 - sp["survivors"] / sp["candidates"], 4), "skipped")
