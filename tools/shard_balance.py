"""Row-shard load balance of the cfg2 product on one GPU: survivors and GEMM
ms per shard at levels 1-3 (python tools/shard_balance.py)."""
import sys
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2005_10680_b200 import _native as nat
from paper_2005_10680_b200.inputs import log_grid
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, 64, 3.0, 0.1, 2005, 10680, 1e-10)
taus = log_grid(32)
C, st, b = nat.spamm_with_error_control(ctx, A, A, 1e-5, taus)
tau = st["tau"]
tot = st["spamm"]["survivors"]
print("total", tot, "gemm ms", st["spamm"]["ms_gemm"])
for level in (1, 2, 3):
    s = []
    ms = []
    for g in range(2 ** level):
        Cs, sts = nat.spamm_shard(ctx, A, A, tau, level, g)
        s.append(sts["survivors"]); ms.append(sts["ms_gemm"])
        del Cs
    print(level, "survivors max/mean %.4f" % (max(s) / (sum(s) / len(s))), "gemm ms max/mean %.4f" % (max(ms) / (sum(ms) / len(ms))), [round(x) for x in ms])
