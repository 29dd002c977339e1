import sys; sys.path.insert(0, "/root/repo")
from paper_2005_10680_b200 import _native as nat
from paper_2005_10680_b200.inputs import log_grid
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, 32, 3.0, 0.1, 2005, 10680, 1e-10)
for _ in range(2):
    C, st, _ = nat.spamm_with_error_control(ctx, A, A, 1e-6, log_grid(128, 1e-2, 1e-14)); del C
sp = st["spamm"]; print("gemm %.1f ms %.2f TF/s" % (sp["ms_gemm"], sp["flops"]/sp["ms_gemm"]/1e9))
