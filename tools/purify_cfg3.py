"""BASELINE config 3 at full size on one GPU: SP2 purification of the config-2
style 3-D cluster Hamiltonian with N = 65536 (L = 64), 25 iterations, every
multiply through the tau-sweep with delta_i = 1e-4/25.  H is built on the
device (no dense host copy): the cluster matrix's off-diagonal part scaled to
max absolute row sum 0.45, plus a diagonal that puts half the states in
[-1+r_i, -0.025-r_i] and half in [0.025+r_i, 1-r_i] (r_i its off-diagonal row
sum): disjoint Gershgorin unions, spectrum in [-1,-0.025] U [0.025,1], gap 0.05
at mu = 0.  X0 = (I - H)/2.

    python tools/purify_cfg3.py [N] [iterations]
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 25
L = 64
ctx = nat.Context(0)
t0 = time.perf_counter()
A = nat.synth_cluster_device(ctx, N, L, 3.0, 0.1, 2005, 10680, 1e-10)
diag_a, rowsum = nat.row_data(A)
off = rowsum - np.abs(diag_a)
s = 0.45 / off.max()
r = s * off
rng = np.random.default_rng(3)
occupied = rng.permutation(N) < N // 2
u = rng.uniform(size=N)
lo = np.where(occupied, -1.0 + r, 0.025 + r)
hi = np.where(occupied, -0.025 - r, 1.0 - r)
Hoff = nat.axpby(ctx, s, A, -s, nat.from_diagonal(ctx, diag_a, L))  # s (A - diag A)
del A
H = nat.axpby(ctx, 1.0, Hoff, 1.0, nat.from_diagonal(ctx, lo + u * (hi - lo), L))
del Hoff
X0 = nat.axpby(ctx, 0.5, nat.identity(ctx, N, L), -0.5, H)
del H
ctx.synchronize()
gen_s = time.perf_counter() - t0
deltas = np.full(iters, 1e-4 / iters)
t1 = time.perf_counter()
D, log, conv, its = nat.purify(ctx, X0, "spamm", N // 2, epsilon=1e-4, max_iterations=iters,
                               taus=log_grid(32), budget=(0.0, deltas), measure_error=False)
ctx.synchronize()
wall = time.perf_counter() - t1
flops = sum(rec["flops"] for rec in log)
out = {
    "workload": f"BASELINE config 3: SP2 purification, 3-D cluster H, N={N}, L={L}",
    "iterations": its, "converged": conv, "wall_s": round(wall, 3),
    "leaf_gemm_tflops_over_wall": round(flops / wall / 1e12, 3), "flops": flops,
    "trace": nat.trace(D), "occupation": N // 2, "x0_leaves": X0.nnz_blocks,
    "density_leaves": D.nnz_blocks, "gen_s": round(gen_s, 1),
    "per_iteration": [{k: rec[k] for k in ("iteration", "chosen_tau", "nnz_blocks_out", "status",
                                            "trace", "t_spamm", "t_cse", "flops")}
                      for rec in log],
}
print(json.dumps(out))
