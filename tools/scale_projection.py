"""Strong-scaling projection of the config-2 step from per-rank measurements
on one GPU: for N = 1, 2, 4, 8 every rank's share of the step (its sweep
share spg_cse_shard + the host finish, its rows' task list + GEMM +
finalize via spg_spamm_shard) is run and timed alone on this GPU; the
projected N-GPU step is the slowest rank plus the partials' all-gather
(<= 4^s N_tau doubles, not modelled).  Output: one JSON line per N with the
per-rank times, the projected whole-job TFLOP/s and efficiency against N x
the one-GPU value.  Ranks on real GPUs also contend for nothing (replicated
operands), so the projection's only approximation is the collective.

    python tools/scale_projection.py
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, 64, 3.0, 0.1, 2005, 10680, 1e-10)
taus = log_grid(32)
delta = 1e-5
C, st, bounds = nat.spamm_with_error_control(ctx, A, A, delta, taus)  # warm-up + reference
tau = st["tau"]
flops_total = st["spamm"]["flops"]
del C
base = None
def run_ranks(n, level):
    ranks, parts = [], []
    for g in range(n):
        ctx.synchronize()
        t0 = time.perf_counter()
        if level:
            parts.append(nat.cse_shard(ctx, A, A, taus, level, g))
        ctx.synchronize()
        sweep_ms = 1e3 * (time.perf_counter() - t0) if level else st["ms_cse"]
        Cs, ss = nat.spamm_shard(ctx, A, A, tau, level, g) if level else (None, st["spamm"])
        ms = ss["ms_tasklist"] + ss["ms_gemm"] + ss["ms_finalize"]
        ranks.append({"rank": g, "sweep_ms": round(sweep_ms, 3), "product_ms": round(ms, 2),
                      "survivors": ss["survivors"], "flops": ss["flops"]})
        del Cs
    return ranks, parts


for n in (1, 2, 4, 8):
    level = n.bit_length() - 1
    run_ranks(n, level)  # warm-up pass (pool sizes, kernel attributes)
    ranks, parts = run_ranks(n, level)
    if level:
        b2 = nat.cse_finish(level, nat.top_norms(A, level), nat.top_norms(A, level), np.stack(parts))
        assert np.array_equal(b2.view(np.uint64), bounds.view(np.uint64))
    step = max(r["sweep_ms"] + r["product_ms"] for r in ranks)
    tf = flops_total / (step / 1e3) / 1e12
    if base is None:
        base = tf
    print(json.dumps({"n_gpus": n, "projected_step_ms": round(step, 2),
                      "projected_tflops": round(tf, 2),
                      "projected_efficiency": round(tf / (n * base), 4),
                      "max_over_mean_product": round(
                          max(r["product_ms"] for r in ranks) /
                          (sum(r["product_ms"] for r in ranks) / n), 4),
                      "ranks": ranks}), flush=True)
