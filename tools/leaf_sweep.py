"""BASELINE config 5's sweep on one GPU at N=32768 (the 3-D cluster of config
2): leaf size L in {32, 64, 128} x delta in {1e-8, 1e-6, 1e-4}, 128 candidate
taus log-spaced over [1e-14, 1e-2] (extended below 1e-12 so delta=1e-8 does
not fall back to tau=0).  Reports the skipped fraction, leaf-GEMM TFLOP/s
(fraction of the DMMA peak) and sweep time / effective GB/s per cell.

    python tools/leaf_sweep.py [N]
"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
PEAK = 37.1
ctx = nat.Context(0)
taus = log_grid(128, 1e-2, 1e-14)
rows = []
for L in (32, 64, 128):
    A = nat.synth_cluster_device(ctx, N, L, 3.0, 0.1, 2005, 10680, 1e-10)
    for delta in (1e-8, 1e-6, 1e-4):
        C, st, _ = nat.spamm_with_error_control(ctx, A, A, delta, taus)  # warm-up
        del C
        C, st, _ = nat.spamm_with_error_control(ctx, A, A, delta, taus)
        sp = st["spamm"]
        gemm_tf = sp["flops"] / (sp["ms_gemm"] / 1e3) / 1e12 if sp["ms_gemm"] > 0 else 0.0
        step_ms = st["ms_cse"] + sp["ms_tasklist"] + sp["ms_gemm"] + sp["ms_finalize"]
        row = {"L": L, "delta": delta, "tau": st["tau"], "tau_index": st["tau_index"],
               "bound": st["bound"], "candidates": sp["candidates"], "survivors": sp["survivors"],
               "skipped_fraction": round(1 - sp["survivors"] / max(sp["candidates"], 1), 4),
               "gemm_tflops": round(gemm_tf, 2), "dmma_frac": round(gemm_tf / PEAK, 3),
               "sweep_ms": round(st["ms_cse"], 3),
               "sweep_eff_gbs": round(12 * sp["candidates"] / (st["ms_cse"] / 1e3) / 1e9, 1),
               "step_ms": round(step_ms, 1),
               "step_tflops": round(sp["flops"] / (step_ms / 1e3) / 1e12, 2)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del C
    del A
