"""Leaf-GEMM tiling variants on the config-5 matrix (3-D cluster, N=32768) for
one leaf size: python tools/gemm_variants.py L  (runs each SPG_GEMM* setting
in its own process; prints TFLOP/s of the GEMM phase)."""
import os
import subprocess
import sys

L = int(sys.argv[1]) if len(sys.argv) > 1 else 64
var = {32: ("SPG_GEMM32", [9, 6, 2, 8, 1, 7]), 64: ("SPG_GEMM", [4, 5, 6, 8]),
       128: ("SPG_GEMM128", [9, 3, 4, 1, 2])}[L]
code = f"""
import sys
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
from paper_2005_10680_b200 import _native as nat
from paper_2005_10680_b200.inputs import log_grid
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, {L}, 3.0, 0.1, 2005, 10680, 1e-10)
for _ in range(2):
    C, st, _ = nat.spamm_with_error_control(ctx, A, A, 1e-6, log_grid(128, 1e-2, 1e-14))
    del C
sp = st["spamm"]
print(round(sp["flops"] / sp["ms_gemm"] / 1e9, 2), round(sp["ms_gemm"], 1))
"""
for v in var[1]:
    env = dict(os.environ, **{var[0]: str(v)})
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(L, var[0], v, out.stdout.strip() or out.stderr[-300:], flush=True)
