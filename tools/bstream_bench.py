"""B streamed from host memory vs B resident, on
the config-2 matrix: N=32768, L=64, 3-D cluster, delta=1e-5, 32 taus.

For each panel height: creation time (norm pass over all panels), the
streamed controlled product's GEMM-phase time and TFLOP/s, against the
resident product; C is checked bitwise equal.

    python tools/bstream_bench.py [N]
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
L = 64
ctx = nat.Context(0)
t0 = time.perf_counter()
rows, cols, pay = nat.synth_cluster_host(N, L, 3.0, 0.1, 2005, 10680, 1e-10)
rows, cols, pay = nat.sort_by_block_row(rows, cols, pay)
gen_s = time.perf_counter() - t0
A = nat.upload(ctx, N, L, rows, cols, pay)
taus = log_grid(32)
delta = 1e-5


def sig(C):
    r, c, p, n = C.download()
    return r.tobytes(), c.tobytes(), p.view(np.uint64).sum(dtype=np.uint64), n.tobytes()


C0, st0, b0 = nat.spamm_with_error_control(ctx, A, A, delta, taus)  # warm-up
del C0
C0, st0, b0 = nat.spamm_with_error_control(ctx, A, A, delta, taus)
ref = sig(C0)
del C0
sp = st0["spamm"]
print(json.dumps({"mode": "resident", "N": N, "leaves": int(len(rows)),
                  "B_bytes": int(pay.nbytes), "gen_s": round(gen_s, 1),
                  "ms_gemm": round(sp["ms_gemm"], 1),
                  "tflops": round(sp["flops"] / sp["ms_gemm"] / 1e9, 2),
                  "ms_tasklist": round(sp["ms_tasklist"], 2)}), flush=True)
for panel_rows in (8, 32, 128):
    t1 = time.perf_counter()
    bs = nat.BStream(ctx, N, L, rows, cols, pay, panel_rows, register_host=True)
    create_s = time.perf_counter() - t1
    C1, st1, b1 = nat.spamm_with_error_control_streamed(ctx, A, bs, delta, taus)  # warm-up
    del C1
    C1, st1, b1 = nat.spamm_with_error_control_streamed(ctx, A, bs, delta, taus)
    same = sig(C1) == ref and np.array_equal(b0.view(np.uint64), b1.view(np.uint64))
    del C1
    s1 = st1["spamm"]
    npan, mx = bs.panels()
    print(json.dumps({"mode": "streamed", "panel_block_rows": panel_rows, "panels": npan,
                      "max_panel_MB": round(mx * L * L * 8 / 1e6, 1),
                      "create_s": round(create_s, 3),
                      "h2d_GBps_create": round(pay.nbytes / create_s / 1e9, 1),
                      "ms_gemm": round(s1["ms_gemm"], 1),
                      "tflops": round(s1["flops"] / s1["ms_gemm"] / 1e9, 2),
                      "vs_resident": round(sp["ms_gemm"] / s1["ms_gemm"], 3),
                      "bitwise_equal": bool(same)}), flush=True)
    bs.free()
