"""Host wall time of the pieces of bench.py's pipelined end-to-end step on cfg2
(stage the next input, finish the staged one, controlled product streamed to
pinned host buffers):  python tools/e2e_probe.py
Measured (final round-2 library): finish 1.4 ms, stage() 0.0 ms (asynchronous),
product 1382 ms of which GEMM + streaming 1380 ms (resident GEMM: 1359 ms)."""
import sys, time, ctypes as C
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import numpy as np, torch
from paper_2005_10680_b200 import _native as nat
from paper_2005_10680_b200.inputs import CONFIGS, log_grid
w = CONFIGS["cfg2"]
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed, w.value_seed, w.drop)
taus = log_grid(32, 1e-2, 1e-12)
rows, cols, pay, _ = A.download(payload=True)
n, LL = len(rows), w.leaf * w.leaf
h_rows = torch.from_numpy(rows).pin_memory(); h_cols = torch.from_numpy(cols).pin_memory()
h_pay = torch.empty((n, LL), dtype=torch.float64).pin_memory(); h_pay.numpy()[:] = pay
cap = (w.n // w.leaf + 1) ** 2
o_rows = torch.empty(cap, dtype=torch.int32).pin_memory(); o_cols = torch.empty(cap, dtype=torch.int32).pin_memory()
o_norm = torch.empty(cap, dtype=torch.float64).pin_memory(); o_pay = torch.empty((cap, LL), dtype=torch.float64).pin_memory()
outs = (o_rows.numpy(), o_cols.numpy(), o_pay.numpy(), o_norm.numpy())
del A
def stage(): return nat.Staged(ctx, w.n, w.leaf, n, h_rows.data_ptr(), h_cols.data_ptr(), h_pay.data_ptr())
staged = stage()
for i in range(6):
    t0 = time.perf_counter(); Ah = staged.finish(); t1 = time.perf_counter()
    staged = stage(); t2 = time.perf_counter()
    out, st, _ = nat.spamm_with_error_control_to_host(ctx, Ah, Ah, w.delta, taus, out=outs); t3 = time.perf_counter()
    del Ah; t4 = time.perf_counter()
    print(f"step {i}: finish {1e3*(t1-t0):.1f} ms, stage() {1e3*(t2-t1):.1f} ms, product {1e3*(t3-t2):.1f} ms (gemm {st['spamm']['ms_gemm']:.1f}, tasklist {st['spamm']['ms_tasklist']:.2f}, cse {st['ms_cse']:.2f}), free {1e3*(t4-t3):.1f} ms", flush=True)
