"""Time the pieces of the e2e path on cfg2 (developer tool)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch

from paper_2005_10680_b200 import _native as nat
from paper_2005_10680_b200.inputs import CONFIGS, log_grid

w = CONFIGS["cfg2"]
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed, w.value_seed, w.drop)
rows, cols, pay, _ = A.download()
n, LL = len(rows), w.leaf * w.leaf
h_pay = torch.empty((n, LL), dtype=torch.float64).pin_memory()
h_pay.numpy()[:] = pay
d = torch.empty((n, LL), dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h_pay, non_blocking=True); torch.cuda.synchronize()
    print("torch pinned H2D %.1f GB/s" % (h_pay.numel() * 8 / (time.perf_counter() - t) / 1e9))
    torch.cuda.synchronize(); t = time.perf_counter(); h_pay.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print("torch pinned D2H %.1f GB/s" % (h_pay.numel() * 8 / (time.perf_counter() - t) / 1e9))
del d
h_rows = torch.from_numpy(rows).pin_memory(); h_cols = torch.from_numpy(cols).pin_memory()
taus = log_grid(w.n_taus)
cap = (w.n // w.leaf) ** 2
outs = (torch.empty(cap, dtype=torch.int32).pin_memory().numpy(), torch.empty(cap, dtype=torch.int32).pin_memory().numpy(),
        torch.empty((cap, LL), dtype=torch.float64).pin_memory().numpy(), torch.empty(cap, dtype=torch.float64).pin_memory().numpy())
for rep in range(3):
    t0 = time.perf_counter()
    Ah = nat.upload(ctx, w.n, w.leaf, h_rows.numpy(), h_cols.numpy(), h_pay.numpy())
    t1 = time.perf_counter()
    C, st, _ = nat.spamm_with_error_control(ctx, Ah, Ah, w.delta, taus)
    t2 = time.perf_counter()
    r = C.download()
    t3 = time.perf_counter()
    del C
    out, st2, _ = nat.spamm_with_error_control_to_host(ctx, Ah, Ah, w.delta, taus, out=outs)
    t4 = time.perf_counter()
    print("upload %.0f ms | product %.0f ms | download %.0f ms | streamed product %.0f ms" % (
        1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3)))
    del Ah
