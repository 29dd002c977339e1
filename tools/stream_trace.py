import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2005_10680_b200 import _native as nat
from paper_2005_10680_b200.inputs import CONFIGS, log_grid
w = CONFIGS["cfg2"]
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed, w.value_seed, w.drop)
taus = log_grid(w.n_taus)
cap = (w.n // w.leaf) ** 2; LL = w.leaf * w.leaf
pin = (torch.empty(cap, dtype=torch.int32).pin_memory().numpy(), torch.empty(cap, dtype=torch.int32).pin_memory().numpy(),
       torch.empty((cap, LL), dtype=torch.float64).pin_memory().numpy(), torch.empty(cap, dtype=torch.float64).pin_memory().numpy())
for i in range(2):
    t = time.perf_counter(); out, st, _ = nat.spamm_with_error_control_to_host(ctx, A, A, w.delta, taus, out=pin)
    print("streamed total %.0f ms" % (1e3 * (time.perf_counter() - t)), st["ms_cse"], st["spamm"]["ms_tasklist"], st["spamm"]["ms_gemm"], file=sys.stderr)
