"""cfg2 tau-sweep only: builds the config-2 matrix on the device and runs
spg_cse a few times (for ncu captures of the sweep kernels).
    python tools/cse_probe.py [n_taus] [reps] [lowest tau]"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, 64, 3.0, 0.1, 2005, 10680, 1e-10)
lo = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-12
taus = log_grid(nt, 1e-2, lo)
for _ in range(reps):
    ctx.synchronize()
    t0 = time.perf_counter()
    b = nat.cse(ctx, A, A, taus)
    print("cse ms", round(1e3 * (time.perf_counter() - t0), 3), flush=True)
