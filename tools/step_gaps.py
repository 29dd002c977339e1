"""Wall time of one controlled product step (config 2) against the sum of its
device phases, to find host-side gaps: python tools/step_gaps.py [steps]"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import CONFIGS, log_grid  # noqa: E402

w = CONFIGS["cfg2"]
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed, w.value_seed, w.drop)
taus = log_grid(w.n_taus)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    ctx.synchronize()
    t0 = time.perf_counter()
    C, st, _ = nat.spamm_with_error_control(ctx, A, A, w.delta, taus)
    ctx.synchronize()
    t1 = time.perf_counter()
    del C
    ctx.synchronize()
    t2 = time.perf_counter()
    sp = st["spamm"]
    dev = st["ms_cse"] + sp["ms_tasklist"] + sp["ms_gemm"] + sp["ms_finalize"]
    print(f"step {i}: wall {1e3 * (t1 - t0):.2f} ms, device phases {dev:.2f} ms "
          f"(cse {st['ms_cse']:.2f} tasklist {sp['ms_tasklist']:.2f} gemm {sp['ms_gemm']:.2f} "
          f"finalize {sp['ms_finalize']:.2f}), free C {1e3 * (t2 - t1):.2f} ms", flush=True)
