"""One error-controlled SpAMM step on a BASELINE workload, for ncu captures
(python tools/profile_step.py [cfg1|cfg2] [warmup])."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import CONFIGS, log_grid  # noqa: E402

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = nat.Context(0)
if w.kind == "cluster":
    A = nat.synth_cluster_device(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed, w.value_seed,
                                 w.drop)
else:
    A = nat.synth_chain_device(ctx, w.n, w.leaf, w.ell, w.value_seed, w.drop)
taus = log_grid(w.n_taus)
for _ in range(warm + 1):
    C, st, _ = nat.spamm_with_error_control(ctx, A, A, w.delta, taus)
    del C
print(st)
