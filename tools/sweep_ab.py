"""tau-sweep A/B on the cfg2 matrix: host wall time of spg_cse (bounds on the
host) over several grids, plus a digest of the bound bits so two builds or two
kernel versions can be compared bit for bit.
    python tools/sweep_ab.py [reps]   -> one JSON line per grid"""
import hashlib
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ctx = nat.Context(0)
A = nat.synth_cluster_device(ctx, 32768, 64, 3.0, 0.1, 2005, 10680, 1e-10)
cand = 134119838
for nt, lo in ((32, 1e-12), (64, 1e-12), (128, 1e-14)):
    taus = log_grid(nt, 1e-2, lo)
    b0 = nat.cse(ctx, A, A, taus)
    ts = []
    for _ in range(reps):
        ctx.synchronize()
        t0 = time.perf_counter()
        b = nat.cse(ctx, A, A, taus)
        ts.append(1e3 * (time.perf_counter() - t0))
        assert np.array_equal(b.view(np.uint64), b0.view(np.uint64)), "run-to-run bits differ"
    ms = float(np.median(ts))
    print(json.dumps({"n_taus": nt, "grid": [1e-2, lo], "ms_median": round(ms, 4),
                      "ms_min": round(min(ts), 4), "gbs_effective": round(12 * cand / ms / 1e6, 1),
                      "digest": hashlib.sha256(b0.tobytes()).hexdigest()[:16]}), flush=True)
