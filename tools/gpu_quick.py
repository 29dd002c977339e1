"""Quick GPU shakeout: parity of every hot-path kernel against the oracle on
small random cases + cfg1, then cfg2 timing.  Developer tool (not a test)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

import oracle
from paper_2005_10680_b200 import _native as nat
from paper_2005_10680_b200 import inputs

ctx = nat.Context(0)
P = oracle.Oracle("port")
rng = np.random.default_rng(1)
bad = 0


def bits_equal(x, y):
    return np.array_equal(np.asarray(x, np.float64).view(np.uint64),
                          np.asarray(y, np.float64).view(np.uint64))


def check_case(n, L, da, db, taus, tag):
    global bad
    la, lb = nat.dense_to_leaves(da, L), nat.dense_to_leaves(db, L)
    A, B = nat.upload(ctx, n, L, *la), nat.upload(ctx, n, L, *lb)
    oa, ob = P.build(n, L, *la), P.build(n, L, *lb)
    for lvl in range(oa.depth() + 1):
        if not bits_equal(A.level_norms(lvl), oa.level_norms(lvl)):
            bad += 1
            print(tag, "level norm mismatch at", lvl)
            break
    g = nat.cse(ctx, A, B, taus)
    o = P.cse(oa, ob, taus)
    if not bits_equal(g, o):
        bad += 1
        diff = np.nonzero(g != o)[0]
        print(tag, "CSE mismatch", diff[:5], g[diff[:3]], o[diff[:3]])
    tau = float(taus[rng.integers(0, len(taus))])
    sg = nat.survivors(ctx, A, B, tau)
    so = P.survivors(oa, ob, tau)
    if not np.array_equal(sg, so):
        bad += 1
        print(tag, "survivor mismatch", len(sg), len(so))
    C, st = nat.spamm(ctx, A, B, tau)
    oc = P.spamm(oa, ob, tau)
    rg, cg, pg, ng = C.download()
    ro, co, po, no = oc.leaves()
    dg = nat.leaves_to_dense(n, L, rg, cg, pg)
    do = nat.leaves_to_dense(n, L, ro, co, po)
    rel = np.linalg.norm(dg - do) / max(np.linalg.norm(do), 1e-300)
    if rel > 1e-12 or not np.array_equal(rg, ro) or not np.array_equal(cg, co):
        bad += 1
        print(tag, "C mismatch rel", rel, len(rg), len(ro))
    return st


for trial in range(40):
    L = int(rng.choice([2, 4, 8, 16, 32, 64]))
    nb = int(rng.integers(1, 9))
    n = max(1, nb * L - int(rng.integers(0, L)))
    fill = rng.uniform(0.05, 1.0)
    def rd():
        d = rng.uniform(-1, 1, (n, n)) * (rng.uniform(size=(n, n)) < fill)
        d *= np.exp(-np.abs(np.subtract.outer(np.arange(n), np.arange(n))) / rng.uniform(1, 30))
        return d
    taus = inputs.geometric_grid(1.0, float(rng.uniform(0.3, 0.9)), int(rng.integers(1, 60)))
    check_case(n, L, rd(), rd(), taus, f"trial{trial}(n={n},L={L})")
print("random trials done, failures:", bad)

# cfg1
w = inputs.CONFIGS["cfg1"]
t0 = time.time()
rows, cols, pay = nat.synth_chain_host(w.n, w.leaf, w.ell, w.value_seed, w.drop)
print("cfg1 host gen", time.time() - t0, "s, leaves", len(rows))
A = nat.upload(ctx, w.n, w.leaf, rows, cols, pay)
oa = P.build(w.n, w.leaf, rows, cols, pay)
taus = inputs.log_grid(w.n_taus)
t0 = time.time()
o = P.cse(oa, oa, taus)
print("oracle cse", time.time() - t0)
g = nat.cse(ctx, A, A, taus)
print("cfg1 cse bitwise:", bits_equal(g, o))
k = P.select_index(o, w.delta)
tau = taus[k]
t0 = time.time()
so = P.survivors(oa, oa, tau)
sg = nat.survivors(ctx, A, A, tau)
print("cfg1 tau", tau, "k", k, "survivors", len(sg), len(so), "equal:", np.array_equal(sg, so))
C, st, bounds = nat.spamm_with_error_control(ctx, A, A, w.delta, taus)
print("cfg1 controlled:", st)
t0 = time.time()
oc = P.spamm(oa, oa, tau)
print("oracle spamm", time.time() - t0)
rg, cg, pg, ng = C.download()
ro, co, po, no = oc.leaves()
print("cfg1 C structure equal:", np.array_equal(rg, ro) and np.array_equal(cg, co))
print("cfg1 C rel err:", np.linalg.norm(pg - po) / np.linalg.norm(po))
for _ in range(3):
    C, st, bounds = nat.spamm_with_error_control(ctx, A, A, w.delta, taus)
    print("cfg1 timing: cse %.3f ms tasklist %.3f gemm %.3f final %.3f  TF/s(gemm) %.2f" % (
        st["ms_cse"], st["spamm"]["ms_tasklist"], st["spamm"]["ms_gemm"], st["spamm"]["ms_finalize"],
        st["spamm"]["flops"] / st["spamm"]["ms_gemm"] / 1e9))

# cfg2
w = inputs.CONFIGS["cfg2"]
t0 = time.time()
A = nat.synth_cluster_device(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed, w.value_seed, w.drop)
ctx.synchronize()
print("cfg2 device gen %.2f s, nnzb %d frob %.6g" % (time.time() - t0, A.nnz_blocks, A.frobenius_norm))
taus = inputs.log_grid(w.n_taus)
for _ in range(3):
    C, st, bounds = nat.spamm_with_error_control(ctx, A, A, w.delta, taus)
    s = st["spamm"]
    print("cfg2: tau %.3g k %d bound %.3g | cse %.3f ms | tasklist %.3f gemm %.3f final %.3f ms | surv %d of %d | gemm %.2f TF/s" % (
        st["tau"], st["tau_index"], st["bound"], st["ms_cse"], s["ms_tasklist"], s["ms_gemm"],
        s["ms_finalize"], s["survivors"], s["candidates"], s["flops"] / s["ms_gemm"] / 1e9))
    del C
print("bounds", bounds)
print("launches", ctx.launch_count())
print("FAILURES", bad)
