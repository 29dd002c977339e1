"""Pin BASELINE configs 3-5 at full size against the reference.

Run on a B200 box (needs the GPU for the inputs, which are generated on the
device, and oracle/_ref for the reference):

    python tests/golden/make_large_pins.py [case ...]     # cases of tests/large_cases.py, or cfg3

For each case it runs the GPU side (tests/large_cases.py: the 8-rank
machinery on one GPU) and the REFERENCE (oracle/_ref: the unmodified
reference sources) on the same leaf-norm tables and operand bits:
  * reference cse (error_control.cpp:160-166) on norm-only trees of the full
    matrices, all host threads (exec::set_max_threads(64): the reference's
    widest fork-join), and select_tolerance per delta;
  * the reference's survivor decisions (spamm_node) as (count, digest);
  * reference spamm_multiply on A restricted to row i and B to column j for
    the sampled blocks (tests/large_cases.sample_blocks).
It checks the GPU against them here and writes tests/golden/large/<case>.json
(+ .npz with the reference blocks), which tests/test_gpu_pins.py replays
against the GPU path without the reference.

cfg3 (SP2 purification, N = 65536, delta_i = 1e-4/25, 32 tau): for the first
three iterations, the tau the GPU driver (spg_purify) chose for X_i * X_i and
the GPU's bounds of that product vs the reference cse + select_tolerance on
X_i's leaf-norm table.
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from large_cases import CASES, GpuCase, sample_blocks, table_digest  # noqa: E402
from paper_2005_10680_b200 import _native as nat  # noqa: E402

OUT = HERE / "large"
THREADS = os.cpu_count() or 1


def hexbits(x):
    return [f"{v:016x}" for v in np.ascontiguousarray(x, np.float64).view(np.uint64)]


def select(bounds, delta):
    return next((k for k, b in enumerate(bounds) if b < delta), -1)


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def pin_case(ctx, case):
    R = oracle.Oracle("ref")
    t0 = time.perf_counter()
    g = GpuCase(ctx, case)
    n, L = g.n, g.L
    out = {"case": case, "n": n, "leaf": L, "n_taus": g.n_taus, "deltas": g.deltas,
           "taus": hexbits(g.taus), "leaves_A": int(len(g.ta[0])), "leaves_B": int(len(g.tb[0])),
           "table_digest_A": table_digest(g.ta), "table_digest_B": table_digest(g.tb),
           "candidates": g.candidates(), "threads": THREADS}
    log(f"{case}: tables {time.perf_counter() - t0:.1f} s, {out['candidates']:.3e} candidates")
    one, sharded = g.bounds()
    assert np.array_equal(one.view(np.uint64), sharded.view(np.uint64)), "sharded != one-GPU"
    # the reference on norm-only trees of the same tables
    RA = R.build_norm_only(n, L, *g.ta)
    RB = R.build_norm_only(n, L, *g.tb)
    R.set_threads(64)
    t1 = time.perf_counter()
    rb = R.cse(RA, RB, g.taus)
    out["ref_cse_s"] = round(time.perf_counter() - t1, 1)
    log(f"{case}: reference cse {out['ref_cse_s']} s")
    out["bounds"] = hexbits(rb)
    out["gpu_bounds_equal"] = bool(np.array_equal(one.view(np.uint64), rb.view(np.uint64)))
    assert out["gpu_bounds_equal"], "GPU bounds differ from the reference"
    out["per_delta"] = []
    for delta in g.deltas:
        k = select(rb, delta)
        tau = float(g.taus[k]) if k >= 0 else 0.0
        t1 = time.perf_counter()
        rc, rd = R.survivor_digest(RA, RB, tau, THREADS)
        ref_s = time.perf_counter() - t1
        gc, gd, lvl = g.survivor_digest(tau)
        log(f"{case} delta {delta}: k {k} tau {tau:.4g} survivors ref {rc} gpu {gc} "
            f"digest {'=' if rd == gd else '!='} ({ref_s:.1f} s)")
        assert (rc, rd) == (gc, gd), "survivor set differs from the reference"
        out["per_delta"].append({"delta": delta, "tau_index": k, "tau": tau,
                                 "bound": float(rb[k]) if k >= 0 else 0.0, "survivors": rc,
                                 "digest": f"{rd:016x}", "digest_shards_level": lvl})
    del RA, RB
    blocks = {}
    if g.sample_at is not None:
        pd = out["per_delta"][g.sample_at]
        tau = pd["tau"]
        samples = sample_blocks(g.nb)
        out["samples"] = []
        rows_done = {}
        for i, j in samples:
            if i not in rows_done:
                rows_done[i] = (g.product_row(i, tau)[0], g.product_row(i, 0.0)[0])
            approx, exact = rows_done[i]
            (ra, ca, pa), (rb_, cb, pb) = g.reference_operands(i, j)
            TA = R.build(n, L, ra, ca, pa)
            TB = R.build(n, L, rb_, cb, pb)
            rr, rc_, rp, _ = R.spamm(TA, TB, tau).leaves()
            assert len(rr) <= 1 and (len(rr) == 0 or (rr[0], rc_[0]) == (i, j))
            ref_blk = rp[0] if len(rr) else np.zeros(L * L)
            mine = approx.get(j, np.zeros(L * L))
            rel = float(np.linalg.norm(mine - ref_blk) / max(np.linalg.norm(ref_blk), 1e-300))
            blocks[f"b{i}_{j}"] = ref_blk
            # realized error of row i against the GPU's exact (tau = 0) row
            keys = set(approx) | set(exact)
            err = float(np.sqrt(sum(float(np.sum((approx.get(q, 0.0) - exact.get(q, 0.0)) ** 2))
                                    for q in keys)))
            out["samples"].append({"i": i, "j": j, "rel_err": rel, "row_realized_error": err,
                                   "ref_block_nonnull": bool(len(rr))})
            log(f"{case}: block ({i},{j}) rel {rel:.2e}, row {i} realized error {err:.3e}")
            assert rel < 1e-12 and err < pd["delta"] and err <= pd["bound"] * (1 + 1e-9)
    out["wall_s"] = round(time.perf_counter() - t0, 1)
    OUT.mkdir(exist_ok=True)
    (OUT / f"{case}.json").write_text(json.dumps(out, indent=1) + "\n")
    if blocks:
        np.savez(OUT / f"{case}.npz", **blocks)
    log(f"{case}: written ({out['wall_s']} s)")


def cfg3_operator(ctx, N=65536, L=64):
    """tools/purify_cfg3.py's X0 = (I - H)/2 (gapped 3-D cluster Hamiltonian)."""
    A = nat.synth_cluster_device(ctx, N, L, 3.0, 0.1, 2005, 10680, 1e-10)
    diag_a, rowsum = nat.row_data(A)
    off = rowsum - np.abs(diag_a)
    s = 0.45 / off.max()
    r = s * off
    rng = np.random.default_rng(3)
    occupied = rng.permutation(N) < N // 2
    u = rng.uniform(size=N)
    lo = np.where(occupied, -1.0 + r, 0.025 + r)
    hi = np.where(occupied, -0.025 - r, 1.0 - r)
    Hoff = nat.axpby(ctx, s, A, -s, nat.from_diagonal(ctx, diag_a, L))
    del A
    H = nat.axpby(ctx, 1.0, Hoff, 1.0, nat.from_diagonal(ctx, lo + u * (hi - lo), L))
    del Hoff
    return nat.axpby(ctx, 0.5, nat.identity(ctx, N, L), -0.5, H)


def pin_cfg3(ctx, iterations=3, N=65536, L=64):
    from paper_2005_10680_b200.inputs import log_grid
    from paper_2005_10680_b200.sharded import leaf_table
    R = oracle.Oracle("ref")
    R.set_threads(64)
    t0 = time.perf_counter()
    X0 = cfg3_operator(ctx, N, L)
    taus = log_grid(32)
    deltas = np.full(25, 1e-4 / 25)
    out = {"case": "cfg3", "n": N, "leaf": L, "taus": hexbits(taus), "delta_i": 1e-4 / 25,
           "iterations": []}
    # X_0's table and GPU bounds; then per m: spg_purify(m iterations) -> X_m and
    # the log, whose entry m-1 is the tau the driver chose for X_{m-1}^2
    prev_table = leaf_table(X0)
    prev_bounds = nat.cse(ctx, X0, X0, taus)
    for m in range(1, iterations + 1):
        X, logs, _, _ = nat.purify(ctx, X0, "spamm", N // 2, epsilon=1e-4, max_iterations=m,
                                   taus=taus, budget=(0.0, deltas), measure_error=False)
        tau_gpu = logs[m - 1]["chosen_tau"]
        t = prev_table
        T = R.build_norm_only(N, L, *t)
        t1 = time.perf_counter()
        rb = R.cse(T, T, taus)
        ref_s = time.perf_counter() - t1
        del T
        k = select(rb, deltas[m - 1])
        tau_ref = float(taus[k]) if k >= 0 else 0.0
        rec = {"iteration": m, "leaves": int(len(t[0])), "table_digest": table_digest(t),
               "bounds": hexbits(rb), "tau_index": k, "tau": tau_ref, "tau_gpu_driver": tau_gpu,
               "gpu_bounds_equal": bool(np.array_equal(prev_bounds.view(np.uint64),
                                                       rb.view(np.uint64))),
               "ref_cse_s": round(ref_s, 1), "trace": logs[m - 1]["trace"]}
        log(f"cfg3 iteration {m}: tau ref {tau_ref:.4g} gpu {tau_gpu:.4g}, bounds equal "
            f"{rec['gpu_bounds_equal']} ({ref_s:.1f} s)")
        assert rec["gpu_bounds_equal"] and tau_ref == tau_gpu
        out["iterations"].append(rec)
        prev_table = leaf_table(X)
        prev_bounds = nat.cse(ctx, X, X, taus)
        del X
    out["wall_s"] = round(time.perf_counter() - t0, 1)
    OUT.mkdir(exist_ok=True)
    (OUT / "cfg3.json").write_text(json.dumps(out, indent=1) + "\n")
    log(f"cfg3: written ({out['wall_s']} s)")


def main():
    if not oracle.available("ref"):
        sys.exit("oracle/_ref not built (make -C oracle ref)")
    ctx = nat.Context(0)
    cases = sys.argv[1:] or ["cfg5-L128", "cfg5-L64", "cfg3", "cfg4x", "cfg4", "cfg5-L32"]
    for case in cases:
        if case == "cfg3":
            pin_cfg3(ctx)
        else:
            pin_case(ctx, case)


if __name__ == "__main__":
    main()
