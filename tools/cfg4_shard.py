"""BASELINE configs 4 and 5 at full size: one shard of the 8-GPU run, on one B200.

Config 4 (N = 262144, L = 64, 3-D cluster with ell = 4 A, A and B with
independent value seeds, 64 log-spaced tau, delta = 1e-6) and config 5 (the
config-4 form at N = 131072, L in {32, 64, 128}, delta in {1e-8, 1e-6, 1e-4},
128 tau) are sharded by output block row over 8 GPUs.  This
runs everything rank `rank` of those 8 would do, on one GPU:
  * the leaf-norm tables of every shard's A and B rows, each generated on the
    device shard by shard (what the all-gather of the tables delivers), and
    the global norm-only matrices built from them;
  * the rank's sweep share (spg_cse_shard), the other ranks' partials (what
    the partial all-gather delivers), spg_cse_finish -> bounds, tau;
  * the rank's rows of C~ through ONE C-ABI call (spg_spamm_panels), which
    row-chunks the task list itself when it would not fit, B arriving in
    block-row panels through its fetch callback -- generated on the device
    here, where on 8 GPUs the owner would broadcast them.
A's rows stay resident (the rank's own shard).  The single-GPU sweep of the
whole problem runs too, and its bounds must equal the sharded ones bit for bit.
One JSON line per delta.

    python tools/cfg4_shard.py                       # config 4, delta 1e-6, grid [1e-12, 1e-2]
    python tools/cfg4_shard.py --tau-lo 1e-16        # grid extended so delta = 1e-6 skips
    python tools/cfg4_shard.py --config 5 --leaf 32  # config 5, one leaf size, all three deltas

At delta = 1e-6 no tau of [1e-12, 1e-2] meets the bound on config 4 (exact
fallback, tau = 0), so the grid can be extended downwards as for config 5
(tools/leaf_sweep.py uses [1e-14, 1e-2]).
"""
import argparse
import json
import time

import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2005_10680_b200 import _native as nat  # noqa: E402
from paper_2005_10680_b200.inputs import log_grid  # noqa: E402
from paper_2005_10680_b200.sharded import leaf_table, merge_tables  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4, choices=[4, 5])
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--leaf", type=int, default=64)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--panel-rows", type=int, default=None)
ap.add_argument("--task-budget", type=float, default=0,
                help="task-list bytes before the library row-chunks a product (0: auto)")
ap.add_argument("--tau-lo", type=float, default=None)
ap.add_argument("--deltas", default=None)
ap.add_argument("--all-ranks", action="store_true",
                help="run every rank's share in turn (tables built once): the projected "
                     "8-GPU time is the slowest rank")
args = ap.parse_args()
cfg5 = args.config == 5
N = args.n or (131072 if cfg5 else 262144)
L = args.leaf
NT = 128 if cfg5 else 64
tau_lo = args.tau_lo or (1e-14 if cfg5 else 1e-12)
deltas = [float(x) for x in (args.deltas or ("1e-8,1e-6,1e-4" if cfg5 else "1e-6")).split(",")]
# panels of ~24 GB of dense leaves: every panel GEMM launch pays a per-block
# accumulator reload, which weighs more the fewer products a block has per
# panel (config 5, L = 64, delta = 1e-4: 22.7 TFLOP/s with 128-row panels,
# 28.4 with 512-row panels)
panel_rows = args.panel_rows or max(8, (24 << 30) // (N * L * 8))
rank, ranks = args.rank, args.ranks
ELL, DENS, SITE, SEED_A, SEED_B, DROP = 4.0, 0.1, 2005, 10680, 10681, 1e-10
level = ranks.bit_length() - 1
assert (1 << level) == ranks

ctx = nat.Context(0)
base = {"workload": f"cfg{args.config}-cluster3d-N{N}-L{L}-ell{ELL}", "rank": rank,
        "ranks": ranks, "n_taus": NT, "tau_grid": [1e-2, tau_lo], "panel_rows": panel_rows,
        "task_budget": args.task_budget or "auto"}
t0 = time.perf_counter()
sA = nat.synth_cluster_scale(ctx, N, ELL, DENS, SITE, SEED_A)
sB = nat.synth_cluster_scale(ctx, N, ELL, DENS, SITE, SEED_B)
nb = N // L
rows_per = nb // ranks
tabA, tabB, A_local = [], [], None
run_ranks = list(range(ranks)) if args.all_ranks else [rank]
for g in range(ranks):
    lo, hi = g * rows_per, (g + 1) * rows_per
    Ag = nat.synth_cluster_device_rows_scaled(ctx, N, L, ELL, DENS, SITE, SEED_A, DROP, sA, lo, hi)
    tabA.append(leaf_table(Ag))
    if g == run_ranks[0]:
        A_local = Ag
    else:
        Ag.free()
    Bg = nat.synth_cluster_device_rows_scaled(ctx, N, L, ELL, DENS, SITE, SEED_B, DROP, sB, lo, hi)
    tabB.append(leaf_table(Bg))
    Bg.free()
ta, tb = merge_tables(tabA), merge_tables(tabB)
A_norms = nat.from_leaf_norms(ctx, N, L, *ta)
B_norms = nat.from_leaf_norms(ctx, N, L, *tb)
ctx.synchronize()
base["tables_s"] = round(time.perf_counter() - t0, 2)
base["leaves_A"], base["leaves_B"] = int(len(ta[0])), int(len(tb[0]))
base["leaves_A_rank"] = int(A_local.nnz_blocks)

taus = log_grid(NT, 1e-2, tau_lo)
nat.cse_shard(ctx, A_norms, B_norms, taus, level, rank)  # warm-up (kernel attributes, pool)
ctx.synchronize()
t1 = time.perf_counter()
mine = nat.cse_shard(ctx, A_norms, B_norms, taus, level, rank)
ctx.synchronize()
base["sweep_shard_ms"] = round(1e3 * (time.perf_counter() - t1), 3)
parts = np.stack([mine if g == rank else nat.cse_shard(ctx, A_norms, B_norms, taus, level, g)
                  for g in range(ranks)])
bounds = nat.cse_finish(level, nat.top_norms(A_norms, level), nat.top_norms(B_norms, level), parts)
ctx.synchronize()
t2 = time.perf_counter()
full = nat.cse(ctx, A_norms, B_norms, taus)
ctx.synchronize()
base["sweep_one_gpu_ms"] = round(1e3 * (time.perf_counter() - t2), 3)
base["sharded_bounds_equal_one_gpu"] = bool(np.array_equal(full.view(np.uint64),
                                                           bounds.view(np.uint64)))
base["bound_at_smallest_tau"] = float(bounds[-1])


def cfetch(r0, r1, dst, count, stream):
    # spg_spamm_panels' callback: the owner's broadcast on 8 GPUs; here the
    # panel is generated in place and its leaves gathered into dst on `stream`
    try:
        Bp = nat.synth_cluster_device_rows_scaled(ctx, N, L, ELL, DENS, SITE, SEED_B, DROP, sB, r0, r1)
    except MemoryError:
        free, total = torch.cuda.mem_get_info()
        print(f"[cfg4_shard] panel [{r0}, {r1}) generation out of memory: device free "
              f"{free / 2**30:.1f} of {total / 2**30:.1f} GiB", file=sys.stderr, flush=True)
        raise
    ctx.synchronize()
    nat.gather_rows(Bp, r0, r1, dst, count, stream)
    torch.cuda.ExternalStream(stream).synchronize()  # before Bp's memory is reused
    Bp.free()


if args.task_budget:
    nat.set_task_budget(ctx, args.task_budget)
for rk in run_ranks:
    if A_local is None:
        A_local = nat.synth_cluster_device_rows_scaled(ctx, N, L, ELL, DENS, SITE, SEED_A, DROP, sA,
                                                       rk * rows_per, (rk + 1) * rows_per)
    if rk != rank:
        ctx.synchronize()
        t1 = time.perf_counter()
        nat.cse_shard(ctx, A_norms, B_norms, taus, level, rk)
        ctx.synchronize()
        base["sweep_shard_ms"] = round(1e3 * (time.perf_counter() - t1), 3)
    base["rank"] = rk
    base["leaves_A_rank"] = int(A_local.nnz_blocks)
    for delta in deltas:
        out = dict(base)
        out["delta"] = delta
        tau, k = nat.select_tolerance(bounds, taus, delta)
        out["tau"], out["tau_index"] = tau, k
        out["bound"] = float(bounds[k]) if k >= 0 else 0.0
        tot = {"candidates": 0, "survivors": 0, "flops": 0.0, "ms_gemm": 0.0, "ms_tasklist": 0.0,
               "ms_finalize": 0.0, "output_blocks": 0}
        t3 = time.perf_counter()
        # one C-ABI call: the library sizes the task-list row chunks itself
        # (spg_context_set_task_budget; ~6e9 products per rank do not fit one)
        C, st = nat.spamm_panels(ctx, A_local, B_norms, tau, cfetch, level, rk, panel_rows,
                                 rows_per, a_norms=A_norms)
        for key in tot:
            tot[key] += st[key]
        C.free()
        ctx.synchronize()
        out["product_wall_s"] = round(time.perf_counter() - t3, 2)
        out.update({k2: (round(v, 1) if isinstance(v, float) else v) for k2, v in tot.items()})
        out["skipped_fraction"] = round(1 - tot["survivors"] / max(tot["candidates"], 1), 4)
        # ms_gemm: the panel GEMM launches' kernel time; the wall time also holds
        # generating the B panels on the device (the owners' broadcasts on 8 GPUs)
        out["gemm_tflops"] = (round(tot["flops"] / tot["ms_gemm"] / 1e9, 2) if tot["ms_gemm"]
                              else 0.0)
        out["wall_tflops_incl_panel_generation"] = round(
            tot["flops"] / out["product_wall_s"] / 1e12, 2)
        out["sweep_shard_eff_gbs"] = round(
            12 * tot["candidates"] / (out["sweep_shard_ms"] / 1e3) / 1e9, 1)
        print(json.dumps(out), flush=True)
    A_local.free()
    A_local = None
