#!/usr/bin/env python
"""Benchmark of the B200-native SpAMM hot path (BASELINE.json north_star).

One step = spamm_with_error_control(A, A, delta, taus) on HBM-resident
matrices (norm tables cached, as in the reference where norms are built at
construction, error_control.cpp:207-209): the CSE tau-sweep, tolerance
selection, task-list build, DMMA leaf GEMM and C finalisation.  Workload =
BASELINE.json configs[1] (3-D cluster, N=32768, L=64, delta=1e-5, 32 taus),
seeded synthetic input; A = 8.6 GB >> 126 MB L2, so no
L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  value = performed leaf-GEMM FP64 TFLOP/s of
the whole step (2 L^3 |S(tau)| / step time); e2e = the same metric through
the C ABI with pinned host buffers (upload + controlled product + download of
C each step); roofline = the DMMA leaf-GEMM kernel against the measured FP64
DMMA peak; cpu_baseline / --impl reference = the reference implementation
(oracle/_ref, compiled from the unmodified reference sources) on a bounded
sample of the same workload using all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "SpAMM FP64 TFLOP/s (performed leaf GEMMs, % peak) + τ-sweep ms; 1/2/4/8 GPU"
# FP64 DMMA.8x8x4 peak measured on this pool's B200 (tools/microbench/fp64_peak.cu,
# profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json carries no FP64 figure.
DMMA_PEAK_TFLOPS = 37.1
PEAK_SOURCE = "measured DMMA microbenchmark (profiles/r01_fp64_peak.txt); cuBLAS DGEMM 35.5"


def hbm_peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), \
            "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2"])
    p.add_argument("--operands", default="replicated", choices=["replicated", "distributed"],
                   help="distributed: each rank holds only its block rows of A and B; B panels "
                        "are broadcast by their owners (SURVEY 8e, configs 4/5)")
    p.add_argument("--panel-rows", type=int, default=32)
    p.add_argument("--transport", default="broadcast", choices=["peer", "broadcast"],
                   help="distributed operands: B panels broadcast by their owners (each leaf "
                        "crosses NVLink once per product) or read in place from the owners' "
                        "memory by one GEMM (CUDA IPC / NVLink; every L2 miss crosses the link)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-rows", type=int, default=1,
                   help="block rows per fork-join row group in the bounded CPU sample "
                        "(sample_rows)")
    return p.parse_args()


# ----------------------------------------------------------------- distributed
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = self.local_rank
        self.pg = None
        self.backend = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            # SPG_DIST_BACKEND=gloo: host-side collectives (lets a 1-GPU box run
            # the sharded path with ranks time-sharing the device; no rank's
            # kernels ever wait on another rank's)
            self.backend = os.environ.get("SPG_DIST_BACKEND") or (
                "nccl" if torch.cuda.is_available() else "gloo")
            if torch.cuda.is_available():
                self.device = self.local_rank % torch.cuda.device_count()
                torch.cuda.set_device(self.device)
            dist.init_process_group(self.backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def _dev(self):
        return "cuda" if self.backend == "nccl" else "cpu"

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self._dev())
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self._dev())
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def all_gather_np(self, arr):
        """NCCL all-gather of a small host array -> (world, *arr.shape)."""
        import torch
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(self._dev())
        if self.backend == "nccl":
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.pg.all_gather_into_tensor(out, t)
            return out.cpu().numpy()
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.pg.all_gather(parts, t)
        return torch.stack(parts).numpy()

    def all_gather_arrays(self, arrays):
        """Per-rank lists of numpy arrays (any dtype, per-rank lengths) ->
        [rank][i] on every rank, through device-buffer collectives (NCCL
        all_gather_into_tensor on the GPUs; gloo on CPU): the byte counts
        first, then one padded byte buffer per array.  Replaces pickling with
        all_gather_object (leaf-norm tables are ~200 MB per rank on config 4)."""
        if not self.pg:
            return [list(arrays)]
        import torch
        dev = self._dev()
        flat = [np.ascontiguousarray(a) for a in arrays]
        nbytes = torch.tensor([a.nbytes for a in flat], dtype=torch.int64, device=dev)
        sizes = self._gather(nbytes).cpu().numpy()  # (world, n_arrays)
        out = [[None] * len(flat) for _ in range(self.world)]
        for i, a in enumerate(flat):
            width = max(int(sizes[:, i].max()), 1)
            buf = torch.zeros(width, dtype=torch.uint8, device=dev)
            if a.nbytes:
                buf[:a.nbytes] = torch.from_numpy(a.reshape(-1).view(np.uint8)).to(dev)
            host = self._gather(buf).cpu().numpy()
            for r in range(self.world):
                v = host[r, :int(sizes[r, i])].view(a.dtype)
                out[r][i] = v.reshape((-1,) + a.shape[1:]).copy()
        return out

    def _gather(self, t):
        if self.backend == "nccl":
            out = t.new_empty((self.world,) + tuple(t.shape))
            self.pg.all_gather_into_tensor(out, t)
            return out
        parts = [t.new_empty(t.shape) for _ in range(self.world)]
        self.pg.all_gather(parts, t)
        import torch
        return torch.stack(parts)

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------- workload
def make_matrix(nat, ctx, w):
    if w.kind == "cluster":
        return nat.synth_cluster_device(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed,
                                        w.value_seed, w.drop)
    return nat.synth_chain_device(ctx, w.n, w.leaf, w.ell, w.value_seed, w.drop)


def spawn_levels(threads: int) -> int:
    """The reference's fork-join depth (execution.cpp:17-23): 4^levels tasks."""
    levels, cap = 0, 1
    while cap < threads and levels < 3:
        cap *= 4
        levels += 1
    return levels


def sample_rows(nb: int, threads: int, per_group: int = 1):
    """Block rows of the bounded CPU sample, spread so that every task the
    reference spawns has work: spawn_levels(threads) levels of 4-way spawning
    split C into 2^levels x 2^levels output quadrants (multiply.cpp:79-84,
    error_control.cpp:59-66), so `per_group` rows in each of the 2^levels row
    groups give every quadrant task a row (e.g. rows 0,128,256,384 of 512 for
    16 threads)."""
    groups = 1 << spawn_levels(threads)
    padded = 1 << max(0, (nb - 1).bit_length())
    per = max(padded // groups, 1)
    return sorted({g * per + o for g in range(groups) for o in range(per_group)
                   if o < per and g * per + o < nb})


class ReferenceSample:
    """The reference CPU implementation (oracle/_ref: the unmodified reference
    sources; `port` = the C restatement when the reference is not built) on
    the workload: its own cse over the FULL matrices picks tau* (the
    reference's tau-sweep, timed whole), and spamm_multiply runs on a bounded
    sample of block rows (A_rows * B, exactly those rows of C~: same leaf
    decisions, same per-block k order), timed and scaled by the survivor
    counts to the full product.  One step estimate =
        t_cse(full) + t_spamm(sample) * S(tau*) / S_sample(tau*)
    and value = 2 L^3 S(tau*) / step estimate.  Mirrors
    spamm_with_error_control's two timed phases (error_control.cpp:207-217)."""

    def __init__(self, w, rows, cols, pay, taus, threads, per_group=1):
        import oracle
        self.kind = "ref" if oracle.available("ref") else "port"
        self.threads = threads if self.kind == "ref" else 1
        R = oracle.Oracle(self.kind)
        R.set_threads(self.threads)
        self.R, self.w, self.taus = R, w, taus
        self.full = R.build(w.n, w.leaf, rows, cols, pay)
        nb = -(-w.n // w.leaf)
        self.rows = sample_rows(nb, self.threads, per_group)
        sel = np.isin(rows, self.rows)
        self.part = R.build(w.n, w.leaf, rows[sel], cols[sel], pay[sel])
        self.tau = None

    def step(self):
        """(t_cse, t_spamm_sample, bounds): one timed cse + sampled spamm."""
        t0 = time.perf_counter()
        bounds = self.R.cse(self.full, self.full, self.taus)
        t_cse = time.perf_counter() - t0
        k = next((i for i, b in enumerate(bounds) if b < self.w.delta), -1)
        tau = float(self.taus[k]) if k >= 0 else 0.0
        if self.tau is None:  # survivor counts at the reference's own tau*
            self.tau, self.k = tau, k
            self.s_total = int(self.R._surv(self.full.h, self.full.h, tau, None, 0))
            self.s_sample = int(self.R._surv(self.part.h, self.full.h, tau, None, 0))
        t0 = time.perf_counter()
        self.R.spamm(self.part, self.full, tau)
        t_spamm = time.perf_counter() - t0
        return t_cse, t_spamm, bounds

    def estimate(self, t_cse, t_spamm):
        scale = self.s_total / max(self.s_sample, 1)
        step_s = t_cse + t_spamm * scale
        flops = 2.0 * self.w.leaf ** 3 * self.s_total
        return flops / step_s / 1e12, step_s, flops

    def describe(self, t_cse, t_spamm):
        return (f"{self.w.name}: reference cse(A, A) over the full matrix (tau*={self.tau:.4g}, "
                f"k={self.k}) + spamm_multiply(A_rows, A, tau*) on block rows "
                f"{self.rows} of {-(-self.w.n // self.w.leaf)} ({self.s_sample} of "
                f"{self.s_total} leaf products), scaled by S/S_sample = "
                f"{self.s_total / max(self.s_sample, 1):.1f}; fork-join on {self.threads} "
                f"threads ({4 ** spawn_levels(self.threads)} tasks, each with work); "
                f"t_cse {t_cse:.3f} s, t_spamm(sample) {t_spamm:.3f} s")


def ncu_entry(key):
    """The ncu capture summarised for `key` in profiles/ncu_summary.json (or {})."""
    try:
        return json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get(key, {})
    except Exception:
        return {}


def traffic_from_profile():
    return ncu_entry("leaf_gemm_dmma").get("dram_bytes_per_launch")


def run_ours(args, dist):
    import torch
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import CONFIGS, log_grid

    from paper_2005_10680_b200.sharded import (DistributedOperands, controlled_product_shard,
                                               torch_fetch)

    w = CONFIGS[args.workload]
    torch.cuda.set_device(dist.device)
    ctx = nat.Context(dist.device)
    stream = torch.cuda.ExternalStream(ctx.stream)
    taus = log_grid(w.n_taus)
    # N = 2^s ranks: output block-row shards + NCCL all-gather of the level-s
    # CSE vectors; other N: independent replicas
    level = dist.world.bit_length() - 1
    distributed = args.operands == "distributed"
    if distributed and 2 ** level != dist.world:
        raise SystemExit("--operands distributed needs a power-of-two GPU count")
    sharded = dist.world > 1 and 2 ** level == dist.world and not distributed
    split = sharded or distributed  # per-rank stats summed over ranks
    if distributed:
        nb = -(-w.n // w.leaf)
        rows_per = (1 << max(0, (nb - 1).bit_length())) >> level
        lo, hi = min(dist.rank * rows_per, nb), min((dist.rank + 1) * rows_per, nb)
        if w.kind == "cluster":
            A = nat.synth_cluster_device_rows(ctx, w.n, w.leaf, w.ell, w.density, w.site_seed,
                                              w.value_seed, w.drop, lo, hi)
        else:
            A = nat.synth_chain_device_rows(ctx, w.n, w.leaf, w.ell, w.value_seed, w.drop, lo, hi)

        ops = DistributedOperands(ctx, A, A, level, dist.rank, dist.all_gather_arrays,
                                  args.transport)
        fetch = torch_fetch(dist.backend or "none", dist.rank, A, w.leaf)
    else:
        A = make_matrix(nat, ctx, w)

    def step():
        if distributed:
            t0 = time.perf_counter()
            C, st, b = ops.controlled_product(w.delta, taus, fetch, args.panel_rows)
            st["ms_cse"] = None
            st["ms_step_host"] = 1e3 * (time.perf_counter() - t0)
            return C, st, b
        if not sharded:
            return nat.spamm_with_error_control(ctx, A, A, w.delta, taus)
        t0 = time.perf_counter()
        C, st, b = controlled_product_shard(ctx, A, A, w.delta, taus, level, dist.rank,
                                            dist.all_gather_np)
        st["ms_cse"] = None
        st["ms_step_host"] = 1e3 * (time.perf_counter() - t0)
        return C, st, b

    for _ in range(args.warmup):
        C, st, _ = step()
        del C
    ctx.synchronize()
    dist.barrier()
    clocks = Clocks(dist.device)
    clocks.start()
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    ctx.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        C, st, bounds = step()
        stats.append(st)
        del C
    ev1.record(stream)
    torch.cuda.synchronize()
    ctx.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    ms_local = ev0.elapsed_time(ev1)
    ms = dist.max(ms_local)
    flops_local = sum(s["spamm"]["flops"] for s in stats)
    flops = dist.sum(flops_local)
    value = flops / (ms / 1e3) / 1e12
    st = stats[-1]
    sp = st["spamm"]
    gemm_ms = sum(s["spamm"]["ms_gemm"] for s in stats) / len(stats)
    if split:  # sweep = step minus the product phases (host-measured)
        cse_ms = sum(s["ms_step_host"] - s["spamm"]["ms_tasklist"] - s["spamm"]["ms_gemm"] -
                     s["spamm"]["ms_finalize"] for s in stats) / len(stats)
        cse_ms = dist.max(cse_ms)
    else:
        cse_ms = sum(s["ms_cse"] for s in stats) / len(stats)
    achieved = sp["flops"] / (max(gemm_ms, 1e-6) / 1e3) / 1e12
    A_bytes = float(A.nnz_blocks) * w.leaf * w.leaf * 8
    hbm, hbm_src = hbm_peak()
    cand = dist.sum(float(sp["candidates"])) if split else float(sp["candidates"])
    surv = dist.sum(float(sp["survivors"])) if split else float(sp["survivors"])
    sweep_bytes = 12.0 * cand
    sweep_gbs = sweep_bytes / (cse_ms / 1e3) / 1e9

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "strong" if split else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": (f"synthetic: seeded {'3-D cluster' if w.kind == 'cluster' else '1-D chain'} "
                 f"decay matrix (DESIGN.md Inputs), generated on device"),
        "config": {"workload": w.name, "n": w.n, "leaf": w.leaf, "ell": w.ell,
                   "density": w.density, "delta": w.delta, "n_taus": w.n_taus,
                   "tau_grid": "log-spaced [1e-12, 1e-2]", "drop": w.drop,
                   "parallelism": (f"distributed operands x{dist.world} (level {level}): "
                                   f"block-row shards of A and B, all-gathered norm tables, "
                                   + ("B leaves read in place from the owners' memory (CUDA IPC "
                                      "over NVLink) by one GEMM"
                                      if args.transport == "peer" else
                                      f"B panels of {args.panel_rows} block rows broadcast by "
                                      f"their owners ({dist.backend or 'local'})")
                                   if distributed else
                                   f"row-shards x{dist.world} (level {level}), "
                                   f"{dist.backend} all-gather of level-{level} CSE vectors"
                                   if sharded else
                                   f"replicas x{dist.world}" if dist.world > 1 else "single"),
                   "l2": (f"no flush: each step streams {A_bytes / 1e9:.1f} GB of leaves "
                          f"(>> 126 MB L2)" if A_bytes > 1e9 else
                          f"no flush: {A_bytes / 1e6:.0f} MB of leaves")},
        "pct_peak": round(100.0 * value / DMMA_PEAK_TFLOPS, 2),
        "sweep_ms": round(cse_ms, 4),
        # the reference's cse_seconds is host wall time (error_control.cpp:207-209): launch
        # overhead and the bound copy included
        "sweep_wall_ms": (round(1e3 * sum(s["cse_seconds"] for s in stats) / len(stats), 4)
                          if all(s.get("cse_seconds") for s in stats) else None),
        "tau": st["tau"], "tau_index": st["tau_index"], "bound": st["bound"],
        "candidates": int(cand), "survivors": int(surv),
        "skipped_fraction": round(1.0 - surv / max(cand, 1), 6),
        "phase_ms": {"cse": round(cse_ms, 3),
                     "tasklist": round(sum(s["spamm"]["ms_tasklist"] for s in stats) / len(stats), 3),
                     "gemm": round(gemm_ms, 3),
                     "finalize": round(sum(s["spamm"]["ms_finalize"] for s in stats) / len(stats), 3)},
        "roofline": {"kernel": "leaf_gemm_dmma<64>", "bound": "tensor",
                     "achieved": round(achieved, 3), "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": round(achieved / DMMA_PEAK_TFLOPS, 4),
                     "traffic": traffic_from_profile() if w.name.startswith("cfg2") else None,
                     "peak_source": PEAK_SOURCE,
                     "algorithmic": "2*L^3*|S(tau)| flops per launch (one launch per step)"},
        "sweep_roofline": {"kernel": "cse (tile + reduce)", "bound": "hbm",
                           "achieved": round(sweep_gbs, 2), "peak": hbm, "unit": "GB/s",
                           "frac": round(sweep_gbs / hbm, 5), "peak_source": hbm_src,
                           "algorithmic": "12 B per candidate leaf product (SURVEY 8d)",
                           # a tiled sweep is FP64-ALU bound -- the ncu capture
                           # (profiles/) of its tile kernel, for the other side of the picture
                           "ncu_tile_kernel": {k: ncu_entry("cse_tile_kernel").get(k) for k in (
                               "duration", "dram_bytes_per_launch", "fp64_pipe_active_pct",
                               "issue_active_pct")}},
        "gpu_launches": launches,
    }
    if clk:
        out["clocks"] = clk
    # K1 (leaf norms, block_norm) on A: the norm-table kernel's HBM roofline
    # (8 L^2 bytes read per leaf; best of 3 timed passes)
    norm_ms = min(A.norm_pass_ms() for _ in range(3))
    norm_bytes = float(A.nnz_blocks) * w.leaf * w.leaf * 8  # non-null leaves (conservative)
    out["norm_roofline"] = {"kernel": "leaf_norm_kernel (K1)", "bound": "hbm",
                            "achieved": round(norm_bytes / (norm_ms / 1e3) / 1e9, 1),
                            "peak": hbm, "unit": "GB/s",
                            "frac": round(norm_bytes / (norm_ms / 1e3) / 1e9 / hbm, 4),
                            "peak_source": hbm_src + " (a copy: read+write; this kernel only "
                                                     "reads)",
                            "frac_of_spec_7700": round(norm_bytes / (norm_ms / 1e3) / 1e9 / 7700.0,
                                                       4),
                            "ms": round(norm_ms, 3), "algorithmic": "8 L^2 B read per leaf"}
    # K4 (task list: skip tests of every level, survivors grouped by output
    # block with k ascending): 8 B key + 8 B slot pair per survivor
    tl_ms = out["phase_ms"]["tasklist"]
    if tl_ms > 0:
        tl_gbs = 16.0 * surv / (tl_ms / 1e3) / 1e9
        out["tasklist_roofline"] = {"kernel": "tl_valid + tl_tile<count> + scan + tl_tile<write> (K4)",
                                    "bound": "hbm", "achieved": round(tl_gbs, 1), "peak": hbm,
                                    "unit": "GB/s", "frac": round(tl_gbs / hbm, 4),
                                    "peak_source": hbm_src, "ms": tl_ms,
                                    "algorithmic": "8 B key + 8 B pair per surviving leaf product"}
    if distributed:
        out["panel_bytes_per_step"] = int(st["panel_bytes"])
    if not split:  # SURVEY 8a parity audit: how close the decisions are to ties
        ties, cands = nat.parity_audit(ctx, A, A, st["tau"], 4)
        out["parity_audit"] = {"near_ties_4ulp": ties, "candidates": cands,
                               "bound_margin": (w.delta - st["bound"]) / w.delta}

    host = None
    if not args.no_e2e and not split:
        out["e2e"], host = run_e2e(args, nat, ctx, stream, A, w, taus)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline and not distributed:
        out["cpu_baseline"] = run_cpu_baseline(args, nat, A, w, taus, st["tau"], host)
    if distributed:  # every rank done reading the others' B before any unmaps
        ops.close(barrier=dist.barrier if dist.world > 1 else None)
    return out


def run_e2e(args, nat, ctx, stream, A, w, taus):
    """The controlled product through the C ABI with pinned host buffers:
    every step uploads A (leaf coordinates + payload, H2D), runs
    spg_spamm_with_error_control, and downloads C (coordinates, payload,
    norms, D2H).  `value`: the steps pipelined -- step i+1's input is staged
    (spg_matrix_stage, upload stream) while step i's product runs and streams
    C out (copy stream), so both directions of the host link overlap the
    GEMM; every step's copies stay inside the timed region.  `serial`: the
    same steps one after the other (upload, then product)."""
    import ctypes as C
    import torch
    rows, cols, pay, _ = A.download(payload=True)
    n, LL = len(rows), w.leaf * w.leaf
    h_rows = torch.from_numpy(rows).pin_memory()
    h_cols = torch.from_numpy(cols).pin_memory()
    h_pay = torch.empty((n, LL), dtype=torch.float64).pin_memory()
    h_pay.numpy()[:] = pay
    cap = (w.n // w.leaf + 1) ** 2
    o_rows = torch.empty(cap, dtype=torch.int32).pin_memory()
    o_cols = torch.empty(cap, dtype=torch.int32).pin_memory()
    o_norm = torch.empty(cap, dtype=torch.float64).pin_memory()
    o_pay = torch.empty((cap, LL), dtype=torch.float64).pin_memory()
    lib = nat.lib()
    i32p, dp = C.POINTER(C.c_int32), C.POINTER(C.c_double)
    outs = (o_rows.numpy(), o_cols.numpy(), o_pay.numpy(), o_norm.numpy())

    def upload():
        h = C.c_void_p()
        nat._check(lib.spg_matrix_upload(ctx.handle, w.n, w.leaf, n,
                                         C.cast(h_rows.data_ptr(), i32p),
                                         C.cast(h_cols.data_ptr(), i32p),
                                         C.cast(h_pay.data_ptr(), dp), C.byref(h)))
        return nat.Matrix(ctx, h)

    def stage():
        return nat.Staged(ctx, w.n, w.leaf, n, h_rows.data_ptr(), h_cols.data_ptr(),
                          h_pay.data_ptr())

    def product(Ah):
        # the controlled product with C streamed into the pinned host buffers
        # while the GEMM runs (spg_spamm_with_error_control_to_host)
        out, st, _ = nat.spamm_with_error_control_to_host(ctx, Ah, Ah, w.delta, taus, out=outs)
        return st, len(out[0]) * (LL * 8 + 4 + 4 + 8)

    def timed(run_steps, k):
        ctx.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        flops, d2h = run_steps(k)
        ev1.record(stream)
        torch.cuda.synchronize()
        ctx.synchronize()
        return ev0.elapsed_time(ev1), flops, d2h

    def serial(k):
        flops, d2h = 0.0, 0
        for _ in range(k):
            st, d2h = product(upload())
            flops += st["spamm"]["flops"]
        return flops, d2h

    def pipelined(k):
        flops, d2h = 0.0, 0
        staged = stage()
        for i in range(k):
            Ah = staged.finish()
            staged = stage() if i + 1 < k else None
            st, d2h = product(Ah)
            del Ah
            flops += st["spamm"]["flops"]
        return flops, d2h

    warm = max(1, min(args.warmup, 2))
    serial(warm)
    ms_s, flops_s, _ = timed(serial, args.steps)
    pipelined(warm)
    ms, flops, d2h = timed(pipelined, args.steps)
    h2d = n * (LL * 8 + 4 + 4)
    return ({"value": round(flops / (ms / 1e3) / 1e12, 4), "unit": "TFLOP/s",
             "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
             "ms_per_step": round(ms / args.steps, 3),
             "path": "C ABI: spg_matrix_stage (pinned H2D of step i+1 on the upload stream) -> "
                     "spg_matrix_stage_finish -> spg_spamm_with_error_control_to_host (C "
                     "streamed D2H during the GEMM)",
             "serial": {"value": round(flops_s / (ms_s / 1e3) / 1e12, 4),
                        "ms_per_step": round(ms_s / args.steps, 3),
                        "path": "spg_matrix_upload then the product, no overlap"}},
            (rows, cols, pay))


def run_cpu_baseline(args, nat, A, w, taus, tau_star, host=None):
    """The reference beside the GPU arm (rank 0, N = 1): one ReferenceSample
    step on the same input bits (downloaded from the device)."""
    if host is None:
        rows, cols, pay, _ = A.download(payload=True)
    else:
        rows, cols, pay = host
    threads = os.cpu_count() or 1
    ref = ReferenceSample(w, rows, cols, pay, taus, threads, args.cpu_rows)
    t_cse, t_spamm, _ = ref.step()
    tf, step_s, _ = ref.estimate(t_cse, t_spamm)
    return {"value": tf, "unit": "TFLOP/s", "cores": ref.threads,
            "kind": "reference" if ref.kind == "ref" else "port",
            "step_seconds_estimate": round(step_s, 3), "seconds_cse": round(t_cse, 3),
            "seconds_spamm_sample": round(t_spamm, 3),
            "tau_matches_gpu": ref.tau == tau_star,
            "sample": ref.describe(t_cse, t_spamm)}


def run_reference(args, dist):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    unmodified reference sources) on the same workload / metric with all host
    threads: each step = its full cse + a sampled spamm_multiply scaled to the
    full product (ReferenceSample).  The input comes from the host generator in
    oracle/ (bitwise the product's host generator; the GPU arm's device
    generator differs from it only through exp()) -- the product library is
    never loaded.  Rank 0 only."""
    if dist.rank != 0:
        return None
    from paper_2005_10680_b200.inputs import CONFIGS, log_grid  # pure Python
    import oracle
    w = CONFIGS[args.workload]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    rows, cols, pay = oracle.host_inputs(w, threads)
    t_gen = time.perf_counter() - t0
    taus = log_grid(w.n_taus)
    ref = ReferenceSample(w, rows, cols, pay, taus, threads, args.cpu_rows)
    del rows, cols, pay
    for _ in range(min(args.warmup, 1)):
        ref.step()
    cses, spamms = [], []
    for _ in range(args.steps):
        t_cse, t_spamm, _ = ref.step()
        cses.append(t_cse)
        spamms.append(t_spamm)
    t_cse, t_spamm = sum(cses) / len(cses), sum(spamms) / len(spamms)
    value, step_s, flops = ref.estimate(t_cse, t_spamm)
    sample = ref.describe(t_cse, t_spamm)
    return {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # measured wall time of one timed step (full cse + the sampled spamm);
        # value is the full product's throughput estimated from it
        "ms_per_step": round(1e3 * (t_cse + t_spamm), 3),
        "full_step_estimate_ms": round(1e3 * step_s, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": (f"synthetic: seeded {'3-D cluster' if w.kind == 'cluster' else '1-D chain'} "
                 f"decay matrix (DESIGN.md Inputs), host generator (oracle/libinputs.so, "
                 f"{t_gen:.1f} s)"),
        "config": {"workload": w.name, "n": w.n, "leaf": w.leaf, "ell": w.ell,
                   "density": w.density, "delta": w.delta, "n_taus": w.n_taus,
                   "tau_grid": "log-spaced [1e-12, 1e-2]", "drop": w.drop},
        "impl": "reference",
        "tau": ref.tau, "tau_index": ref.k, "survivors": ref.s_total,
        "sweep_ms": round(1e3 * t_cse, 3),
        "phase_s": {"cse": round(t_cse, 3), "spamm_sample": round(t_spamm, 3),
                    "spamm_full_estimate": round(step_s - t_cse, 3)},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": ref.threads,
                         "kind": "reference" if ref.kind == "ref" else "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def launch_ranks(n: int) -> int:
    """`--gpus N` without a torch.distributed launcher: start the N ranks
    ourselves, one process per GPU, exactly as the driver's torchrun command
    would (127.0.0.1 rendezvous), and return the launcher's exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator set-up (transport, NVLS) on stderr
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    dist = Dist()
    try:
        if args.impl == "reference":
            out = run_reference(args, dist)
        else:
            out = run_ours(args, dist)
        if dist.rank == 0 and out is not None:
            print(json.dumps(out), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
