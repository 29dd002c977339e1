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
    p.add_argument("--cpu-rows", type=int, default=4,
                   help="block-rows of A in the bounded CPU sample")
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


def cpu_sample(kind, rows, cols, pay, w, taus, tau_star, sample_rows, threads):
    """The reference CPU implementation on a bounded slice of the workload:
    spamm_with_error_control's two phases -- cse(A_rows, A) and
    spamm_multiply(A_rows, A, tau*) -- for the first `sample_rows` block-rows of
    A (A_rows = A restricted to those rows, B = the full A), with tau* the
    full problem's selected tolerance.  Returns (tflops, seconds, flops)."""
    import oracle
    R = oracle.Oracle(kind)
    R.set_threads(threads)
    full = R.build(w.n, w.leaf, rows, cols, pay)
    sel = rows < sample_rows
    part = R.build(w.n, w.leaf, rows[sel], cols[sel], pay[sel])
    surv = len(R.survivors(part, full, tau_star))
    flops = 2.0 * w.leaf ** 3 * surv
    t0 = time.perf_counter()
    R.cse(part, full, taus)
    R.spamm(part, full, tau_star)
    dt = time.perf_counter() - t0
    return flops / dt / 1e12, dt, flops, surv


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

        def allgather(arrays):
            if dist.world == 1:
                return [arrays]
            out = [None] * dist.world
            dist.pg.all_gather_object(out, arrays)
            return out
        ops = DistributedOperands(ctx, A, A, level, dist.rank, allgather, args.transport)
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
    import oracle
    if host is None:
        rows, cols, pay, _ = A.download(payload=True)
    else:
        rows, cols, pay = host
    kind = "ref" if oracle.available("ref") else "port"
    threads = os.cpu_count() or 1
    tf, dt, flops, surv = cpu_sample(kind, rows, cols, pay, w, taus, tau_star, args.cpu_rows,
                                     threads)
    return {"value": tf, "unit": "TFLOP/s", "cores": threads if kind == "ref" else 1,
            "kind": "reference" if kind == "ref" else "port",
            "seconds": round(dt, 3),
            "sample": f"{w.name}: cse(A_rows, A) + spamm_multiply(A_rows, A, tau*={tau_star:.4g}) "
                      f"for block-rows [0,{args.cpu_rows}) of {w.n // w.leaf} "
                      f"({surv} leaf products, {flops / 1e9:.1f} GFLOP)"}


def run_reference(args, dist):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    unmodified reference sources) on the same workload/metric, all host
    threads, each step a bounded sample.  Rank 0 only."""
    if dist.rank != 0:
        return None
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import CONFIGS, log_grid
    import oracle
    w = CONFIGS[args.workload]
    # Input generation (not timed, not on the measured path): the same seeded
    # matrix bits the GPU arm uses, produced by the device generator.
    ctx = nat.Context(dist.device)
    A = make_matrix(nat, ctx, w)
    taus = log_grid(w.n_taus)
    rows, cols, pay, _ = A.download(payload=True)
    bounds = nat.cse(ctx, A, A, taus)
    tau_star, _ = nat.select_tolerance(bounds, taus, w.delta)
    del A
    ctx.close()
    kind = "ref" if oracle.available("ref") else "port"
    threads = os.cpu_count() or 1
    R = oracle.Oracle(kind)
    R.set_threads(threads)
    full = R.build(w.n, w.leaf, rows, cols, pay)
    sel = rows < args.cpu_rows
    part = R.build(w.n, w.leaf, rows[sel], cols[sel], pay[sel])
    surv = len(R.survivors(part, full, tau_star))
    flops = 2.0 * w.leaf ** 3 * surv
    for _ in range(min(args.warmup, 1)):
        R.cse(part, full, taus)
        R.spamm(part, full, tau_star)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        R.cse(part, full, taus)
        R.spamm(part, full, tau_star)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = flops * args.steps / total / 1e12
    sample = (f"{w.name}: cse(A_rows, A) + spamm_multiply(A_rows, A, tau*={tau_star:.4g}) for "
              f"block-rows [0,{args.cpu_rows}) of {w.n // w.leaf} ({surv} leaf products)")
    return {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded 3-D cluster decay matrix (DESIGN.md Inputs)",
        "config": {"workload": w.name, "n": w.n, "leaf": w.leaf, "delta": w.delta,
                   "n_taus": w.n_taus},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "TFLOP/s",
                         "cores": threads if kind == "ref" else 1,
                         "kind": "reference" if kind == "ref" else "port", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
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
