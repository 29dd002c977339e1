"""Row-sharded error-controlled product across GPUs.

Rank r of 2^s ranks owns output block-rows [r nb/2^s, (r+1) nb/2^s):
  1. spg_cse_shard      -- level-s partial bound vectors of its row quadtree
  2. gather(partial)    -- all-gather of the 4^s x N_tau vectors (NCCL over
                           NVLink in bench.py; <= 128 KB per rank at s=3,
                           N_tau=64)
  3. spg_cse_finish     -- every rank combines the top s levels in reference
                           order: bounds and tau bit-identical to one GPU
  4. spg_spamm_shard    -- its block-rows of C~ (same per-block k order as
                           one GPU, so C~ bits do not depend on the GPU count)
"""
from __future__ import annotations

from . import _native as nat


def controlled_product_shard(ctx, A, B, delta: float, taus, level: int, shard: int, gather):
    """`gather(partial) -> array (2^level, 4^level, n_taus)` in shard order."""
    import numpy as np
    if not (delta > 0.0):
        raise ValueError("spamm_with_error_control: delta must be positive")
    taus = np.ascontiguousarray(taus, np.float64)
    nat.tolerance_grid_check(taus)
    partial = nat.cse_shard(ctx, A, B, taus, level, shard)
    parts = np.ascontiguousarray(gather(partial), np.float64)
    bounds = nat.cse_finish(level, nat.top_norms(A, level), nat.top_norms(B, level), parts)
    tau, k = nat.select_tolerance(bounds, taus, delta)
    C, st = nat.spamm_shard(ctx, A, B, tau, level, shard)
    return C, {"tau": tau, "tau_index": k, "bound": float(bounds[k]) if k >= 0 else 0.0,
               "spamm": st}, bounds
