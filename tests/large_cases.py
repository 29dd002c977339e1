"""BASELINE configs 3-5 at full size: the GPU side of the reference pins.

Shared by tests/golden/make_large_pins.py (runs the GPU side AND the reference
on the box, writes tests/golden/large/<case>.{json,npz}) and
tests/test_gpu_pins.py (re-runs the GPU side and checks it against those
fixtures).  SURVEY.md 8c(i)-(iii):
  (i)   the reference's own cse / select_tolerance (error_control.cpp:160-172)
        and spamm_node decisions (multiply.cpp:70-92) on norm-only trees built
        from the leaf-norm tables the GPUs computed (block_norm, checked
        bitwise on config 2 in full) -> bounds bitwise, tau, survivor count and
        the survivor-set digest (spg_survivor_digest / ref_survivor_digest);
  (ii)  sampled blocks C~(i, j) by the reference's spamm_multiply on A
        restricted to row i and B to column j (the same leaf decisions and the
        same k order as the full product) vs the GPU's rows of C~, 1e-12;
  (iii) the realized error of the sampled rows against the GPU's tau = 0
        product of the same rows, < delta and <= the bound.
The GPU side runs the 8-GPU sharding's machinery on one GPU: per-shard
device generation of the row panels, all-gathered (here: concatenated)
leaf-norm tables -> global norm-only matrices, spg_cse_shard x 8 +
spg_cse_finish (== the one-GPU sweep, bitwise), the task list by row
sub-shards, and row plans fed by B panels (spg_plan_*).
"""
from __future__ import annotations

import hashlib
import math

import numpy as np

ELL, DENS, SITE, SEED_A, SEED_B, DROP = 4.0, 0.1, 2005, 10680, 10681, 1e-10

# name -> (N, L, n_taus, tau_lo, deltas, sample delta index or None)
CASES = {
    # a small case of the same form (pipeline check; depth 8)
    "mini": (16384, 64, 64, 1e-14, [1e-6], 0),
    # config 4 as BASELINE.json states it (64 tau over the config-1 range):
    # no tau meets delta = 1e-6 -> tau = 0, the exact product
    "cfg4": (262144, 64, 64, 1e-12, [1e-6], None),
    # config 4 with the grid extended to 1e-16 so that delta = 1e-6 skips
    "cfg4x": (262144, 64, 64, 1e-16, [1e-6], 0),
    "cfg5-L128": (131072, 128, 128, 1e-14, [1e-8, 1e-6, 1e-4], 1),
    "cfg5-L64": (131072, 64, 128, 1e-14, [1e-8, 1e-6, 1e-4], 1),
    "cfg5-L32": (131072, 32, 128, 1e-14, [1e-8, 1e-6, 1e-4], 1),
}
RANKS = 8


def taus_of(case):
    from paper_2005_10680_b200.inputs import log_grid
    n, L, nt, lo, _, _ = CASES[case]
    return log_grid(nt, 1e-2, lo)


def table_digest(t) -> str:
    h = hashlib.sha256()
    for x in t:
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


def sample_blocks(nb: int):
    """Two spread rows, two columns each (the diagonal block and a far one)."""
    rows = [nb // 5, (3 * nb) // 4]
    return [(i, j) for i in rows for j in (i, (i + nb // 2 + 7) % nb)]


class GpuCase:
    """Everything the 8-rank run computes for one case, on one GPU."""

    def __init__(self, ctx, case):
        from paper_2005_10680_b200 import _native as nat
        from paper_2005_10680_b200.sharded import leaf_table, merge_tables
        self.nat, self.ctx, self.case = nat, ctx, case
        self.n, self.L, self.n_taus, _, self.deltas, self.sample_at = CASES[case]
        self.nb = self.n // self.L
        self.depth = int(math.log2(self.nb))
        self.sA = nat.synth_cluster_scale(ctx, self.n, ELL, DENS, SITE, SEED_A)
        self.sB = nat.synth_cluster_scale(ctx, self.n, ELL, DENS, SITE, SEED_B)
        per = self.nb // RANKS
        ta, tb = [], []
        for g in range(RANKS):  # each rank's rows, generated and normed on "its" GPU
            for seed, s, out in ((SEED_A, self.sA, ta), (SEED_B, self.sB, tb)):
                M = self.rows(seed, s, g * per, (g + 1) * per)
                out.append(leaf_table(M))
                M.free()
        self.ta, self.tb = merge_tables(ta), merge_tables(tb)
        self.A_norms = nat.from_leaf_norms(ctx, self.n, self.L, *self.ta)
        self.B_norms = nat.from_leaf_norms(ctx, self.n, self.L, *self.tb)
        self.taus = taus_of(case)

    def rows(self, seed, scale, r0, r1):
        return self.nat.synth_cluster_device_rows_scaled(self.ctx, self.n, self.L, ELL, DENS, SITE,
                                                         seed, DROP, scale, r0, r1)

    def candidates(self) -> int:
        colA = np.bincount(self.ta[1], minlength=self.nb).astype(np.int64)
        rowB = np.bincount(self.tb[0], minlength=self.nb).astype(np.int64)
        return int(colA @ rowB)

    def bounds(self):
        """(one-GPU sweep, sharded sweep) of the whole problem."""
        nat = self.nat
        one = nat.cse(self.ctx, self.A_norms, self.B_norms, self.taus)
        level = RANKS.bit_length() - 1
        parts = np.stack([nat.cse_shard(self.ctx, self.A_norms, self.B_norms, self.taus, level, g)
                          for g in range(RANKS)])
        sharded = nat.cse_finish(level, nat.top_norms(self.A_norms, level),
                                 nat.top_norms(self.B_norms, level), parts)
        return one, sharded

    def survivor_digest(self, tau):
        """(count, digest) summed over row sub-shards sized for the task list."""
        cand = self.candidates()
        level = min(self.depth, max(RANKS.bit_length() - 1,
                                    math.ceil(math.log2(max(cand / 4e8, 1)))))
        count, dig = 0, 0
        for s in range(1 << level):
            c, d = self.nat.survivor_digest(self.ctx, self.A_norms, self.B_norms, tau, level, s)
            count += c
            dig = (dig + d) & 0xFFFFFFFFFFFFFFFF
        return count, dig, level

    def product_row(self, i, tau):
        """Row i of C~ through a one-row plan (the shard at the leaf level) with
        B arriving in block-row panels generated on the device, where the
        owning GPUs would broadcast them.  -> {j: block (L x L, column-major)}"""
        from paper_2005_10680_b200.sharded import panel_schedule, run_panels
        nat = self.nat
        A_i = self.rows(SEED_A, self.sA, i, i + 1)
        plan = nat.Plan(self.ctx, A_i, self.B_norms, tau, self.depth, i, a_norms=self.A_norms)
        panel_rows = max(8, (16 << 30) // (self.n * self.L * 8))

        def fetch(r0, r1, owner, buf, count, stream):
            Bp = self.rows(SEED_B, self.sB, r0, r1)
            self.ctx.synchronize()
            nat.gather_rows(Bp, r0, r1, buf.data_ptr(), count, stream.cuda_stream)
            stream.synchronize()
            Bp.free()

        run_panels(self.ctx, plan, panel_schedule(self.n, self.L, 0, panel_rows), fetch, self.L)
        C, st = plan.finish()
        plan.free()
        r, c, p, _ = C.download()
        assert np.all(r == i)
        A_i.free()
        return {int(j): p[t] for t, j in enumerate(c)}, st

    def reference_operands(self, i, j):
        """Host copies (device generator bits) of A's row i and B's column j
        (B is symmetric: column j = transposed leaves of row j)."""
        A_i = self.rows(SEED_A, self.sA, i, i + 1)
        ra, ca, pa, _ = A_i.download()
        A_i.free()
        B_j = self.rows(SEED_B, self.sB, j, j + 1)
        rb, cb, pb, _ = B_j.download()
        B_j.free()
        L = self.L
        pbT = pb.reshape(-1, L, L).transpose(0, 2, 1).reshape(-1, L * L)
        return (ra, ca, pa), (cb, rb, np.ascontiguousarray(pbT))
