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


# --------------------------------------------------------------------------
# Operands distributed by block row: rank g holds
# only its shard's block rows of A and of B.  Every rank all-gathers the two
# leaf-norm tables (block_norm values computed by the owning GPU, so the
# global norm pyramids are bit-exact), runs the sweep on its shard, and then
# builds its rows of C~ from B panels broadcast by their owners -- ascending
# block rows, double-buffered against the panel GEMMs (spg_plan_*).  C~ is
# bitwise the single-GPU product's rows.

def leaf_table(M):
    """(rows, cols, norms) of M's non-null leaves, sorted by (row, col)."""
    import numpy as np
    r, c, _, nrm = M.download(payload=False)
    order = np.lexsort((c, r))
    return r[order], c[order], nrm[order]


def merge_tables(tables):
    """Union of per-rank leaf tables (disjoint block rows) in (row, col) order."""
    import numpy as np
    r = np.concatenate([t[0] for t in tables]).astype(np.int32)
    c = np.concatenate([t[1] for t in tables]).astype(np.int32)
    n = np.concatenate([t[2] for t in tables]).astype(np.float64)
    order = np.lexsort((c, r))
    r, c, n = r[order], c[order], n[order]
    if len(r) > 1:
        dup = (r[1:] == r[:-1]) & (c[1:] == c[:-1])
        if dup.any():
            raise ValueError("leaf tables overlap: shards must own disjoint block rows")
    return r, c, n


def panel_schedule(n: int, leaf: int, level: int, panel_rows: int):
    """[(r0, r1, owner)] tiling block rows [0, ceil(n/L)) in ascending order;
    a panel never crosses a shard boundary (owner = shard of its rows)."""
    if panel_rows < 1:
        raise ValueError("panel_rows must be positive")
    nb = -(-n // leaf)
    depth = 0
    while (leaf << depth) < n:
        depth += 1
    rows_per = (1 << depth) >> level
    out = []
    for g in range(1 << level):
        lo, hi = g * rows_per, min((g + 1) * rows_per, nb)
        for r in range(lo, hi, panel_rows):
            out.append((r, min(r + panel_rows, hi), g))
    return out


def run_panels(ctx, plan, schedule, fetch, leaf: int):
    """Feed `plan` the B panels of `schedule`, two in flight: fetch(r0, r1,
    owner, buf, count, stream) fills buf (count leaves) on `stream`; the
    panel GEMM waits for that stream, and the buffer's next fill waits for
    the GEMM (stream-ordered, no host synchronisation)."""
    import torch
    LL = leaf * leaf
    counts = [plan.panel_slots(r0, r1)[1] for r0, r1, _ in schedule]
    cap = max(counts, default=0)
    dev = torch.device("cuda", ctx.device)
    bufs = [torch.empty(max(cap * LL, 1), dtype=torch.float64, device=dev) for _ in range(2)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    live = [q for q, cnt in enumerate(counts) if cnt > 0]
    slot = {q: i % 2 for i, q in enumerate(live)}

    def issue(q):
        r0, r1, owner = schedule[q]
        i = slot[q]
        with torch.cuda.stream(streams[i]):
            fetch(r0, r1, owner, bufs[i], counts[q], streams[i])

    nxt = iter(live)
    pending = next(nxt, None)
    if pending is not None:
        issue(pending)
        pending = next(nxt, None)
    for q, (r0, r1, owner) in enumerate(schedule):
        if counts[q] == 0:
            plan.accumulate(r0, r1, None)
            continue
        if pending is not None:  # panel after this one goes in flight first
            issue(pending)
            pending = next(nxt, None)
        i = slot[q]
        plan.accumulate(r0, r1, bufs[i].data_ptr(), streams[i].cuda_stream)
    ctx.synchronize()
    return sum(counts) * LL * 8


def torch_fetch(comm_backend: str, rank: int, B_local, leaf: int):
    """fetch() for run_panels over torch.distributed: the owner gathers its
    rows of B into the buffer, then a broadcast from the owner (NCCL on the
    buffer's stream; gloo through host memory)."""
    import torch
    import torch.distributed as dist
    LL = leaf * leaf

    def fetch(r0, r1, owner, buf, count, stream):
        view = buf[: count * LL]
        if owner == rank:
            nat.gather_rows(B_local, r0, r1, buf.data_ptr(), count, stream.cuda_stream)
        if comm_backend not in ("nccl", "gloo"):  # one rank: the panel is local
            return
        if comm_backend == "nccl":
            dist.broadcast(view, src=owner)
        else:
            stream.synchronize()
            host = view.cpu() if owner == rank else torch.empty(count * LL, dtype=torch.float64)
            dist.broadcast(host, src=owner)
            if owner != rank:
                view.copy_(host)
            stream.synchronize()
    return fetch


class DistributedOperands:
    """A and B distributed by block row: rank `rank` of 2^level holds its
    shard's rows (A_local, B_local).  Construction all-gathers the leaf-norm
    tables into global norm-only matrices (the cached norms, as the resident
    matrices cache theirs); allgather(list_of_arrays) -> per-rank lists.

    transport "broadcast": B panels are broadcast by their owners (run_panels
    with a fetch()); "peer": every rank maps the other ranks' B payloads into
    its address space (CUDA IPC; over NVLink between GPUs) and ONE GEMM reads
    each B leaf in place (spg_plan_run_table) -- the all-gather fused into the
    product, no staging buffers.  Ranks must call close() together."""

    def __init__(self, ctx, A_local, B_local, level: int, rank: int, allgather,
                 transport: str = "broadcast"):
        import numpy as np
        if transport not in ("broadcast", "peer"):
            raise ValueError("transport must be 'broadcast' or 'peer'")
        self.ctx, self.A, self.B = ctx, A_local, B_local
        self.level, self.rank = level, rank
        self.allgather = allgather
        self.transport = transport
        self.n, self.L = A_local.dimension, A_local.leaf_size
        self.opened = []
        ta = merge_tables(allgather(list(leaf_table(A_local))))
        if transport == "peer":
            # B table with (owner, payload slot) per leaf, merged in (row, col) order
            r, c, _, nrm = B_local.download(payload=False)
            sl = B_local.payload_slots() if len(r) else np.empty(0, np.int32)
            handle = nat.ipc_export(B_local) if len(r) else bytes(64)
            parts = allgather([r, c, nrm, sl, np.frombuffer(handle, np.uint8)])
            owner = np.concatenate([np.full(len(p[0]), k, np.int32) for k, p in enumerate(parts)])
            rows = np.concatenate([p[0] for p in parts]).astype(np.int32)
            cols = np.concatenate([p[1] for p in parts]).astype(np.int32)
            norms = np.concatenate([p[2] for p in parts]).astype(np.float64)
            local = np.concatenate([p[3] for p in parts]).astype(np.int32)
            order = np.lexsort((cols, rows))
            tb = (rows[order], cols[order], norms[order])
            self.slot_owner, self.slot_local = owner[order], local[order]
            self.bases = []
            for k, p in enumerate(parts):
                if k == rank:
                    self.bases.append(B_local.payload_ptr() if len(r) else 0)
                elif len(p[0]):
                    ptr = nat.ipc_open(ctx, p[4].tobytes())
                    self.opened.append(ptr)
                    self.bases.append(ptr)
                else:
                    self.bases.append(0)
            self.A_norms = nat.from_leaf_norms(ctx, self.n, self.L, *ta)
            self.B_norms = nat.from_leaf_norms(ctx, self.n, self.L, *tb)
            return
        tb = ta if B_local is A_local else merge_tables(allgather(list(leaf_table(B_local))))
        self.A_norms = nat.from_leaf_norms(ctx, self.n, self.L, *ta)
        self.B_norms = (self.A_norms if B_local is A_local
                        else nat.from_leaf_norms(ctx, self.n, self.L, *tb))

    def close(self, barrier=None):
        """Unmap the peers' payloads; with `barrier`, first wait until every
        rank is done reading this rank's B."""
        if barrier is not None:
            barrier()
        for ptr in self.opened:
            nat.ipc_close(self.ctx, ptr)
        self.opened = []

    def _panels(self, tau, fetch, panel_rows):
        """Broadcast transport: spg_spamm_panels with fetch(r0, r1, owner, buf,
        count, stream) adapted from the C callback (device pointer -> torch
        view, stream pointer -> torch stream).  The library row-chunks the
        rank's rows when the task list would exceed the context's task budget
        (spg_context_set_task_budget), each chunk receiving the panels again."""
        import torch
        LL = self.L * self.L
        owner_rows = (1 << nat_depth(self.n, self.L)) >> self.level
        dev = torch.device("cuda", self.ctx.device)
        moved = [0]

        def cfetch(r0, r1, dst, count, stream):
            owner = r0 // owner_rows
            buf = torch.as_tensor(nat.DevicePtr(dst, max(count, 1) * LL), device=dev)
            s = torch.cuda.ExternalStream(stream, device=dev)
            with torch.cuda.stream(s):
                fetch(r0, r1, owner, buf, count, s)
            moved[0] += count * LL * 8

        C, st = nat.spamm_panels(self.ctx, self.A, self.B_norms, tau, cfetch, self.level,
                                 self.rank, panel_rows, owner_rows, a_norms=self.A_norms)
        return C, st, moved[0]

    def controlled_product(self, delta: float, taus, fetch=None, panel_rows: int = 8,
                           row_chunks: int = 1):
        """This rank's rows of spamm_with_error_control(A, B, delta, taus).

        Broadcast transport: one spg_spamm_panels call; the library splits the
        rank's rows into task-list chunks by itself when the task list (~40 B
        per candidate) would not fit (config 4: ~6e9 products per rank), each
        chunk receiving B's panels again.  Peer transport: row_chunks = 2^c
        consecutive sub-shards, one task list and one table-addressed GEMM
        each (B read in place either way); returns the list of chunk matrices
        in row order when row_chunks > 1."""
        import numpy as np
        if not (delta > 0.0):
            raise ValueError("spamm_with_error_control: delta must be positive")
        c = max(0, int(row_chunks).bit_length() - 1)
        if row_chunks < 1 or (1 << c) != row_chunks:
            raise ValueError("row_chunks must be a power of two")
        taus = np.ascontiguousarray(taus, np.float64)
        nat.tolerance_grid_check(taus)
        level = self.level
        if level == 0:
            bounds = nat.cse(self.ctx, self.A_norms, self.B_norms, taus)
        else:
            partial = nat.cse_shard(self.ctx, self.A_norms, self.B_norms, taus, level, self.rank)
            parts = np.stack([p[0] for p in self.allgather([partial])])
            bounds = nat.cse_finish(level, nat.top_norms(self.A_norms, level),
                                    nat.top_norms(self.B_norms, level), parts)
        tau, k = nat.select_tolerance(bounds, taus, delta)
        if self.transport == "broadcast":
            # the whole panel loop in C (spg_spamm_panels): B panels from the
            # owners through fetch(), row chunks sized by the task budget
            C, st, moved = self._panels(tau, fetch, panel_rows)
            return C, {"tau": tau, "tau_index": k,
                       "bound": float(bounds[k]) if k >= 0 else 0.0, "spamm": st,
                       "panel_bytes": moved}, bounds
        pieces, stats = [], []
        moved = 0
        for sub in range(1 << c):
            plan = nat.Plan(self.ctx, self.A, self.B_norms, tau, level + c,
                            (self.rank << c) + sub, a_norms=self.A_norms)
            plan.run_table(self.bases, self.slot_owner, self.slot_local)
            C, st = plan.finish()
            plan.free()
            pieces.append(C)
            stats.append(st)
        st = dict(stats[0])
        for key in ("candidates", "survivors", "output_blocks", "flops", "ms_tasklist", "ms_gemm",
                    "ms_finalize"):
            st[key] = sum(x[key] for x in stats)
        mine = self.slot_owner == self.rank
        moved = int((~mine).sum()) * self.L * self.L * 8  # leaves read remotely (distinct)
        return (pieces[0] if c == 0 else pieces), \
            {"tau": tau, "tau_index": k, "bound": float(bounds[k]) if k >= 0 else 0.0,
             "spamm": st, "panel_bytes": moved}, bounds


def nat_depth(n: int, leaf: int) -> int:
    d = 0
    while (leaf << d) < n:
        d += 1
    return d


def controlled_product_distributed(ctx, A_local, B_local, delta: float, taus, level: int,
                                   rank: int, allgather, fetch, panel_rows: int = 8):
    """One-shot DistributedOperands(...).controlled_product(...)."""
    ops = DistributedOperands(ctx, A_local, B_local, level, rank, allgather)
    return ops.controlled_product(delta, taus, fetch, panel_rows)
