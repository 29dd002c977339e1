"""Operands distributed by block row, B panels broadcast by their owners
(A and B too large for one GPU).

Rank g holds only its shard's block rows of A and B.  Bars: the global norm
pyramids rebuilt from the all-gathered leaf tables, the bounds, tau, and
every rank's rows of C~ are BITWISE those of the single-GPU computation on
the whole matrices.

* CPU: panel schedule and table merge (host logic).
* GPU, one process: every shard's plan fed from its owners' matrices through
  spg_matrix_gather_rows (the broadcast replaced by a direct read).
* GPU, one process: the one-GEMM leaf-table path (spg_plan_run_table) with B
  split over two owner allocations.
* GPU, two processes (gloo, host-side collectives; the ranks time-share the
  one GPU and never wait on each other's kernels): the full driver, with B
  panels broadcast by their owners or read in place from the other process's
  memory through CUDA IPC (transport "peer")."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, bits_equal


def test_panel_schedule_tiles_rows_by_owner(built):
    from paper_2005_10680_b200.sharded import panel_schedule
    for n, L, level, pr in [(1000, 16, 2, 3), (4096, 64, 3, 1), (4096, 64, 0, 100),
                            (777, 8, 1, 5)]:
        sch = panel_schedule(n, L, level, pr)
        nb = -(-n // L)
        depth = max(0, int(np.ceil(np.log2(nb)))) if nb > 1 else 0
        rows_per = (1 << depth) >> level
        assert sch[0][0] == 0 and sch[-1][1] == nb
        for (a0, a1, ga), (b0, b1, gb) in zip(sch, sch[1:]):
            assert a1 == b0 and ga <= gb
        for r0, r1, g in sch:
            assert 0 < r1 - r0 <= pr
            assert r0 // rows_per == g and (r1 - 1) // rows_per == g
    with pytest.raises(ValueError):
        panel_schedule(100, 10, 1, 0)


def test_merge_tables_orders_and_rejects_overlap(built):
    from paper_2005_10680_b200.sharded import merge_tables
    t0 = (np.array([0, 0, 1]), np.array([3, 1, 0]), np.array([1.0, 2.0, 3.0]))
    t1 = (np.array([2, 2]), np.array([1, 0]), np.array([4.0, 5.0]))
    r, c, n = merge_tables([t1, t0])
    assert list(r) == [0, 0, 1, 2, 2] and list(c) == [1, 3, 0, 0, 1]
    assert list(n) == [2.0, 1.0, 3.0, 5.0, 4.0]
    with pytest.raises(ValueError):
        merge_tables([t0, t0])


def _shard_case(ctx, nat, n, L, level):
    """Whole A, B (two seeds of the 3-D cluster) and their row shards."""
    A = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10)
    B = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10)
    nb = -(-n // L)
    depth = max(0, int(np.ceil(np.log2(nb)))) if nb > 1 else 0
    rows_per = (1 << depth) >> level
    As, Bs = [], []
    for g in range(1 << level):
        lo, hi = min(g * rows_per, nb), min((g + 1) * rows_per, nb)
        As.append(nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10, lo, hi))
        Bs.append(nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10, lo, hi))
    return A, B, As, Bs


@pytest.mark.gpu
@pytest.mark.parametrize("level,L,panel_rows", [(1, 64, 4), (2, 32, 3), (3, 64, 1)])
def test_plan_panels_from_owners_bitwise(ctx, level, L, panel_rows):
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    from paper_2005_10680_b200.sharded import leaf_table, merge_tables, panel_schedule, run_panels
    n = 2048
    A, B, As, Bs = _shard_case(ctx, nat, n, L, level)
    ta = merge_tables([leaf_table(x) for x in As])
    tb = merge_tables([leaf_table(x) for x in Bs])
    # the row generator + owners' block_norm reproduce the whole matrix's table
    for t, M in ((ta, A), (tb, B)):
        full = leaf_table(M)
        assert all(np.array_equal(x, y) for x, y in zip(t[:2], full[:2]))
        assert bits_equal(t[2], full[2])
    A_norms = nat.from_leaf_norms(ctx, n, L, *ta)
    B_norms = nat.from_leaf_norms(ctx, n, L, *tb)
    for lvl in range(A.info().depth + 1):
        assert bits_equal(A_norms.level_norms(lvl), A.level_norms(lvl))
        assert bits_equal(B_norms.level_norms(lvl), B.level_norms(lvl))
    taus = log_grid(32)
    full_bounds = nat.cse(ctx, A, B, taus)
    parts = np.stack([nat.cse_shard(ctx, A_norms, B_norms, taus, level, g)
                      for g in range(1 << level)])
    bounds = nat.cse_finish(level, nat.top_norms(A_norms, level), nat.top_norms(B_norms, level),
                            parts)
    assert bits_equal(bounds, full_bounds)
    tau, _ = nat.select_tolerance(bounds, taus, 1e-6)
    schedule = panel_schedule(n, L, level, panel_rows)

    def fetch(r0, r1, owner, buf, count, stream):
        nat.gather_rows(Bs[owner], r0, r1, buf.data_ptr(), count, stream.cuda_stream)

    C, st = nat.spamm(ctx, A, B, tau)
    r, c, p, nrm = C.download()
    got = {}
    surv = 0
    for g in range(1 << level):
        plan = nat.Plan(ctx, As[g], B_norms, tau, level, g, a_norms=A_norms)
        run_panels(ctx, plan, schedule, fetch, L)
        Cg, sg = plan.finish()
        ref, sref = nat.spamm_shard(ctx, A, B, tau, level, g)
        assert sg["survivors"] == sref["survivors"]
        rg, cg, pg, ng = Cg.download()
        r2, c2, p2, n2 = ref.download()
        assert np.array_equal(rg, r2) and np.array_equal(cg, c2)
        assert bits_equal(pg, p2) and bits_equal(ng, n2)
        surv += sg["survivors"]
        for i in range(len(rg)):
            got[(rg[i], cg[i])] = (pg[i], ng[i])
    assert surv == st["survivors"] and len(got) == len(r)
    for i in range(len(r)):
        assert bits_equal(got[(r[i], c[i])][0], p[i])


@pytest.mark.gpu
def test_plan_contract_errors(ctx):
    from paper_2005_10680_b200 import _native as nat
    n, L = 512, 32
    A, B, As, Bs = _shard_case(ctx, nat, n, L, 1)
    from paper_2005_10680_b200.sharded import leaf_table
    Bn = nat.from_leaf_norms(ctx, n, L, *leaf_table(B))
    with pytest.raises(ValueError):  # resident B is not a panel source
        nat.Plan(ctx, A, B, 0.0)
    plan = nat.Plan(ctx, A, Bn, 0.0)
    lo, cnt = plan.panel_slots(0, 4)
    assert lo == 0 and cnt > 0
    with pytest.raises(ValueError):  # must start at row 0
        plan.accumulate(4, 8, None)
    with pytest.raises(ValueError):  # leaves but no buffer
        plan.accumulate(0, 4, None)
    with pytest.raises(ValueError):  # rows not covered
        plan.finish()
    with pytest.raises(ValueError):  # unsorted leaf table
        r, c, nr = leaf_table(B)
        nat.from_leaf_norms(ctx, n, L, r[::-1], c[::-1], nr[::-1])
    r, c, nr = leaf_table(B)
    row0 = np.flatnonzero(r == r[0])
    assert len(row0) > 1
    with pytest.raises(ValueError):  # rows sorted, columns not (gather_rows pairs by order)
        sw = np.arange(len(r))
        sw[row0[0]], sw[row0[1]] = row0[1], row0[0]
        nat.from_leaf_norms(ctx, n, L, r[sw], c[sw], nr[sw])
    with pytest.raises(ValueError):  # duplicate leaf
        nat.from_leaf_norms(ctx, n, L, np.r_[r[:1], r], np.r_[c[:1], c], np.r_[nr[:1], nr])
    # a_norms listing a shard-row leaf the local A lacks: refused, no wild read
    An = nat.from_leaf_norms(ctx, n, L, *leaf_table(A))
    ra, ca, pa, _ = As[0].download()
    keep = np.ones(len(ra), bool)
    keep[len(ra) // 2] = False
    A_hole = nat.upload(ctx, n, L, ra[keep], ca[keep], pa[keep])
    with pytest.raises(ValueError, match="a_norms"):
        nat.Plan(ctx, A_hole, Bn, 0.0, 1, 0, a_norms=An)
    nat.Plan(ctx, As[0], Bn, 0.0, 1, 0, a_norms=An)  # the consistent shard is accepted


@pytest.mark.gpu
@pytest.mark.parametrize("L", [16, 32, 64, 128])
def test_plan_leaf_table_one_gemm_bitwise(ctx, L):
    """spg_plan_run_table: every product in one GEMM with B leaves read through
    a per-leaf address table (the NVLink peer path's kernel) == resident
    product, bitwise; B split over two owner allocations."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    n = 40 * L // 4 + 3
    A = nat.synth_cluster_device(ctx, n - n % 4, L, 3.0, 0.1, 2005, 1, 1e-10)
    n = A.dimension
    nb = -(-n // L)
    half = nb // 2
    Bs = [nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10, 0, half),
          nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10, half, nb)]
    B = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10)
    rows, cols, norms, owner, local = [], [], [], [], []
    for k, M in enumerate(Bs):
        r, c, _, nr = M.download(payload=False)
        rows.append(r); cols.append(c); norms.append(nr)
        owner.append(np.full(len(r), k, np.int32)); local.append(M.payload_slots())
    rows, cols, norms = (np.concatenate(x) for x in (rows, cols, norms))
    owner, local = np.concatenate(owner), np.concatenate(local)
    order = np.lexsort((cols, rows))
    Bn = nat.from_leaf_norms(ctx, n, L, rows[order], cols[order], norms[order])
    taus = log_grid(32)
    bounds = nat.cse(ctx, A, B, taus)
    assert bits_equal(nat.cse(ctx, A, Bn, taus), bounds)
    for tau in (nat.select_tolerance(bounds, taus, 1e-6)[0], 0.0):
        plan = nat.Plan(ctx, A, Bn, tau)
        plan.run_table([M.payload_ptr() for M in Bs], owner[order], local[order])
        C1, s1 = plan.finish()
        C0, s0 = nat.spamm(ctx, A, B, tau)
        r0, c0, p0, n0 = C0.download()
        r1, c1, p1, n1 = C1.download()
        assert np.array_equal(r0, r1) and np.array_equal(c0, c1)
        assert bits_equal(p0, p1) and bits_equal(n0, n1)
        assert s0["survivors"] == s1["survivors"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    from paper_2005_10680_b200.sharded import controlled_product_distributed, torch_fetch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = nat.Context(0)
    n, L, level = 2048, 64, 1
    nb = n // L
    lo, hi = rank * nb // world, (rank + 1) * nb // world
    A = nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10, lo, hi)
    B = nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10, lo, hi)

    def allgather(arrays):
        out = [None] * world
        dist.all_gather_object(out, arrays)
        return out

    C, st, bounds = controlled_product_distributed(
        ctx, A, B, 1e-6, log_grid(32), level, rank, allgather,
        torch_fetch("gloo", rank, B, L), panel_rows=3)
    r, c, p, nrm = C.download()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), r=r, c=c, p=p, n=nrm, bounds=bounds,
             tau=st["tau"], surv=st["spamm"]["survivors"])
    dist.barrier()
    dist.destroy_process_group()


def _peer_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    from paper_2005_10680_b200.sharded import DistributedOperands
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = nat.Context(0)
    n, L, level = 2048, 64, 1
    nb = n // L
    lo, hi = rank * nb // world, (rank + 1) * nb // world
    A = nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10, lo, hi)
    B = nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10, lo, hi)

    def allgather(arrays):
        out = [None] * world
        dist.all_gather_object(out, arrays)
        return out

    ops = DistributedOperands(ctx, A, B, level, rank, allgather, transport="peer")
    C, st, bounds = ops.controlled_product(1e-6, log_grid(32))
    r, c, p, nrm = C.download()
    ops.close(barrier=dist.barrier)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), r=r, c=c, p=p, n=nrm, bounds=bounds,
             tau=st["tau"], surv=st["spamm"]["survivors"])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["broadcast", "peer"])
def test_two_ranks_gloo_distributed_driver(ctx, tmp_path, transport):
    """Two processes on the one GPU, host-side (gloo) collectives; 'peer' maps
    the other process's B payload with CUDA IPC and reads it inside the GEMM."""
    import torch.multiprocessing as mp
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    worker = _peer_worker if transport == "peer" else _worker
    mp.spawn(worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    n, L = 2048, 64
    A = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10)
    B = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10)
    C, st, bounds = nat.spamm_with_error_control(ctx, A, B, 1e-6, log_grid(32))
    r, c, p, nrm = C.download()
    got = [np.load(tmp_path / f"rank{k}.npz") for k in range(2)]
    for g in got:
        assert bits_equal(g["bounds"], bounds) and float(g["tau"]) == st["tau"]
    assert sum(int(g["surv"]) for g in got) == st["spamm"]["survivors"]
    rr = np.concatenate([g["r"] for g in got])
    cc = np.concatenate([g["c"] for g in got])
    pp = np.concatenate([g["p"] for g in got])
    key = np.lexsort((cc, rr))
    key0 = np.lexsort((c, r))
    assert np.array_equal(rr[key], r[key0]) and np.array_equal(cc[key], c[key0])
    assert bits_equal(pp[key], p[key0])


@pytest.mark.gpu
@pytest.mark.parametrize("chunks", [1, 2, 8])
def test_peer_row_chunks_bitwise(ctx, chunks):
    """DistributedOperands(transport="peer") on one rank with the rows split in
    2^c task-list chunks: the chunk products, in row order, are the resident
    product's blocks, bitwise."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    from paper_2005_10680_b200.sharded import DistributedOperands
    n, L = 2048, 32
    A = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10)
    B = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10)
    ops = DistributedOperands(ctx, A, B, 0, 0, lambda arrays: [arrays], transport="peer")
    C, st, bounds = ops.controlled_product(1e-6, log_grid(32), row_chunks=chunks)
    ops.close()
    ref, sref, bref = nat.spamm_with_error_control(ctx, A, B, 1e-6, log_grid(32))
    assert bits_equal(bounds, bref) and st["tau"] == sref["tau"]
    assert st["spamm"]["survivors"] == sref["spamm"]["survivors"]
    pieces = C if isinstance(C, list) else [C]
    assert len(pieces) == chunks
    got = [p.download() for p in pieces]
    r = np.concatenate([g[0] for g in got])
    c = np.concatenate([g[1] for g in got])
    p = np.concatenate([g[2] for g in got])
    r0, c0, p0, _ = ref.download()
    k, k0 = np.lexsort((c, r)), np.lexsort((c0, r0))
    assert np.array_equal(r[k], r0[k0]) and np.array_equal(c[k], c0[k0])
    assert bits_equal(p[k], p0[k0])
    with pytest.raises(ValueError):
        ops.controlled_product(1e-6, log_grid(32), row_chunks=3)


@pytest.mark.gpu
@pytest.mark.parametrize("L", [32, 64, 128])
def test_broadcast_row_chunks_bitwise(ctx, L):
    """Broadcast transport through spg_spamm_panels with the task budget set
    so the library splits the rows into task-list chunks (4 where a chunk
    keeps whole tile rows; each chunk receives the B panels again): C~ is the
    resident product, bitwise."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    from paper_2005_10680_b200.sharded import DistributedOperands
    n = 2048
    A = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10)
    B = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10)
    ref, sref, _ = nat.spamm_with_error_control(ctx, A, B, 1e-6, log_grid(32))
    ops = DistributedOperands(ctx, A, B, 0, 0, lambda arrays: [arrays])

    def fetch(r0, r1, owner, buf, count, stream):
        nat.gather_rows(B, r0, r1, buf.data_ptr(), count, stream.cuda_stream)

    # the library charges 16 B per candidate for the dense task-list walk, 24 B
    # for the L = 32 super-block entries (spamm.cu chunk_bits): a budget of a
    # quarter -> 4 chunks
    per = 24 if L == 32 else 16
    nat.set_task_budget(ctx, -(-per * sref["spamm"]["candidates"] // 4))
    try:
        C, st, bounds = ops.controlled_product(1e-6, log_grid(32), fetch, panel_rows=4)
    finally:
        nat.set_task_budget(ctx, 0)
    assert st["spamm"]["survivors"] == sref["spamm"]["survivors"]
    r, c, p, nr = C.download()
    r0, c0, p0, n0 = ref.download()
    assert np.array_equal(r, r0) and np.array_equal(c, c0)
    assert bits_equal(p, p0) and bits_equal(nr, n0)
    # every chunk receives B once; at L = 128 (depth 4) a quarter of the rows is
    # thinner than a tile row, so the library falls back to the expansion's
    # charge there and splits further
    chunks, rest = divmod(st["panel_bytes"], int(ops.B_norms.nnz_blocks) * L * L * 8)
    assert rest == 0 and (chunks == 4 if L < 128 else chunks >= 2)


@pytest.mark.gpu
@pytest.mark.parametrize("L", [32, 64, 128])
def test_resident_product_row_chunks_bitwise(ctx, L):
    """spg_spamm / spg_spamm_with_error_control with a task budget too small
    for the task list: the library runs the product in row chunks (super
    blocks at L = 32, sub-products at L = 128 included) -- bitwise the same C,
    same stats."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    n = 2048
    A = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 1, 1e-10)
    B = nat.synth_cluster_device(ctx, n, L, 3.0, 0.1, 2005, 2, 1e-10)
    C0, s0, b0 = nat.spamm_with_error_control(ctx, A, B, 1e-6, log_grid(32))
    E0, _ = nat.multiply_exact(ctx, A, B)
    for budget in (40 * s0["spamm"]["candidates"] // 3, 4096):
        nat.set_task_budget(ctx, budget)
        try:
            C1, s1, b1 = nat.spamm_with_error_control(ctx, A, B, 1e-6, log_grid(32))
            E1, _ = nat.multiply_exact(ctx, A, B)
        finally:
            nat.set_task_budget(ctx, 0)
        assert bits_equal(b0, b1) and s0["tau"] == s1["tau"]
        for k in ("survivors", "output_blocks", "candidates"):
            assert s0["spamm"][k] == s1["spamm"][k]
        for X, Y in ((C0, C1), (E0, E1)):
            x, y = X.download(), Y.download()
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
            assert bits_equal(x[2], y[2]) and bits_equal(x[3], y[3])


@pytest.mark.gpu
def test_scaled_row_generator_is_bit_identical(ctx):
    """spg_synth_cluster_device_rows_scaled with spg_synth_cluster_scale's
    value reproduces spg_synth_cluster_device_rows bit for bit (the panel
    generator of tools/cfg4_shard.py)."""
    from paper_2005_10680_b200 import _native as nat
    n, L = 4096, 64
    scale = nat.synth_cluster_scale(ctx, n, 3.0, 0.1, 2005, 7)
    for lo, hi in ((0, 16), (16, 40), (40, 64)):
        a = nat.synth_cluster_device_rows(ctx, n, L, 3.0, 0.1, 2005, 7, 1e-10, lo, hi)
        b = nat.synth_cluster_device_rows_scaled(ctx, n, L, 3.0, 0.1, 2005, 7, 1e-10, scale, lo, hi)
        ra, ca, pa, na = a.download()
        rb, cb, pb, nb_ = b.download()
        assert np.array_equal(ra, rb) and np.array_equal(ca, cb)
        assert bits_equal(pa, pb) and bits_equal(na, nb_)
