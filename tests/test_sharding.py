"""Row-sharded (multi-GPU) path, SURVEY.md 8e.

CPU (gloo, world_size 2): each rank computes its shards' level-s partial bound
vectors (oracle), the partials are all-gathered over torch.distributed, and
every rank runs the library's host-only spg_cse_finish -- the bounds must be
bit-identical to the single-process sweep on every rank.  GPU: the CUDA
shards reproduce spg_cse / spg_spamm exactly."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, bits_equal


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, level, out_dir):
    import sys
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = oracle.Oracle("port")
    n, L = 768, 16
    rows, cols, pay = nat.synth_chain_host(n, L, 12.0, 99, 1e-10)
    t = P.build(n, L, rows, cols, pay)
    taus = log_grid(32)
    shards = 2 ** level
    mine = [s for s in range(shards) if s % world == rank]
    local = {s: P.shard_partials(t, t, taus, level, s) for s in mine}
    # all-gather: every rank contributes a fixed-size slab per owned shard
    per_rank = shards // world
    slab = torch.from_numpy(np.stack([local[s] for s in mine]))
    gathered = [torch.empty_like(slab) for _ in range(world)]
    dist.all_gather(gathered, slab)
    partials = np.empty((shards, 4 ** level, len(taus)))
    for r in range(world):
        for i, s in enumerate([s for s in range(shards) if s % world == r]):
            partials[s] = gathered[r][i].numpy()
    top = np.concatenate([t.level_norms(l) for l in range(level)])
    bounds = nat.cse_finish(level, top, top, partials)
    np.save(os.path.join(out_dir, f"bounds_{level}_{rank}.npy"), bounds)
    # survivors of the row shards partition the full set (host logic)
    tau = float(taus[P.select_index(P.cse(t, t, taus), 1e-6)])
    surv = P.survivors(t, t, tau)
    nb_shard = (t.depth() and (2 ** t.depth()) // shards) or 1
    mine_rows = np.isin(surv[:, 0] // nb_shard, mine)
    np.save(os.path.join(out_dir, f"surv_{level}_{rank}.npy"), surv[mine_rows])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("level", [1, 2])
def test_gloo_two_ranks_bitwise_bounds(tmp_path, port, level):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), level, str(tmp_path)), nprocs=world, join=True)
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rows, cols, pay = nat.synth_chain_host(768, 16, 12.0, 99, 1e-10)
    t = port.build(768, 16, rows, cols, pay)
    taus = log_grid(32)
    full = port.cse(t, t, taus)
    for r in range(world):
        assert bits_equal(np.load(tmp_path / f"bounds_{level}_{r}.npy"), full)
    tau = float(taus[port.select_index(full, 1e-6)])
    surv = port.survivors(t, t, tau)
    parts = np.concatenate([np.load(tmp_path / f"surv_{level}_{r}.npy") for r in range(world)])
    assert len(parts) == len(surv)
    assert {tuple(x) for x in parts} == {tuple(x) for x in surv}


def test_finish_rejects_bad_shapes(built):
    from paper_2005_10680_b200 import _native as nat
    with pytest.raises(ValueError):
        nat.cse_finish(1, np.zeros(1), np.zeros(1), np.zeros((2, 3, 4)))
    with pytest.raises(ValueError):
        nat.cse_finish(0, np.zeros(1), np.zeros(1), np.zeros((1, 1, 4)))


@pytest.mark.gpu
@pytest.mark.parametrize("level", [1, 2, 3])
def test_gpu_shards_reproduce_single_gpu(ctx, level):
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rows, cols, pay = nat.synth_chain_host(4096, 64, 40.0, 12345, 1e-10)
    A = nat.upload(ctx, 4096, 64, rows, cols, pay)
    taus = log_grid(32)
    full = nat.cse(ctx, A, A, taus)
    parts = np.stack([nat.cse_shard(ctx, A, A, taus, level, s) for s in range(2 ** level)])
    top = nat.top_norms(A, level)
    assert bits_equal(nat.cse_finish(level, top, top, parts), full)
    tau, _ = nat.select_tolerance(full, taus, 1e-6)
    C, st = nat.spamm(ctx, A, A, tau)
    r, c, p, nrm = C.download()
    got = {}
    total = 0
    for s in range(2 ** level):
        Cs, sts = nat.spamm_shard(ctx, A, A, tau, level, s)
        total += sts["survivors"]
        rs, cs, ps, ns = Cs.download()
        nb = 64 // (2 ** level)
        assert np.all(rs // nb == s)
        for i in range(len(rs)):
            got[(rs[i], cs[i])] = (ps[i], ns[i])
    assert total == st["survivors"]
    assert sum(nat.spamm_shard(ctx, A, A, tau, level, s)[1]["candidates"]
               for s in range(2 ** level)) == st["candidates"]
    assert len(got) == len(r)
    for i in range(len(r)):
        gp, gn = got[(r[i], c[i])]
        assert bits_equal(gp, p[i]) and bits_equal(gn, nrm[i])


@pytest.mark.gpu
def test_sharded_controlled_product_matches_single_gpu(ctx):
    """The per-rank step bench.py runs under torchrun (gather emulated in-process:
    every shard's partial computed on this GPU)."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    from paper_2005_10680_b200.sharded import controlled_product_shard
    rows, cols, pay = nat.synth_chain_host(4096, 64, 40.0, 12345, 1e-10)
    A = nat.upload(ctx, 4096, 64, rows, cols, pay)
    taus = log_grid(32)
    C, st, bounds = nat.spamm_with_error_control(ctx, A, A, 1e-6, taus)
    level = 3
    gather = lambda _p: np.stack([nat.cse_shard(ctx, A, A, taus, level, s) for s in range(8)])
    surv = 0
    for s in range(8):
        Cs, sts, bs = controlled_product_shard(ctx, A, A, 1e-6, taus, level, s, gather)
        assert bits_equal(bs, bounds)
        assert sts["tau"] == st["tau"] and sts["tau_index"] == st["tau_index"]
        assert sts["bound"] == st["bound"]
        surv += sts["spamm"]["survivors"]
    assert surv == st["spamm"]["survivors"]
