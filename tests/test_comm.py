"""Multi-GPU inside the C ABI and the C++ drop-in (the
reference's fork-join over host threads, execution.cpp:11-23).

* CPU: the drop-in's multi-rank test program compiles against the reference
  API plus include/spamm/distributed.hpp.
* GPU, one process: an NCCL communicator (dlopen'd libnccl) of one rank; the
  sharded entry points equal the plain ones bitwise.
* GPU, two processes on the one GPU (host all-gather over gloo; ranks never
  wait on each other's kernels): spg_spamm_with_error_control_sharded with and
  without the C gather, spg_cse_sharded, spg_spamm_sharded -- bounds, tau and
  C~ bitwise the single-GPU results; each rank's rows partition C~.
* GPU, the drop-in: tests/cpp/test_multi.cpp (two forked ranks) runs the
  unchanged reference calls and compares them with single-GPU calls bitwise.
NCCL between two physical GPUs is not exercised here (one GPU per box)."""
import os
import socket
import subprocess

import numpy as np
import pytest

from conftest import ROOT, bits_equal

BIN = ROOT / "tests" / "cpp" / "bin" / "test_multi"
LIB = ROOT / "paper_2005_10680_b200" / "lib"


def compile_multi():
    BIN.parent.mkdir(parents=True, exist_ok=True)
    src = ROOT / "tests" / "cpp" / "test_multi.cpp"
    if BIN.exists() and BIN.stat().st_mtime > max(src.stat().st_mtime,
                                                  (LIB / "libspamm_ec.so").stat().st_mtime):
        return BIN
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT / 'include'}",
                    str(src), "-o", str(BIN), f"-L{LIB}", "-lspamm_ec", "-lspamm_gpu",
                    "-pthread", f"-Wl,-rpath,{LIB}"], check=True)
    return BIN


def test_multi_rank_dropin_compiles(built):
    assert compile_multi().exists()


@pytest.mark.gpu
def test_dropin_two_ranks_bitwise(built):
    res = subprocess.run([str(compile_multi())], capture_output=True, text=True, timeout=600)
    print(res.stdout, res.stderr[-3000:])
    assert res.returncode == 0
    assert "0 of 2 ranks failed" in res.stdout


def _case(nat, ctx):
    A = nat.synth_cluster_device(ctx, 4096, 64, 3.0, 0.1, 2005, 1, 1e-10)
    B = nat.synth_cluster_device(ctx, 4096, 64, 3.0, 0.1, 2005, 2, 1e-10)
    return A, B


@pytest.mark.gpu
def test_nccl_single_rank_comm(ctx):
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    comm = nat.Comm.nccl(ctx, 1, 0, nat.Comm.unique_id())
    assert comm.info() == (1, 0, True)
    A, B = _case(nat, ctx)
    taus = log_grid(32)
    C1, s1, b1 = nat.spamm_with_error_control(ctx, A, B, 1e-6, taus)
    C2, s2, b2 = nat.spamm_with_error_control_sharded(comm, A, B, 1e-6, taus, gather=True)
    assert bits_equal(b1, b2) and s1["tau"] == s2["tau"]
    r1, c1, p1, n1 = C1.download()
    r2, c2, p2, n2 = C2.download()
    assert np.array_equal(r1, r2) and np.array_equal(c1, c2) and bits_equal(p1, p2)
    comm.close()


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allgather(blob: bytes):
        t = torch.frombuffer(bytearray(blob), dtype=torch.uint8) if blob else \
            torch.empty(0, dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.numpy().tobytes() for p in parts]

    ctx = nat.Context(0)
    comm = nat.Comm.host(ctx, world, rank, allgather)
    A, B = _case(nat, ctx)
    taus = log_grid(32)
    res = {}
    C, st, b = nat.spamm_with_error_control(ctx, A, B, 1e-6, taus)
    res["single"] = C.download() + (b, st["tau"])
    Cg, sg, bg = nat.spamm_with_error_control_sharded(comm, A, B, 1e-6, taus, gather=True)
    res["gathered"] = Cg.download() + (bg, sg["tau"])
    Cs, ss, bs = nat.spamm_with_error_control_sharded(comm, A, B, 1e-6, taus, gather=False)
    res["shard"] = Cs.download() + (bs, ss["tau"])
    res["cse"] = nat.cse_sharded(comm, A, B, taus)
    Ex, _ = nat.spamm_sharded(comm, A, B, 0.0, skip_test=False, gather=True)
    E1, _ = nat.multiply_exact(ctx, A, B)
    res["exact_equal"] = all(np.array_equal(x, y) for x, y in zip(Ex.download(), E1.download()))
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(res, dtype=object), allow_pickle=True)
    comm.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_host_comm_bitwise(built, tmp_path):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item() for r in range(2)]
    for r, res in enumerate(got):
        r1, c1, p1, n1, b1, t1 = res["single"]
        r2, c2, p2, n2, b2, t2 = res["gathered"]
        assert bits_equal(b1, b2) and t1 == t2 and bits_equal(res["cse"], b1)
        assert np.array_equal(r1, r2) and np.array_equal(c1, c2)
        assert bits_equal(p1, p2) and bits_equal(n1, n2)
        assert res["exact_equal"]
        # the rank's own rows: block rows [r nb/2, (r+1) nb/2) of C~, bitwise
        rs, cs, ps, ns, bs, ts = res["shard"]
        half = 32  # 4096 / 64 / 2
        mine = (r1 >= r * half) & (r1 < (r + 1) * half)
        k1 = np.lexsort((c1[mine], r1[mine]))
        ks = np.lexsort((cs, rs))
        assert np.array_equal(rs[ks], r1[mine][k1]) and np.array_equal(cs[ks], c1[mine][k1])
        assert bits_equal(ps[ks], p1[mine][k1])
