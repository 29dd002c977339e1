"""CPU: bench.py's host-side machinery.

* the reference arm's input generator (oracle/libinputs.so) reproduces the
  product's host generator bit for bit, without loading the product library;
* the bounded CPU sample gives every fork-join task of the reference work
  (execution.cpp:17-23, multiply.cpp:79-84);
* `bench.py --gpus N` starts N ranks itself (torch.distributed.run) and refuses
  a mismatched WORLD_SIZE;
* the device-buffer all-gather used for the leaf-norm tables (gloo, world 2).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def test_host_inputs_equal_product_host_generator(built):
    import oracle
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import Workload
    cases = [Workload("c", "cluster", 512, 16, 3.0, 1e-5, 32),
             Workload("c", "cluster", 1000, 32, 2.0, 1e-5, 32, drop=1e-6, value_seed=3),
             Workload("h", "chain", 700, 32, 40.0, 1e-6, 32, value_seed=12345),
             Workload("h", "chain", 257, 8, 5.0, 1e-6, 32, drop=1e-4, value_seed=1)]
    for w in cases:
        for threads in (1, 7):
            got = oracle.host_inputs(w, threads)
            if w.kind == "cluster":
                want = nat.synth_cluster_host(w.n, w.leaf, w.ell, w.density, w.site_seed,
                                              w.value_seed, w.drop)
            else:
                want = nat.synth_chain_host(w.n, w.leaf, w.ell, w.value_seed, w.drop)
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
            assert got[2].tobytes() == want[2].tobytes()


def test_sample_rows_feed_every_task():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.spawn_levels(1) == 0 and bench.spawn_levels(4) == 1
    assert bench.spawn_levels(16) == 2 and bench.spawn_levels(17) == 3
    assert bench.spawn_levels(1000) == 3
    assert bench.sample_rows(512, 16) == [0, 128, 256, 384]
    assert bench.sample_rows(512, 16, 2) == [0, 1, 128, 129, 256, 257, 384, 385]
    assert bench.sample_rows(512, 64) == list(range(0, 512, 64))
    assert bench.sample_rows(64, 8) == [0, 16, 32, 48]
    assert bench.sample_rows(5, 16) == [0, 2, 4]  # padded 8 -> groups of 2; row 6 absent
    # every level-`levels` output quadrant row gets a sampled row
    for nb, threads in ((512, 16), (300, 64), (33, 4)):
        lv = bench.spawn_levels(threads)
        padded = 1 << max(0, (nb - 1).bit_length())
        groups = {r // (padded >> lv) for r in bench.sample_rows(nb, threads)}
        assert groups == {g for g in range(1 << lv) if g * (padded >> lv) < nb}


def test_bench_reference_arm_spawns_ranks(built):
    """`bench.py --gpus 2` with no launcher around it starts two ranks; rank 0
    alone runs the reference arm and prints one JSON line with n_gpus 2."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT"):
        env.pop(k, None)
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", "cfg1", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["impl"] == "reference"
    assert out["cpu_baseline"]["kind"] in ("reference", "port")
    assert out["tau_index"] == 19 and out["survivors"] == 29448  # config 1 (DESIGN.md Inputs)
    assert out["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_refuses_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", "cfg1", "--gpus", "2"], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert res.returncode != 0 and "WORLD_SIZE" in res.stderr


def _gather_worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank), SPG_DIST_BACKEND="gloo")
    import bench
    d = bench.Dist()
    rng = np.random.default_rng(rank)
    n = 5 + 3 * rank  # per-rank lengths differ
    arrays = [rng.integers(0, 100, n).astype(np.int32), rng.normal(size=n),
              rng.normal(size=(2 + rank, 4)), np.empty(0, np.float64) if rank else np.ones(1)]
    got = d.all_gather_arrays(arrays)
    np.save(os.path.join(out_dir, f"mine_{rank}.npy"), np.array(arrays, dtype=object),
            allow_pickle=True)
    np.save(os.path.join(out_dir, f"got_{rank}.npy"), np.array(got, dtype=object),
            allow_pickle=True)
    d.close()


def test_all_gather_arrays_gloo(tmp_path):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_gather_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    mine = [np.load(tmp_path / f"mine_{r}.npy", allow_pickle=True) for r in range(2)]
    for r in range(2):
        got = np.load(tmp_path / f"got_{r}.npy", allow_pickle=True)
        for src in range(2):
            for a, b in zip(got[src], mine[src]):
                assert a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a, b)
