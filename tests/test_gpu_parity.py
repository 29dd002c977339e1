"""GPU parity: the CUDA path through the C ABI against the oracle.

Bars (BASELINE.json north_star / SURVEY.md 8a P1-P5): node norms, CSE bounds,
selected tau and surviving product set bit-exact; C~ within 1e-12 relative
Frobenius of the reference product with the identical block structure."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal, golden_names, load_golden

pytestmark = pytest.mark.gpu

REL_TOL = 1e-12  # P5: DMMA fuses and reorders the k-sum (test_multiply.cpp:55,122)


def rel_fro(x, y):
    ny = np.linalg.norm(y)
    return np.linalg.norm(x - y) / (ny if ny > 0 else 1.0)


def upload_golden(nat, ctx, g, tag):
    return nat.upload(ctx, int(g["n"]), int(g["L"]), g[f"{tag}_rows"], g[f"{tag}_cols"],
                      g[f"{tag}_payload"])


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "cfg1"])
def test_golden_case_on_gpu(ctx, name):
    from paper_2005_10680_b200 import _native as nat
    g = load_golden(name)
    n, L = int(g["n"]), int(g["L"])
    A, B = upload_golden(nat, ctx, g, "a"), upload_golden(nat, ctx, g, "b")
    lvl = 0
    while f"a_level{lvl}" in g:
        assert bits_equal(A.level_norms(lvl), g[f"a_level{lvl}"]), lvl
        assert bits_equal(B.level_norms(lvl), g[f"b_level{lvl}"]), lvl
        lvl += 1
    bounds = nat.cse(ctx, A, B, g["taus"])
    assert bits_equal(bounds, g["bounds"])
    i = 0
    while f"delta{i}" in g:
        tau, k = nat.select_tolerance(bounds, g["taus"], float(g[f"delta{i}"]))
        assert k == int(g[f"select{i}"])
        i += 1
    i = 0
    while f"tau{i}" in g:
        tau = float(g[f"tau{i}"])
        assert np.array_equal(nat.survivors(ctx, A, B, tau), g[f"surv{i}"])
        C, st = nat.spamm(ctx, A, B, tau)
        r, c, p, nrm = C.download()
        assert np.array_equal(r, g[f"c{i}_rows"]) and np.array_equal(c, g[f"c{i}_cols"])
        assert rel_fro(p, g[f"c{i}_payload"]) < REL_TOL
        assert st["survivors"] == len(g[f"surv{i}"])
        i += 1


def test_cfg1_on_gpu_matches_reference_golden(ctx):
    """BASELINE.json config 1 (N=4096, L=64, 32 taus, delta=1e-6) end to end."""
    import hashlib
    from paper_2005_10680_b200 import _native as nat
    meta = json.loads((GOLDEN / "cfg1.json").read_text())
    g = load_golden("cfg1")
    rows, cols, pay = nat.synth_chain_host(meta["n"], meta["leaf"], meta["ell"], meta["seed"],
                                           meta["drop"])
    A = nat.upload(ctx, meta["n"], meta["leaf"], rows, cols, pay)
    for lvl in range(7):
        assert bits_equal(A.level_norms(lvl), g[f"a_level{lvl}"])
    C, st, bounds = nat.spamm_with_error_control(ctx, A, A, meta["delta"], g["taus"])
    assert bits_equal(bounds, g["bounds"])
    assert st["tau_index"] == meta["tau_index"] and st["tau"] == meta["tau"]
    assert st["bound"] == meta["bound"]
    surv = nat.survivors(ctx, A, A, meta["tau"])
    assert hashlib.sha256(np.ascontiguousarray(surv).tobytes()).hexdigest() == \
        meta["survivors_sha256"]
    assert st["spamm"]["survivors"] == meta["survivors"]
    r, c, p, nrm = C.download()
    assert np.array_equal(r, g["c_rows"]) and np.array_equal(c, g["c_cols"])
    assert abs(C.frobenius_norm - float(g["c_frob"])) <= 1e-12 * float(g["c_frob"])
    # delta bound against an exact dense product (error_control.hpp:73-75)
    d = nat.leaves_to_dense(meta["n"], meta["leaf"], rows, cols, pay)
    exact = d @ d
    approx = nat.leaves_to_dense(meta["n"], meta["leaf"], r, c, p)
    realized = np.linalg.norm(approx - exact)
    assert realized < meta["delta"]
    assert realized <= st["bound"] * (1 + 1e-9) + 1e-10 * np.linalg.norm(d) ** 2 * 1e-6


def test_cfg1_c_elementwise_vs_reference(ctx, ref):
    """Config 1's C~ block by block against the reference's own
    spamm_multiply (oracle/_ref, all host threads) at the reference's tau*:
    identical block structure, every block within 1e-12 relative Frobenius,
    every C~ leaf norm within the same tolerance."""
    import os
    from paper_2005_10680_b200 import _native as nat
    meta = json.loads((GOLDEN / "cfg1.json").read_text())
    rows, cols, pay = nat.synth_chain_host(meta["n"], meta["leaf"], meta["ell"], meta["seed"],
                                           meta["drop"])
    A = nat.upload(ctx, meta["n"], meta["leaf"], rows, cols, pay)
    g = load_golden("cfg1")
    C, st, _ = nat.spamm_with_error_control(ctx, A, A, meta["delta"], g["taus"])
    ref.set_threads(os.cpu_count() or 1)
    T = ref.build(meta["n"], meta["leaf"], rows, cols, pay)
    rr, rc, rp, rn = ref.spamm(T, T, st["tau"]).leaves()
    r, c, p, nrm = C.download()
    assert np.array_equal(r, rr) and np.array_equal(c, rc)
    assert rel_fro(p, rp) < REL_TOL
    per_block = np.linalg.norm(p - rp, axis=1) / np.maximum(np.linalg.norm(rp, axis=1), 1e-300)
    assert per_block.max() < REL_TOL, per_block.max()
    assert np.all(np.abs(nrm - rn) <= REL_TOL * rn)


def _random_case(rng, n, L, fill, decay):
    d = np.where(rng.uniform(size=(n, n)) < fill, rng.uniform(-1, 1, (n, n)), 0.0)
    if decay:
        d *= np.exp(-np.abs(np.subtract.outer(np.arange(n), np.arange(n))) / decay)
    return d


@pytest.mark.parametrize("L", [2, 3, 4, 8, 12, 16, 24, 32, 48, 64, 128])
def test_random_vs_oracle_all_leaf_sizes(ctx, port, L):
    """Every GEMM instantiation (generic, DMMA L=32/64/128) and ragged sizes."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    rng = np.random.default_rng(1000 + L)
    for trial in range(4):
        nb = int(rng.integers(1, 6 if L >= 64 else 9))
        n = max(1, nb * L - int(rng.integers(0, L)))
        da = _random_case(rng, n, L, rng.uniform(0.05, 1.0), rng.uniform(1, 3 * L))
        db = _random_case(rng, n, L, rng.uniform(0.05, 1.0), rng.uniform(1, 3 * L))
        la, lb = nat.dense_to_leaves(da, L), nat.dense_to_leaves(db, L)
        A, B = nat.upload(ctx, n, L, *la), nat.upload(ctx, n, L, *lb)
        ta, tb = port.build(n, L, *la), port.build(n, L, *lb)
        for lvl in range(ta.depth() + 1):
            assert bits_equal(A.level_norms(lvl), ta.level_norms(lvl))
        taus = geometric_grid(1.0, float(rng.uniform(0.2, 0.9)), int(rng.integers(1, 80)))
        assert bits_equal(nat.cse(ctx, A, B, taus), port.cse(ta, tb, taus))
        for tau in (float(taus[rng.integers(0, len(taus))]), 0.0):
            assert np.array_equal(nat.survivors(ctx, A, B, tau), port.survivors(ta, tb, tau))
            C, _ = nat.spamm(ctx, A, B, tau)
            r, c, p, _ = C.download()
            ro, co, po, _ = port.spamm(ta, tb, tau).leaves()
            assert np.array_equal(r, ro) and np.array_equal(c, co)
            assert rel_fro(p, po) < REL_TOL


def test_many_taus_and_piece_batches(ctx, port):
    """Grids far larger than the tile's piece batch (350 = geometric default,
    error_control.hpp:21, and 4000) still give bit-identical bounds."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    rng = np.random.default_rng(5)
    n, L = 512, 16
    da = _random_case(rng, n, L, 1.0, 20.0)
    la = nat.dense_to_leaves(da, L)
    A = nat.upload(ctx, n, L, *la)
    t = port.build(n, L, *la)
    for taus in (geometric_grid(), geometric_grid(1.0, 0.99, 4000)):
        assert bits_equal(nat.cse(ctx, A, A, taus), port.cse(t, t, taus))


@pytest.mark.parametrize("n_taus", [1, 2, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129])
def test_sweep_kernel_variants_every_grid_size(ctx, port, n_taus):
    """Depth >= 3 trees run the windowed tile kernel for N_tau <= 128 (1-4
    windows of 32, the F-in-last-column case across windows) and the
    breakpoint-window kernel above: bounds bit-identical for log-spaced and
    very fine grids, with null and zero-norm leaves in the tiles."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid, log_grid
    rng = np.random.default_rng(100 + n_taus)
    n, L = 700, 16
    da = _random_case(rng, n, L, 0.7, 25.0)
    da[:, 100:140] = 0.0                       # null leaves
    da[200:216, 300:316] = 1e-300 * rng.uniform(size=(16, 16))  # underflowing products
    db = _random_case(rng, n, L, 0.9, 60.0)
    la, lb = nat.dense_to_leaves(da, L), nat.dense_to_leaves(db, L)
    A, B = nat.upload(ctx, n, L, *la), nat.upload(ctx, n, L, *lb)
    ta, tb = port.build(n, L, *la), port.build(n, L, *lb)
    grids = [log_grid(n_taus, 10.0, 1e-6) if n_taus > 1 else np.array([1e-2]),
             geometric_grid(float(np.sqrt(ta.level_norms(0)[0] * tb.level_norms(0)[0])), 0.97,
                            n_taus)]
    for taus in grids:
        assert bits_equal(nat.cse(ctx, A, B, taus), port.cse(ta, tb, taus))
    # a grid spanning ~2000 binades (no bucket table: other kernels)
    wide = np.logspace(300, -300, n_taus) if n_taus > 1 else np.array([1.0])
    assert bits_equal(nat.cse(ctx, A, B, wide), port.cse(ta, tb, wide))


@pytest.mark.parametrize("n_taus", [32, 64, 128])
def test_sweep_wide_breakpoint_ranges(ctx, port, n_taus):
    """Leaf blocks whose norms spread over ten decades inside every quadtree
    node: a level d-1 node's live tau range then spans most of the grid, a
    half-tile holds more items than the tile kernel's flat array and is
    evaluated one level d-2 group at a time -- still bit-identical."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rng = np.random.default_rng(900 + n_taus)
    n, L = 512, 8
    nb = n // L
    scale = np.repeat(np.repeat(10.0 ** rng.uniform(-10, 0, (nb, nb)), L, 0), L, 1)
    da = rng.uniform(-1, 1, (n, n)) * scale
    db = rng.uniform(-1, 1, (n, n)) * scale.T
    la, lb = nat.dense_to_leaves(da, L), nat.dense_to_leaves(db, L)
    A, B = nat.upload(ctx, n, L, *la), nat.upload(ctx, n, L, *lb)
    ta, tb = port.build(n, L, *la), port.build(n, L, *lb)
    taus = log_grid(n_taus, 1.0, 1e-14)
    assert bits_equal(nat.cse(ctx, A, B, taus), port.cse(ta, tb, taus))
    assert bits_equal(nat.cse(ctx, A, A, taus), port.cse(ta, ta, taus))


def test_sweep_branch_free_sqrt_is_correctly_rounded(ctx):
    """The tile kernels take square roots through the builtin's fast path with
    one shared range check per group of evaluations (csrc/cse.cu sqrt_fast);
    4e9 bit patterns over every exponent, sign and special value, and perfect
    squares +-1 ulp, give sqrt.rn.f64's bits."""
    from paper_2005_10680_b200 import _native as nat
    assert nat.selftest_sqrt(ctx, 2_000_000_000, 20051068) == 0
    assert nat.selftest_sqrt(ctx, 1000, 7) == 0


@pytest.mark.parametrize("n_taus,scale", [(32, 1e-75), (32, 1e-78), (128, 1e-77), (64, 1e-150)])
def test_sweep_tiny_norms_take_the_sqrt_slow_path(ctx, port, n_taus, scale):
    """Norm products around 1e-150: their squares fall below 2^-970 (the range
    the fast square root covers), into the subnormals, or underflow to zero."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rng = np.random.default_rng(77)
    n, L = 256, 4
    nb = n // L
    spread = np.repeat(np.repeat(10.0 ** rng.uniform(-6, 0, (nb, nb)), L, 0), L, 1)
    da = rng.uniform(-1, 1, (n, n)) * spread * scale
    db = rng.uniform(-1, 1, (n, n)) * spread.T * scale
    la, lb = nat.dense_to_leaves(da, L), nat.dense_to_leaves(db, L)
    A, B = nat.upload(ctx, n, L, *la), nat.upload(ctx, n, L, *lb)
    ta, tb = port.build(n, L, *la), port.build(n, L, *lb)
    taus = log_grid(n_taus, scale * scale * 10.0, scale * scale * 1e-12)
    got, want = nat.cse(ctx, A, B, taus), port.cse(ta, tb, taus)
    assert bits_equal(got, want)
    assert scale < 1e-100 or np.count_nonzero(want) > 0


@pytest.mark.parametrize("env", [{"SPG_CSE_LISTS": "1"}, {"SPG_CSE_FOLD": "2"},
                                 {"SPG_CSE_FOLD": "2", "SPG_CSE_LISTS": "1"},
                                 {"SPG_CSE_FOLD": "0"}, {"SPG_CSE": "4"},
                                 {"SPG_CSE_SYNC": "1", "SPG_CSE_LISTS": "1"},
                                 {"SPG_CSE_SYNC": "1", "SPG_CSE_LISTS": "1", "SPG_CSE": "4"}])
def test_sweep_paths_in_subprocesses(port, env):
    """Every sweep path (pair lists instead of dense enumeration, level s-1
    folded into the tile CTAs or not, the general tile kernel of grids the
    bucket table cannot hold, the host-synchronised list path) gives the oracle's bounds
    bit for bit; the path is fixed per process, so each runs in a child."""
    import os
    import subprocess
    import sys as _sys
    from pathlib import Path
    from paper_2005_10680_b200 import _native as nat
    here = Path(__file__).resolve().parent
    _sys.path.insert(0, str(here))
    import sweep_paths_case as spc
    out = subprocess.run([_sys.executable, str(here / "sweep_paths_case.py")],
                         env={**os.environ, **env}, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    got = dict(line.split() for line in out.stdout.strip().splitlines())
    for name, n, L, da, db, taus in spc.cases():
        ta = port.build(n, L, *nat.dense_to_leaves(da, L))
        tb = port.build(n, L, *nat.dense_to_leaves(db, L))
        want = port.cse(ta, tb, taus).view(np.uint64).tobytes().hex()
        assert got[name] == want, (env, name)


@pytest.mark.parametrize("env", [{"SPG_GEMM32": "6"}, {"SPG_SUPER32_QUAD": "0"}, {"SPG_GEMM128": "3"},
                                 {"SPG_TASKLIST": "lists"}])
def test_gemm_paths_in_subprocesses(env):
    """Leaf-GEMM variants that keep every block's products in ascending k and
    the same DMMA k-steps give C~ bit for bit equal to each other: the L = 32
    super-block kernel (default) against per-block tilings, L = 128 leaves as
    L = 64 sub-products against the L = 128 kernel; likewise the two task-list
    builders (sort-free dense walk, default, against expansion + radix sort:
    same survivors in the same order); the variant is fixed per process."""
    import os
    import subprocess
    import sys as _sys
    from pathlib import Path
    script = Path(__file__).resolve().parent / "gemm_paths_case.py"

    def run(extra):
        out = subprocess.run([_sys.executable, str(script)], env={**os.environ, **extra},
                             capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        return out.stdout.split("\n")

    assert run(env) == run({})


@pytest.mark.parametrize("n,L", [(16384, 2), (32768, 2), (24000, 4)])
def test_deep_trees_task_list_and_sweep(ctx, port, n, L):
    """Quadtrees of depth 13 and 14 (the deepest the Morton grids allow), banded
    with decaying blocks: the dense task-list walk (flags per (tile, K) up to
    8^11) gives the oracle's survivor set, the product its C~, and the sweep
    (pair lists at this depth) its bounds."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rng = np.random.default_rng(n + L)
    nb = -(-n // L)
    off = np.arange(-3, 4)
    r = np.repeat(np.arange(nb), len(off))
    c = r + np.tile(off, nb)
    keep = (c >= 0) & (c < nb) & (rng.random(len(r)) < 0.9)
    r, c = r[keep].astype(np.int32), c[keep].astype(np.int32)
    pay = rng.uniform(-1, 1, (len(r), L * L)) * (10.0 ** (-1.5 * np.abs(r - c)))[:, None]
    if n % L:  # zero padding of the ragged last block row / column
        blk = pay.reshape(len(r), L, L)  # column-major leaves: [col][row]
        blk[r == nb - 1, :, n % L:] = 0.0
        blk[c == nb - 1, n % L:, :] = 0.0
    A = nat.upload(ctx, n, L, r, c, pay)
    ta = port.build(n, L, r, c, pay)
    tau = 1e-3
    got = nat.survivors(ctx, A, A, tau)
    want = port.survivors(ta, ta, tau)
    assert len(got) == len(want) and len(want) > 0
    key = lambda t: np.lexsort((t[:, 2], t[:, 1], t[:, 0]))  # noqa: E731
    assert np.array_equal(got[key(got)], want[key(want)])
    C, st = nat.spamm(ctx, A, A, tau)
    assert st["survivors"] == len(want) and st["survivors"] < st["candidates"]
    rc, cc, pc, _ = C.download()
    wr, wc, wp, _ = port.spamm(ta, ta, tau).leaves()
    assert np.array_equal(rc, wr) and np.array_equal(cc, wc)
    assert rel_fro(pc, wp) < REL_TOL
    taus = log_grid(32, 1.0, 1e-10)
    assert bits_equal(nat.cse(ctx, A, A, taus), port.cse(ta, ta, taus))


def test_run_to_run_determinism(ctx):
    """SPEC determinism (test_multiply.cpp:140-156 analogue): repeated calls are
    bitwise identical."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rows, cols, pay = nat.synth_chain_host(2048, 64, 40.0, 3, 1e-10)
    A = nat.upload(ctx, 2048, 64, rows, cols, pay)
    outs = []
    for _ in range(3):
        C, st, b = nat.spamm_with_error_control(ctx, A, A, 1e-6, log_grid(32))
        outs.append((b, C.download()))
    for b, (r, c, p, nrm) in outs[1:]:
        assert bits_equal(b, outs[0][0])
        assert bits_equal(p, outs[0][1][2]) and bits_equal(nrm, outs[0][1][3])


@pytest.mark.parametrize("L", [16, 64])
def test_streamed_to_host_equals_device_product(ctx, L):
    """spg_spamm_with_error_control_to_host (chunked GEMM + overlapped D2H) ==
    spg_spamm_with_error_control + spg_matrix_download, bit for bit."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    n = 64 * L
    rows, cols, pay = nat.synth_chain_host(n, L, 40.0, 7, 1e-10)
    A = nat.upload(ctx, n, L, rows, cols, pay)
    taus = log_grid(32)
    C, st, b = nat.spamm_with_error_control(ctx, A, A, 1e-6, taus)
    r, c, p, nrm = C.download()
    (hr, hc, hp, hn), hst, hb = nat.spamm_with_error_control_to_host(ctx, A, A, 1e-6, taus)
    assert bits_equal(b, hb) and hst["tau"] == st["tau"]
    assert np.array_equal(r, hr) and np.array_equal(c, hc)
    assert bits_equal(p, hp) and bits_equal(nrm, hn)
    with pytest.raises(ValueError):
        nat.spamm_with_error_control_to_host(
            ctx, A, A, 1e-6, taus, out=(np.empty(1, np.int32), np.empty(1, np.int32),
                                        np.empty((1, L * L)), np.empty(1)))


def test_parity_audit_counts(ctx, port):
    """The near-tie audit counts candidates exactly (oracle candidate count) and
    finds a product placed exactly on tau."""
    from paper_2005_10680_b200 import _native as nat
    rows, cols, pay = nat.synth_chain_host(1024, 32, 20.0, 3, 1e-10)
    A = nat.upload(ctx, 1024, 32, rows, cols, pay)
    t = port.build(1024, 32, rows, cols, pay)
    ties, cands = nat.parity_audit(ctx, A, A, 1e-6, 4)
    assert cands == port._cand(t.h, t.h)
    _, _, _, norms = A.download(payload=False)
    tau = float(norms[0] * norms[0])  # the (0,0,0) leaf product itself
    ties, _ = nat.parity_audit(ctx, A, A, tau, 0)
    assert ties >= 1


def test_staged_upload_equals_upload_and_overlaps_a_product(ctx):
    """spg_matrix_stage / stage_finish: the same matrix as spg_matrix_upload
    (bitwise), also when staged while a product is queued on the context."""
    import torch
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rows, cols, pay = nat.synth_chain_host(2048, 64, 40.0, 9, 1e-10)
    h_rows = torch.from_numpy(rows).pin_memory()
    h_cols = torch.from_numpy(cols).pin_memory()
    h_pay = torch.from_numpy(np.ascontiguousarray(pay)).pin_memory()
    A = nat.upload(ctx, 2048, 64, rows, cols, pay)
    st = nat.Staged(ctx, 2048, 64, len(rows), h_rows.data_ptr(), h_cols.data_ptr(),
                    h_pay.data_ptr())
    S = st.finish()
    for lvl in range(6):
        assert bits_equal(S.level_norms(lvl), A.level_norms(lvl))
    ra, ca, pa, na = A.download()
    rs, cs, ps, ns = S.download()
    assert np.array_equal(ra, rs) and np.array_equal(ca, cs) and bits_equal(pa, ps)
    taus = log_grid(32)
    C0, s0, b0 = nat.spamm_with_error_control(ctx, A, A, 1e-6, taus)
    nxt = nat.Staged(ctx, 2048, 64, len(rows), h_rows.data_ptr(), h_cols.data_ptr(),
                     h_pay.data_ptr())
    C1, s1, b1 = nat.spamm_with_error_control(ctx, S, S, 1e-6, taus)  # runs while nxt copies
    N = nxt.finish()
    C2, s2, b2 = nat.spamm_with_error_control(ctx, N, N, 1e-6, taus)
    for Ck, bk in ((C1, b1), (C2, b2)):
        assert bits_equal(bk, b0)
        assert bits_equal(Ck.download()[2], C0.download()[2])
    abandoned = nat.Staged(ctx, 2048, 64, len(rows), h_rows.data_ptr(), h_cols.data_ptr(),
                           h_pay.data_ptr())
    del abandoned  # spg_staged_free waits for its copies


def test_nan_entries_follow_the_reference(ctx, ref):
    """A NaN entry makes its leaf norm NaN (non-null, block_norm): the sweep
    treats the leaf's products as never skipped-error (NaN < tau is false at
    every k), the skip test keeps them (!(NaN < tau)); bounds, survivors and
    norms match the reference bit for bit."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid, log_grid
    rng = np.random.default_rng(31)
    n, L = 300, 8
    d = _random_case(rng, n, L, 0.6, 30.0)
    d[17, 40] = np.nan
    d[250, 3] = np.nan
    lv = nat.dense_to_leaves(d, L)
    A = nat.upload(ctx, n, L, *lv)
    tr = ref.build(n, L, *lv)
    for lvl in range(tr.depth() + 1):
        assert bits_equal(A.level_norms(lvl), tr.level_norms(lvl))
    for taus in (log_grid(32, 1.0, 1e-8), geometric_grid(10.0, 0.8, 60)):
        b = nat.cse(ctx, A, A, taus)
        assert bits_equal(b, ref.cse(tr, tr, taus))
        tau = float(taus[len(taus) // 2])
        assert np.array_equal(nat.survivors(ctx, A, A, tau), ref.survivors(tr, tr, tau))
