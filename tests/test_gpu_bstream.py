"""B resident in host memory, streamed to the GPU in panels of block rows
(SURVEY.md 8e, configs 4/5).

Property: with the panels in ascending k and the accumulator reloaded exactly,
every result -- B's norms, the CSE bounds, the selected tau, the surviving
products and C~ (payload and norms) -- is BITWISE identical to the same call
with B resident on the device, for any panel height.  The resident path is
itself pinned to the oracle by test_gpu_parity.py; here one case is also
checked against the oracle directly."""
import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu


def _random_case(rng, n, fill, decay):
    d = np.where(rng.uniform(size=(n, n)) < fill, rng.uniform(-1, 1, (n, n)), 0.0)
    if decay:
        d *= np.exp(-np.abs(np.subtract.outer(np.arange(n), np.arange(n))) / decay)
    return d


def _same_matrix(x, y):
    rx, cx, px, nx = x.download()
    ry, cy, py, ny = y.download()
    return (np.array_equal(rx, ry) and np.array_equal(cx, cy) and bits_equal(px, py)
            and bits_equal(nx, ny) and x.frobenius_norm == y.frobenius_norm)


@pytest.mark.parametrize("L", [4, 12, 16, 32, 64, 128])
def test_streamed_product_bitwise_equals_resident(ctx, L):
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    rng = np.random.default_rng(7000 + L)
    for trial in range(3):
        nb = int(rng.integers(2, 6 if L >= 64 else 12))
        n = max(1, nb * L - int(rng.integers(0, L)))
        da = _random_case(rng, n, rng.uniform(0.1, 1.0), rng.uniform(1, 3 * L))
        db = _random_case(rng, n, rng.uniform(0.1, 1.0), rng.uniform(1, 3 * L))
        la = nat.dense_to_leaves(da, L)
        rows, cols, pay = nat.sort_by_block_row(*nat.dense_to_leaves(db, L))
        A = nat.upload(ctx, n, L, *la)
        B = nat.upload(ctx, n, L, rows, cols, pay)
        taus = geometric_grid(1.0, float(rng.uniform(0.2, 0.9)), int(rng.integers(2, 60)))
        for panel_rows in (1, 3, 1 << 20):
            bs = nat.BStream(ctx, n, L, rows, cols, pay, panel_rows)
            npanels, _ = bs.panels()
            assert npanels >= 1
            depth = B.info().depth
            for lvl in range(depth + 1):
                assert bits_equal(bs.norms.level_norms(lvl), B.level_norms(lvl)), lvl
            assert bits_equal(nat.cse(ctx, A, bs.norms, taus), nat.cse(ctx, A, B, taus))
            for tau in (float(taus[rng.integers(0, len(taus))]), 0.0):
                C0, s0 = nat.spamm(ctx, A, B, tau)
                C1, s1 = nat.spamm_streamed(ctx, A, bs, tau)
                assert _same_matrix(C0, C1)
                assert s0["survivors"] == s1["survivors"]
                assert s0["candidates"] == s1["candidates"]
                assert s0["output_blocks"] == s1["output_blocks"]
            delta = float(rng.uniform(1e-3, 1.0)) * B.frobenius_norm * A.frobenius_norm
            if delta > 0:
                C0, st0, b0 = nat.spamm_with_error_control(ctx, A, B, delta, taus)
                C1, st1, b1 = nat.spamm_with_error_control_streamed(ctx, A, bs, delta, taus)
                assert bits_equal(b0, b1)
                assert st0["tau"] == st1["tau"] and st0["tau_index"] == st1["tau_index"]
                assert _same_matrix(C0, C1)
            bs.free()


def test_streamed_product_against_oracle(ctx, port):
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    rng = np.random.default_rng(99)
    n, L = 700, 32
    da = _random_case(rng, n, 0.6, 40.0)
    la = nat.dense_to_leaves(da, L)
    lb = nat.sort_by_block_row(*la)
    A = nat.upload(ctx, n, L, *la)
    bs = nat.BStream(ctx, n, L, *lb, panel_block_rows=5)
    ta = port.build(n, L, *la)
    taus = geometric_grid(1.0, 0.5, 40)
    assert bits_equal(nat.cse(ctx, A, bs.norms, taus), port.cse(ta, ta, taus))
    tau = float(taus[12])
    C, st = nat.spamm_streamed(ctx, A, bs, tau)
    r, c, p, _ = C.download()
    ro, co, po, _ = port.spamm(ta, ta, tau).leaves()
    assert np.array_equal(r, ro) and np.array_equal(c, co)
    assert np.linalg.norm(p - po) <= 1e-12 * np.linalg.norm(po)
    assert st["survivors"] == len(port.survivors(ta, ta, tau))


def test_streamed_cluster_matrix_pinned_torch_payload(ctx):
    """BASELINE cfg2-style input (3-D cluster decay, L=64), pinned torch host
    payload, 8-block-row panels."""
    import torch
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    n, L = 4096, 64
    rows, cols, pay = nat.synth_cluster_host(n, L, 3.0, 0.1, 2005, 10680, 1e-10)
    rows, cols, pay = nat.sort_by_block_row(rows, cols, pay)
    A = nat.upload(ctx, n, L, rows, cols, pay)
    host = torch.from_numpy(pay).pin_memory()
    bs = nat.BStream(ctx, n, L, rows, cols, host, panel_block_rows=8)
    assert bs.panels()[0] == 8
    taus = log_grid(32)
    C0, st0, b0 = nat.spamm_with_error_control(ctx, A, A, 1e-6, taus)
    C1, st1, b1 = nat.spamm_with_error_control_streamed(ctx, A, bs, 1e-6, taus)
    assert bits_equal(b0, b1) and st0["tau"] == st1["tau"]
    assert st0["spamm"]["survivors"] == st1["spamm"]["survivors"] > 0
    assert _same_matrix(C0, C1)


def test_streamed_edge_cases(ctx):
    from paper_2005_10680_b200 import _native as nat
    L, n = 16, 100
    rng = np.random.default_rng(3)
    d = _random_case(rng, n, 0.5, 10.0)
    rows, cols, pay = nat.sort_by_block_row(*nat.dense_to_leaves(d, L))
    A = nat.upload(ctx, n, L, rows, cols, pay)
    # unsorted leaves are rejected
    with pytest.raises(ValueError):
        nat.BStream(ctx, n, L, rows[::-1], cols[::-1], pay[::-1], 2)
    with pytest.raises(ValueError):
        nat.BStream(ctx, n, L, rows, cols, pay, 0)
    # out-of-range coordinate
    bad = rows.copy()
    bad[-1] = 64
    with pytest.raises(IndexError):
        nat.BStream(ctx, n, L, bad, cols, pay, 2)
    # nonzero padding of a boundary leaf
    pay2 = pay.copy()
    edge = np.nonzero(rows == rows.max())[0][0]
    pay2[edge].reshape(L, L)[L - 1, :] = 1.0  # row L-1 of the last block row is padding
    with pytest.raises(ValueError):
        nat.BStream(ctx, n, L, rows, cols, pay2, 2)
    # the norm-only matrix refuses payload uses
    bs = nat.BStream(ctx, n, L, rows, cols, pay, 2)
    with pytest.raises(ValueError):
        nat.spamm(ctx, A, bs.norms, 0.0)
    with pytest.raises(ValueError):
        bs.norms.to_dense()
    with pytest.raises(ValueError):
        nat.truncate(ctx, bs.norms, 0.1)
    r, c, _, nrm = bs.norms.download(payload=False)
    assert len(r) == A.nnz_blocks
    # empty B: empty product
    empty = nat.BStream(ctx, n, L, np.empty(0, np.int32), np.empty(0, np.int32),
                        np.empty((0, L * L)), 2)
    C, st = nat.spamm_streamed(ctx, A, empty, 0.0)
    assert C.nnz_blocks == 0 and st["survivors"] == 0
    # zero leaves collapse to null (make_leaf) exactly as on upload
    pz = pay.copy()
    pz[0] = 0.0
    bz = nat.BStream(ctx, n, L, rows, cols, pz, 1)
    Bz = nat.upload(ctx, n, L, rows, cols, pz)
    assert bz.norms.nnz_blocks == Bz.nnz_blocks == A.nnz_blocks - 1
    assert _same_matrix(nat.spamm_streamed(ctx, A, bz, 0.0)[0], nat.spamm(ctx, A, Bz, 0.0)[0])
