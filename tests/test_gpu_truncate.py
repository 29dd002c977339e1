"""GPU block truncation and the approximate-square variants (SURVEY.md 8f row
1): bit-exact removed set, removed-norm bound and resulting norms against the
reference; the reference's truncation tests (test_error_control.cpp:148-236)
restated; truncmul/spamm/hybrid (experiment.cpp:47-82) against the oracle
composition."""
import numpy as np
import pytest

from conftest import bits_equal, golden_names, load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "cfg1"])
def test_truncate_golden(ctx, name):
    from paper_2005_10680_b200 import _native as nat
    g = load_golden(name)
    A = nat.upload(ctx, int(g["n"]), int(g["L"]), g["a_rows"], g["a_cols"], g["a_payload"])
    i = 0
    while f"trunc{i}_delta" in g:
        T, rn, rc = nat.truncate(ctx, A, float(g[f"trunc{i}_delta"]))
        assert rc == int(g[f"trunc{i}_removed_count"])
        assert bits_equal(rn, g[f"trunc{i}_removed_norm"])
        r, c, _, nrm = T.download(payload=False)
        assert np.array_equal(r, g[f"trunc{i}_rows"]) and np.array_equal(c, g[f"trunc{i}_cols"])
        assert bits_equal(nrm, g[f"trunc{i}_norms"])
        lvl = 0
        while f"a_level{lvl}" in g:  # inner norms rebuilt exactly
            T.level_norms(lvl)
            lvl += 1
        i += 1


def test_truncate_reference_cases(ctx, port):
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(31)
    d = np.where(rng.uniform(size=(32, 32)) < 0.4, rng.uniform(-1, 1, (32, 32)), 0.0)
    x = nat.from_dense(ctx, d, 8)
    same, rn, rc = nat.truncate(ctx, x, 0.0)  # :148-160
    assert rc == 0 and rn == 0.0 and same.nnz_blocks == x.nnz_blocks
    empt, rn, rc = nat.truncate(ctx, x, x.frobenius_norm * 1.01)
    assert empt.nnz_blocks == 0 and rc == x.nnz_blocks and rn < x.frobenius_norm * 1.01
    with pytest.raises(ValueError):
        nat.truncate(ctx, x, -1.0)
    e = np.zeros((8, 8))  # :162-175 greedy KAT
    e[0, 0], e[0, 4], e[4, 0] = 0.9, 0.1, 0.2
    t, rn, rc = nat.truncate(ctx, nat.from_dense(ctx, e, 4), 0.25)
    assert rc == 2 and rn == pytest.approx(np.sqrt(0.05), rel=1e-14)
    expect = np.zeros((8, 8))
    expect[0, 0] = 0.9
    assert bits_equal(t.to_dense(), expect)


def test_truncate_contract_and_parity_random(ctx, port):  # :177-236
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(61)
    for trial in range(60):
        n = 8 * int(rng.integers(1, 7))
        L = int(rng.choice([2, 4, 8]))
        d = np.where(rng.uniform(size=(n, n)) < 0.3, rng.uniform(-1, 1, (n, n)), 0.0)
        la = nat.dense_to_leaves(d, L)
        x = nat.upload(ctx, n, L, *la)
        tx = port.build(n, L, *la)
        delta = float(rng.uniform() * 1.2 * (x.frobenius_norm + 0.1))
        T, rn, rc = nat.truncate(ctx, x, delta)
        To, rno, rco = port.truncate(tx, delta)
        assert rc == rco and bits_equal(rn, rno)
        r, c, p, nrm = T.download()
        ro, co, po, no = To.leaves()
        assert np.array_equal(r, ro) and np.array_equal(c, co)
        assert bits_equal(p, po) and bits_equal(nrm, no)
        removed = np.linalg.norm(d - T.to_dense())
        assert removed < delta + (1e-300 if delta == 0 else 0.0)
        assert rn <= delta


@pytest.mark.parametrize("variant", ["truncmul", "spamm", "hybrid"])
def test_approximate_square_variants(ctx, port, variant):
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import log_grid
    rows, cols, pay = nat.synth_chain_host(1024, 32, 20.0, 11, 1e-10)
    X = nat.upload(ctx, 1024, 32, rows, cols, pay)
    tx = port.build(1024, 32, rows, cols, pay)
    taus = log_grid(32)
    delta = 1e-6
    Y, st = nat.approximate_square(ctx, X, variant, delta, taus)
    # oracle composition of the same protocol
    if variant == "truncmul":
        mid = port.multiply_exact(tx, tx)
        want, _, _ = port.truncate(mid, delta)
    else:
        dm = delta / 2 if variant == "hybrid" else delta
        k = port.select_index(port.cse(tx, tx, taus), dm)
        tau = float(taus[k]) if k >= 0 else 0.0
        assert st["chosen_tau"] == tau
        mid = port.spamm(tx, tx, tau)
        want = port.truncate(mid, delta / 2)[0] if variant == "hybrid" else mid
    r, c, p, _ = Y.download()
    ro, co, po, _ = want.leaves()
    if variant == "spamm":
        assert np.array_equal(r, ro) and np.array_equal(c, co)
    d = nat.leaves_to_dense(1024, 32, rows, cols, pay)
    realized = np.linalg.norm(nat.leaves_to_dense(1024, 32, r, c, p) - d @ d)
    assert realized < delta
    rel = np.linalg.norm(nat.leaves_to_dense(1024, 32, r, c, p) -
                         nat.leaves_to_dense(1024, 32, ro, co, po)) / np.linalg.norm(po)
    assert rel < 1e-10  # truncation decisions near ties may differ only by rounding of C~
