"""GPU: the reference's own hot-path tests (test_multiply.cpp,
test_error_control.cpp) restated against the CUDA path via the C ABI."""
import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu


def rd(rng, n, fill=1.0):
    # np.where, not a product: u * 0 would give -0.0 entries, which the
    # reference generator (support.hpp:32-39) never produces
    return np.where(rng.uniform(size=(n, n)) < fill, rng.uniform(-1, 1, (n, n)), 0.0)


def test_identity_product_exact(ctx):  # test_multiply.cpp:30-36
    from paper_2005_10680_b200 import _native as nat
    d = rd(np.random.default_rng(41), 24, 0.5)
    A = nat.from_dense(ctx, d, 8)
    I = nat.from_dense(ctx, np.eye(24), 8)
    assert bits_equal(nat.multiply_exact(ctx, A, I)[0].to_dense(), d)
    assert bits_equal(nat.multiply_exact(ctx, I, A)[0].to_dense(), d)


def test_zero_product(ctx):  # test_multiply.cpp:38-44
    from paper_2005_10680_b200 import _native as nat
    A = nat.from_dense(ctx, rd(np.random.default_rng(42), 16), 8)
    Z = nat.zero(ctx, 16, 8)
    assert nat.multiply_exact(ctx, A, Z)[0].nnz_blocks == 0
    assert nat.multiply_exact(ctx, Z, A)[0].nnz_blocks == 0
    assert nat.spamm(ctx, A, Z, 0.0)[0].nnz_blocks == 0


def test_exact_vs_dense(ctx):  # test_multiply.cpp:46-57
    from paper_2005_10680_b200 import _native as nat
    for seed in (1, 2, 3):
        rng = np.random.default_rng(seed)
        da, db = rd(rng, 64, 0.6), rd(rng, 64, 0.6)
        C, _ = nat.multiply_exact(ctx, nat.from_dense(ctx, da, 16), nat.from_dense(ctx, db, 16))
        ref = da @ db
        assert np.linalg.norm(C.to_dense() - ref) / np.linalg.norm(ref) < 1e-12


def test_tau_zero_equals_exact_bitwise(ctx):  # test_multiply.cpp:59-66
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(7)
    A = nat.from_dense(ctx, rd(rng, 48, 0.4), 16)
    B = nat.from_dense(ctx, rd(rng, 48, 0.4), 16)
    assert bits_equal(nat.spamm(ctx, A, B, 0.0)[0].to_dense(),
                      nat.multiply_exact(ctx, A, B)[0].to_dense())


def test_tau_above_root_skips_everything(ctx):  # test_multiply.cpp:68-73
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(9)
    A = nat.from_dense(ctx, rd(rng, 16), 8)
    B = nat.from_dense(ctx, rd(rng, 16), 8)
    root = A.frobenius_norm * B.frobenius_norm
    assert nat.spamm(ctx, A, B, root * 1.0001)[0].nnz_blocks == 0


def test_quadrant_pair_dropped(ctx):  # test_multiply.cpp:75-109
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(55)
    da = rng.uniform(0.5, 1.0, (8, 8))
    db = rng.uniform(0.5, 1.0, (8, 8))
    da[:4, 4:] *= 1e-4
    db[4:, :4] *= 1e-4
    small = np.linalg.norm(da[:4, 4:]) * np.linalg.norm(db[4:, :4])
    C, _ = nat.spamm(ctx, nat.from_dense(ctx, da, 4), nat.from_dense(ctx, db, 4), small * 50)
    expect = da @ db
    expect[:4, :4] -= da[:4, 4:] @ db[4:, :4]
    assert np.linalg.norm(C.to_dense() - expect) < 1e-13


def test_larger_tau_structural_subset(ctx):  # test_multiply.cpp:126-138
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(13)
    A = nat.from_dense(ctx, rd(rng, 64, 0.3), 8)
    B = nat.from_dense(ctx, rd(rng, 64, 0.3), 8)
    tau1 = 1e-4
    for _ in range(6):
        tau2 = tau1 * 10
        s2 = {tuple(x) for x in nat.survivors(ctx, A, B, tau2)}
        s1 = {tuple(x) for x in nat.survivors(ctx, A, B, tau1)}
        assert s2 <= s1
        tau1 = tau2


def test_conformability(ctx):  # test_multiply.cpp:158-163
    from paper_2005_10680_b200 import _native as nat
    a = nat.zero(ctx, 16, 8)
    with pytest.raises(ValueError):
        nat.multiply_exact(ctx, a, nat.zero(ctx, 24, 8))
    with pytest.raises(ValueError):
        nat.spamm(ctx, a, nat.zero(ctx, 16, 4), 0.0)
    with pytest.raises(ValueError):
        nat.spamm(ctx, a, a, -1.0)
    with pytest.raises(ValueError):
        nat.cse(ctx, a, nat.zero(ctx, 24, 8), [1.0])


def test_upload_errors(ctx):  # quadtree.cpp:202-216
    from paper_2005_10680_b200 import _native as nat
    blk = np.ones((1, 16))
    with pytest.raises(IndexError):
        nat.upload(ctx, 8, 4, [2], [0], blk)
    with pytest.raises(ValueError):
        nat.upload(ctx, 8, 4, [0, 0], [1, 1], np.ones((2, 16)))
    with pytest.raises(ValueError):
        nat.zero(ctx, 0, 4)


def test_cse_zero_factor(ctx):  # test_error_control.cpp:35-42
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    z = nat.zero(ctx, 16, 8)
    a = nat.from_dense(ctx, rd(np.random.default_rng(1), 16), 8)
    g = geometric_grid(1.0, 0.5, 20)
    assert np.all(nat.cse(ctx, z, a, g) == 0.0)
    assert np.all(nat.cse(ctx, a, z, g) == 0.0)


def test_single_leaf_bound(ctx):  # test_error_control.cpp:44-54
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(5)
    a = nat.from_dense(ctx, rd(rng, 8), 8)
    b = nat.from_dense(ctx, rd(rng, 8), 8)
    p = a.frobenius_norm * b.frobenius_norm
    bounds = nat.cse(ctx, a, b, [p * 4, p * 2, p * 0.5, p * 0.25])
    assert bounds[0] == p and bounds[1] == p and bounds[2] == 0.0 and bounds[3] == 0.0


def test_two_level_quadrature_attained(ctx):  # test_error_control.cpp:56-88
    from paper_2005_10680_b200 import _native as nat
    def single(vals):
        d = np.zeros((4, 4))
        for (br, bc), v in vals.items():
            d[2 * br, 2 * bc] = v
        return d
    da = single({(0, 0): 0.1, (0, 1): 0.1, (1, 0): 10.0, (1, 1): 1.0})
    db = single({(0, 0): 0.1, (0, 1): 10.0, (1, 0): 0.1, (1, 1): 0.011})
    a, b = nat.from_dense(ctx, da, 2), nat.from_dense(ctx, db, 2)
    bound = nat.cse(ctx, a, b, [0.02])[0]
    expected = np.sqrt((0.01 + 0.01) ** 2 + 0.0011 ** 2 + 0.011 ** 2)
    assert bound == pytest.approx(expected, rel=1e-12)
    realized = np.linalg.norm(nat.spamm(ctx, a, b, 0.02)[0].to_dense() - da @ db)
    assert realized == pytest.approx(expected, rel=1e-12)


def test_bounds_monotone_and_sweep_consistent(ctx):  # test_error_control.cpp:105-117
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    rng = np.random.default_rng(21)
    a = nat.from_dense(ctx, rd(rng, 48, 0.4), 8)
    b = nat.from_dense(ctx, rd(rng, 48, 0.4), 8)
    g = geometric_grid(1.0, 0.6, 40)
    joint = nat.cse(ctx, a, b, g)
    assert np.all(joint[1:] <= joint[:-1])
    for k in range(0, 40, 7):
        assert nat.cse(ctx, a, b, [g[k]])[0] == joint[k]  # exactly


def test_soundness(ctx):  # test_error_control.cpp:126-146
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    g = geometric_grid(1.0, 0.5, 50)
    checked = 0
    for seed in range(100):
        rng = np.random.default_rng(2000 + seed)
        n = 16 * (1 + seed % 4)
        da, db = rd(rng, n, 0.5), rd(rng, n, 0.5)
        a, b = nat.from_dense(ctx, da, 16), nat.from_dense(ctx, db, 16)
        bounds = nat.cse(ctx, a, b, g)
        exact = da @ db
        slack = 1e-10 * a.frobenius_norm * b.frobenius_norm
        for k in range(0, 50, 5):
            realized = np.linalg.norm(nat.spamm(ctx, a, b, g[k])[0].to_dense() - exact)
            assert realized <= bounds[k] + slack
            checked += 1
    assert checked >= 1000


def test_controlled_product_cases(ctx):  # test_error_control.cpp:238-285
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    z = nat.zero(ctx, 16, 8)
    C, st, _ = nat.spamm_with_error_control(ctx, z, z, 0.5, geometric_grid(1.0, 0.5, 10))
    assert C.nnz_blocks == 0 and st["tau"] == 1.0 and st["bound"] == 0.0

    rng = np.random.default_rng(71)
    d = rd(rng, 16)
    a = nat.from_dense(ctx, d, 8)
    huge = a.frobenius_norm ** 2 * 10
    C, st, _ = nat.spamm_with_error_control(ctx, a, a, huge, geometric_grid())
    assert st["bound"] < huge and np.linalg.norm(C.to_dense() - d @ d) < huge

    # decay pair at delta = 1e-5 (generate_decay_matrix-like 1-D decay)
    rng = np.random.default_rng(17)
    f = rd(rng, 96) * np.exp(-0.5 * np.abs(np.subtract.outer(np.arange(96), np.arange(96))))
    f = (f + f.T) / 2
    q = nat.from_dense(ctx, f, 16)
    C, st, _ = nat.spamm_with_error_control(ctx, q, q, 1e-5, geometric_grid())
    assert np.linalg.norm(C.to_dense() - f @ f) < 1e-5 and st["bound"] < 1e-5

    # impossible budget -> exact fallback, bitwise
    d = rd(np.random.default_rng(72), 16)
    d[:8, 8:] = 0.0
    d[0, 8] = 1e-30
    a = nat.from_dense(ctx, d, 8)
    C, st, _ = nat.spamm_with_error_control(ctx, a, a, 1e-300, geometric_grid(1.0, 0.5, 40))
    assert st["tau"] == 0.0 and st["bound"] == 0.0 and st["tau_index"] == -1
    assert bits_equal(C.to_dense(), nat.multiply_exact(ctx, a, a)[0].to_dense())

    with pytest.raises(ValueError):
        nat.spamm_with_error_control(ctx, z, z, 0.0, geometric_grid())


def test_underflow_corner_matches_oracle(ctx, port):
    """Subnormal squares make a parent norm smaller than a child norm
    (sqrt(fl(x*x)) < x); the top-down skip test and the p == 0 early-outs must
    still follow the reference recursion exactly."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    rng = np.random.default_rng(99)
    n, L = 32, 4
    da = rd(rng, n) * 1e-160
    da[:8, :8] = rd(rng, 8)
    db = rd(rng, n) * 1e150
    la, lb = nat.dense_to_leaves(da, L), nat.dense_to_leaves(db, L)
    A, B = nat.upload(ctx, n, L, *la), nat.upload(ctx, n, L, *lb)
    ta, tb = port.build(n, L, *la), port.build(n, L, *lb)
    for lvl in range(4):
        assert bits_equal(A.level_norms(lvl), ta.level_norms(lvl))
    g = geometric_grid(1e160, 1e-3, 110)
    assert bits_equal(nat.cse(ctx, A, B, g), port.cse(ta, tb, g))
    for tau in (1e-15, 1e-8, 1e-3, 0.0):
        assert np.array_equal(nat.survivors(ctx, A, B, tau), port.survivors(ta, tb, tau))
