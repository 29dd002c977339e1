"""SP2 purification over the GPU product (BASELINE
config 3's caller): the reference's purification tests
(test_purification.cpp) restated through the C ABI, plus a per-iteration
comparison with the reference driver itself (oracle/_ref) on a decay model."""
import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu

VARIANTS = ["truncmul", "spamm", "hybrid"]


def diagonal(nat, ctx, values, leaf):
    return nat.from_dense(ctx, np.diag(np.asarray(values, np.float64)), leaf)


def decay_matrix(n, alpha, seed, low=0.0, high=2.0, scale=0.3):
    """Symmetric decay model with Gershgorin-placed diagonal (the idea of
    oracle.cpp:156-189; own numpy generator)."""
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    env = scale * np.exp(-alpha * np.abs(np.subtract.outer(i, i)))
    a = np.triu(rng.uniform(-1, 1, (n, n)) * env, 1)
    a = a + a.T
    radius = np.abs(a).sum(axis=1)
    width = high - low
    assert np.all(2 * radius <= width)
    a[i, i] = low + radius + rng.uniform(size=n) * (width - 2 * radius)
    return a


def initial_transform(nat, ctx, f, lo, hi, leaf):  # purification.cpp:49-57 on the device
    F = nat.from_dense(ctx, f, leaf)
    I = nat.identity(ctx, f.shape[0], leaf)
    shifted = nat.axpby(ctx, hi, I, -1.0, F)
    return nat.axpby(ctx, 1.0 / (hi - lo), shifted)


def test_device_algebra_matches_reference_semantics(ctx):
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(3)
    a = np.where(rng.uniform(size=(40, 40)) < 0.3, rng.uniform(-1, 1, (40, 40)), 0.0)
    b = np.where(rng.uniform(size=(40, 40)) < 0.3, rng.uniform(-1, 1, (40, 40)), 0.0)
    A, B = nat.from_dense(ctx, a, 8), nat.from_dense(ctx, b, 8)
    assert bits_equal(nat.axpby(ctx, 2.0, A, -1.0, B).to_dense(), 2.0 * a + (-1.0) * b)
    assert nat.axpby(ctx, 1.0, A, -1.0, A).nnz_blocks == 0
    assert nat.axpby(ctx, 0.0, A).nnz_blocks == 0
    assert nat.nnz(A) == np.count_nonzero(a)
    # trace in node_trace's association (pairwise over diagonal blocks)
    blocks = [sum(a[8 * k + i, 8 * k + i] for i in range(8)) for k in range(5)] + [0.0] * 3
    while len(blocks) > 1:
        blocks = [blocks[2 * i] + blocks[2 * i + 1] for i in range(len(blocks) // 2)]
    assert nat.trace(A) == blocks[0]
    assert bits_equal(nat.identity(ctx, 13, 4).to_dense(), np.eye(13))


def test_initial_transform_and_sp2_cases(ctx):  # test_purification.cpp:33-88
    from paper_2005_10680_b200 import _native as nat
    x0 = initial_transform(nat, ctx, np.diag([-1.0, 0.0, 3.0]), -1.0, 3.0, 4)
    expect = np.zeros((3, 3))
    expect[0, 0], expect[1, 1] = 1.0, 0.75
    assert bits_equal(x0.to_dense(), expect)
    assert initial_transform(nat, ctx, 2.0 * np.eye(8), 0.0, 2.0, 4).nnz_blocks == 0
    p = diagonal(nat, ctx, [1.0, 1.0, 0.0, 0.0], 4)
    p2, _ = nat.multiply_exact(ctx, p, p)
    assert bits_equal(p2.to_dense(), p.to_dense())
    assert bits_equal(nat.axpby(ctx, 2.0, p, -1.0, p2).to_dense(), p.to_dense())


def test_budget_geometric():  # test_purification.cpp:90-104
    from paper_2005_10680_b200 import _native as nat
    d0, d = nat.error_budget_geometric(1e-5, 40)
    assert d0 == 5e-6 and np.all(d > 0) and np.all(np.diff(d) < 0)
    assert d.sum() == pytest.approx(5e-6, rel=1e-12)
    with pytest.raises(ValueError):
        nat.error_budget_geometric(0.0, 10)
    with pytest.raises(ValueError):
        nat.error_budget_geometric(1e-5, 0)


@pytest.mark.parametrize("variant", VARIANTS)
def test_idempotent_and_diagonal_starts(ctx, variant):  # :106-142
    from paper_2005_10680_b200 import _native as nat
    p = diagonal(nat, ctx, [1.0, 1.0, 0.0, 0.0], 4)
    D, log, conv, its = nat.purify(ctx, p, variant, 2, epsilon=1e-6)
    assert conv and its == 0 and log[-1]["status"] == "converged"
    assert bits_equal(D.to_dense(), p.to_dense())
    x0 = diagonal(nat, ctx, [0.9, 0.8, 0.2, 0.1], 4)
    D, log, conv, its = nat.purify(ctx, x0, variant, 2, epsilon=1e-6)
    assert conv
    assert np.linalg.norm(D.to_dense() - np.diag([1.0, 1.0, 0.0, 0.0])) < 1e-6
    for rec in log:
        if rec["status"] != "converged":
            assert rec["status"] == "ok" and rec["realized_error"] < rec["tolerance"]


def test_zero_budget_variant_equivalence(ctx):  # :144-183
    from paper_2005_10680_b200 import _native as nat
    f = decay_matrix(48, 0.6, 5)
    x0 = initial_transform(nat, ctx, f, 0.0, 2.0, 16)
    finals, counts, traces = [], [], []
    for v in VARIANTS:
        D, log, conv, its = nat.purify(ctx, x0, v, 12, epsilon=1e-9,
                                       budget=(0.0, np.zeros(100)))
        assert conv
        finals.append(D.to_dense())
        counts.append(its)
        traces.append([r["trace"] for r in log])
    assert counts[1] == counts[0] == counts[2]
    assert bits_equal(finals[1], finals[0]) and bits_equal(finals[2], finals[0])
    assert traces[1] == traces[0] == traces[2]


@pytest.mark.parametrize("variant", VARIANTS)
def test_decay_model_tracks_eigensolver(ctx, variant):  # :185-204
    from paper_2005_10680_b200 import _native as nat
    f = decay_matrix(128, 0.55, 9)
    w, v = np.linalg.eigh(f)
    ref = v[:, :32] @ v[:, :32].T
    x0 = initial_transform(nat, ctx, f, 0.0, 2.0, 32)
    D, log, conv, its = nat.purify(ctx, x0, variant, 32, epsilon=1e-5)
    assert conv
    d = D.to_dense()
    assert np.linalg.norm(d - ref) < 1e-5
    assert abs(np.trace(d) - 32.0) < 1e-3
    for rec in log:
        if rec["status"] != "converged":
            # late deltas shrink below the FP64 rounding of the product sums
            # themselves (~1e-17 here): below that floor the comparison measures
            # summation-order noise, not skipped products
            assert rec["realized_error"] < max(rec["tolerance"], 1e-15)


def test_iteration_cap_and_validation(ctx):  # :206-223
    from paper_2005_10680_b200 import _native as nat
    f = decay_matrix(64, 0.5, 21)
    x0 = initial_transform(nat, ctx, f, 0.0, 2.0, 32)
    D, log, conv, its = nat.purify(ctx, x0, "hybrid", 16, epsilon=1e-6, max_iterations=2)
    assert not conv and its == 2 and len(log) >= 2
    x = diagonal(nat, ctx, [1.0, 0.0], 2)
    for kw in ({"occupation": 0}, {"occupation": 2}, {"occupation": 1, "epsilon": 0.0},
               {"occupation": 1, "max_iterations": 0}):
        args = dict(epsilon=1e-6, max_iterations=10)
        args.update(kw)
        occ = args.pop("occupation")
        with pytest.raises(ValueError):
            nat.purify(ctx, x, "hybrid", occ, **args)


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_against_reference_driver(ctx, ref, variant):
    """Same x0 bits, same budget: the reference's purify and ours agree on the
    polynomial path, the first iteration's tau bit for bit, and the density."""
    from paper_2005_10680_b200 import _native as nat
    from paper_2005_10680_b200.inputs import geometric_grid
    f = decay_matrix(256, 0.5, 77)
    x0 = initial_transform(nat, ctx, f, 0.0, 2.0, 16)
    r, c, p, _ = x0.download()
    tx = ref.build(256, 16, r, c, p)
    taus = geometric_grid()
    d0, deltas = nat.error_budget_geometric(1e-5, 60)
    name = ["truncmul", "spamm", "hybrid"][variant]
    D, log, conv, its = nat.purify(ctx, x0, name, 64, epsilon=1e-5, max_iterations=60,
                                   taus=taus, budget=(d0, deltas))
    T, rlog, rconv, rits = ref.purify(tx, variant, 64, 60, 1e-5, taus, d0, deltas)
    assert conv == rconv and its == rits and len(log) == len(rlog)
    first = 1 if variant != 1 else 0
    assert log[first]["chosen_tau"] == rlog[first][2]
    for mine, theirs in zip(log, rlog):
        assert mine["trace"] == pytest.approx(theirs[3], abs=1e-9)
        assert mine["status"] == ("ok", "violation", "converged")[int(theirs[1])]
    rr, rc_, rp, _ = T.leaves()
    dr = nat.leaves_to_dense(256, 16, rr, rc_, rp)
    assert np.linalg.norm(D.to_dense() - dr) < 1e-9


def test_row_data_and_diagonal_matrices(ctx):
    """spg_matrix_rows (diagonal, sum_j |a_ij|) and spg_matrix_from_diagonal
    against numpy, ragged last block included."""
    from paper_2005_10680_b200 import _native as nat
    rng = np.random.default_rng(4)
    n, L = 333, 16
    d = np.where(rng.uniform(size=(n, n)) < 0.3, rng.uniform(-1, 1, (n, n)), 0.0)
    d[:, 50:70] = 0.0
    A = nat.from_dense(ctx, d, L)
    diag, rs = nat.row_data(A)
    assert np.array_equal(diag, np.diag(d))
    ref = np.array([sum(abs(x) for x in row) for row in d])  # ascending j, sequential
    assert np.array_equal(rs, ref)
    v = rng.uniform(-2, 2, n)
    D = nat.from_diagonal(ctx, v, L)
    assert np.array_equal(D.to_dense(), np.diag(v))
    assert nat.trace(D) == pytest.approx(v.sum(), rel=1e-14)


def test_gershgorin_bounds_match_reference(ctx):
    """spg_matrix_gershgorin (device row scan, j != i) equals the reference's
    oracle::gershgorin_bounds on the dense matrix bit for bit
    (oracle.cpp:191-200), ragged last block and empty block columns included."""
    import ctypes
    import oracle
    from paper_2005_10680_b200 import _native as nat
    if not oracle.available("ref"):
        pytest.skip("reference build (oracle/_ref) not present")
    R = oracle.Oracle("ref")
    f = R.L.ref_gershgorin
    f.restype = None
    f.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                  ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    rng = np.random.default_rng(9)
    for n, L in ((333, 16), (64, 64), (1000, 32)):
        d = np.where(rng.uniform(size=(n, n)) < 0.3, rng.uniform(-1, 1, (n, n)), 0.0)
        d = d + d.T + np.diag(rng.uniform(-3, 3, n))
        d[:, n // 3:n // 3 + 20] = 0.0
        d = np.ascontiguousarray(d)
        lo, hi = ctypes.c_double(), ctypes.c_double()
        f(d.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, ctypes.byref(lo),
          ctypes.byref(hi))
        got = nat.gershgorin(nat.from_dense(ctx, d, L))
        assert got == (lo.value, hi.value)


def test_device_algebra_matches_reference_build(ctx):
    """trace / nnz / scale / add on the device (spg_matrix_trace, _nnz, _axpby:
    what the drop-in's QuadTreeMatrix::trace/nnz/scale and spamm::add call)
    against the reference build's own QuadTreeMatrix methods (quadtree.cpp:
    231-261): trace bitwise, nnz exact, every leaf's payload and norm bitwise,
    the same null leaves (zero-collapse included)."""
    import oracle
    from paper_2005_10680_b200 import _native as nat
    if not oracle.available("ref"):
        pytest.skip("reference build (oracle/_ref) not present")
    R = oracle.Oracle("ref")
    rng = np.random.default_rng(21)
    for n, L in ((333, 16), (256, 32), (100, 8)):
        a = np.where(rng.uniform(size=(n, n)) < 0.2, rng.uniform(-1, 1, (n, n)), 0.0)
        b = np.where(rng.uniform(size=(n, n)) < 0.2, rng.uniform(-1, 1, (n, n)), 0.0)
        b[: n // 2, : n // 2] = -a[: n // 2, : n // 2]  # a + b cancels -> leaves collapse
        b[n // 2:, :] = 0.0
        A, B = nat.from_dense(ctx, a, L), nat.from_dense(ctx, b, L)
        r, c, p, _ = A.download()
        RA = R.build(n, L, r, c, p)
        r, c, p, _ = B.download()
        RB = R.build(n, L, r, c, p)
        assert nat.trace(A) == R.trace(RA)
        assert nat.nnz(A) == R.nnz(RA)
        for alpha, beta, use_b in ((1.0, 1.0, True), (2.5, -0.75, True), (-1.0, 0.0, False),
                                   (1e-300, 0.0, False)):
            got = nat.axpby(ctx, alpha, A, beta, B) if use_b else nat.axpby(ctx, alpha, A)
            want = R.axpby(alpha, RA, beta, RB if use_b else None)
            gr, gc, gp, gn = got.download()
            wr, wc, wp, wn = want.leaves()
            assert np.array_equal(gr, wr) and np.array_equal(gc, wc)
            assert gp.tobytes() == wp.tobytes() and gn.tobytes() == wn.tobytes()
            assert nat.trace(got) == R.trace(want) and nat.nnz(got) == R.nnz(want)
