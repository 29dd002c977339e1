// test_dropin.cpp -- the reference's hot-path unit tests, restated against the
// spamm-b200 C++ drop-in (include/spamm/*.hpp), i.e. the same API a caller of
// the reference (purification.cpp, experiment.cpp) would link against.
// Reference cases: /root/reference/proj/tests/test_multiply.cpp,
// test_error_control.cpp, test_quadtree.cpp.  No doctest in this image, so a
// minimal CHECK harness stands in.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "spamm/error_control.hpp"
#include "spamm/execution.hpp"
#include "spamm/multiply.hpp"
#include "spamm/oracle.hpp"
#include "spamm/purification.hpp"
#include "spamm/quadtree.hpp"

using spamm::CoordinateEntry;
using spamm::DenseMatrix;
using spamm::ErrorBoundVector;
using spamm::QuadTreeMatrix;
using spamm::SpammTolerance;
using spamm::ToleranceGrid;

static int g_checks = 0, g_failures = 0;
static const char* g_case = "";
#define CHECK(cond)                                                                   \
  do {                                                                                \
    ++g_checks;                                                                       \
    if (!(cond)) {                                                                    \
      ++g_failures;                                                                   \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond); \
    }                                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                     \
  do {                                                  \
    bool thrown = false;                                \
    try {                                               \
      (void)(expr);                                     \
    } catch (const type&) {                             \
      thrown = true;                                    \
    } catch (...) {                                     \
    }                                                   \
    CHECK(thrown && #type);                             \
  } while (0)

struct Case {
  const char* name;
  std::function<void()> fn;
};
static std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
#define TEST(id, name)                         \
  static void test_##id();                     \
  static Reg reg_##id(name, test_##id);        \
  static void test_##id()

// ---- test support (own restatement of the usual helpers) -------------------
struct Rng {
  std::mt19937_64 e;
  explicit Rng(uint64_t s) : e(s) {}
  double u01() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * u01(); }
  int uniform_int(int lo, int hi) { return lo + static_cast<int>(e() % static_cast<uint64_t>(hi - lo + 1)); }
};

static DenseMatrix random_dense(int n, uint64_t seed, double fill = 1.0) {
  Rng r(seed);
  DenseMatrix a(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (fill >= 1.0 || r.u01() < fill) a(i, j) = r.uniform(-1.0, 1.0);
  return a;
}
static bool bitwise_equal(const DenseMatrix& a, const DenseMatrix& b) {
  return a.dimension() == b.dimension() && std::memcmp(a.data(), b.data(), a.size() * 8) == 0;
}
static double frob(const DenseMatrix& a) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a.data()[i] * a.data()[i];
  return std::sqrt(s);
}
static double diff_frob(const DenseMatrix& a, const DenseMatrix& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double d = a.data()[i] - b.data()[i];
    s += d * d;
  }
  return std::sqrt(s);
}
static DenseMatrix dense_multiply(const DenseMatrix& a, const DenseMatrix& b) {
  const int n = a.dimension();
  DenseMatrix c(n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) c(i, j) += a(i, k) * b(k, j);
  return c;
}
static DenseMatrix padded(const DenseMatrix& a, int leaf) {
  int p = leaf;
  while (p < a.dimension()) p *= 2;
  DenseMatrix o(p);
  for (int i = 0; i < a.dimension(); ++i)
    for (int j = 0; j < a.dimension(); ++j) o(i, j) = a(i, j);
  return o;
}
static double region_norm(const DenseMatrix& a, int r0, int c0, int s) {
  double t = 0;
  for (int i = r0; i < r0 + s; ++i)
    for (int j = c0; j < c0 + s; ++j) t += a(i, j) * a(i, j);
  return std::sqrt(t);
}
// Independent dense recursions: skip decisions and bounds re-derived from
// region norms recomputed from raw entries (never touches the quadtree).
static void dense_spamm(const DenseMatrix& a, int ar, int ac, const DenseMatrix& b, int br, int bc,
                        int size, int leaf, double tau, DenseMatrix& out, int orow, int ocol) {
  const double na = region_norm(a, ar, ac, size), nb = region_norm(b, br, bc, size);
  if (na == 0.0 || nb == 0.0 || na * nb < tau) return;
  if (size == leaf) {
    for (int i = 0; i < leaf; ++i)
      for (int j = 0; j < leaf; ++j) {
        double s = 0;
        for (int k = 0; k < leaf; ++k) s += a(ar + i, ac + k) * b(br + k, bc + j);
        out(orow + i, ocol + j) += s;
      }
    return;
  }
  const int h = size / 2;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k)
        dense_spamm(a, ar + i * h, ac + k * h, b, br + k * h, bc + j * h, h, leaf, tau, out,
                    orow + i * h, ocol + j * h);
}
static std::vector<double> dense_cse(const DenseMatrix& a, int ar, int ac, const DenseMatrix& b,
                                     int br, int bc, int size, int leaf,
                                     const std::vector<double>& taus) {
  std::vector<double> e(taus.size(), 0.0);
  const double p = region_norm(a, ar, ac, size) * region_norm(b, br, bc, size);
  if (p == 0.0) return e;
  if (size == leaf) {
    for (size_t k = 0; k < taus.size(); ++k)
      if (p < taus[k]) e[k] = p;
    return e;
  }
  const int h = size / 2;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      auto e1 = dense_cse(a, ar + i * h, ac, b, br, bc + j * h, h, leaf, taus);
      auto e2 = dense_cse(a, ar + i * h, ac + h, b, br + h, bc + j * h, h, leaf, taus);
      for (size_t k = 0; k < e.size(); ++k) e[k] += (e1[k] + e2[k]) * (e1[k] + e2[k]);
    }
  for (double& v : e) v = std::sqrt(v);
  return e;
}
static DenseMatrix unpad(const DenseMatrix& a, int n) {
  DenseMatrix o(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) o(i, j) = a(i, j);
  return o;
}
static bool approx(double a, double b, double rel) {
  return std::fabs(a - b) <= rel * std::max(std::fabs(a), std::fabs(b)) + 1e-300;
}

// ---- quadtree ------------------------------------------------------------------
static void norm_walk(const QuadTreeMatrix::NodePtr& n, const DenseMatrix& pad, int r0, int c0,
                      int size, int leaf) {
  if (!n) {
    CHECK(region_norm(pad, r0, c0, size) == 0.0);
    return;
  }
  CHECK(approx(n->norm, region_norm(pad, r0, c0, size), 1e-12));
  CHECK(n->norm > 0.0);
  if (n->is_leaf()) {
    CHECK(static_cast<int>(n->block.size()) == leaf * leaf);
    return;
  }
  const int h = size / 2;
  for (int q = 0; q < 4; ++q) norm_walk(n->child[q], pad, r0 + (q >> 1) * h, c0 + (q & 1) * h, h, leaf);
}

TEST(quadtree_norm_cache, "cached norms match recomputed region norms; no all-zero nodes") {
  for (int leaf : {4, 8, 16}) {
    const DenseMatrix d = random_dense(50, 3 + leaf, 0.3);
    const auto q = QuadTreeMatrix::from_dense(d, leaf);
    norm_walk(q.root(), padded(d, leaf), 0, 0, q.padded_dimension(), leaf);
    CHECK(bitwise_equal(q.to_dense(), d));
    CHECK(approx(q.frobenius_norm(), frob(d), 1e-12));
  }
}

TEST(quadtree_coordinates, "from_coordinates validation and round trip") {
  std::vector<CoordinateEntry> e{{0, 0, 1.5}, {7, 3, -2.0}, {12, 12, 0.25}};
  const auto q = QuadTreeMatrix::from_coordinates(e, 13, 4);
  CHECK(q.to_dense()(7, 3) == -2.0 && q.nnz() == 3);
  CHECK(q.trace() == 1.75);
  std::vector<CoordinateEntry> bad{{13, 0, 1.0}};
  CHECK_THROWS_AS(QuadTreeMatrix::from_coordinates(bad, 13, 4), std::out_of_range);
  std::vector<CoordinateEntry> dup{{1, 1, 1.0}, {1, 1, 2.0}};
  CHECK_THROWS_AS(QuadTreeMatrix::from_coordinates(dup, 13, 4), std::invalid_argument);
  CHECK_THROWS_AS(QuadTreeMatrix::zero(0, 4), std::invalid_argument);
}

// ---- multiply (test_multiply.cpp) ---------------------------------------------
TEST(identity, "product with the identity reproduces the operand exactly") {
  const DenseMatrix d = random_dense(24, 41, 0.5);
  const auto a = QuadTreeMatrix::from_dense(d, 8);
  const auto id = QuadTreeMatrix::identity(24, 8);
  CHECK(bitwise_equal(multiply_exact(a, id).to_dense(), d));
  CHECK(bitwise_equal(multiply_exact(id, a).to_dense(), d));
}

TEST(zero_product, "product with zero is zero") {
  const auto a = QuadTreeMatrix::from_dense(random_dense(16, 42), 8);
  const auto z = QuadTreeMatrix::zero(16, 8);
  CHECK(multiply_exact(a, z).is_zero());
  CHECK(multiply_exact(z, a).is_zero());
  CHECK(spamm_multiply(a, z, {0.0}).is_zero());
}

TEST(exact_vs_dense, "exact product matches the dense oracle") {
  for (uint64_t seed : {1u, 2u, 3u}) {
    const DenseMatrix da = random_dense(64, seed, 0.6), db = random_dense(64, seed + 100, 0.6);
    const auto c = multiply_exact(QuadTreeMatrix::from_dense(da, 16), QuadTreeMatrix::from_dense(db, 16));
    const DenseMatrix r = dense_multiply(da, db);
    CHECK(diff_frob(c.to_dense(), r) / frob(r) < 1e-12);
  }
}

TEST(tau_zero_exact, "tau = 0 is bitwise identical to the exact product") {
  const auto a = QuadTreeMatrix::from_dense(random_dense(48, 7, 0.4), 16);
  const auto b = QuadTreeMatrix::from_dense(random_dense(48, 8, 0.4), 16);
  CHECK(bitwise_equal(spamm_multiply(a, b, {0.0}).to_dense(), multiply_exact(a, b).to_dense()));
}

TEST(tau_above_root, "tau above the root norm product skips everything") {
  const auto a = QuadTreeMatrix::from_dense(random_dense(16, 9), 8);
  const auto b = QuadTreeMatrix::from_dense(random_dense(16, 10), 8);
  CHECK(spamm_multiply(a, b, {a.frobenius_norm() * b.frobenius_norm() * 1.0001}).is_zero());
}

TEST(quadrant_pair, "a quadrant pair under tau is dropped, everything else kept") {
  DenseMatrix da(8), db(8);
  Rng rng(55);
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      da(i, j) = rng.uniform(0.5, 1.0) * ((i < 4 && j >= 4) ? 1e-4 : 1.0);
      db(i, j) = rng.uniform(0.5, 1.0) * ((i >= 4 && j < 4) ? 1e-4 : 1.0);
    }
  const double tau = region_norm(da, 0, 4, 4) * region_norm(db, 4, 0, 4) * 50.0;
  const DenseMatrix approx_c =
      spamm_multiply(QuadTreeMatrix::from_dense(da, 4), QuadTreeMatrix::from_dense(db, 4), {tau}).to_dense();
  DenseMatrix expect = dense_multiply(da, db);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double drop = 0;
      for (int k = 0; k < 4; ++k) drop += da(i, 4 + k) * db(4 + k, j);
      expect(i, j) -= drop;
    }
  CHECK(diff_frob(approx_c, expect) < 1e-13);
  DenseMatrix ref(8);
  dense_spamm(da, 0, 0, db, 0, 0, 8, 4, tau, ref, 0, 0);
  CHECK(diff_frob(approx_c, ref) < 1e-13);
}

TEST(random_vs_dense_recursion, "dense recursion agrees with spamm on random instances and taus") {
  Rng rng(77);
  for (int trial = 0; trial < 20; ++trial) {
    const int n = 8 * rng.uniform_int(2, 6);
    const DenseMatrix da = random_dense(n, 200 + trial, 0.5), db = random_dense(n, 300 + trial, 0.5);
    const double tau = std::pow(10.0, rng.uniform(-3.0, 1.0));
    const DenseMatrix got =
        spamm_multiply(QuadTreeMatrix::from_dense(da, 8), QuadTreeMatrix::from_dense(db, 8), {tau}).to_dense();
    const DenseMatrix pa = padded(da, 8), pb = padded(db, 8);
    DenseMatrix want(pa.dimension());
    dense_spamm(pa, 0, 0, pb, 0, 0, pa.dimension(), 8, tau, want, 0, 0);
    CHECK(diff_frob(got, unpad(want, n)) < 1e-12 * (1.0 + frob(want)));
  }
}

static void subset(const QuadTreeMatrix::NodePtr& sparser, const QuadTreeMatrix::NodePtr& denser) {
  if (!sparser) return;
  CHECK(denser != nullptr);
  if (!denser || sparser->is_leaf()) return;
  for (int q = 0; q < 4; ++q) subset(sparser->child[q], denser->child[q]);
}

TEST(monotone_structure, "larger tau keeps a subset of the structure") {
  const auto a = QuadTreeMatrix::from_dense(random_dense(64, 13, 0.3), 8);
  const auto b = QuadTreeMatrix::from_dense(random_dense(64, 14, 0.3), 8);
  double tau1 = 1e-4;
  for (int s = 0; s < 6; ++s) {
    const double tau2 = tau1 * 10;
    const auto c2 = spamm_multiply(a, b, {tau2});
    const auto c1 = spamm_multiply(a, b, {tau1});
    subset(c2.root(), c1.root());
    tau1 = tau2;
  }
}

TEST(thread_knob, "results are bitwise identical for every thread setting") {
  const auto a = QuadTreeMatrix::from_dense(random_dense(96, 15, 0.5), 16);
  const auto b = QuadTreeMatrix::from_dense(random_dense(96, 16, 0.5), 16);
  spamm::exec::set_max_threads(1);
  const DenseMatrix e1 = multiply_exact(a, b).to_dense(), s1 = spamm_multiply(a, b, {1e-3}).to_dense();
  spamm::exec::set_max_threads(8);
  CHECK(spamm::exec::spawn_levels() == 2);
  const DenseMatrix e8 = multiply_exact(a, b).to_dense(), s8 = spamm_multiply(a, b, {1e-3}).to_dense();
  spamm::exec::set_max_threads(1);
  CHECK(bitwise_equal(e1, e8) && bitwise_equal(s1, s8));
}

TEST(conformability, "conformability is enforced") {
  const auto a = QuadTreeMatrix::zero(16, 8);
  CHECK_THROWS_AS(multiply_exact(a, QuadTreeMatrix::zero(24, 8)), std::invalid_argument);
  CHECK_THROWS_AS(spamm_multiply(a, QuadTreeMatrix::zero(16, 4), {0.0}), std::invalid_argument);
  CHECK_THROWS_AS(spamm_multiply(a, a, {-1.0}), std::invalid_argument);
}

// ---- error control (test_error_control.cpp) -----------------------------------
TEST(grid, "grid validation") {
  const ToleranceGrid g = ToleranceGrid::geometric();
  CHECK(g.size() == 350 && g.taus().front() == 1.0);
  CHECK(approx(g.taus().back(), std::pow(0.9, 349), 1e-12));
  CHECK_THROWS_AS(ToleranceGrid({}), std::invalid_argument);
  CHECK_THROWS_AS(ToleranceGrid({1.0, 1.0}), std::invalid_argument);
  CHECK_THROWS_AS(ToleranceGrid({1.0, -0.5}), std::invalid_argument);
  CHECK_THROWS_AS(ToleranceGrid::geometric(1.0, 1.5, 10), std::invalid_argument);
  CHECK_THROWS_AS(ToleranceGrid::geometric(0.0, 0.9, 10), std::invalid_argument);
  CHECK_THROWS_AS(ToleranceGrid::geometric(1.0, 0.9, 0), std::invalid_argument);
}

TEST(cse_zero, "cse returns zeros when either factor is zero") {
  const auto z = QuadTreeMatrix::zero(16, 8);
  const auto a = QuadTreeMatrix::from_dense(random_dense(16, 1), 8);
  for (double v : cse(z, a, ToleranceGrid::geometric(1.0, 0.5, 20)).bounds) CHECK(v == 0.0);
  for (double v : cse(a, z, ToleranceGrid::geometric(1.0, 0.5, 20)).bounds) CHECK(v == 0.0);
}

TEST(single_leaf, "single-leaf bound is the norm product below tau, zero above") {
  const auto a = QuadTreeMatrix::from_dense(random_dense(8, 5), 8);
  const auto b = QuadTreeMatrix::from_dense(random_dense(8, 6), 8);
  const double p = a.frobenius_norm() * b.frobenius_norm();
  const ErrorBoundVector e = cse(a, b, ToleranceGrid({p * 4.0, p * 2.0, p * 0.5, p * 0.25}));
  CHECK(e.bounds[0] == p && e.bounds[1] == p && e.bounds[2] == 0.0 && e.bounds[3] == 0.0);
}

TEST(two_level, "two-level bound combines quadrant sums in quadrature") {
  auto put = [](std::vector<CoordinateEntry>& e, int br, int bc, double v) { e.push_back({2 * br, 2 * bc, v}); };
  std::vector<CoordinateEntry> ea, eb;
  put(ea, 0, 0, 0.1); put(ea, 0, 1, 0.1); put(ea, 1, 0, 10.0); put(ea, 1, 1, 1.0);
  put(eb, 0, 0, 0.1); put(eb, 0, 1, 10.0); put(eb, 1, 0, 0.1); put(eb, 1, 1, 0.011);
  const auto a = QuadTreeMatrix::from_coordinates(ea, 4, 2);
  const auto b = QuadTreeMatrix::from_coordinates(eb, 4, 2);
  const double bound = cse(a, b, ToleranceGrid({0.02})).bounds[0];
  const double expected = std::sqrt(0.02 * 0.02 + 0.0011 * 0.0011 + 0.011 * 0.011);
  CHECK(approx(bound, expected, 1e-12));
  const double realized = diff_frob(spamm_multiply(a, b, {0.02}).to_dense(),
                                    dense_multiply(a.to_dense(), b.to_dense()));
  CHECK(approx(realized, expected, 1e-12));
}

TEST(cse_vs_dense, "cse agrees with the independent dense recursion") {
  const ToleranceGrid g = ToleranceGrid::geometric(1.0, 0.4, 30);
  for (uint64_t seed = 0; seed < 8; ++seed) {
    const int n = 8 * (2 + static_cast<int>(seed % 5));
    const DenseMatrix da = random_dense(n, 900 + seed, 0.35), db = random_dense(n, 950 + seed, 0.35);
    const auto got = cse(QuadTreeMatrix::from_dense(da, 8), QuadTreeMatrix::from_dense(db, 8), g);
    const DenseMatrix pa = padded(da, 8), pb = padded(db, 8);
    const auto want = dense_cse(pa, 0, 0, pb, 0, 0, pa.dimension(), 8, g.taus());
    for (size_t k = 0; k < want.size(); ++k) CHECK(approx(got.bounds[k], want[k], 1e-12));
  }
}

TEST(monotone_bounds, "bounds are monotone in tau and sweep-consistent") {
  const ToleranceGrid g = ToleranceGrid::geometric(1.0, 0.6, 40);
  const auto a = QuadTreeMatrix::from_dense(random_dense(48, 21, 0.4), 8);
  const auto b = QuadTreeMatrix::from_dense(random_dense(48, 22, 0.4), 8);
  const ErrorBoundVector joint = cse(a, b, g);
  for (size_t k = 1; k < g.size(); ++k) CHECK(joint.bounds[k] <= joint.bounds[k - 1]);
  for (size_t k = 0; k < g.size(); k += 7)
    CHECK(cse(a, b, ToleranceGrid({g.taus()[k]})).bounds[0] == joint.bounds[k]);
}

TEST(select, "select_tolerance picks the largest candidate under delta") {
  const ToleranceGrid g({1.0, 0.1, 0.01});
  CHECK(select_tolerance(ErrorBoundVector{{0.5, 0.09, 0.0}}, g, 0.1).tau == 0.1);
  CHECK(select_tolerance(ErrorBoundVector{{0.0, 0.0, 0.0}}, g, 1e-9).tau == 1.0);
  CHECK(select_tolerance(ErrorBoundVector{{0.5, 0.2, 0.1}}, g, 0.05).tau == 0.0);
}

TEST(soundness, "soundness: realized error never exceeds the bound") {
  const ToleranceGrid g = ToleranceGrid::geometric(1.0, 0.5, 50);
  int checked = 0;
  for (uint64_t seed = 0; seed < 100; ++seed) {
    const int n = 16 * (1 + static_cast<int>(seed % 4));
    const DenseMatrix da = random_dense(n, 2000 + seed, 0.5), db = random_dense(n, 3000 + seed, 0.5);
    const auto a = QuadTreeMatrix::from_dense(da, 16), b = QuadTreeMatrix::from_dense(db, 16);
    const ErrorBoundVector e = cse(a, b, g);
    const DenseMatrix exact = dense_multiply(da, db);
    const double slack = 1e-10 * a.frobenius_norm() * b.frobenius_norm();
    for (size_t k = 0; k < g.size(); k += 5) {
      CHECK(diff_frob(spamm_multiply(a, b, {g.taus()[k]}).to_dense(), exact) <= e.bounds[k] + slack);
      ++checked;
    }
  }
  CHECK(checked >= 1000);
}

TEST(controlled, "error-controlled product meets its budget") {
  {
    const auto z = QuadTreeMatrix::zero(16, 8);
    const auto r = spamm_with_error_control(z, z, 0.5, ToleranceGrid::geometric(1.0, 0.5, 10));
    CHECK(r.matrix.is_zero() && r.chosen_tau.tau == 1.0 && r.bound == 0.0);
    CHECK_THROWS_AS(spamm_with_error_control(z, z, 0.0, ToleranceGrid::geometric()), std::invalid_argument);
  }
  {
    const auto a = QuadTreeMatrix::from_dense(random_dense(16, 71), 8);
    const double huge = a.frobenius_norm() * a.frobenius_norm() * 10.0;
    const auto r = spamm_with_error_control(a, a, huge, ToleranceGrid::geometric());
    CHECK(r.bound < huge);
    CHECK(diff_frob(r.matrix.to_dense(), dense_multiply(a.to_dense(), a.to_dense())) < huge);
  }
  {
    DenseMatrix d = random_dense(16, 72);
    for (int i = 0; i < 8; ++i)
      for (int j = 8; j < 16; ++j) d(i, j) = 0.0;
    d(0, 8) = 1e-30;
    const auto a = QuadTreeMatrix::from_dense(d, 8);
    const auto r = spamm_with_error_control(a, a, 1e-300, ToleranceGrid::geometric(1.0, 0.5, 40));
    CHECK(r.chosen_tau.tau == 0.0 && r.bound == 0.0);
    CHECK(bitwise_equal(r.matrix.to_dense(), multiply_exact(a, a).to_dense()));
  }
}

TEST(truncate_cases, "truncate: identity at zero budget, greedy prefix otherwise") {
  const auto x = QuadTreeMatrix::from_dense(random_dense(32, 31, 0.4), 8);
  const auto same = spamm::truncate(x, 0.0);
  CHECK(same.matrix.root() == x.root() && same.removed_block_count == 0);
  const auto all = spamm::truncate(x, x.frobenius_norm() * 1.01);
  CHECK(all.matrix.is_zero() && all.removed_block_count == x.nnz_blocks());
  std::vector<CoordinateEntry> e{{0, 0, 0.9}, {0, 4, 0.1}, {4, 0, 0.2}};
  const auto r = spamm::truncate(QuadTreeMatrix::from_coordinates(e, 8, 4), 0.25);
  CHECK(r.removed_block_count == 2 && approx(r.removed_norm_bound, std::sqrt(0.05), 1e-14));
  CHECK_THROWS_AS(spamm::truncate(x, -1.0), std::invalid_argument);
}

TEST(add_scale, "add and scale follow the reference semantics") {
  const DenseMatrix da = random_dense(40, 5, 0.3), db = random_dense(40, 6, 0.3);
  const auto a = QuadTreeMatrix::from_dense(da, 8), b = QuadTreeMatrix::from_dense(db, 8);
  const DenseMatrix s = spamm::add(a, b).to_dense();
  bool ok = true;
  for (int i = 0; i < 40; ++i)
    for (int j = 0; j < 40; ++j) ok = ok && s(i, j) == da(i, j) + db(i, j);
  CHECK(ok);
  CHECK(spamm::add(a, a.scale(-1.0)).is_zero());
  CHECK(a.scale(0.0).is_zero());
}

// ---- purification (test_purification.cpp) -------------------------------------
static QuadTreeMatrix diag_matrix(const std::vector<double>& v, int leaf) {
  std::vector<CoordinateEntry> e;
  for (size_t i = 0; i < v.size(); ++i) e.push_back({static_cast<int>(i), static_cast<int>(i), v[i]});
  return QuadTreeMatrix::from_coordinates(e, static_cast<int>(v.size()), leaf);
}

TEST(purify_transform, "initial transform maps the spectrum into [0, 1] reversed") {
  const auto id = QuadTreeMatrix::identity(8, 4);
  CHECK(bitwise_equal(spamm::initial_transform(id.scale(0.0), {0.0, 2.0}).to_dense(), id.to_dense()));
  CHECK(spamm::initial_transform(id.scale(2.0), {0.0, 2.0}).is_zero());
  DenseMatrix expect(3);
  expect(0, 0) = 1.0;
  expect(1, 1) = 0.75;
  CHECK(bitwise_equal(spamm::initial_transform(diag_matrix({-1.0, 0.0, 3.0}, 4), {-1.0, 3.0}).to_dense(), expect));
  CHECK_THROWS_AS(spamm::initial_transform(id, {1.0, 1.0}), std::invalid_argument);
}

TEST(purify_sp2, "sp2 selection, budget, and convergence to the projector") {
  CHECK(spamm::sp2_step(diag_matrix({0.9, 0.3}, 2), 1).polynomial == spamm::Sp2Polynomial::square);
  CHECK(spamm::sp2_step(diag_matrix({1.5, 0.5}, 2), 2).polynomial ==
        spamm::Sp2Polynomial::trace_correcting);
  const auto b = spamm::ErrorBudget::geometric(1e-5, 40);
  CHECK(b.initial_delta == 5e-6 && approx(b.total(), 1e-5, 1e-12));
  DenseMatrix expect(4);
  expect(0, 0) = 1.0;
  expect(1, 1) = 1.0;
  for (auto v : {spamm::Variant::truncmul, spamm::Variant::spamm, spamm::Variant::hybrid}) {
    spamm::PurificationConfig cfg;
    cfg.variant = v;
    cfg.occupation = 2;
    cfg.epsilon = 1e-6;
    const auto r = spamm::purify(diag_matrix({0.9, 0.8, 0.2, 0.1}, 4), cfg);
    CHECK(r.converged);
    CHECK(diff_frob(r.density.to_dense(), expect) < 1e-6);
    CHECK(!r.log.empty() && r.log.back().status == "converged");
  }
  spamm::PurificationConfig bad;
  bad.occupation = 0;
  CHECK_THROWS_AS(spamm::purify(diag_matrix({1.0, 0.0}, 2), bad), std::invalid_argument);
}

static const spamm::Variant kVariants[] = {spamm::Variant::truncmul, spamm::Variant::spamm,
                                           spamm::Variant::hybrid};

TEST(purify_idempotent_start, "an idempotent start with the right trace converges at once") {
  const auto proj = diag_matrix({1.0, 1.0, 0.0, 0.0}, 4);
  for (auto v : kVariants) {
    spamm::PurificationConfig cfg;
    cfg.variant = v;
    cfg.occupation = 2;
    cfg.epsilon = 1e-6;
    const auto r = spamm::purify(proj, cfg);
    CHECK(r.converged && r.iterations == 0);
    CHECK(bitwise_equal(r.density.to_dense(), proj.to_dense()));
    CHECK(!r.log.empty() && r.log.back().status == "converged");
  }
}

TEST(purify_per_iteration, "each logged iteration meets its own tolerance") {
  for (auto v : kVariants) {
    spamm::PurificationConfig cfg;
    cfg.variant = v;
    cfg.occupation = 2;
    cfg.epsilon = 1e-6;
    const auto r = spamm::purify(diag_matrix({0.9, 0.8, 0.2, 0.1}, 4), cfg);
    for (const auto& rec : r.log)
      if (rec.status != "converged") CHECK(rec.status == "ok" && rec.realized_error < rec.tolerance);
  }
}

TEST(purify_zero_budget, "a zero budget makes every variant exact and identical") {
  spamm::oracle::DecayModelSpec spec;
  spec.dimension = 48;
  spec.alpha = 0.6;
  spec.seed = 5;
  const DenseMatrix f = spamm::oracle::generate_decay_matrix(spec);
  const auto x0 = spamm::initial_transform(QuadTreeMatrix::from_dense(f, 16), {0.0, 2.0});
  std::vector<DenseMatrix> dens;
  std::vector<int> its;
  std::vector<std::vector<double>> tr;
  for (auto v : kVariants) {
    spamm::PurificationConfig cfg;
    cfg.variant = v;
    cfg.occupation = 12;
    cfg.epsilon = 1e-9;
    cfg.budget = [](double, int n) {
      spamm::ErrorBudget b;
      b.deltas.assign(static_cast<size_t>(n), 0.0);
      return b;
    };
    const auto r = spamm::purify(x0, cfg);
    CHECK(r.converged);
    dens.push_back(r.density.to_dense());
    its.push_back(r.iterations);
    std::vector<double> t;
    for (const auto& rec : r.log) t.push_back(rec.trace);
    tr.push_back(t);
  }
  for (int k = 1; k < 3; ++k) {
    CHECK(its[k] == its[0]);
    CHECK(bitwise_equal(dens[k], dens[0]));
    CHECK(tr[k] == tr[0]);
  }
}

TEST(purify_vs_eigensolver, "decay-model purification matches the eigensolver projector") {
  spamm::oracle::DecayModelSpec spec;
  spec.dimension = 128;
  spec.alpha = 0.55;
  spec.seed = 9;
  const DenseMatrix f = spamm::oracle::generate_decay_matrix(spec);
  const DenseMatrix proj = spamm::oracle::density_matrix_oracle(f, 32);
  const auto x0 = spamm::initial_transform(QuadTreeMatrix::from_dense(f, 32), {0.0, 2.0});
  for (auto v : kVariants) {
    spamm::PurificationConfig cfg;
    cfg.variant = v;
    cfg.occupation = 32;
    cfg.epsilon = 1e-5;
    const auto r = spamm::purify(x0, cfg);
    CHECK(r.converged);
    CHECK(diff_frob(r.density.to_dense(), proj) < 1e-5);
    CHECK(std::abs(r.density.trace() - 32.0) < 1e-3);
    for (const auto& rec : r.log)
      if (rec.status != "converged") CHECK(rec.realized_error < rec.tolerance);
  }
}

TEST(purify_cap_and_validation, "iteration cap reports non-convergence; bad configs throw") {
  spamm::oracle::DecayModelSpec spec;
  spec.dimension = 64;
  spec.alpha = 0.5;
  spec.seed = 21;
  const auto x0 = spamm::initial_transform(
      QuadTreeMatrix::from_dense(spamm::oracle::generate_decay_matrix(spec), 32), {0.0, 2.0});
  spamm::PurificationConfig cfg;
  cfg.variant = spamm::Variant::hybrid;
  cfg.occupation = 16;
  cfg.epsilon = 1e-6;
  cfg.max_iterations = 2;
  const auto r = spamm::purify(x0, cfg);
  CHECK(!r.converged && r.iterations == 2 && r.log.size() >= 2);
  const auto small = diag_matrix({1.0, 0.0}, 2);
  spamm::PurificationConfig bad;
  bad.occupation = 2;  // == dimension
  CHECK_THROWS_AS(spamm::purify(small, bad), std::invalid_argument);
  bad.occupation = 1;
  bad.epsilon = 0.0;
  CHECK_THROWS_AS(spamm::purify(small, bad), std::invalid_argument);
  bad.epsilon = 1e-6;
  bad.max_iterations = 0;
  CHECK_THROWS_AS(spamm::purify(small, bad), std::invalid_argument);
  CHECK_THROWS_AS(spamm::ErrorBudget::geometric(0.0, 10), std::invalid_argument);
  CHECK_THROWS_AS(spamm::ErrorBudget::geometric(1e-5, 0), std::invalid_argument);
}

int main() {
  for (const Case& c : cases()) {
    g_case = c.name;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_failures;
      std::fprintf(stderr, "EXCEPTION [%s]: %s\n", c.name, e.what());
    }
  }
  std::printf("%d cases, %d checks, %d failures\n", static_cast<int>(cases().size()), g_checks, g_failures);
  return g_failures ? 1 : 0;
}
