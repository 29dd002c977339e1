// test_experiment.cpp -- the drop-in's experiment-side modules (SURVEY 8f row
// 4: MatrixMarket I/O, the squaring / purification runners, device Gershgorin
// bounds and RunRecord CSV / JSON output) against the reference itself,
// loaded from oracle/_ref/libspamm_ref.so (the unmodified reference sources,
// namespace-renamed, with C entry points in oracle/ref_adapter.cpp).
//
// The reference's dense test helpers (spamm::oracle::generate_decay_matrix,
// density_matrix_oracle) are NOT in the product library: this program links
// oracle/_ref/libspamm_dense_oracle.so (the unmodified src/oracle.cpp) and
// registers them with spamm::set_experiment_oracle, as a reference caller
// (the CLI) would.
//
//   test_experiment host OUTDIR   -- no GPU: the linked dense oracle is the
//                                    reference's, MatrixMarket reading, emit,
//                                    the unregistered-generator error
//   test_experiment gpu OUTDIR    -- experiments, Gershgorin, MatrixMarket writing
#include <dlfcn.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "spamm/experiment.hpp"
#include "spamm/matrix_market.hpp"
#include "spamm/oracle.hpp"
#include "spamm/quadtree.hpp"

using namespace spamm;

static int g_checks = 0, g_failures = 0;
static std::string g_case;
#define CHECK(cond)                                                                       \
  do {                                                                                    \
    ++g_checks;                                                                           \
    if (!(cond)) {                                                                        \
      ++g_failures;                                                                       \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                     \
  } while (0)

static bool bits_equal(const double* a, const double* b, std::size_t n) {
  return std::memcmp(a, b, n * sizeof(double)) == 0;
}

// ---- the reference, through its C adapter ---------------------------------
struct Ref {
  void* h = nullptr;
  int (*generate_decay)(int, double, double, double, double, std::uint64_t, double*) = nullptr;
  void (*gershgorin)(const double*, int, double*, double*) = nullptr;
  int (*density_oracle)(const double*, int, int, double*) = nullptr;
  int (*mm_read)(const char*, int*, std::int64_t*, std::int32_t*, std::int32_t*, double*,
                 std::int64_t) = nullptr;
  std::int64_t (*mm_write)(const void*, char*, std::int64_t) = nullptr;
  void* (*from_dense)(int, int, const double*) = nullptr;
  void (*free_tree)(void*) = nullptr;
  int (*squaring)(const void*, int, const double*, int, const double*, int, double*) = nullptr;

  explicit Ref(const std::string& path) {
    h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
    };
    sym(generate_decay, "ref_generate_decay");
    sym(gershgorin, "ref_gershgorin");
    sym(density_oracle, "ref_density_oracle");
    sym(mm_read, "ref_mm_read");
    sym(mm_write, "ref_mm_write");
    sym(from_dense, "ref_from_dense");
    sym(free_tree, "ref_free");
    sym(squaring, "ref_squaring");
  }
  bool ok() const { return h && generate_decay && mm_read && squaring; }
};

static int our_status(const std::function<void()>& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::domain_error&) {
    return 2;
  } catch (const std::exception&) {
    return 3;
  }
}

// ---- host-side cases --------------------------------------------------------
// the linked dense oracle is the reference's (same bits as libspamm_ref's copy)
static void test_generator(const Ref& ref) {
  g_case = "generate_decay_matrix";
  struct P {
    int n;
    double alpha, scale, lo, hi;
    std::uint64_t seed;
  };
  const P cases[] = {{1, 0.5, 0.3, 0.0, 2.0, 0}, {37, 0.5, 0.3, 0.0, 2.0, 7},
                     {200, 0.2, 0.1, -1.0, 1.0, 123456789}, {64, 1.5, 0.9, -3.0, 3.0, 42},
                     {50, 0.05, 0.5, 0.0, 1.0, 3} /* infeasible: domain_error */,
                     {0, 0.5, 0.3, 0.0, 2.0, 1} /* invalid */};
  for (const P& p : cases) {
    oracle::DecayModelSpec spec;
    spec.dimension = p.n;
    spec.alpha = p.alpha;
    spec.scale = p.scale;
    spec.spectral_low = p.lo;
    spec.spectral_high = p.hi;
    spec.seed = p.seed;
    DenseMatrix ours;
    const int so = our_status([&] { ours = oracle::generate_decay_matrix(spec); });
    std::vector<double> theirs(static_cast<std::size_t>(std::max(p.n, 1)) * std::max(p.n, 1));
    const int sr = ref.generate_decay(p.n, p.alpha, p.scale, p.lo, p.hi, p.seed, theirs.data());
    CHECK(so == sr);
    if (so == 0 && sr == 0) {
      CHECK(bits_equal(ours.data(), theirs.data(), ours.size()));
    }
  }
}

// a generated-input config with no generator registered fails loudly
static void test_unregistered_generator() {
  g_case = "unregistered generator";
  set_experiment_oracle({});
  ExperimentConfig cfg;
  cfg.generated = oracle::DecayModelSpec{};
  cfg.generated->dimension = 8;
  cfg.tolerances = {1e-3};
  bool threw = false;
  try {
    run_squaring_experiment(cfg);
  } catch (const std::logic_error& e) {
    threw = std::string(e.what()).find("set_experiment_oracle") != std::string::npos;
  }
  CHECK(threw);
}

// spamm::gershgorin_bounds on the device leaves == the reference's dense
// oracle::gershgorin_bounds (oracle.cpp:191-200), bit for bit
static void test_gershgorin(const Ref& ref) {
  g_case = "gershgorin_bounds";
  struct P {
    int n, leaf;
    double alpha, scale, lo, hi;
    std::uint64_t seed;
  };
  const P cases[] = {{1, 4, 0.5, 0.3, 0.0, 2.0, 0}, {37, 4, 0.5, 0.3, 0.0, 2.0, 7},
                     {200, 16, 0.2, 0.1, -1.0, 1.0, 123456789}, {64, 32, 1.5, 0.9, -3.0, 3.0, 42}};
  for (const P& p : cases) {
    oracle::DecayModelSpec spec;
    spec.dimension = p.n;
    spec.alpha = p.alpha;
    spec.scale = p.scale;
    spec.spectral_low = p.lo;
    spec.spectral_high = p.hi;
    spec.seed = p.seed;
    DenseMatrix d = oracle::generate_decay_matrix(spec);
    for (std::size_t i = 3; i < d.size(); i += 11) d.data()[i] = 0.0;  // ragged sparsity
    double lo = 0, hi = 0;
    ref.gershgorin(d.data(), p.n, &lo, &hi);
    const auto b = gershgorin_bounds(QuadTreeMatrix::from_dense(d, p.leaf));
    CHECK(b.first == lo && b.second == hi);
  }
}

// the linked dense oracle is the reference's (same bits as libspamm_ref's copy)
static void test_density_oracle(const Ref& ref) {
  g_case = "density_matrix_oracle";
  oracle::DecayModelSpec spec;
  spec.dimension = 40;
  spec.seed = 11;
  spec.spectral_low = -1.0;
  spec.spectral_high = 1.0;
  const DenseMatrix f = oracle::generate_decay_matrix(spec);
  for (int occ : {0, 1, 17, 40}) {
    const DenseMatrix d = oracle::density_matrix_oracle(f, occ);
    std::vector<double> r(f.size());
    CHECK(ref.density_oracle(f.data(), 40, occ, r.data()) == 0);
    CHECK(bits_equal(d.data(), r.data(), d.size()));
    double tr = 0;
    for (int i = 0; i < 40; ++i) tr += d(i, i);
    CHECK(std::abs(tr - occ) < 1e-10);
  }
  DenseMatrix asym(3);
  asym(0, 1) = 1.0;
  CHECK(our_status([&] { oracle::density_matrix_oracle(asym, 1); }) == 1);
  CHECK(our_status([&] { oracle::density_matrix_oracle(f, 41); }) == 1);
  // dense_multiply / dense_frobenius agree with a plain restatement
  const DenseMatrix p = oracle::dense_multiply(f, f);
  double acc = 0;
  for (int k = 0; k < 40; ++k) acc += f(3, k) * f(k, 5);
  CHECK(std::abs(p(3, 5) - acc) <= 1e-15);
}

static void test_mm_read(const Ref& ref) {
  g_case = "read_matrix_market";
  const std::vector<std::string> texts = {
      "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.5\n3 2 -2e-300\n",
      "%%MATRIXMARKET Matrix Coordinate REAL General\n% comment\n\n2 2 3\n% c\n1 2 0.1\n\n2 1 "
      "3\n2 2 1e308\n",
      "%%MatrixMarket matrix coordinate real general\n4 4 0\n",
      "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 0.30000000000000004\n",
      "",                                                                        // empty
      "%%NotMatrixMarket matrix coordinate real general\n1 1 0\n",               // banner
      "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",               // field
      "%%MatrixMarket matrix coordinate real symmetric\n1 1 0\n",                // symmetry
      "%%MatrixMarket matrix array real general\n1 1\n1\n",                      // format
      "%%MatrixMarket matrix coordinate real general\n2 3 0\n",                  // rectangular
      "%%MatrixMarket matrix coordinate real general\n0 0 0\n",                  // dimension
      "%%MatrixMarket matrix coordinate real general\n% only comments\n",        // no size
      "%%MatrixMarket matrix coordinate real general\nthree 3 1\n",              // bad size
      "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n",           // truncated
      "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 x 1\n",           // bad entry
      "%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n",           // range
      "%%MatrixMarket matrix coordinate real general\n3 3 1\n0 1 1\n",           // range
  };
  for (const std::string& t : texts) {
    std::istringstream in(t);
    CoordinateData ours;
    const int so = our_status([&] { ours = read_matrix_market(in); });
    int dim = 0;
    std::int64_t cnt = 0;
    std::vector<std::int32_t> r(16), c(16);
    std::vector<double> v(16);
    const int sr = ref.mm_read(t.c_str(), &dim, &cnt, r.data(), c.data(), v.data(), 16);
    CHECK(so == sr);
    if (so == 0 && sr == 0) {
      CHECK(ours.dimension == dim && static_cast<std::int64_t>(ours.entries.size()) == cnt);
      for (std::int64_t i = 0; i < cnt && i < static_cast<std::int64_t>(ours.entries.size()); ++i) {
        CHECK(ours.entries[i].row == r[i] && ours.entries[i].col == c[i]);
        CHECK(std::memcmp(&ours.entries[i].value, &v[i], sizeof(double)) == 0);
      }
    }
  }
  CHECK(our_status([] { read_matrix_market_file("/nonexistent/x.mtx"); }) == 3);
}

static std::vector<RunRecord> sample_records() {
  RunRecord a;
  a.variant = "spamm";
  a.iteration = 2;
  a.tolerance = 1e-6;
  a.chosen_tau = 7.4296395075949501e-09;
  a.t_spamm = 0.125;
  a.t_cse = 3.0;
  a.nnz_in = 123;
  a.nnz_mid = 456;
  a.nnz_out = 789;
  a.nnz_blocks_out = 10;
  a.realized_error = 0.1 + 0.2;
  a.status = "ok";
  a.trace = 2.0;
  RunRecord b = a;
  b.variant = "hybrid";
  b.status = "violation";
  b.realized_error = std::numeric_limits<double>::infinity();
  b.iteration = 7;
  return {a, b};
}

static void test_emit(const std::string& outdir) {
  g_case = "emit";
  const auto recs = sample_records();
  std::ostringstream csv;
  emit(recs, csv, OutputFormat::csv);
  const std::string s = csv.str();
  CHECK(s.rfind(std::string(kCsvHeader) + "\n", 0) == 0);
  CHECK(s.find("\nspamm,2,9.9999999999999995e-07,7.4296395075949501e-09,0,0,0.125,3,123,456,789,"
               "10,0.30000000000000004,ok\n") != std::string::npos);
  CHECK(any_violation(recs));
  CHECK(!any_violation({recs[0]}));
  emit_file(recs, outdir + "/records.csv", OutputFormat::csv);
  emit_file(recs, outdir + "/records.json", OutputFormat::json);
  emit_file({}, outdir + "/empty.json", OutputFormat::json);
  CHECK(our_status([&] { emit_file(recs, "/nonexistent/dir/x.csv", OutputFormat::csv); }) == 3);
}

// ---- GPU cases --------------------------------------------------------------
static void test_mm_write(const Ref& ref, const std::string& outdir) {
  g_case = "write_matrix_market";
  for (int n : {1, 45, 100}) {
    oracle::DecayModelSpec spec;
    spec.dimension = n;
    spec.seed = static_cast<std::uint64_t>(n);
    DenseMatrix d = oracle::generate_decay_matrix(spec);
    for (std::size_t i = 0; i < d.size(); i += 7) d.data()[i] = 0.0;  // explicit zeros
    for (int leaf : {4, 16, 32}) {
      const QuadTreeMatrix x = QuadTreeMatrix::from_dense(d, leaf);
      std::ostringstream ours;
      write_matrix_market(ours, x);
      void* t = ref.from_dense(n, leaf, d.data());
      const std::int64_t len = ref.mm_write(t, nullptr, 0);
      std::string theirs(static_cast<std::size_t>(len), '\0');
      ref.mm_write(t, theirs.data(), len);
      ref.free_tree(t);
      CHECK(ours.str() == theirs);
      // and it reads back to the same matrix, bitwise
      std::istringstream in(ours.str());
      const CoordinateData back = read_matrix_market(in);
      const DenseMatrix y = QuadTreeMatrix::from_coordinates(back.entries, back.dimension, leaf)
                                .to_dense();
      CHECK(y == x.to_dense());
    }
  }
  const QuadTreeMatrix z = QuadTreeMatrix::zero(10, 4);
  std::ostringstream zo;
  write_matrix_market(zo, z);
  CHECK(zo.str() == "%%MatrixMarket matrix coordinate real general\n10 10 0\n");
  write_matrix_market_file(outdir + "/z.mtx", z);
  CHECK(read_matrix_market_file(outdir + "/z.mtx").dimension == 10);
}

static void test_squaring(const Ref& ref, const std::string& outdir) {
  g_case = "run_squaring_experiment";
  oracle::DecayModelSpec spec;
  spec.dimension = 300;
  spec.alpha = 0.7;
  spec.scale = 0.2;
  spec.seed = 2005;
  ExperimentConfig cfg;
  cfg.generated = spec;
  cfg.tolerances = {1e-3, 1e-5, 1e-7};
  cfg.leaf_size = 16;
  const auto recs = run_squaring_experiment(cfg);
  CHECK(recs.size() == 9);
  const DenseMatrix d = oracle::generate_decay_matrix(spec);
  void* t = ref.from_dense(spec.dimension, cfg.leaf_size, d.data());
  const std::vector<double> taus(cfg.grid.taus().begin(), cfg.grid.taus().end());
  for (int vi = 0; vi < 3; ++vi) {
    std::vector<double> r9(9 * cfg.tolerances.size());
    CHECK(ref.squaring(t, vi, cfg.tolerances.data(), static_cast<int>(cfg.tolerances.size()),
                       taus.data(), static_cast<int>(taus.size()), r9.data()) == 0);
    for (std::size_t i = 0; i < cfg.tolerances.size(); ++i) {
      const RunRecord& r = recs[vi * cfg.tolerances.size() + i];
      const double* o = &r9[9 * i];
      CHECK(r.variant == std::string(to_string(static_cast<Variant>(vi))));
      CHECK(r.iteration == 2 && r.tolerance == cfg.tolerances[i]);
      CHECK(r.chosen_tau == o[0]);
      CHECK(r.nnz_in == static_cast<std::int64_t>(o[1]));
      CHECK(r.nnz_mid == static_cast<std::int64_t>(o[2]));
      CHECK(r.nnz_out == static_cast<std::int64_t>(o[3]));
      CHECK(r.nnz_blocks_out == static_cast<std::int64_t>(o[4]));
      CHECK(std::abs(r.realized_error - o[5]) <= 1e-6 * o[5] + 1e-15);
      CHECK((r.status == "ok") == (o[6] == 0.0));
      CHECK(std::abs(r.trace - o[7]) <= 1e-12 * std::abs(o[7]));
      CHECK(r.status == "ok");
    }
  }
  ref.free_tree(t);
  emit_file(recs, outdir + "/squaring.csv", OutputFormat::csv);
  // a MatrixMarket input gives the same records as the generated one
  {
    const QuadTreeMatrix x = QuadTreeMatrix::from_dense(d, cfg.leaf_size);
    write_matrix_market_file(outdir + "/decay300.mtx", x);
    ExperimentConfig c2 = cfg;
    c2.generated.reset();
    c2.matrix_file = outdir + "/decay300.mtx";
    c2.variants = {Variant::spamm};
    c2.tolerances = {1e-5};
    const auto r2 = run_squaring_experiment(c2);
    CHECK(r2.size() == 1 && r2[0].chosen_tau == recs[4].chosen_tau &&
          r2[0].nnz_out == recs[4].nnz_out);
  }
  ExperimentConfig bad = cfg;
  bad.tolerances = {};
  CHECK(our_status([&] { run_squaring_experiment(bad); }) == 1);
  bad = cfg;
  bad.tolerances = {0.0};
  CHECK(our_status([&] { run_squaring_experiment(bad); }) == 1);
  bad = cfg;
  bad.matrix_file = "x.mtx";
  CHECK(our_status([&] { run_squaring_experiment(bad); }) == 1);
  bad = cfg;
  bad.generated.reset();
  CHECK(our_status([&] { run_squaring_experiment(bad); }) == 1);
}

static void test_purification(const std::string& outdir) {
  g_case = "run_purification_experiment";
  oracle::DecayModelSpec spec;
  spec.dimension = 160;
  spec.alpha = 0.6;
  spec.scale = 0.05;
  spec.spectral_low = -1.0;
  spec.spectral_high = 1.0;
  spec.seed = 77;
  ExperimentConfig cfg;
  cfg.generated = spec;
  cfg.occupation = 80;
  cfg.epsilon = 1e-5;
  cfg.max_iterations = 60;
  cfg.leaf_size = 16;
  const auto recs = run_purification_experiment(cfg);
  int summaries = 0;
  for (const RunRecord& r : recs) {
    if (r.status.rfind("final", 0) == 0 || r.status == "no-convergence") {
      ++summaries;
      CHECK(r.status == "final-ok");
      CHECK(r.realized_error < cfg.epsilon);
      CHECK(std::abs(r.trace - cfg.occupation) < 1e-3);
    }
  }
  CHECK(summaries == 3);
  CHECK(!any_violation(recs));
  emit_file(recs, outdir + "/purification.json", OutputFormat::json);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  const std::string outdir = argc > 2 ? argv[2] : "/tmp";
  const std::string refpath = argc > 3 ? argv[3] : "oracle/_ref/libspamm_ref.so";
  Ref ref(refpath);
  if (!ref.ok()) {
    std::printf("reference library not loadable (%s): %s\n", refpath.c_str(), dlerror());
    return 2;
  }
  try {
    if (mode == "host") {
      test_unregistered_generator();
      set_experiment_oracle({&oracle::generate_decay_matrix, &oracle::density_matrix_oracle});
      test_generator(ref);
      test_density_oracle(ref);
      test_mm_read(ref);
      test_emit(outdir);
    } else {
      set_experiment_oracle({&oracle::generate_decay_matrix, &oracle::density_matrix_oracle});
      test_gershgorin(ref);
      test_mm_write(ref, outdir);
      test_squaring(ref, outdir);
      test_purification(outdir);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "FAIL [%s] uncaught: %s\n", g_case.c_str(), e.what());
    ++g_failures;
  }
  std::printf("%d checks, %d failures\n", g_checks, g_failures);
  return g_failures ? 1 : 0;
}
