// ref_adapter.cpp -- C entry points over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own core sources (/root/reference/proj/core/src/*.cpp, built in
// place, never copied) into oracle/_ref/libspamm_ref.so with
// -Dspamm=spamm_ref.  It exposes the same C signatures as oracle/spamm_oracle.h
// with a `ref_` prefix so tests can pin the C restatement, and the GPU path,
// against the reference itself.  Trees are assembled with the reference's
// own node helpers (node_ops.hpp:40-63) and QuadTreeMatrix::wrap
// (quadtree.hpp:87-89), so norms follow the reference rule by construction.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <vector>
#include <thread>
#include <atomic>

#include "node_ops.hpp"
#include <sstream>
#include <string>

#include "spamm/error_control.hpp"
#include "spamm/execution.hpp"
#include "spamm/matrix_market.hpp"
#include "spamm/oracle.hpp"
#include "spamm/multiply.hpp"
#include "spamm/purification.hpp"
#include "spamm/quadtree.hpp"

namespace {

using spamm::QuadTreeMatrix;
using NodePtr = QuadTreeMatrix::NodePtr;
using Node = QuadTreeMatrix::Node;

struct RefTree {
  QuadTreeMatrix m;
  int depth = 0;
};

std::uint64_t morton2(std::uint32_t r, std::uint32_t c, int depth) {
  std::uint64_t key = 0;
  for (int b = depth - 1; b >= 0; --b) key = (key << 2) | (((r >> b) & 1u) << 1) | ((c >> b) & 1u);
  return key;
}

int depth_of(int padded, int leaf) {
  int d = 0;
  while ((leaf << d) < padded) ++d;
  return d;
}

struct Builder {
  const std::vector<std::pair<std::uint64_t, std::int64_t>>* order;
  const double* data;
  std::int64_t block;
  int depth;
  bool norm_only;

  NodePtr build(std::int64_t lo, std::int64_t hi, int level) const {
    if (lo >= hi) return nullptr;
    if (level == depth) {
      const std::int64_t src = (*order)[lo].second;
      if (norm_only) {
        const double nrm = data[src];
        if (nrm < 0.0) return nullptr;
        auto n = std::make_shared<Node>();
        n->norm = nrm;
        n->block = {nrm};  // size-1 payload marks a leaf; cse_node never reads it
        return n;
      }
      std::vector<double> blk(data + src * block, data + (src + 1) * block);
      return spamm::detail::make_leaf(std::move(blk));
    }
    const int shift = 2 * (depth - level - 1);
    std::array<NodePtr, 4> child;
    std::int64_t start = lo;
    for (int c = 0; c < 4; ++c) {
      std::int64_t end = start;
      while (end < hi && static_cast<int>(((*order)[end].first >> shift) & 3u) == c) ++end;
      child[c] = build(start, end, level + 1);
      start = end;
    }
    return spamm::detail::make_inner(std::move(child));
  }
};

RefTree* build_common(int dimension, int leaf, std::int64_t n, const std::int32_t* rows,
                      const std::int32_t* cols, const double* data, bool norm_only) {
  try {
    const QuadTreeMatrix zero = QuadTreeMatrix::zero(dimension, leaf);
    const int depth = depth_of(zero.padded_dimension(), leaf);
    const std::int64_t limit = (dimension + leaf - 1) / leaf;
    std::vector<std::pair<std::uint64_t, std::int64_t>> order(static_cast<std::size_t>(n));
    for (std::int64_t t = 0; t < n; ++t) {
      if (rows[t] < 0 || cols[t] < 0 || rows[t] >= limit || cols[t] >= limit) return nullptr;
      order[t] = {morton2(rows[t], cols[t], depth), t};
    }
    std::sort(order.begin(), order.end());
    for (std::size_t t = 1; t < order.size(); ++t)
      if (order[t].first == order[t - 1].first) return nullptr;
    Builder b{&order, data, static_cast<std::int64_t>(leaf) * leaf, depth, norm_only};
    auto* out = new RefTree;
    out->m = QuadTreeMatrix::wrap(b.build(0, n, 0), dimension, leaf);
    out->depth = depth;
    return out;
  } catch (const std::exception&) {
    return nullptr;
  }
}

void walk_leaves(const NodePtr& n, int level, int depth, std::int32_t r, std::int32_t c,
                 std::int64_t block, std::int64_t& next, std::int32_t* rows, std::int32_t* cols,
                 double* payload, double* norms) {
  if (!n) return;
  if (level == depth) {
    const std::int64_t at = next++;
    if (rows) rows[at] = r;
    if (cols) cols[at] = c;
    if (norms) norms[at] = n->norm;
    if (payload) {
      if (static_cast<std::int64_t>(n->block.size()) == block)
        std::memcpy(payload + at * block, n->block.data(), sizeof(double) * block);
      else
        std::memset(payload + at * block, 0, sizeof(double) * block);
    }
    return;
  }
  for (int q = 0; q < 4; ++q)
    walk_leaves(n->child[q], level + 1, depth, 2 * r + (q >> 1), 2 * c + (q & 1), block, next,
                rows, cols, payload, norms);
}

void walk_level(const NodePtr& n, int level, int target, std::uint64_t key, double* out) {
  if (!n) return;
  if (level == target) {
    out[key] = n->norm;
    return;
  }
  for (int q = 0; q < 4; ++q) walk_level(n->child[q], level + 1, target, key * 4 + q, out);
}

std::int64_t count_leaves(const NodePtr& n, int level, int depth) {
  if (!n) return 0;
  if (level == depth) return 1;
  std::int64_t s = 0;
  for (const auto& c : n->child) s += count_leaves(c, level + 1, depth);
  return s;
}

// The decisions of spamm_node (multiply.cpp:70-92) replayed on reference trees.
void surv_walk(const NodePtr& a, const NodePtr& b, int level, int depth, double tau, bool skip,
               std::int32_t I, std::int32_t K, std::int32_t J,
               std::vector<std::array<std::int32_t, 3>>* out, std::int64_t& count) {
  if (!a || !b) return;
  if (skip && a->norm * b->norm < tau) return;
  if (level == depth) {
    ++count;
    if (out) out->push_back({I, K, J});
    return;
  }
  for (int row = 0; row < 2; ++row)
    for (int col = 0; col < 2; ++col)
      for (int h = 0; h < 2; ++h)
        surv_walk(a->child[2 * row + h], b->child[2 * h + col], level + 1, depth, tau, skip,
                  2 * I + row, 2 * K + h, 2 * J + col, out, count);
}

std::uint64_t digest_mix(std::uint64_t z) {  // SplitMix64 finaliser (spg_survivor_digest)
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// spamm_node's decisions (multiply.cpp:70-92) on reference trees, reduced to
// (count, sum of digest_mix(i << 42 | k << 21 | j))
void digest_walk(const NodePtr& a, const NodePtr& b, int level, int depth, double tau,
                 std::uint64_t I, std::uint64_t K, std::uint64_t J, std::int64_t& count,
                 std::uint64_t& sum) {
  if (!a || !b) return;
  if (a->norm * b->norm < tau) return;
  if (level == depth) {
    ++count;
    sum += digest_mix((I << 42) | (K << 21) | J);
    return;
  }
  for (int row = 0; row < 2; ++row)
    for (int col = 0; col < 2; ++col)
      for (int h = 0; h < 2; ++h)
        digest_walk(a->child[2 * row + h], b->child[2 * h + col], level + 1, depth, tau,
                    2 * I + row, 2 * K + h, 2 * J + col, count, sum);
}

struct WalkTask {
  NodePtr a, b;
  std::uint64_t I, K, J;
};

// the surviving level-`top` triples (the same skip test above them)
void collect_tasks(const NodePtr& a, const NodePtr& b, int level, int top, double tau,
                   std::uint64_t I, std::uint64_t K, std::uint64_t J, std::vector<WalkTask>& out) {
  if (!a || !b) return;
  if (a->norm * b->norm < tau) return;
  if (level == top) {
    out.push_back({a, b, I, K, J});
    return;
  }
  for (int row = 0; row < 2; ++row)
    for (int col = 0; col < 2; ++col)
      for (int h = 0; h < 2; ++h)
        collect_tasks(a->child[2 * row + h], b->child[2 * h + col], level + 1, top, tau,
                      2 * I + row, 2 * K + h, 2 * J + col, out);
}

}  // namespace

extern "C" {

// Survivor-set digest of spamm_multiply(a, b, tau): the reference trees' own
// norms and skip rule, walked on `threads` host threads (the sum is order-free)
void ref_survivor_digest(const void* a, const void* b, double tau, int threads,
                         std::int64_t* count, std::uint64_t* digest) {
  const auto* ra = static_cast<const RefTree*>(a);
  const auto* rb = static_cast<const RefTree*>(b);
  const int depth = ra->depth;
  const int top = std::min(depth, 4);
  std::vector<WalkTask> tasks;
  collect_tasks(ra->m.root(), rb->m.root(), 0, top, tau, 0, 0, 0, tasks);
  std::atomic<std::size_t> next{0};
  std::vector<std::int64_t> counts(static_cast<std::size_t>(std::max(threads, 1)), 0);
  std::vector<std::uint64_t> sums(counts.size(), 0);
  std::vector<std::thread> pool;
  for (std::size_t t = 0; t < counts.size(); ++t)
    pool.emplace_back([&, t] {
      for (std::size_t i = next++; i < tasks.size(); i = next++)
        digest_walk(tasks[i].a, tasks[i].b, top, depth, tau, tasks[i].I, tasks[i].K, tasks[i].J,
                    counts[t], sums[t]);
    });
  for (auto& th : pool) th.join();
  *count = 0;
  *digest = 0;
  for (std::size_t t = 0; t < counts.size(); ++t) {
    *count += counts[t];
    *digest += sums[t];
  }
}

void* ref_build(int dimension, int leaf, std::int64_t n, const std::int32_t* rows,
                const std::int32_t* cols, const double* payload) {
  return build_common(dimension, leaf, n, rows, cols, payload, false);
}

void* ref_build_norm_only(int dimension, int leaf, std::int64_t n, const std::int32_t* rows,
                          const std::int32_t* cols, const double* norms) {
  return build_common(dimension, leaf, n, rows, cols, norms, true);
}

// QuadTreeMatrix::from_dense (quadtree.cpp:224-229) on a row-major host array.
void* ref_from_dense(int dimension, int leaf, const double* rowmajor) {
  try {
    spamm::DenseMatrix d(dimension);
    std::memcpy(d.data(), rowmajor, sizeof(double) * d.size());
    auto* out = new RefTree;
    out->m = QuadTreeMatrix::from_dense(d, leaf);
    out->depth = depth_of(out->m.padded_dimension(), leaf);
    return out;
  } catch (const std::exception&) {
    return nullptr;
  }
}

void ref_free(void* t) { delete static_cast<RefTree*>(t); }

void ref_set_max_threads(int threads) { spamm::exec::set_max_threads(threads); }

int ref_depth(const void* t) { return static_cast<const RefTree*>(t)->depth; }
std::int64_t ref_nnz_blocks(const void* t) {
  const auto* r = static_cast<const RefTree*>(t);
  return count_leaves(r->m.root(), 0, r->depth);
}
double ref_frobenius(const void* t) { return static_cast<const RefTree*>(t)->m.frobenius_norm(); }

void ref_leaves(const void* t, std::int32_t* rows, std::int32_t* cols, double* payload,
                double* norms) {
  const auto* r = static_cast<const RefTree*>(t);
  std::int64_t next = 0;
  walk_leaves(r->m.root(), 0, r->depth, 0, 0,
              static_cast<std::int64_t>(r->m.leaf_size()) * r->m.leaf_size(), next, rows, cols,
              payload, norms);
}

void ref_level_norms(const void* t, int level, double* out) {
  const auto* r = static_cast<const RefTree*>(t);
  const std::uint64_t count = 1ull << (2 * level);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = -1.0;
  walk_level(r->m.root(), 0, level, 0, out);
}

// QuadTreeMatrix::trace / nnz (quadtree.cpp:231-233)
double ref_trace(const void* t) { return static_cast<const RefTree*>(t)->m.trace(); }
std::int64_t ref_nnz(const void* t) { return static_cast<const RefTree*>(t)->m.nnz(); }

// add(a.scale(alpha), b.scale(beta)) (quadtree.cpp:249-261); b may be null
void* ref_axpby(double alpha, const void* a, double beta, const void* b) {
  try {
    const auto* ra = static_cast<const RefTree*>(a);
    auto* out = new RefTree;
    out->depth = ra->depth;
    QuadTreeMatrix x = ra->m.scale(alpha);
    if (b) x = spamm::add(x, static_cast<const RefTree*>(b)->m.scale(beta));
    out->m = std::move(x);
    return out;
  } catch (const std::exception&) {
    return nullptr;
  }
}

// spamm::cse (error_control.cpp:160-166)
int ref_cse(const void* a, const void* b, const double* taus, int n, double* bounds) {
  try {
    const spamm::ToleranceGrid grid(std::vector<double>(taus, taus + n));
    const auto e = spamm::cse(static_cast<const RefTree*>(a)->m, static_cast<const RefTree*>(b)->m,
                              grid);
    std::memcpy(bounds, e.bounds.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// cse_node for the pair A(I,K) x B(K,J) at `level`: spamm::cse on the two
// subtrees wrapped as matrices of the subtree size (same recursion).
int ref_cse_subtree(const void* a, const void* b, const double* taus, int n, int level,
                    std::int32_t I, std::int32_t K, std::int32_t J, double* out) {
  try {
    const auto* ra = static_cast<const RefTree*>(a);
    const auto* rb = static_cast<const RefTree*>(b);
    auto at = [&](NodePtr nd, std::int32_t r, std::int32_t c) {
      for (int l = level - 1; l >= 0 && nd; --l) nd = nd->child[2 * ((r >> l) & 1) + ((c >> l) & 1)];
      return nd;
    };
    const int size = ra->m.padded_dimension() >> level;
    const auto sa = QuadTreeMatrix::wrap(at(ra->m.root(), I, K), size, ra->m.leaf_size());
    const auto sb = QuadTreeMatrix::wrap(at(rb->m.root(), K, J), size, rb->m.leaf_size());
    const spamm::ToleranceGrid grid(std::vector<double>(taus, taus + n));
    const auto e = spamm::cse(sa, sb, grid);
    std::memcpy(out, e.bounds.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// spamm::select_tolerance (error_control.cpp:168-172); returns tau (0 = exact).
double ref_select_tolerance(const double* bounds, const double* taus, int n, double delta) {
  const spamm::ToleranceGrid grid(std::vector<double>(taus, taus + n));
  return spamm::select_tolerance(spamm::ErrorBoundVector{std::vector<double>(bounds, bounds + n)},
                                 grid, delta)
      .tau;
}

void* ref_spamm(const void* a, const void* b, double tau, int* status) {
  try {
    auto* out = new RefTree;
    out->m = spamm::spamm_multiply(static_cast<const RefTree*>(a)->m,
                                   static_cast<const RefTree*>(b)->m, spamm::SpammTolerance{tau});
    out->depth = static_cast<const RefTree*>(a)->depth;
    if (status) *status = 0;
    return out;
  } catch (const std::exception&) {
    if (status) *status = -1;
    return nullptr;
  }
}

void* ref_multiply_exact(const void* a, const void* b, int* status) {
  try {
    auto* out = new RefTree;
    out->m = spamm::multiply_exact(static_cast<const RefTree*>(a)->m,
                                   static_cast<const RefTree*>(b)->m);
    out->depth = static_cast<const RefTree*>(a)->depth;
    if (status) *status = 0;
    return out;
  } catch (const std::exception&) {
    if (status) *status = -1;
    return nullptr;
  }
}

// spamm::spamm_with_error_control (error_control.cpp:203-220).
void* ref_spamm_with_error_control(const void* a, const void* b, double delta, const double* taus,
                                   int n, double* tau_out, double* bound_out, double* cse_seconds,
                                   double* spamm_seconds, int* status) {
  try {
    const spamm::ToleranceGrid grid(std::vector<double>(taus, taus + n));
    auto res = spamm::spamm_with_error_control(static_cast<const RefTree*>(a)->m,
                                               static_cast<const RefTree*>(b)->m, delta, grid);
    auto* out = new RefTree;
    out->m = std::move(res.matrix);
    out->depth = static_cast<const RefTree*>(a)->depth;
    if (tau_out) *tau_out = res.chosen_tau.tau;
    if (bound_out) *bound_out = res.bound;
    if (cse_seconds) *cse_seconds = res.cse_seconds;
    if (spamm_seconds) *spamm_seconds = res.spamm_seconds;
    if (status) *status = 0;
    return out;
  } catch (const std::exception&) {
    if (status) *status = -1;
    return nullptr;
  }
}

// spamm::truncate (error_control.cpp:174-201)
void* ref_truncate(const void* x, double delta, double* removed_norm, std::int64_t* removed_count,
                   int* status) {
  try {
    const auto* r = static_cast<const RefTree*>(x);
    auto res = spamm::truncate(r->m, delta);
    auto* out = new RefTree;
    out->m = std::move(res.matrix);
    out->depth = r->depth;
    if (removed_norm) *removed_norm = res.removed_norm_bound;
    if (removed_count) *removed_count = res.removed_block_count;
    if (status) *status = 0;
    return out;
  } catch (const std::exception&) {
    if (status) *status = -1;
    return nullptr;
  }
}

// spamm::purify (purification.cpp:90-202) with an explicit budget.  Writes
// per-record (iteration, status 0 ok/1 violation/2 converged, chosen_tau,
// trace, realized_error, nnz_out) and returns the density tree.
void* ref_purify(const void* x0, int variant, int occupation, int max_iterations, double epsilon,
                 const double* taus, int n_taus, double initial_delta, const double* deltas,
                 double idempotency_threshold, int log_capacity, int* n_log, double* log6,
                 int* converged, int* iterations) {
  try {
    spamm::PurificationConfig cfg;
    cfg.variant = static_cast<spamm::Variant>(variant);
    cfg.occupation = occupation;
    cfg.max_iterations = max_iterations;
    cfg.epsilon = epsilon;
    cfg.grid = spamm::ToleranceGrid(std::vector<double>(taus, taus + n_taus));
    cfg.idempotency_threshold = idempotency_threshold;
    std::vector<double> dv(deltas, deltas + max_iterations);
    cfg.budget = [initial_delta, dv](double, int) {
      spamm::ErrorBudget b;
      b.initial_delta = initial_delta;
      b.deltas = dv;
      return b;
    };
    const auto* r = static_cast<const RefTree*>(x0);
    auto res = spamm::purify(r->m, cfg);
    int k = 0;
    for (const auto& rec : res.log) {
      if (k < log_capacity) {
        double* o = log6 + 6 * k;
        o[0] = rec.iteration;
        o[1] = rec.status == "ok" ? 0 : rec.status == "violation" ? 1 : 2;
        o[2] = rec.chosen_tau;
        o[3] = rec.trace;
        o[4] = rec.realized_error;
        o[5] = static_cast<double>(rec.nnz_out);
      }
      ++k;
    }
    *n_log = k;
    *converged = res.converged;
    *iterations = res.iterations;
    auto* out = new RefTree;
    out->m = std::move(res.density);
    out->depth = r->depth;
    return out;
  } catch (const std::exception&) {
    return nullptr;
  }
}

std::int64_t ref_survivors(const void* a, const void* b, double tau, std::int32_t* triples,
                           std::int64_t capacity) {
  const auto* ra = static_cast<const RefTree*>(a);
  const auto* rb = static_cast<const RefTree*>(b);
  std::vector<std::array<std::int32_t, 3>> out;
  std::int64_t count = 0;
  surv_walk(ra->m.root(), rb->m.root(), 0, ra->depth, tau, true, 0, 0, 0,
            triples ? &out : nullptr, count);
  if (!triples) return count;
  std::sort(out.begin(), out.end(), [&](const auto& x, const auto& y) {
    const auto kx = morton2(x[0], x[2], ra->depth), ky = morton2(y[0], y[2], ra->depth);
    return kx != ky ? kx < ky : x[1] < y[1];
  });
  const std::int64_t n = std::min<std::int64_t>(count, capacity);
  for (std::int64_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) triples[3 * i + c] = out[i][c];
  return count;
}

// ---- experiment-side modules ------------------------------
// status: 0 ok, 1 std::invalid_argument, 2 std::domain_error, 3 other
static int classify(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::domain_error*>(&e)) return 2;
  return 3;
}

// spamm::oracle::generate_decay_matrix (oracle.cpp) -> row-major n x n
int ref_generate_decay(int n, double alpha, double scale, double low, double high,
                       std::uint64_t seed, double* out) {
  try {
    spamm::oracle::DecayModelSpec spec;
    spec.dimension = n;
    spec.alpha = alpha;
    spec.scale = scale;
    spec.spectral_low = low;
    spec.spectral_high = high;
    spec.seed = seed;
    const auto d = spamm::oracle::generate_decay_matrix(spec);
    std::memcpy(out, d.data(), d.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

void ref_gershgorin(const double* a, int n, double* lo, double* hi) {
  spamm::DenseMatrix d(n);
  std::memcpy(d.data(), a, d.size() * sizeof(double));
  const auto b = spamm::oracle::gershgorin_bounds(d);
  *lo = b.first;
  *hi = b.second;
}

int ref_density_oracle(const double* fock, int n, int occupation, double* out) {
  try {
    spamm::DenseMatrix d(n);
    std::memcpy(d.data(), fock, d.size() * sizeof(double));
    const auto p = spamm::oracle::density_matrix_oracle(d, occupation);
    std::memcpy(out, p.data(), p.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// spamm::read_matrix_market (matrix_market.cpp:40-94): returns -1 when cap is
// too small (count written), else the status above (1 invalid_argument, 3
// runtime_error).
int ref_mm_read(const char* text, int* dimension, std::int64_t* count, std::int32_t* rows,
                std::int32_t* cols, double* values, std::int64_t cap) {
  try {
    std::istringstream in{std::string(text)};
    const auto data = spamm::read_matrix_market(in);
    *dimension = data.dimension;
    *count = static_cast<std::int64_t>(data.entries.size());
    if (*count > cap) return -1;
    for (std::int64_t i = 0; i < *count; ++i) {
      rows[i] = data.entries[i].row;
      cols[i] = data.entries[i].col;
      values[i] = data.entries[i].value;
    }
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// spamm::write_matrix_market (matrix_market.cpp:96-111) of a reference tree;
// returns the text length (written up to cap bytes)
std::int64_t ref_mm_write(const void* x, char* buf, std::int64_t cap) {
  std::ostringstream out;
  spamm::write_matrix_market(out, static_cast<const RefTree*>(x)->m);
  const std::string s = out.str();
  if (buf) std::memcpy(buf, s.data(), static_cast<std::size_t>(std::min<std::int64_t>(cap, s.size())));
  return static_cast<std::int64_t>(s.size());
}

// The squaring protocol of run_squaring_experiment (experiment.cpp:92-128;
// the file itself needs nlohmann/json, absent here) restated over the
// reference's own calls: per tolerance, square twice with the variant's
// method and measure the second square against the exact one.
// rec9 per tolerance: chosen_tau, nnz_in, nnz_mid, nnz_out, nnz_blocks_out,
// realized_error, status (0 ok / 1 violation), trace, chosen_tau of square 1.
int ref_squaring(const void* x, int variant, const double* deltas, int n_deltas,
                 const double* taus, int n_taus, double* rec9) {
  try {
    const spamm::ToleranceGrid grid(std::vector<double>(taus, taus + n_taus));
    const auto v = static_cast<spamm::Variant>(variant);
    auto square = [&](const QuadTreeMatrix& in, double delta, double* tau,
                      std::int64_t* nnz_mid) -> QuadTreeMatrix {
      if (v == spamm::Variant::truncmul) {
        QuadTreeMatrix p = spamm::multiply_exact(in, in);
        *nnz_mid = p.nnz();
        *tau = 0.0;
        return std::move(spamm::truncate(p, delta).matrix);
      }
      const double d = v == spamm::Variant::hybrid ? delta / 2.0 : delta;
      auto cp = spamm::spamm_with_error_control(in, in, d, grid);
      *tau = cp.chosen_tau.tau;
      *nnz_mid = cp.matrix.nnz();
      if (v == spamm::Variant::spamm) return std::move(cp.matrix);
      return std::move(spamm::truncate(cp.matrix, d).matrix);
    };
    const auto& input = static_cast<const RefTree*>(x)->m;
    for (int i = 0; i < n_deltas; ++i) {
      double* o = rec9 + 9 * i;
      double tau1 = 0.0, tau2 = 0.0;
      std::int64_t mid1 = 0, mid2 = 0;
      const QuadTreeMatrix x1 = square(input, deltas[i], &tau1, &mid1);
      const QuadTreeMatrix x2 = square(x1, deltas[i], &tau2, &mid2);
      const QuadTreeMatrix exact = spamm::multiply_exact(x1, x1);
      const double err = spamm::add(x2, exact.scale(-1.0)).frobenius_norm();
      o[0] = tau2;
      o[1] = static_cast<double>(x1.nnz());
      o[2] = static_cast<double>(mid2);
      o[3] = static_cast<double>(x2.nnz());
      o[4] = static_cast<double>(x2.nnz_blocks());
      o[5] = err;
      o[6] = err < deltas[i] ? 0.0 : 1.0;
      o[7] = x2.trace();
      o[8] = tau1;
    }
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

}  // extern "C"
