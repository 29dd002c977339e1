// quadtree.cpp -- drop-in QuadTreeMatrix over device-resident matrices.
//
// Construction goes straight to the device (spg_matrix_upload /
// spg_matrix_from_dense): the CUDA norm kernels compute every cached norm with
// the reference rule (node_ops.hpp:24-36).  The host Node tree is built only
// when root() is called, from the downloaded leaves and their device norms;
// inner norms are recombined on the host with the same sequential rule, so
// they equal the device pyramid bit for bit.  trace / nnz / scale / add and the
// Gershgorin bounds run on the device (include/spamm_gpu.h, csrc/algebra.cu):
// no full-matrix host round trip.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>

#include "runtime.hpp"

namespace spamm {

namespace {

using Node = QuadTreeMatrix::Node;
using NodePtr = QuadTreeMatrix::NodePtr;

int padded_for(int dimension, int leaf) {
  if (dimension <= 0) throw std::invalid_argument("dimension must be positive");
  if (leaf <= 0) throw std::invalid_argument("leaf_size must be positive");
  int padded = leaf;
  while (padded < dimension) {
    if (padded > (1 << 29)) throw std::invalid_argument("dimension too large to pad");
    padded *= 2;
  }
  return padded;
}

int depth_for(int padded, int leaf) {
  int d = 0;
  while ((leaf << d) < padded) ++d;
  return d;
}

// combine_child_norms (node_ops.hpp:30-36); built with -ffp-contract=off.
NodePtr make_inner(std::array<NodePtr, 4> child) {
  if (!child[0] && !child[1] && !child[2] && !child[3]) return nullptr;
  double s = 0.0;
  for (const NodePtr& c : child)
    if (c) s += c->norm * c->norm;
  auto n = std::make_shared<Node>();
  n->norm = std::sqrt(s);
  n->child = std::move(child);
  return n;
}

struct Leaves {
  std::vector<int32_t> rows, cols;
  std::vector<double> payload, norms;
};

// Leaves arrive in Morton order; rebuild the tree by splitting on key digits.
NodePtr build_host(const Leaves& lv, const std::vector<uint64_t>& keys, size_t lo, size_t hi,
                   int level, int depth, int64_t block) {
  if (lo >= hi) return nullptr;
  if (level == depth) {
    auto n = std::make_shared<Node>();
    n->norm = lv.norms[lo];
    n->block.assign(lv.payload.begin() + static_cast<int64_t>(lo) * block,
                    lv.payload.begin() + static_cast<int64_t>(lo + 1) * block);
    return n;
  }
  const int shift = 2 * (depth - level - 1);
  std::array<NodePtr, 4> child;
  size_t start = lo;
  for (int c = 0; c < 4; ++c) {
    size_t end = start;
    while (end < hi && static_cast<int>((keys[end] >> shift) & 3u) == c) ++end;
    child[c] = build_host(lv, keys, start, end, level + 1, depth, block);
    start = end;
  }
  return make_inner(std::move(child));
}

uint64_t morton(uint32_t r, uint32_t c, int depth) {
  uint64_t k = 0;
  for (int b = depth - 1; b >= 0; --b) k = (k << 2) | (((r >> b) & 1u) << 1) | ((c >> b) & 1u);
  return k;
}

Leaves download(const spg_matrix* m, int leaf) {
  spg_matrix_info info{};
  b200::check(spg_matrix_get_info(m, &info));
  Leaves lv;
  const size_t n = static_cast<size_t>(info.nnz_blocks);
  lv.rows.resize(n);
  lv.cols.resize(n);
  lv.norms.resize(n);
  lv.payload.resize(n * static_cast<size_t>(leaf) * leaf);
  if (n)
    b200::check(spg_matrix_download(m, lv.rows.data(), lv.cols.data(), lv.payload.data(),
                                    lv.norms.data()));
  return lv;
}

void collect(const NodePtr& n, int level, int depth, int32_t r, int32_t c, Leaves& out) {
  if (!n) return;
  if (level == depth) {
    out.rows.push_back(r);
    out.cols.push_back(c);
    out.payload.insert(out.payload.end(), n->block.begin(), n->block.end());
    return;
  }
  for (int q = 0; q < 4; ++q)
    collect(n->child[q], level + 1, depth, 2 * r + (q >> 1), 2 * c + (q & 1), out);
}

spg_matrix* upload(const Leaves& lv, int dimension, int leaf) {
  spg_matrix* m = nullptr;
  b200::check(spg_matrix_upload(b200::context(), dimension, leaf,
                                static_cast<int64_t>(lv.rows.size()), lv.rows.data(),
                                lv.cols.data(), lv.payload.data(), &m));
  return m;
}

}  // namespace

QuadTreeMatrix adopt_device(spg_matrix* m) {
  spg_matrix_info info{};
  const int rc = spg_matrix_get_info(m, &info);
  if (rc != SPG_OK) {
    spg_matrix_free(m);
    b200::check(rc);
  }
  QuadTreeMatrix q;
  q.dimension_ = info.dimension;
  q.padded_dimension_ = info.padded_dimension;
  q.leaf_size_ = info.leaf_size;
  q.state_ = std::make_shared<QuadTreeMatrix::State>();
  q.state_->dev = m;
  return q;
}

QuadTreeMatrix QuadTreeMatrix::wrap(NodePtr root, int dimension, int leaf_size) {
  QuadTreeMatrix q;
  q.dimension_ = dimension;
  q.padded_dimension_ = padded_for(dimension, leaf_size);
  q.leaf_size_ = leaf_size;
  q.state_ = std::make_shared<State>();
  q.state_->host = std::move(root);
  q.state_->host_ready = true;
  return q;
}

QuadTreeMatrix QuadTreeMatrix::zero(int dimension, int leaf_size) {
  padded_for(dimension, leaf_size);
  return wrap(nullptr, dimension, leaf_size);
}

QuadTreeMatrix QuadTreeMatrix::identity(int dimension, int leaf_size) {
  padded_for(dimension, leaf_size);
  std::vector<CoordinateEntry> diag(static_cast<size_t>(dimension));
  for (int i = 0; i < dimension; ++i) diag[i] = {i, i, 1.0};
  return from_coordinates(diag, dimension, leaf_size);
}

QuadTreeMatrix QuadTreeMatrix::from_coordinates(std::span<const CoordinateEntry> entries,
                                                int dimension, int leaf_size) {
  padded_for(dimension, leaf_size);
  for (const CoordinateEntry& e : entries)  // quadtree.cpp:202-208
    if (e.row < 0 || e.row >= dimension || e.col < 0 || e.col >= dimension)
      throw std::out_of_range("coordinate (" + std::to_string(e.row) + ", " +
                              std::to_string(e.col) + ") outside dimension " +
                              std::to_string(dimension));
  std::vector<CoordinateEntry> sorted(entries.begin(), entries.end());
  std::sort(sorted.begin(), sorted.end(), [](const CoordinateEntry& a, const CoordinateEntry& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  for (size_t i = 1; i < sorted.size(); ++i)  // quadtree.cpp:213-216
    if (sorted[i].row == sorted[i - 1].row && sorted[i].col == sorted[i - 1].col)
      throw std::invalid_argument("duplicate coordinate (" + std::to_string(sorted[i].row) +
                                  ", " + std::to_string(sorted[i].col) + ")");
  // bucket entries into leaf blocks (column-major payload)
  const int L = leaf_size;
  std::vector<std::pair<uint64_t, const CoordinateEntry*>> keyed;
  keyed.reserve(sorted.size());
  for (const CoordinateEntry& e : sorted)
    keyed.push_back({(static_cast<uint64_t>(e.row / L) << 32) | static_cast<uint32_t>(e.col / L), &e});
  std::stable_sort(keyed.begin(), keyed.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  Leaves lv;
  for (size_t i = 0; i < keyed.size();) {
    size_t j = i;
    const int br = static_cast<int>(keyed[i].first >> 32), bc = static_cast<int>(keyed[i].first & 0xffffffffu);
    lv.rows.push_back(br);
    lv.cols.push_back(bc);
    const size_t base = lv.payload.size();
    lv.payload.resize(base + static_cast<size_t>(L) * L, 0.0);
    for (; j < keyed.size() && keyed[j].first == keyed[i].first; ++j) {
      const CoordinateEntry& e = *keyed[j].second;
      lv.payload[base + (e.row - br * L) + static_cast<size_t>(e.col - bc * L) * L] = e.value;
    }
    i = j;
  }
  return adopt_device(upload(lv, dimension, leaf_size));
}

QuadTreeMatrix QuadTreeMatrix::from_dense(const DenseMatrix& dense, int leaf_size) {
  padded_for(dense.dimension(), leaf_size);
  spg_matrix* m = nullptr;
  b200::check(spg_matrix_from_dense(b200::context(), dense.dimension(), leaf_size, dense.data(), &m));
  return adopt_device(m);
}

const QuadTreeMatrix::NodePtr& QuadTreeMatrix::root() const noexcept {
  static const NodePtr kNull;
  if (!state_) return kNull;
  std::lock_guard<std::mutex> lock(state_->mu);
  if (!state_->host_ready) {
    // a device failure here cannot be reported through the noexcept
    // signature; terminate loudly rather than return a wrong tree
    Leaves lv = download(state_->dev, leaf_size_);
    const int depth = depth_for(padded_dimension_, leaf_size_);
    std::vector<uint64_t> keys(lv.rows.size());
    for (size_t i = 0; i < keys.size(); ++i) keys[i] = morton(lv.rows[i], lv.cols[i], depth);
    state_->host = build_host(lv, keys, 0, keys.size(), 0, depth,
                              static_cast<int64_t>(leaf_size_) * leaf_size_);
    state_->host_ready = true;
  }
  return state_->host;
}

const spg_matrix* QuadTreeMatrix::device() const {
  if (!state_) throw std::invalid_argument("empty QuadTreeMatrix");
  std::lock_guard<std::mutex> lock(state_->mu);
  if (!state_->dev) {
    Leaves lv;
    collect(state_->host, 0, depth_for(padded_dimension_, leaf_size_), 0, 0, lv);
    state_->dev = upload(lv, dimension_, leaf_size_);
  }
  return state_->dev;
}

bool QuadTreeMatrix::is_zero() const noexcept {
  if (!state_) return true;
  {
    std::lock_guard<std::mutex> lock(state_->mu);
    if (state_->host_ready) return state_->host == nullptr;
    spg_matrix_info info{};
    if (spg_matrix_get_info(state_->dev, &info) == SPG_OK) return info.nnz_blocks == 0;
  }
  return root() == nullptr;
}

double QuadTreeMatrix::frobenius_norm() const noexcept {
  if (!state_) return 0.0;
  {
    std::lock_guard<std::mutex> lock(state_->mu);
    if (state_->host_ready) return state_->host ? state_->host->norm : 0.0;
    spg_matrix_info info{};
    if (spg_matrix_get_info(state_->dev, &info) == SPG_OK) return info.frobenius_norm;
  }
  return root() ? root()->norm : 0.0;
}

namespace {
void write_dense(const NodePtr& n, DenseMatrix& out, int r0, int c0, int size, int leaf, int limit) {
  if (!n) return;
  if (n->is_leaf()) {
    for (int j = 0; j < leaf && c0 + j < limit; ++j)
      for (int i = 0; i < leaf && r0 + i < limit; ++i)
        out(r0 + i, c0 + j) = n->block[i + static_cast<size_t>(j) * leaf];
    return;
  }
  const int h = size / 2;
  for (int q = 0; q < 4; ++q)
    write_dense(n->child[q], out, r0 + (q >> 1) * h, c0 + (q & 1) * h, h, leaf, limit);
}
}  // namespace

// node_trace (quadtree.cpp:128-138): per diagonal leaf a sequential sum, then
// trace(child 0) + trace(child 3) level by level -- spg_matrix_trace
double QuadTreeMatrix::trace() const {
  if (!state_) return 0.0;
  double t = 0.0;
  b200::check(spg_matrix_trace(device(), &t));
  return t;
}

// node_nnz (quadtree.cpp:140-151): stored entries != 0, counted on the device
std::int64_t QuadTreeMatrix::nnz() const {
  if (!state_) return 0;
  int64_t n = 0;
  b200::check(spg_matrix_nnz(device(), &n));
  return n;
}

std::int64_t QuadTreeMatrix::nnz_blocks() const {
  if (!state_) return 0;
  spg_matrix_info info{};
  b200::check(spg_matrix_get_info(device(), &info));
  return info.nnz_blocks;
}

DenseMatrix QuadTreeMatrix::to_dense() const {
  DenseMatrix out(dimension_);
  write_dense(root(), out, 0, 0, padded_dimension_, leaf_size_, dimension_);
  return out;
}

DenseMatrix QuadTreeMatrix::to_dense_padded() const {
  DenseMatrix out(padded_dimension_);
  write_dense(root(), out, 0, 0, padded_dimension_, leaf_size_, padded_dimension_);
  return out;
}

// scale_node (quadtree.cpp:153-171,249-252): fl(alpha * v) per entry, leaf
// norms recomputed, all-zero leaves collapse -- spg_matrix_axpby(alpha, a, 0, -)
QuadTreeMatrix QuadTreeMatrix::scale(double alpha) const {
  if (alpha == 0.0 || !state_) return zero(dimension_, leaf_size_);
  spg_matrix* out = nullptr;
  b200::check(spg_matrix_axpby(b200::context(), alpha, device(), 0.0, nullptr, &out));
  return adopt_device(out);
}

// add_nodes (quadtree.cpp:24-36,254-261): a + b where both leaves exist, the
// present leaf otherwise (fl(1 * v) = v) -- spg_matrix_axpby(1, a, 1, b)
QuadTreeMatrix add(const QuadTreeMatrix& a, const QuadTreeMatrix& b) {
  if (a.dimension() != b.dimension() || a.leaf_size() != b.leaf_size())
    throw std::invalid_argument("add: dimension or leaf size mismatch");
  if (a.is_zero()) return b;
  if (b.is_zero()) return a;
  spg_matrix* out = nullptr;
  b200::check(spg_matrix_axpby(b200::context(), 1.0, a.device(), 1.0, b.device(), &out));
  return adopt_device(out);
}

std::pair<double, double> gershgorin_bounds(const QuadTreeMatrix& a) {
  if (a.is_zero()) {
    // all diagonal entries and radii are 0 (oracle.cpp:191-200 on a zero matrix)
    return {0.0, 0.0};
  }
  double lo = 0.0, hi = 0.0;
  b200::check(spg_matrix_gershgorin(a.device(), &lo, &hi));
  return {lo, hi};
}

}  // namespace spamm
