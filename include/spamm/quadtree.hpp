#pragma once
//
// spamm-b200 drop-in: quadtree sparse matrix with cached Frobenius norms.
//
// Same public interface and semantics as the reference's QuadTreeMatrix
// (/root/reference/proj/core/include/spamm/quadtree.hpp:34-101): null child =
// identically zero quadrant, column-major dense leaves, cached norm per node,
// padding to leaf * 2^k, immutable values.
//
// B200 design: a QuadTreeMatrix is a handle to a device-resident matrix
// (include/spamm_gpu.h: packed FP64 leaf payload + dense Morton norm pyramid
// in HBM) built by the CUDA norm kernels.  The host Node tree that root()
// exposes is materialised lazily, only when a caller walks it; products,
// the CSE sweep, tolerance selection, trace, nnz, scale and add never leave
// the device.  Host trees assembled with wrap() are uploaded on first use.
//
#include <array>
#include <cstdint>
#include <memory>
#include <span>
#include <utility>
#include <vector>

#include "spamm/dense_matrix.hpp"

struct spg_matrix;

namespace spamm {

struct CoordinateEntry {
  int row = 0;
  int col = 0;
  double value = 0.0;
};

class QuadTreeMatrix {
 public:
  static constexpr int kDefaultLeafSize = 32;

  struct Node;
  using NodePtr = std::shared_ptr<const Node>;

  struct Node {
    double norm = 0.0;
    std::vector<double> block;       // leaf payload, column-major; empty on inner nodes
    std::array<NodePtr, 4> child{};  // inner payload, indexed [2*row + col]
    bool is_leaf() const noexcept { return !block.empty(); }
  };

  QuadTreeMatrix() = default;

  static QuadTreeMatrix zero(int dimension, int leaf_size = kDefaultLeafSize);
  static QuadTreeMatrix identity(int dimension, int leaf_size = kDefaultLeafSize);
  /// Throws std::out_of_range for indices outside [0, dimension) and
  /// std::invalid_argument for duplicate (row, col) pairs.
  static QuadTreeMatrix from_coordinates(std::span<const CoordinateEntry> entries, int dimension,
                                         int leaf_size = kDefaultLeafSize);
  static QuadTreeMatrix from_dense(const DenseMatrix& dense, int leaf_size = kDefaultLeafSize);

  int dimension() const noexcept { return dimension_; }
  int padded_dimension() const noexcept { return padded_dimension_; }
  int leaf_size() const noexcept { return leaf_size_; }
  /// Host view of the tree (materialised from the device on first call).
  const NodePtr& root() const noexcept;
  bool is_zero() const noexcept;
  double frobenius_norm() const noexcept;

  double trace() const;
  std::int64_t nnz() const;
  std::int64_t nnz_blocks() const;
  DenseMatrix to_dense() const;
  DenseMatrix to_dense_padded() const;
  QuadTreeMatrix scale(double alpha) const;

  static QuadTreeMatrix wrap(NodePtr root, int dimension, int leaf_size);

  /// B200 extension: the device matrix behind this value (uploaded on demand).
  const spg_matrix* device() const;

  struct State;  // shared device handle + lazily materialised host tree

 private:
  int dimension_ = 0;
  int padded_dimension_ = 0;
  int leaf_size_ = 0;
  std::shared_ptr<State> state_;

  friend QuadTreeMatrix adopt_device(spg_matrix* m);
};

/// Entrywise sum (add_nodes, quadtree.cpp:24-36), computed on the device.
QuadTreeMatrix add(const QuadTreeMatrix& a, const QuadTreeMatrix& b);

/// B200 extension: Gershgorin spectral bounds {low, high} computed from the
/// device leaves -- bitwise the reference's oracle::gershgorin_bounds on
/// a.to_dense() (oracle.cpp:191-200) without building the dense matrix.
std::pair<double, double> gershgorin_bounds(const QuadTreeMatrix& a);

/// B200 extension: wrap a device matrix returned by the C ABI.
QuadTreeMatrix adopt_device(spg_matrix* m);

}  // namespace spamm
