#pragma once
//
// spamm-b200 drop-in: exact quadtree product and SpAMM norm-product skipping
// (/root/reference/proj/core/include/spamm/multiply.hpp:15-29), executed by the
// CUDA task-list builder and DMMA leaf GEMM (include/spamm_gpu.h).
//
#include "spamm/quadtree.hpp"

namespace spamm {

struct SpammTolerance {
  double tau = 0.0;
};

/// C = A * B.  Throws std::invalid_argument on dimension or leaf size mismatch.
QuadTreeMatrix multiply_exact(const QuadTreeMatrix& a, const QuadTreeMatrix& b);

/// Skips every subtree product with fl(||A||_F * ||B||_F) < tau, tested at
/// every level; the surviving product set is bit-identical to the reference.
/// Throws std::invalid_argument on mismatch or tau < 0.
QuadTreeMatrix spamm_multiply(const QuadTreeMatrix& a, const QuadTreeMatrix& b,
                              SpammTolerance tolerance);

}  // namespace spamm
