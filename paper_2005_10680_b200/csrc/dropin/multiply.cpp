// multiply.cpp -- drop-in products (multiply.hpp:15-29) on the GPU path:
// K4 task-list builder + K5 DMMA leaf GEMM through the C ABI; row-sharded over
// the job's GPUs while a spamm::distributed communicator is set.
#include "spamm/multiply.hpp"

#include <stdexcept>

#include "runtime.hpp"

namespace spamm {

namespace {
void check_conformable(const QuadTreeMatrix& a, const QuadTreeMatrix& b) {  // multiply.cpp:94-98
  if (a.dimension() != b.dimension() || a.leaf_size() != b.leaf_size())
    throw std::invalid_argument("multiply: dimension or leaf size mismatch");
}
}  // namespace

QuadTreeMatrix multiply_exact(const QuadTreeMatrix& a, const QuadTreeMatrix& b) {
  check_conformable(a, b);
  spg_matrix* c = nullptr;
  if (spg_comm* comm = b200::communicator())  // row shards on every rank's GPU, C gathered
    b200::check(spg_spamm_sharded(comm, a.device(), b.device(), 0.0, 0, 1, &c, nullptr));
  else
    b200::check(spg_multiply_exact(b200::context(), a.device(), b.device(), &c, nullptr));
  return adopt_device(c);
}

QuadTreeMatrix spamm_multiply(const QuadTreeMatrix& a, const QuadTreeMatrix& b,
                              SpammTolerance tolerance) {
  check_conformable(a, b);
  if (tolerance.tau < 0.0) throw std::invalid_argument("spamm: tau must be nonnegative");
  spg_matrix* c = nullptr;
  if (spg_comm* comm = b200::communicator())
    b200::check(spg_spamm_sharded(comm, a.device(), b.device(), tolerance.tau, 1, 1, &c, nullptr));
  else
    b200::check(spg_spamm(b200::context(), a.device(), b.device(), tolerance.tau, &c, nullptr));
  return adopt_device(c);
}

}  // namespace spamm
