// error_control.cpp -- drop-in CSE sweep, selection, truncation and
// controlled product (error_control.hpp:18-77), all on the GPU path.
#include "spamm/error_control.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <utility>

#include "runtime.hpp"

namespace spamm {

ToleranceGrid::ToleranceGrid(std::vector<double> taus) : taus_(std::move(taus)) {
  // error_control.cpp:139-150 (same messages, same exception type)
  if (taus_.empty()) throw std::invalid_argument("tolerance grid must be nonempty");
  for (size_t k = 0; k < taus_.size(); ++k) {
    if (!(taus_[k] > 0.0)) throw std::invalid_argument("tolerance grid entries must be positive");
    if (k > 0 && !(taus_[k] < taus_[k - 1]))
      throw std::invalid_argument("tolerance grid must be strictly decreasing");
  }
}

ToleranceGrid ToleranceGrid::geometric(double start, double ratio, int count) {
  if (!(start > 0.0)) throw std::invalid_argument("grid start must be positive");
  if (!(ratio > 0.0 && ratio < 1.0)) throw std::invalid_argument("grid ratio must be in (0, 1)");
  if (count < 1) throw std::invalid_argument("grid count must be at least 1");
  std::vector<double> taus(static_cast<size_t>(count));
  double tau = start;  // repeated multiplication, not pow (error_control.cpp:152-158)
  for (int k = 0; k < count; ++k) {
    taus[k] = tau;
    tau *= ratio;
  }
  return ToleranceGrid(std::move(taus));
}

ErrorBoundVector cse(const QuadTreeMatrix& a, const QuadTreeMatrix& b, const ToleranceGrid& grid) {
  if (a.dimension() != b.dimension() || a.leaf_size() != b.leaf_size())
    throw std::invalid_argument("cse: dimension or leaf size mismatch");
  ErrorBoundVector out{std::vector<double>(grid.size())};
  if (spg_comm* comm = b200::communicator())
    b200::check(spg_cse_sharded(comm, a.device(), b.device(), grid.taus().data(),
                                static_cast<int32_t>(grid.size()), out.bounds.data()));
  else
    b200::check(spg_cse(b200::context(), a.device(), b.device(), grid.taus().data(),
                        static_cast<int32_t>(grid.size()), out.bounds.data()));
  return out;
}

SpammTolerance select_tolerance(const ErrorBoundVector& bounds, const ToleranceGrid& grid,
                                double delta) {
  double tau = 0.0;
  int32_t k = -1;
  b200::check(spg_select_tolerance(bounds.bounds.data(), grid.taus().data(),
                                   static_cast<int32_t>(grid.size()), delta, &tau, &k));
  return SpammTolerance{tau};
}

TruncationResult truncate(const QuadTreeMatrix& x, double delta) {
  // GPU greedy truncation (spg_truncate): same removed set, bound and norms as
  // error_control.cpp:174-201; the result shares x's leaf payload.
  if (delta < 0.0) throw std::invalid_argument("truncate: delta must be nonnegative");
  spg_matrix* m = nullptr;
  double removed = 0.0;
  int64_t count = 0;
  b200::check(spg_truncate(b200::context(), x.device(), delta, &m, &removed, &count));
  TruncationResult result{x, removed, count};
  if (count > 0) {
    result.matrix = adopt_device(m);
  } else {
    spg_matrix_free(m);  // nothing removed: share x itself (root() identity, :197-198)
  }
  return result;
}

ControlledProduct spamm_with_error_control(const QuadTreeMatrix& a, const QuadTreeMatrix& b,
                                           double delta, const ToleranceGrid& grid) {
  if (!(delta > 0.0))
    throw std::invalid_argument("spamm_with_error_control: delta must be positive");
  if (a.dimension() != b.dimension() || a.leaf_size() != b.leaf_size())
    throw std::invalid_argument("cse: dimension or leaf size mismatch");
  spg_matrix* c = nullptr;
  spg_controlled_stats st{};
  if (spg_comm* comm = b200::communicator())  // row shards, C gathered on every rank
    b200::check(spg_spamm_with_error_control_sharded(
        comm, a.device(), b.device(), delta, grid.taus().data(),
        static_cast<int32_t>(grid.size()), 1, &c, nullptr, &st));
  else
    b200::check(spg_spamm_with_error_control(b200::context(), a.device(), b.device(), delta,
                                             grid.taus().data(),
                                             static_cast<int32_t>(grid.size()), &c, nullptr, &st));
  ControlledProduct out;
  out.matrix = adopt_device(c);
  out.chosen_tau = SpammTolerance{st.tau};
  out.bound = st.bound;
  out.cse_seconds = st.cse_seconds;
  out.spamm_seconds = st.spamm_seconds;
  return out;
}

}  // namespace spamm
