// purification.cpp -- drop-in SP2 drivers (purification.hpp) over spg_purify:
// the whole iteration (squares, truncations, traces, 2X - X^2) runs on the
// device; this file only maps the C++ configuration and the RunRecord log.
#include "spamm/purification.hpp"

#include <cmath>
#include <limits>
#include <stdexcept>

#include "runtime.hpp"

namespace spamm {

std::string_view to_string(Variant v) {
  switch (v) {
    case Variant::truncmul: return "truncmul";
    case Variant::spamm: return "spamm";
    case Variant::hybrid: return "hybrid";
  }
  return "unknown";
}

std::optional<Variant> parse_variant(std::string_view name) {
  if (name == "truncmul") return Variant::truncmul;
  if (name == "spamm") return Variant::spamm;
  if (name == "hybrid") return Variant::hybrid;
  return std::nullopt;
}

QuadTreeMatrix initial_transform(const QuadTreeMatrix& fock, const SpectralTransform& t) {
  // X0 = (lambda_max I - F) / (lambda_max - lambda_min)  (purification.cpp:49-57)
  if (!(t.lambda_max > t.lambda_min))
    throw std::invalid_argument("initial_transform: lambda_max must exceed lambda_min");
  spg_context* ctx = b200::context();
  spg_matrix* id = nullptr;
  b200::check(spg_matrix_identity(ctx, fock.dimension(), fock.leaf_size(), &id));
  const QuadTreeMatrix identity = adopt_device(id);
  spg_matrix* shifted = nullptr;
  b200::check(spg_matrix_axpby(ctx, t.lambda_max, identity.device(), -1.0, fock.device(), &shifted));
  const QuadTreeMatrix s = adopt_device(shifted);
  spg_matrix* out = nullptr;
  b200::check(spg_matrix_axpby(ctx, 1.0 / (t.lambda_max - t.lambda_min), s.device(), 0.0, nullptr,
                               &out));
  return adopt_device(out);
}

Sp2Choice sp2_step(const QuadTreeMatrix& x, int occupation) {
  double tr = 0.0;
  b200::check(spg_matrix_trace(x.device(), &tr));
  if (tr > static_cast<double>(occupation)) return {Sp2Polynomial::square, "x^2"};
  return {Sp2Polynomial::trace_correcting, "2x - x^2"};
}

ErrorBudget ErrorBudget::geometric(double epsilon, int iterations, double ratio) {
  ErrorBudget b;
  b.deltas.resize(iterations > 0 ? static_cast<size_t>(iterations) : 1);
  b200::check(spg_error_budget_geometric(epsilon, iterations, ratio, &b.initial_delta,
                                         b.deltas.data()));
  b.deltas.resize(static_cast<size_t>(iterations));
  return b;
}

double ErrorBudget::total() const {
  double sum = initial_delta;
  for (const double d : deltas) sum += d;
  return sum;
}

PurificationResult purify(const QuadTreeMatrix& x0, const PurificationConfig& config) {
  if (config.occupation <= 0 || config.occupation >= x0.dimension())
    throw std::invalid_argument("purify: occupation must lie strictly between 0 and the dimension");
  if (config.max_iterations < 1) throw std::invalid_argument("purify: max_iterations must be positive");
  if (!(config.epsilon > 0.0)) throw std::invalid_argument("purify: epsilon must be positive");
  const ErrorBudget budget = config.budget ? config.budget(config.epsilon, config.max_iterations)
                                           : ErrorBudget::geometric(config.epsilon,
                                                                    config.max_iterations);
  if (static_cast<int>(budget.deltas.size()) < config.max_iterations)
    throw std::invalid_argument("purify: budget provides fewer deltas than max_iterations");
  spg_purify_config cfg{};
  cfg.variant = static_cast<int32_t>(config.variant);
  cfg.occupation = config.occupation;
  cfg.max_iterations = config.max_iterations;
  cfg.epsilon = config.epsilon;
  cfg.idempotency_threshold = config.idempotency_threshold;
  cfg.taus = config.grid.taus().data();
  cfg.n_taus = static_cast<int32_t>(config.grid.size());
  cfg.initial_delta = budget.initial_delta;
  cfg.deltas = budget.deltas.data();
  cfg.n_deltas = static_cast<int32_t>(budget.deltas.size());
  cfg.measure_error = 1;
  std::vector<spg_run_record> log(static_cast<size_t>(config.max_iterations) + 2);
  spg_matrix* density = nullptr;
  int32_t n_log = 0, converged = 0, iterations = 0;
  b200::check(spg_purify(b200::context(), x0.device(), &cfg, &density, log.data(),
                         static_cast<int32_t>(log.size()), &n_log, &converged, &iterations));
  PurificationResult out;
  out.density = adopt_device(density);
  out.converged = converged != 0;
  out.iterations = iterations;
  static const char* kStatus[] = {"ok", "violation", "converged"};
  for (int32_t i = 0; i < n_log && i < static_cast<int32_t>(log.size()); ++i) {
    const spg_run_record& r = log[i];
    RunRecord rec;
    rec.variant = std::string(to_string(config.variant));
    rec.iteration = r.iteration;
    rec.tolerance = r.tolerance;
    rec.chosen_tau = r.chosen_tau;
    rec.t_mul = r.t_mul;
    rec.t_trunc = r.t_trunc;
    rec.t_spamm = r.t_spamm;
    rec.t_cse = r.t_cse;
    rec.nnz_in = r.nnz_in;
    rec.nnz_mid = r.nnz_mid;
    rec.nnz_out = r.nnz_out;
    rec.nnz_blocks_out = r.nnz_blocks_out;
    rec.realized_error = r.realized_error;
    rec.status = kStatus[r.status];
    rec.trace = r.trace;
    out.log.push_back(std::move(rec));
  }
  return out;
}

PurificationResult purify_fock(const QuadTreeMatrix& fock, const SpectralTransform& t,
                               const PurificationConfig& config) {
  return purify(initial_transform(fock, t), config);
}

}  // namespace spamm
