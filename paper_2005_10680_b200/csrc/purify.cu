// purify.cu -- SP2 density-matrix purification over the GPU product
// (purification.cpp:49-202, BASELINE config 3).
//
// Same driver as the reference: error budget (ErrorBudget::geometric,
// purification.cpp:66-82, or caller-supplied deltas), initial truncation for
// the truncmul/hybrid variants, trace-steered polynomial choice (sp2_step
// :59-64), squaring by multiply_exact (truncmul / exact mode) or
// spamm_with_error_control (spamm: delta_i, hybrid: delta_i/2), idempotency
// stop |tr X - tr X^2| < eta, 2X - X^2 as fl(fl(2x) + fl(-x^2)) (apply_polynomial
// :21-25), truncation (truncmul: delta_i, hybrid: delta_i/2) and the
// measurement-only realized error ||X_i - f(X_{i-1})||_F against an exact
// product.  Every matrix stays on the device; traces and counts are the only
// host transfers per iteration.
#include <chrono>
#include <cmath>
#include <limits>
#include <memory>
#include <vector>

#include "common.cuh"

namespace spg {
namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

using MatPtr = std::unique_ptr<spg_matrix, void (*)(spg_matrix*)>;
MatPtr own(spg_matrix* m) { return MatPtr(m, matrix_destroy); }

// apply_polynomial (purification.cpp:21-25)
MatPtr apply_poly(spg_context* ctx, int square, const spg_matrix* x, const spg_matrix* x2) {
  if (square) return own(axpby_device(ctx, 1.0, x2, 0.0, nullptr));  // an owned copy of x^2
  return own(axpby_device(ctx, 2.0, x, -1.0, x2));
}

}  // namespace
}  // namespace spg

using namespace spg;

extern "C" {

int spg_error_budget_geometric(double epsilon, int32_t iterations, double ratio,
                               double* initial_delta, double* deltas) {
  SPG_API_BEGIN
  // ErrorBudget::geometric (purification.cpp:66-82)
  if (!(epsilon > 0.0)) fail(SPG_EINVAL, "budget: epsilon must be positive");
  if (iterations < 1) fail(SPG_EINVAL, "budget: iteration count must be positive");
  if (!(ratio > 0.0 && ratio < 1.0)) fail(SPG_EINVAL, "budget: ratio must be in (0, 1)");
  if (!initial_delta || !deltas) fail(SPG_EINVAL, "null argument");
  *initial_delta = epsilon / 2.0;
  const double half = epsilon / 2.0;
  const double geometric_mass = 1.0 - std::pow(ratio, iterations);
  double term = (1.0 - ratio) / geometric_mass;
  for (int i = 0; i < iterations; ++i) {
    volatile double d = half * term;
    deltas[i] = std::max(static_cast<double>(d), std::numeric_limits<double>::min());
    term *= ratio;
  }
  SPG_API_END
}

int spg_purify(spg_context* ctx, const spg_matrix* x0, const spg_purify_config* cfg,
               spg_matrix** density, spg_run_record* log, int32_t log_capacity, int32_t* n_log,
               int32_t* converged, int32_t* iterations) {
  SPG_API_BEGIN
  if (!ctx || !x0 || !cfg || !density) fail(SPG_EINVAL, "null argument");
  *density = nullptr;
  // purification.cpp:91-104
  if (cfg->occupation <= 0 || cfg->occupation >= x0->dimension)
    fail(SPG_EINVAL, "purify: occupation must lie strictly between 0 and the dimension");
  if (cfg->max_iterations < 1) fail(SPG_EINVAL, "purify: max_iterations must be positive");
  if (!(cfg->epsilon > 0.0)) fail(SPG_EINVAL, "purify: epsilon must be positive");
  if (cfg->variant < SPG_VARIANT_TRUNCMUL || cfg->variant > SPG_VARIANT_HYBRID)
    fail(SPG_EINVAL, "purify: unknown variant");
  if (!cfg->deltas || cfg->n_deltas < cfg->max_iterations)
    fail(SPG_EINVAL, "purify: budget provides fewer deltas than max_iterations");
  int rc = spg_tolerance_grid_check(cfg->taus, cfg->n_taus);
  if (rc != SPG_OK) return rc;
  const double eta =
      cfg->idempotency_threshold > 0.0 ? cfg->idempotency_threshold : cfg->epsilon / 10.0;
  CtxGuard g(ctx);
  int32_t nl = 0;
  auto push = [&](const spg_run_record& r) {
    if (log && nl < log_capacity) log[nl] = r;
    ++nl;
  };

  MatPtr cur = own(axpby_device(ctx, 1.0, x0, 0.0, nullptr));  // X (owned copy of x0)
  if (cfg->variant != SPG_VARIANT_SPAMM && cfg->initial_delta > 0.0) {  // :109-126
    spg_run_record rec{};
    rec.iteration = 0;
    rec.tolerance = cfg->initial_delta;
    rec.nnz_in = nnz_device(ctx, x0);
    const auto t0 = Clock::now();
    double removed = 0.0;
    int64_t count = 0;
    MatPtr t = own(truncate_device(ctx, x0, cfg->initial_delta, &removed, &count));
    rec.t_trunc = seconds_since(t0);
    rec.nnz_mid = rec.nnz_in;
    cur = std::move(t);
    rec.nnz_out = nnz_device(ctx, cur.get());
    rec.nnz_blocks_out = cur->nnzb;
    rec.realized_error = removed;
    rec.status = SPG_STATUS_OK;
    rec.trace = trace_device(ctx, cur.get());
    push(rec);
  }

  int32_t done = 0, its = 0;
  for (int i = 1; i <= cfg->max_iterations; ++i) {
    const double delta = cfg->deltas[i - 1];
    const bool exact_mode = !(delta > 0.0);
    const spg_matrix* prev = cur.get();
    const double tr_prev = trace_device(ctx, prev);
    const int square = tr_prev > static_cast<double>(cfg->occupation);  // sp2_step :59-64
    spg_run_record rec{};
    rec.iteration = i;
    rec.tolerance = delta;
    rec.polynomial = square ? 0 : 1;
    rec.nnz_in = nnz_device(ctx, prev);

    MatPtr squared = own(nullptr);
    if (cfg->variant == SPG_VARIANT_TRUNCMUL || exact_mode) {
      const auto t0 = Clock::now();
      spg_spamm_stats ss{};
      squared = own(spamm_device(ctx, prev, prev, 0.0, false, &ss));
      rec.t_mul = seconds_since(t0);
      rec.flops = ss.flops;
    } else {
      const double md = cfg->variant == SPG_VARIANT_HYBRID ? delta / 2.0 : delta;
      spg_controlled_stats cs{};
      squared = own(controlled_product(ctx, prev, prev, md, cfg->taus, cfg->n_taus, nullptr, &cs));
      rec.chosen_tau = cs.tau;
      rec.t_cse = cs.cse_seconds;
      rec.t_spamm = cs.spamm_seconds;
      rec.flops = cs.spamm.flops;
    }
    const double tr_sq = trace_device(ctx, squared.get());
    if (std::abs(tr_prev - tr_sq) < eta) {  // idempotency stop :156-168
      rec.nnz_mid = nnz_device(ctx, squared.get());
      rec.nnz_out = rec.nnz_in;
      rec.nnz_blocks_out = prev->nnzb;
      rec.realized_error = 0.0;
      rec.status = SPG_STATUS_CONVERGED;
      rec.trace = tr_prev;
      push(rec);
      done = 1;
      its = i - 1;
      break;
    }
    MatPtr iterate = apply_poly(ctx, square, prev, squared.get());
    rec.nnz_mid = nnz_device(ctx, iterate.get());
    if (!exact_mode && cfg->variant != SPG_VARIANT_SPAMM) {  // :173-180
      const double td = cfg->variant == SPG_VARIANT_HYBRID ? delta / 2.0 : delta;
      const auto t0 = Clock::now();
      double removed = 0.0;
      int64_t count = 0;
      iterate = own(truncate_device(ctx, iterate.get(), td, &removed, &count));
      rec.t_trunc = seconds_since(t0);
    }
    rec.nnz_out = nnz_device(ctx, iterate.get());
    rec.nnz_blocks_out = iterate->nnzb;
    if (cfg->measure_error) {  // measurement only (:184-191)
      MatPtr exact_sq = own(spamm_device(ctx, prev, prev, 0.0, false, nullptr));
      MatPtr exact_step = apply_poly(ctx, square, prev, exact_sq.get());
      MatPtr diff = own(axpby_device(ctx, 1.0, iterate.get(), -1.0, exact_step.get()));
      rec.realized_error = diff->frob;
      rec.status = (rec.realized_error < delta || (exact_mode && rec.realized_error == 0.0))
                       ? SPG_STATUS_OK
                       : SPG_STATUS_VIOLATION;
    } else {
      rec.realized_error = -1.0;
      rec.status = SPG_STATUS_OK;
    }
    rec.trace = trace_device(ctx, iterate.get());
    push(rec);
    cur = std::move(iterate);
    its = i;
  }
  if (n_log) *n_log = nl;
  if (converged) *converged = done;
  if (iterations) *iterations = its;
  *density = cur.release();
  SPG_API_END
}

}  // extern "C"
