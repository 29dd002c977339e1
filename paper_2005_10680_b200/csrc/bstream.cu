// bstream.cu -- B resident in host memory, streamed to the GPU in panels of
// block rows (configs 4/5, where B does not fit next to A and C
// in one GPU's HBM).
//
// The reference holds B as a host quadtree (quadtree.cpp:198-222) and its
// recursion reads leaves as it reaches them; here the leaves stay in the
// caller's host buffer sorted by block row, so a panel of block rows
// [r0, r1) is one contiguous byte range.  Creation streams every panel once
// through K1 (leaf norms, bit-exact block_norm) to build B's norm pyramid on
// the device; CSE and the task list need nothing else.  The product
// (spamm_streamed_device, spamm.cu) streams the panels again, double
// buffered, and continues each output block's accumulator per panel.
#include <algorithm>
#include <chrono>
#include <memory>
#include <vector>

#include "common.cuh"

namespace spg {
namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

void bstream_destroy(spg_bstream* bs) {
  if (!bs) return;
  matrix_destroy(bs->norms);
  if (bs->registered) cudaHostUnregister(const_cast<double*>(bs->host_payload));
  delete bs;
}

spg_bstream* bstream_create(spg_context* ctx, int32_t dimension, int32_t leaf, int64_t n,
                            const int32_t* rows, const int32_t* cols, const double* payload,
                            int32_t panel_rows, bool register_host) {
  int32_t padded = 0, depth = 0;
  check_shape(dimension, leaf, &padded, &depth);
  if (n < 0) fail(SPG_EINVAL, "negative leaf count");
  if (n && (!rows || !cols || !payload)) fail(SPG_EINVAL, "null argument");
  if (panel_rows < 1) fail(SPG_EINVAL, "panel_block_rows must be positive");
  for (int64_t t = 1; t < n; ++t)
    if (rows[t] < rows[t - 1]) fail(SPG_EINVAL, "bstream: leaves must be sorted by block row");
  const int64_t LL = static_cast<int64_t>(leaf) * leaf;
  std::unique_ptr<spg_bstream, void (*)(spg_bstream*)> bs(new spg_bstream, bstream_destroy);
  bs->ctx = ctx;
  bs->host_payload = payload;
  const int32_t nb = 1 << depth;
  for (int32_t r = 0; r < nb; r += panel_rows) bs->panel_row.push_back(r);
  bs->panel_row.push_back(nb);
  for (int32_t r : bs->panel_row)
    bs->panel_leaf.push_back(std::lower_bound(rows, rows + n, r) - rows);
  // leaves with a row outside [0, nb) fall outside every panel; the scatter
  // below rejects them (SPG_ERANGE) like spg_matrix_upload
  for (size_t p = 0; p + 1 < bs->panel_leaf.size(); ++p)
    bs->max_panel_leaves =
        std::max(bs->max_panel_leaves, bs->panel_leaf[p + 1] - bs->panel_leaf[p]);
  if (register_host && n) {
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, payload) == cudaSuccess &&
                        attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (!pinned) {
      void* host = const_cast<double*>(payload);
      const size_t bytes = static_cast<size_t>(n) * LL * sizeof(double);
      if (cudaHostRegister(host, bytes, cudaHostRegisterReadOnly) != cudaSuccess) {
        cudaGetLastError();
        SPG_CUDA(cudaHostRegister(host, bytes, cudaHostRegisterDefault));
      }
      bs->registered = true;
    }
  }
  DevBuf<int32_t> d_rows(std::max<int64_t>(n, 1), ctx), d_cols(std::max<int64_t>(n, 1), ctx);
  DevBuf<double> norms(std::max<int64_t>(n, 1), ctx);
  DevBuf<uint8_t> nonzero(std::max<int64_t>(n, 1), ctx);
  DevBuf<int> bad(1, ctx);
  SPG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), ctx->stream));
  if (n) {
    SPG_CUDA(cudaMemcpyAsync(d_rows.get(), rows, n * sizeof(int32_t), cudaMemcpyHostToDevice,
                             ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(d_cols.get(), cols, n * sizeof(int32_t), cudaMemcpyHostToDevice,
                             ctx->stream));
  }
  // norm pass: panel q+1 copies (copy stream) while K1 runs on panel q
  const int32_t nb_logical = (dimension + leaf - 1) / leaf;
  const int64_t cap = bs->max_panel_leaves;
  if (cap) {
    DevBuf<double> buf[2] = {DevBuf<double>(cap * LL, ctx), DevBuf<double>(cap * LL, ctx)};
    cudaEvent_t ev[4];
    for (auto& e : ev) SPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct Guard {
      cudaEvent_t* e;
      ~Guard() {
        for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
      }
    } guard{ev};
    SPG_CUDA(cudaEventRecord(ev[2], ctx->stream));
    SPG_CUDA(cudaEventRecord(ev[3], ctx->stream));
    std::vector<int> live;
    for (size_t p = 0; p + 1 < bs->panel_leaf.size(); ++p)
      if (bs->panel_leaf[p + 1] > bs->panel_leaf[p]) live.push_back(static_cast<int>(p));
    auto issue_copy = [&](size_t q) {
      const int p = live[q], i = static_cast<int>(q & 1);
      const int64_t lo = bs->panel_leaf[p], cnt = bs->panel_leaf[p + 1] - lo;
      SPG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev[2 + i], 0));
      SPG_CUDA(cudaMemcpyAsync(buf[i].get(), payload + lo * LL, cnt * LL * sizeof(double),
                               cudaMemcpyHostToDevice, ctx->copy_stream));
      SPG_CUDA(cudaEventRecord(ev[i], ctx->copy_stream));
    };
    if (!live.empty()) issue_copy(0);
    for (size_t q = 0; q < live.size(); ++q) {
      if (q + 1 < live.size()) issue_copy(q + 1);
      const int p = live[q], i = static_cast<int>(q & 1);
      const int64_t lo = bs->panel_leaf[p], cnt = bs->panel_leaf[p + 1] - lo;
      SPG_CUDA(cudaStreamWaitEvent(ctx->stream, ev[i], 0));
      leaf_norms(ctx, buf[i].get(), cnt, leaf, dimension, nb_logical, d_rows.get() + lo,
                 d_cols.get() + lo, norms.get() + lo, nonzero.get() + lo, bad.get());
      SPG_CUDA(cudaEventRecord(ev[2 + i], ctx->stream));
    }
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  int h_bad = 0;
  SPG_CUDA(cudaMemcpy(&h_bad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost));
  bs->norms = matrix_from_leaf_norms(ctx, dimension, leaf, n, rows, d_rows.get(), d_cols.get(),
                                     norms.get(), nonzero.get());
  if (h_bad) fail(SPG_EINVAL, "nonzero entry in the padding region of a boundary leaf");
  return bs.release();
}

// spamm_with_error_control (error_control.cpp:203-220) with B streamed:
// cse -> select (first k with bound < delta) -> streamed spamm_multiply.
spg_matrix* controlled_product_streamed(spg_context* ctx, const spg_matrix* a,
                                        const spg_bstream* bs, double delta, const double* taus,
                                        int n_taus, double* bounds,
                                        spg_controlled_stats* stats) {
  std::vector<double> local(static_cast<size_t>(n_taus));
  double* bv = bounds ? bounds : local.data();
  float cse_ms = 0.0f;
  const auto t0 = Clock::now();
  cse_device(ctx, a, bs->norms, taus, n_taus, bv, &cse_ms);
  const double cse_seconds = seconds_since(t0);
  int32_t k = -1;
  for (int32_t i = 0; i < n_taus; ++i)
    if (bv[i] < delta) {
      k = i;
      break;
    }
  const double tau = k >= 0 ? taus[k] : 0.0;
  spg_spamm_stats ss{};
  const auto t1 = Clock::now();
  spg_matrix* c = spamm_streamed_device(ctx, a, bs, tau, stats ? &ss : nullptr);
  const double spamm_seconds = seconds_since(t1);
  if (stats) {
    stats->tau = tau;
    stats->tau_index = k;
    stats->bound = k >= 0 ? bv[k] : 0.0;
    stats->cse_seconds = cse_seconds;
    stats->spamm_seconds = spamm_seconds;
    stats->ms_cse = cse_ms;
    stats->spamm = ss;
  }
  return c;
}

}  // namespace
}  // namespace spg

using namespace spg;

extern "C" {

int spg_bstream_create(spg_context* ctx, int32_t dimension, int32_t leaf_size, int64_t n_leaves,
                       const int32_t* block_rows, const int32_t* block_cols,
                       const double* payload, int32_t panel_block_rows, int32_t register_host,
                       spg_bstream** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  CtxGuard g(ctx);
  *out = bstream_create(ctx, dimension, leaf_size, n_leaves, block_rows, block_cols, payload,
                        panel_block_rows, register_host != 0);
  SPG_API_END
}

int spg_bstream_matrix(const spg_bstream* bs, const spg_matrix** norms) {
  SPG_API_BEGIN
  if (!bs || !norms) fail(SPG_EINVAL, "null argument");
  *norms = bs->norms;
  SPG_API_END
}

int spg_bstream_panels(const spg_bstream* bs, int32_t* n_panels, int64_t* max_panel_leaves) {
  SPG_API_BEGIN
  if (!bs) fail(SPG_EINVAL, "null argument");
  if (n_panels) *n_panels = static_cast<int32_t>(bs->panel_row.size()) - 1;
  if (max_panel_leaves) *max_panel_leaves = bs->max_panel_leaves;
  SPG_API_END
}

void spg_bstream_free(spg_bstream* bs) {
  if (!bs) return;
  try {
    CtxGuard g(bs->ctx);
    bstream_destroy(bs);
  } catch (...) {
  }
}

int spg_spamm_streamed(spg_context* ctx, const spg_matrix* a, const spg_bstream* b, double tau,
                       spg_matrix** c, spg_spamm_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  if (a->ctx != ctx || b->ctx != ctx) fail(SPG_EINVAL, "operands belong to another context");
  CtxGuard g(ctx);
  *c = spamm_streamed_device(ctx, a, b, tau, stats);
  SPG_API_END
}

int spg_spamm_with_error_control_streamed(spg_context* ctx, const spg_matrix* a,
                                          const spg_bstream* b, double delta, const double* taus,
                                          int32_t n_taus, spg_matrix** c, double* bounds,
                                          spg_controlled_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  if (a->ctx != ctx || b->ctx != ctx) fail(SPG_EINVAL, "operands belong to another context");
  if (!(delta > 0.0)) fail(SPG_EINVAL, "spamm_with_error_control: delta must be positive");
  int rc = spg_tolerance_grid_check(taus, n_taus);
  if (rc != SPG_OK) return rc;
  CtxGuard g(ctx);
  *c = controlled_product_streamed(ctx, a, b, delta, taus, n_taus, bounds, stats);
  SPG_API_END
}

}  // extern "C"
