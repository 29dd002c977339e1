// truncate.cu -- greedy block truncation (error_control.cpp:93-134,174-201) and
// the approximate-square variants of the experiment protocol
// (experiment.cpp:47-82: truncmul, spamm, hybrid).  SURVEY.md 8f "next" row 1.
//
// Truncation semantics, bit for bit: leaves ordered by (norm, row-major block
// position) ascending; walking that order a leaf is removed while
// sqrt(fl(s + fl(n*n))) < delta, with s accumulating fl(s + fl(n*n)) in the
// same order.  The running sum is inherently sequential: one thread runs its
// add chain chunk by chunk while the block checks the stop test in parallel
// (trunc_walk); the sort is the other parallel part.  Removed leaves become null; inner norms are rebuilt by
// K2 (combine_child_norms), which equals the reference's make_inner on the
// changed paths and its cached norms everywhere else.  The result shares the
// input's leaf payload -- nothing is copied.
#include <cub/cub.cuh>

#include <chrono>

#include "common.cuh"

namespace spg {

namespace {

__global__ void trunc_positions(const uint64_t* __restrict__ keys, int64_t n, int side_bits,
                                uint64_t* __restrict__ position, int64_t* __restrict__ index) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint64_t key = keys[t];
  position[t] = (static_cast<uint64_t>(morton_row(key)) << side_bits) | morton_col(key);
  index[t] = t;
}

// norm bits (non-negative doubles order like their bit patterns) of the
// leaves in position order
__global__ void trunc_gather_norms(const int64_t* __restrict__ index, int64_t n,
                                   const uint64_t* __restrict__ keys,
                                   const double* __restrict__ leaf_level,
                                   uint64_t* __restrict__ norm_bits) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  norm_bits[t] = static_cast<uint64_t>(__double_as_longlong(leaf_level[keys[index[t]]]));
}

// The greedy walk.  The running sum is a sequential FP recurrence, but the
// stop test is not part of it: s_c = fl(s_{c-1} + fl(n_c^2)) is the plain
// prefix sum up to the first c with !(sqrt(s_c) < delta), and the removed
// count is that c.  So one thread runs only the DADD chain for a chunk of
// kWalkChunk leaves into shared memory, then the block tests the chunk's
// prefix sums in parallel (correctly rounded sqrt, same comparison) and
// stops at the first failure -- bit-identical to the one-leaf-at-a-time
// loop, with the square root and the branch off the dependency chain.
constexpr int kWalkChunk = 4096;

__global__ void __launch_bounds__(256) trunc_walk(const uint64_t* __restrict__ sorted_norm_bits,
                                                  int64_t n, double delta,
                                                  int64_t* __restrict__ count,
                                                  double* __restrict__ removed) {
  __shared__ double pref[kWalkChunk];
  __shared__ int first_fail;
  __shared__ double carry;  // prefix sum before the chunk
  if (threadIdx.x == 0) carry = 0.0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += kWalkChunk) {
    const int len = static_cast<int>(n - base < kWalkChunk ? n - base : kWalkChunk);
    // squares in parallel (coalesced loads), then the add chain alone
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const double v = __longlong_as_double(static_cast<long long>(sorted_norm_bits[base + i]));
      pref[i] = __dmul_rn(v, v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = carry;
      first_fail = len;
      for (int i = 0; i < len; ++i) {
        s = __dadd_rn(s, pref[i]);
        pref[i] = s;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += blockDim.x)
      if (!(__dsqrt_rn(pref[i]) < delta)) atomicMin(&first_fail, i);
    __syncthreads();
    const int f = first_fail;
    if (f < len) {
      if (threadIdx.x == 0) {
        *count = base + f;
        *removed = __dsqrt_rn(f > 0 ? pref[f - 1] : carry);
      }
      return;
    }
    if (threadIdx.x == 0) carry = pref[len - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *count = n;
    *removed = __dsqrt_rn(carry);
  }
}

__global__ void trunc_slot_flags(const uint64_t* __restrict__ keys,
                                 const int32_t* __restrict__ slots, int64_t n,
                                 const double* __restrict__ leaf_level,
                                 double* __restrict__ slot_norms, uint8_t* __restrict__ keep) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t s = slots[t];
  slot_norms[s] = leaf_level[keys[t]];
  keep[s] = 1;
}

__global__ void trunc_mark_removed(const int64_t* __restrict__ sorted_index, int64_t n,
                                   const int64_t* __restrict__ count,
                                   const int32_t* __restrict__ slots, uint8_t* __restrict__ keep) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n || t >= *count) return;
  keep[slots[sorted_index[t]]] = 0;
}

}  // namespace

spg_matrix* truncate_device(spg_context* ctx, const spg_matrix* x, double delta,
                            double* removed_norm, int64_t* removed_count) {
  if (delta < 0.0) fail(SPG_EINVAL, "truncate: delta must be nonnegative");  // :175
  require_payload(x);
  const int64_t n = x->nnzb;
  const int d = x->depth;
  const double* leaf_level = x->pyramid + level_offset(d);
  DevBuf<int64_t> d_count(1, ctx);
  DevBuf<double> d_removed(1, ctx);
  SPG_CUDA(cudaMemsetAsync(d_count.get(), 0, sizeof(int64_t), ctx->stream));
  SPG_CUDA(cudaMemsetAsync(d_removed.get(), 0, sizeof(double), ctx->stream));
  DevBuf<double> slot_norms(std::max<int64_t>(x->n_slots, 1), ctx);
  DevBuf<uint8_t> keep(std::max<int64_t>(x->n_slots, 1), ctx);
  SPG_CUDA(cudaMemsetAsync(keep.get(), 0, std::max<int64_t>(x->n_slots, 1), ctx->stream));
  if (n > 0) {
    DevBuf<uint64_t> pos(n, ctx), pos_sorted(n, ctx), nbits(n, ctx), nbits_sorted(n, ctx);
    DevBuf<int64_t> idx(n, ctx), idx_pos(n, ctx), idx_sorted(n, ctx);
    trunc_positions<<<grid_for(n, 256), 256, 0, ctx->stream>>>(x->keys, n, d, pos.get(),
                                                               idx.get());
    SPG_CHECK_LAUNCH(ctx);
    const int pos_bits = std::max(1, 2 * d);
    size_t b1 = 0, b2 = 0;
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, pos.get(), pos_sorted.get(), idx.get(),
                                             idx_pos.get(), n, 0, pos_bits, ctx->stream));
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, nbits.get(), nbits_sorted.get(),
                                             idx_pos.get(), idx_sorted.get(), n, 0, 64,
                                             ctx->stream));
    DevBuf<uint8_t> tmp(std::max<size_t>(std::max(b1, b2), 1), ctx);
    size_t bytes = tmp.n;
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, pos.get(), pos_sorted.get(),
                                             idx.get(), idx_pos.get(), n, 0, pos_bits,
                                             ctx->stream));
    ctx->lib_calls++;
    trunc_gather_norms<<<grid_for(n, 256), 256, 0, ctx->stream>>>(idx_pos.get(), n, x->keys,
                                                                  leaf_level, nbits.get());
    SPG_CHECK_LAUNCH(ctx);
    bytes = tmp.n;  // stable: equal norms keep the position order
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, nbits.get(), nbits_sorted.get(),
                                             idx_pos.get(), idx_sorted.get(), n, 0, 64,
                                             ctx->stream));
    ctx->lib_calls++;
    trunc_walk<<<1, 256, 0, ctx->stream>>>(nbits_sorted.get(), n, delta, d_count.get(),
                                          d_removed.get());
    SPG_CHECK_LAUNCH(ctx);
    trunc_slot_flags<<<grid_for(n, 256), 256, 0, ctx->stream>>>(x->keys, x->slots, n, leaf_level,
                                                                slot_norms.get(), keep.get());
    SPG_CHECK_LAUNCH(ctx);
    trunc_mark_removed<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        idx_sorted.get(), n, d_count.get(), x->slots, keep.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  SPG_CUDA(cudaMemcpyAsync(removed_count, d_count.get(), sizeof(int64_t), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaMemcpyAsync(removed_norm, d_removed.get(), sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  return matrix_keep_slots(ctx, x, slot_norms.get(), keep.get());
}

}  // namespace spg

using namespace spg;

namespace {
using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}
}  // namespace

extern "C" {

int spg_truncate(spg_context* ctx, const spg_matrix* x, double delta, spg_matrix** out,
                 double* removed_norm_bound, int64_t* removed_block_count) {
  SPG_API_BEGIN
  if (!ctx || !x || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  CtxGuard g(ctx);
  double rn = 0.0;
  int64_t rc = 0;
  *out = truncate_device(ctx, x, delta, &rn, &rc);
  if (removed_norm_bound) *removed_norm_bound = rn;
  if (removed_block_count) *removed_block_count = rc;
  SPG_API_END
}

int spg_approximate_square(spg_context* ctx, const spg_matrix* x, int32_t variant, double delta,
                           const double* taus, int32_t n_taus, spg_matrix** out,
                           spg_square_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !x || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (variant != SPG_VARIANT_TRUNCMUL && variant != SPG_VARIANT_SPAMM &&
      variant != SPG_VARIANT_HYBRID)
    fail(SPG_EINVAL, "approximate_square: unknown variant");
  spg_square_stats st{};
  st.variant = variant;
  if (variant == SPG_VARIANT_TRUNCMUL) {  // experiment.cpp:50-60
    CtxGuard g(ctx);
    const auto t0 = Clock::now();
    spg_spamm_stats ss{};
    spg_matrix* prod = spamm_device(ctx, x, x, 0.0, false, &ss);
    st.t_mul = seconds_since(t0);
    st.nnz_blocks_mid = prod->nnzb;
    const auto t1 = Clock::now();
    try {
      *out = truncate_device(ctx, prod, delta, &st.removed_norm_bound, &st.removed_blocks);
    } catch (...) {
      matrix_destroy(prod);
      throw;
    }
    matrix_destroy(prod);
    st.t_trunc = seconds_since(t1);
    st.chosen_tau = 0.0;
    st.flops = ss.flops;
  } else {  // spamm (:61-68) or hybrid (:69-79): delta/2 to the product, delta/2 to truncation
    const double d_mul = variant == SPG_VARIANT_HYBRID ? delta / 2.0 : delta;
    spg_matrix* prod = nullptr;
    spg_controlled_stats cs{};
    int rc = spg_spamm_with_error_control(ctx, x, x, d_mul, taus, n_taus, &prod, nullptr, &cs);
    if (rc != SPG_OK) return rc;
    st.t_cse = cs.cse_seconds;
    st.t_spamm = cs.spamm_seconds;
    st.chosen_tau = cs.tau;
    st.flops = cs.spamm.flops;
    {
      CtxGuard g(ctx);
      st.nnz_blocks_mid = prod->nnzb;
      if (variant == SPG_VARIANT_HYBRID) {
        const auto t1 = Clock::now();
        try {
          *out = truncate_device(ctx, prod, delta / 2.0, &st.removed_norm_bound,
                                 &st.removed_blocks);
        } catch (...) {
          matrix_destroy(prod);
          throw;
        }
        matrix_destroy(prod);
        st.t_trunc = seconds_since(t1);
      } else {
        *out = prod;
      }
    }
  }
  if (stats) *stats = st;
  SPG_API_END
}

}  // extern "C"
