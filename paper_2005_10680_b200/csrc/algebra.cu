// algebra.cu -- device matrix algebra used by the callers of the hot path
// (SP2 purification): trace, nnz, alpha*A + beta*B,
// identity.  Same results as the reference's host operations:
//   trace   node_trace (quadtree.cpp:128-138): leaf = sequential diagonal sum,
//           inner = trace(child 0) + trace(child 3)  (pairwise over the
//           diagonal blocks, null = 0)
//   nnz     node_nnz (quadtree.cpp:140-151)
//   axpby   add(A.scale(alpha), B.scale(beta)) (quadtree.cpp:24-36,153-171,
//           254-261): fl(fl(alpha a) + fl(beta b)) where both leaves exist,
//           the scaled leaf where one does; all-zero leaves collapse (K1)
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <limits>
#include <vector>

#include "common.cuh"

namespace spg {

namespace {

__global__ void diag_leaf_traces(const int32_t* __restrict__ grid_slot, int32_t nb,
                                 const double* __restrict__ payload, int L,
                                 double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const int32_t s = grid_slot[morton2(i, i)];
  double t = 0.0;
  if (s >= 0) {
    const double* blk = payload + static_cast<int64_t>(s) * L * L;
    for (int k = 0; k < L; ++k) t = __dadd_rn(t, blk[k + static_cast<int64_t>(k) * L]);
  }
  out[i] = t;
}

__global__ void count_nonzero(const double* __restrict__ payload,
                              const int32_t* __restrict__ slots, int64_t n, int64_t LL,
                              unsigned long long* __restrict__ total) {
  unsigned long long local = 0;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n * LL;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t leaf = t / LL, e = t - leaf * LL;
    local += payload[static_cast<int64_t>(slots[leaf]) * LL + e] != 0.0;
  }
  for (int off = 16; off; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(total, local);
}

struct InEither {
  const int32_t* ga;
  const int32_t* gb;
  __host__ __device__ bool operator()(const uint64_t& p) const {
    return ga[p] >= 0 || (gb && gb[p] >= 0);
  }
};

__global__ void axpby_blocks(const uint64_t* __restrict__ keys, int64_t n, double alpha,
                             const int32_t* __restrict__ ga, const double* __restrict__ pa,
                             double beta, const int32_t* __restrict__ gb,
                             const double* __restrict__ pb, int64_t LL,
                             double* __restrict__ out) {
  for (int64_t blk = blockIdx.x; blk < n; blk += gridDim.x) {
    const uint64_t key = keys[blk];
    const int32_t sa = ga[key];
    const int32_t sb = gb ? gb[key] : -1;
    const double* a = sa >= 0 ? pa + static_cast<int64_t>(sa) * LL : nullptr;
    const double* b = sb >= 0 ? pb + static_cast<int64_t>(sb) * LL : nullptr;
    double* o = out + blk * LL;
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) {
      double v;
      if (a && b) v = __dadd_rn(__dmul_rn(alpha, a[e]), __dmul_rn(beta, b[e]));
      else if (a) v = __dmul_rn(alpha, a[e]);
      else v = __dmul_rn(beta, b[e]);
      o[e] = v;
    }
  }
}

// per row i: the diagonal entry and sum_j |a_ij| in ascending j (deterministic);
// off_diagonal: j == i left out, as oracle.cpp's off_diagonal_row_sum does
__global__ void row_scan_kernel(const int32_t* __restrict__ grid_slot, int32_t dimension,
                                int32_t nb_logical, const double* __restrict__ payload, int L,
                                double* __restrict__ diag, double* __restrict__ abs_sum,
                                bool off_diagonal = false) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dimension) return;
  const uint32_t br = static_cast<uint32_t>(i / L);
  const int r = i % L;
  const int64_t LL = static_cast<int64_t>(L) * L;
  double s = 0.0, dv = 0.0;
  for (uint32_t bc = 0; bc < static_cast<uint32_t>(nb_logical); ++bc) {
    const int32_t slot = grid_slot[morton2(br, bc)];
    if (slot < 0) continue;
    const double* blk = payload + static_cast<int64_t>(slot) * LL + r;
    const int jn = min(L, dimension - static_cast<int>(bc) * L);
    for (int j = 0; j < jn; ++j) {
      const double v = blk[static_cast<int64_t>(j) * L];
      const bool on_diag = bc == br && j == r;
      if (!(off_diagonal && on_diag)) s = __dadd_rn(s, fabs(v));
      if (on_diag) dv = v;
    }
  }
  if (diag) diag[i] = dv;
  if (abs_sum) abs_sum[i] = s;
}

}  // namespace

double trace_device(spg_context* ctx, const spg_matrix* m) {
  require_payload(m);
  const int32_t nb = 1 << m->depth;
  DevBuf<double> t(nb, ctx);
  diag_leaf_traces<<<grid_for(nb, 128), 128, 0, ctx->stream>>>(m->grid_slot, nb, m->payload,
                                                               m->leaf, t.get());
  SPG_CHECK_LAUNCH(ctx);
  std::vector<double> h(static_cast<size_t>(nb));
  SPG_CUDA(cudaMemcpyAsync(h.data(), t.get(), nb * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  // node_trace's association: trace(child 0) + trace(child 3), level by level
  for (int32_t w = nb; w > 1; w >>= 1)
    for (int32_t i = 0; i < w / 2; ++i) {
      volatile double s = h[2 * i] + h[2 * i + 1];
      h[i] = s;
    }
  return h[0];
}

int64_t nnz_device(spg_context* ctx, const spg_matrix* m) {
  require_payload(m);
  if (m->nnzb == 0) return 0;
  DevBuf<unsigned long long> total(1, ctx);
  SPG_CUDA(cudaMemsetAsync(total.get(), 0, sizeof(unsigned long long), ctx->stream));
  const int64_t LL = static_cast<int64_t>(m->leaf) * m->leaf;
  count_nonzero<<<grid_for(m->nnzb * LL, 256, int64_t(ctx->sm_count) * 32), 256, 0, ctx->stream>>>(
      m->payload, m->slots, m->nnzb, LL, total.get());
  SPG_CHECK_LAUNCH(ctx);
  unsigned long long h = 0;
  SPG_CUDA(cudaMemcpyAsync(&h, total.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  return static_cast<int64_t>(h);
}

spg_matrix* axpby_device(spg_context* ctx, double alpha, const spg_matrix* a, double beta,
                         const spg_matrix* b) {
  require_payload(a);
  require_payload(b);
  if (b && (a->dimension != b->dimension || a->leaf != b->leaf))
    fail(SPG_EINVAL, "add: dimension or leaf size mismatch");
  // QuadTreeMatrix::scale(0) is the zero matrix (quadtree.cpp:249-252)
  const bool use_a = alpha != 0.0;
  const bool use_b = b != nullptr && beta != 0.0;
  const spg_matrix* first = use_a ? a : (use_b ? b : a);
  const int64_t cells = int64_t(1) << (2 * a->depth);
  const int64_t LL = static_cast<int64_t>(a->leaf) * a->leaf;
  if (!use_a && !use_b) {
    return matrix_from_morton_blocks(ctx, a->dimension, a->leaf, 0, nullptr,
                                     dev_alloc<double>(1, ctx));
  }
  const spg_matrix* second = (use_a && use_b) ? b : nullptr;
  const double s1 = use_a ? alpha : beta, s2 = beta;
  DevBuf<uint64_t> keys(std::max<int64_t>(cells, 1), ctx);
  DevBuf<int64_t> n_sel(1, ctx);
  thrust::counting_iterator<uint64_t> it(0);
  InEither pred{first->grid_slot, second ? second->grid_slot : nullptr};
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, keys.get(), n_sel.get(), cells, pred,
                                 ctx->stream));
  DevBuf<uint8_t> tmp(std::max<size_t>(bytes, 1), ctx);
  SPG_CUDA(cub::DeviceSelect::If(tmp.get(), bytes, it, keys.get(), n_sel.get(), cells, pred,
                                 ctx->stream));
  ctx->lib_calls++;
  const int64_t n = copy_scalar_to_host_i64(ctx, n_sel.get());
  double* payload = dev_alloc<double>(std::max<int64_t>(n * LL, 1), ctx);
  uint64_t* out_keys = dev_alloc<uint64_t>(std::max<int64_t>(n, 1), ctx);
  if (n) {
    SPG_CUDA(cudaMemcpyAsync(out_keys, keys.get(), n * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    axpby_blocks<<<static_cast<unsigned>(std::min<int64_t>(n, 1 << 20)), 256, 0, ctx->stream>>>(
        out_keys, n, s1, first->grid_slot, first->payload, s2,
        second ? second->grid_slot : nullptr, second ? second->payload : nullptr, LL, payload);
    SPG_CHECK_LAUNCH(ctx);
  }
  return matrix_from_morton_blocks(ctx, a->dimension, a->leaf, n, out_keys, payload);
}

spg_matrix* diagonal_device(spg_context* ctx, int32_t dimension, int32_t leaf,
                            const double* diag) {
  int32_t padded, depth;
  check_shape(dimension, leaf, &padded, &depth);
  const int32_t nb = (dimension + leaf - 1) / leaf;
  const int64_t LL = static_cast<int64_t>(leaf) * leaf;
  std::vector<int32_t> rows(static_cast<size_t>(nb));
  std::vector<double> pay(static_cast<size_t>(nb * LL), 0.0);
  for (int32_t i = 0; i < nb; ++i) {
    rows[i] = i;
    for (int32_t k = 0; k < leaf && i * leaf + k < dimension; ++k)
      pay[i * LL + k + static_cast<int64_t>(k) * leaf] = diag ? diag[i * leaf + k] : 1.0;
  }
  DevBuf<int32_t> d_rows(nb, ctx);
  double* d_pay = dev_alloc<double>(nb * LL, ctx);
  SPG_CUDA(cudaMemcpyAsync(d_rows.get(), rows.data(), nb * sizeof(int32_t),
                           cudaMemcpyHostToDevice, ctx->stream));
  SPG_CUDA(cudaMemcpyAsync(d_pay, pay.data(), nb * LL * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  return matrix_from_device_leaves(ctx, dimension, leaf, nb, d_rows.get(), d_rows.get(), d_pay);
}

spg_matrix* identity_device(spg_context* ctx, int32_t dimension, int32_t leaf) {
  return diagonal_device(ctx, dimension, leaf, nullptr);
}

}  // namespace spg

using namespace spg;

extern "C" {

int spg_matrix_trace(const spg_matrix* m, double* out) {
  SPG_API_BEGIN
  if (!m || !out) fail(SPG_EINVAL, "null argument");
  CtxGuard g(m->ctx);
  *out = trace_device(m->ctx, m);
  SPG_API_END
}

int spg_matrix_nnz(const spg_matrix* m, int64_t* out) {
  SPG_API_BEGIN
  if (!m || !out) fail(SPG_EINVAL, "null argument");
  CtxGuard g(m->ctx);
  *out = nnz_device(m->ctx, m);
  SPG_API_END
}

int spg_matrix_axpby(spg_context* ctx, double alpha, const spg_matrix* a, double beta,
                     const spg_matrix* b, spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !a || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  CtxGuard g(ctx);
  *out = axpby_device(ctx, alpha, a, beta, b);
  SPG_API_END
}

int spg_matrix_from_diagonal(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                             const double* diag, spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out || !diag) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  CtxGuard g(ctx);
  *out = diagonal_device(ctx, dimension, leaf_size, diag);
  SPG_API_END
}

int spg_matrix_rows(const spg_matrix* m, double* diag, double* abs_row_sums) {
  SPG_API_BEGIN
  if (!m) fail(SPG_EINVAL, "null argument");
  require_payload(m);
  spg_context* ctx = m->ctx;
  CtxGuard g(ctx);
  const int32_t n = m->dimension, nb = (n + m->leaf - 1) / m->leaf;
  DevBuf<double> d(n, ctx), a(n, ctx);
  row_scan_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(m->grid_slot, n, nb, m->payload,
                                                             m->leaf, d.get(), a.get());
  SPG_CHECK_LAUNCH(ctx);
  if (diag)
    SPG_CUDA(cudaMemcpyAsync(diag, d.get(), n * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
  if (abs_row_sums)
    SPG_CUDA(cudaMemcpyAsync(abs_row_sums, a.get(), n * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  SPG_API_END
}

int spg_matrix_gershgorin(const spg_matrix* m, double* low, double* high) {
  SPG_API_BEGIN
  if (!m || !low || !high) fail(SPG_EINVAL, "null argument");
  require_payload(m);
  spg_context* ctx = m->ctx;
  CtxGuard g(ctx);
  const int32_t n = m->dimension, nb = (n + m->leaf - 1) / m->leaf;
  DevBuf<double> d(n, ctx), r(n, ctx);
  row_scan_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(m->grid_slot, n, nb, m->payload,
                                                             m->leaf, d.get(), r.get(), true);
  SPG_CHECK_LAUNCH(ctx);
  std::vector<double> hd(static_cast<size_t>(n)), hr(static_cast<size_t>(n));
  SPG_CUDA(cudaMemcpyAsync(hd.data(), d.get(), n * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaMemcpyAsync(hr.data(), r.get(), n * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  // oracle.cpp:191-200: ascending rows, std::min / std::max semantics
  double lo = std::numeric_limits<double>::infinity();
  double hi = -std::numeric_limits<double>::infinity();
  for (int32_t i = 0; i < n; ++i) {
    volatile double a = hd[i] - hr[i], b = hd[i] + hr[i];
    lo = std::min(lo, static_cast<double>(a));
    hi = std::max(hi, static_cast<double>(b));
  }
  *low = lo;
  *high = hi;
  SPG_API_END
}

int spg_matrix_identity(spg_context* ctx, int32_t dimension, int32_t leaf_size, spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  CtxGuard g(ctx);
  *out = identity_device(ctx, dimension, leaf_size);
  SPG_API_END
}

}  // extern "C"
