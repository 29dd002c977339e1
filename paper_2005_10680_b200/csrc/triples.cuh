// triples.cuh -- level-by-level expansion of the (A node, B node) pair tree.
//
// The reference recursions (cse_node error_control.cpp:46-79, spamm_node
// multiply.cpp:70-92) visit node pairs A(I,K) x B(K,J) of one level and
// descend into the 8 child pairs (2I+r, 2K+h, 2J+c).  On the GPU the visited
// pairs of a level are a compacted list ("triples"); a parent is expanded into
// its kept children in child order (r, c, h) -- output quadrant q = 2r+c major,
// k-half h minor -- by a count / exclusive-scan / write pass, so the lists are
// deterministic and every parent's children form one contiguous run (the
// offsets of the scan are kept for the bottom-up CSE reduction).
//
// Keep rules, evaluated on the dense Morton norm pyramids (-1 = null):
//   kSweep  (cse):   both children non-null and fl(nA*nB) != 0   (:49-51)
//   kSkip   (spamm): both non-null and !(fl(nA*nB) < tau)         (:72-73)
//   kExact  (multiply_exact): both non-null                       (:37)
#pragma once

#include <cub/cub.cuh>

#include "common.cuh"

namespace spg {

enum class KeepRule : int { kSweep = 0, kSkip = 1, kExact = 2 };

struct TripleList {
  DevBuf<int32_t> I, K, J;
  DevBuf<int64_t> child_offset;  // n + 1 entries once expanded (children of this level)
  int64_t n = 0;
};

template <KeepRule R>
__device__ __forceinline__ bool keep_pair(double na, double nb, double tau) {
  if (na < 0.0 || nb < 0.0) return false;  // null quadrant (NaN norms are non-null)
  if (R == KeepRule::kExact) return true;
  const double p = __dmul_rn(na, nb);
  if (R == KeepRule::kSweep) return p != 0.0;
  return !(p < tau);
}

template <KeepRule R>
__global__ void expand_count(const int32_t* __restrict__ I, const int32_t* __restrict__ K,
                             const int32_t* __restrict__ J, int64_t n,
                             const double* __restrict__ pa, const double* __restrict__ pb,
                             double tau, uint8_t* __restrict__ masks,
                             int64_t* __restrict__ counts) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t i0 = 2u * I[p], k0 = 2u * K[p], j0 = 2u * J[p];
  unsigned mask = 0;
#pragma unroll
  for (int code = 0; code < 8; ++code) {
    const uint32_t r = code >> 2, c = (code >> 1) & 1, h = code & 1;
    const double na = pa[morton2(i0 + r, k0 + h)];
    const double nb = pb[morton2(k0 + h, j0 + c)];
    if (keep_pair<R>(na, nb, tau)) mask |= 1u << code;
  }
  masks[p] = static_cast<uint8_t>(mask);
  counts[p] = __popc(mask);
}

static __global__ void expand_write(const int32_t* __restrict__ I, const int32_t* __restrict__ K,
                             const int32_t* __restrict__ J, int64_t n,
                             const uint8_t* __restrict__ masks,
                             const int64_t* __restrict__ offsets, int32_t* __restrict__ oI,
                             int32_t* __restrict__ oK, int32_t* __restrict__ oJ) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  unsigned mask = masks[p];
  int64_t at = offsets[p];
  const int32_t i0 = 2 * I[p], k0 = 2 * K[p], j0 = 2 * J[p];
  while (mask) {
    const int code = __ffs(mask) - 1;
    mask &= mask - 1;
    oI[at] = i0 + (code >> 2);
    oJ[at] = j0 + ((code >> 1) & 1);
    oK[at] = k0 + (code & 1);
    ++at;
  }
}

// Leaf-level variant: writes the sort key (Morton(i,j) << kbits) | k.
static __global__ void expand_write_keys(const int32_t* __restrict__ I, const int32_t* __restrict__ K,
                                  const int32_t* __restrict__ J, int64_t n,
                                  const uint8_t* __restrict__ masks,
                                  const int64_t* __restrict__ offsets, int kbits,
                                  uint64_t* __restrict__ keys) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  unsigned mask = masks[p];
  int64_t at = offsets[p];
  const uint32_t i0 = 2u * I[p], k0 = 2u * K[p], j0 = 2u * J[p];
  while (mask) {
    const int code = __ffs(mask) - 1;
    mask &= mask - 1;
    const uint32_t i = i0 + (code >> 2), j = j0 + ((code >> 1) & 1), k = k0 + (code & 1);
    keys[at++] = (morton2(i, j) << kbits) | k;
  }
}

// Exclusive scan of int64 counts into offsets[0..n]; returns the total.
inline int64_t scan_counts(spg_context* ctx, const int64_t* counts, int64_t n, int64_t* offsets) {
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, counts, offsets, n + 1, ctx->stream));
  DevBuf<uint8_t> tmp(bytes, ctx);
  SPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, counts, offsets, n + 1, ctx->stream));
  ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
  int64_t total = 0;
  SPG_CUDA(cudaMemcpyAsync(&total, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  return total;
}

// Expand `parent` (level l) into its kept children (level l+1).  counts has
// n+1 slots so the scan's last entry is the total.
template <KeepRule R>
TripleList expand_level(spg_context* ctx, TripleList& parent, const double* pa_child_level,
                        const double* pb_child_level, double tau) {
  TripleList out;
  const int64_t n = parent.n;
  DevBuf<uint8_t> masks(std::max<int64_t>(n, 1), ctx);
  DevBuf<int64_t> counts(n + 1, ctx);
  parent.child_offset = DevBuf<int64_t>(n + 1, ctx);
  SPG_CUDA(cudaMemsetAsync(counts.get() + n, 0, sizeof(int64_t), ctx->stream));
  if (n) {
    expand_count<R><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        parent.I.get(), parent.K.get(), parent.J.get(), n, pa_child_level, pb_child_level, tau,
        masks.get(), counts.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  const int64_t total = scan_counts(ctx, counts.get(), n, parent.child_offset.get());
  out.n = total;
  out.I = DevBuf<int32_t>(std::max<int64_t>(total, 1), ctx);
  out.K = DevBuf<int32_t>(std::max<int64_t>(total, 1), ctx);
  out.J = DevBuf<int32_t>(std::max<int64_t>(total, 1), ctx);
  if (total) {
    expand_write<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        parent.I.get(), parent.K.get(), parent.J.get(), n, masks.get(),
        parent.child_offset.get(), out.I.get(), out.K.get(), out.J.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  return out;
}

// The root pair (level 0) under rule R, decided from the two root norms.
template <KeepRule R>
TripleList root_list(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau) {
  double na = -1.0, nb = -1.0;
  SPG_CUDA(cudaMemcpyAsync(&na, a->pyramid, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SPG_CUDA(cudaMemcpyAsync(&nb, b->pyramid, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  bool keep = !(na < 0.0) && !(nb < 0.0);
  if (keep && R != KeepRule::kExact) {
    volatile double p = na * nb;  // plain IEEE multiply on the host
    keep = (R == KeepRule::kSweep) ? (p != 0.0) : !(p < tau);
  }
  TripleList out;
  out.n = keep ? 1 : 0;
  out.I = DevBuf<int32_t>(1, ctx);
  out.K = DevBuf<int32_t>(1, ctx);
  out.J = DevBuf<int32_t>(1, ctx);
  SPG_CUDA(cudaMemsetAsync(out.I.get(), 0, sizeof(int32_t), ctx->stream));
  SPG_CUDA(cudaMemsetAsync(out.K.get(), 0, sizeof(int32_t), ctx->stream));
  SPG_CUDA(cudaMemsetAsync(out.J.get(), 0, sizeof(int32_t), ctx->stream));
  return out;
}

// The level-`level` pairs (shard, K, J) of one row shard:
// block-rows [shard * nb / 2^level, (shard+1) * nb / 2^level) of C.  For the
// products every ancestor pair must pass the rule too (the reference prunes
// top-down); the sweep keeps pairs whose own norms pass and lets
// spg_cse_finish apply the ancestors' masks.
template <KeepRule R>
TripleList shard_list(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, int level,
                      int shard, double tau, bool check_ancestors) {
  const int64_t top = level_offset(level + 1);
  std::vector<double> pa(static_cast<size_t>(top)), pb(static_cast<size_t>(top));
  SPG_CUDA(cudaMemcpyAsync(pa.data(), a->pyramid, top * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaMemcpyAsync(pb.data(), b->pyramid, top * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  auto keep = [&](int l, uint32_t I, uint32_t K, uint32_t J) {
    const double na = pa[level_offset(l) + morton2(I, K)];
    const double nb = pb[level_offset(l) + morton2(K, J)];
    if (na < 0.0 || nb < 0.0) return false;
    if (R == KeepRule::kExact) return true;
    volatile double p = na * nb;
    return R == KeepRule::kSweep ? (p != 0.0) : !(p < tau);
  };
  std::vector<int32_t> hI, hK, hJ;
  const uint32_t side = 1u << level;
  for (uint32_t K = 0; K < side; ++K)
    for (uint32_t J = 0; J < side; ++J) {
      bool ok = keep(level, shard, K, J);
      for (int l = level - 1; ok && check_ancestors && l >= 0; --l) {
        const int sh = level - l;
        ok = keep(l, static_cast<uint32_t>(shard) >> sh, K >> sh, J >> sh);
      }
      if (!ok) continue;
      hI.push_back(shard);
      hK.push_back(static_cast<int32_t>(K));
      hJ.push_back(static_cast<int32_t>(J));
    }
  TripleList out;
  out.n = static_cast<int64_t>(hI.size());
  const size_t cap = std::max<size_t>(hI.size(), 1);
  out.I = DevBuf<int32_t>(cap, ctx);
  out.K = DevBuf<int32_t>(cap, ctx);
  out.J = DevBuf<int32_t>(cap, ctx);
  if (out.n) {
    SPG_CUDA(cudaMemcpyAsync(out.I.get(), hI.data(), out.n * 4, cudaMemcpyHostToDevice, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(out.K.get(), hK.data(), out.n * 4, cudaMemcpyHostToDevice, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(out.J.get(), hJ.data(), out.n * 4, cudaMemcpyHostToDevice, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return out;
}

}  // namespace spg
