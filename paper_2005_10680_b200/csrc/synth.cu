// synth.cu -- seeded synthetic inputs for the BASELINE.json configs
// (include/spamm_synth.h).  Input generation only; not part of the hot path.
//
// Recipe:
//   u(seed, a, b) = (mix64(mix64(seed) ^ (a << 32 | b)) >> 11) * 2^-53, with
//   mix64 the SplitMix64 finaliser; a symmetric entry uses (min(i,j), max(i,j))
//   and the same bits->double map as the reference (oracle.cpp:20-21).
//   chain:   A_ij = (2u - 1) * exp(-|i-j| / ell)
//   cluster: sites s = 0..n/4-1 at box * (u(site_seed, s, 0..2)), box =
//            cbrt((n/4) / density); sites sorted by the Morton key of their
//            10-bit quantised coordinates (ties by index); basis b = 4*rank+orb
//            sits on its site; A_ij = (2u - 1) * exp(-d_ij / ell), then divided
//            by max_i sum_j |A_ij| (Gershgorin bound on the spectral norm,
//            oracle.cpp:191-200).
//   |A_ij| < drop -> 0 after scaling; blocks that end up all-zero are null.
// Host and device share every integer and +,-,*,/,sqrt step (no FMA); they
// differ through exp() and the row-sum order only.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "spamm_synth.h"

namespace spg {

namespace {

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ inline double u01(uint64_t seed_mixed, uint32_t a, uint32_t b) {
  const uint64_t h = mix64(seed_mixed ^ ((static_cast<uint64_t>(a) << 32) | b));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

__host__ __device__ inline double signed_u(uint64_t seed_mixed, uint32_t i, uint32_t j) {
  const uint32_t lo = i < j ? i : j, hi = i < j ? j : i;
  return 2.0 * u01(seed_mixed, lo, hi) - 1.0;
}

uint64_t spread3(uint32_t x) {
  uint64_t v = x & 0x3ff;
  v = (v | (v << 16)) & 0x030000FFull;
  v = (v | (v << 8)) & 0x0300F00Full;
  v = (v | (v << 4)) & 0x030C30C3ull;
  v = (v | (v << 2)) & 0x09249249ull;
  return v;
}

// Morton-ordered site centres (host; shared by both generators).
std::vector<double> cluster_sites(int32_t n_sites, double density, uint64_t site_seed,
                                  double* box_out) {
  const double box = std::cbrt(static_cast<double>(n_sites) / density);
  const uint64_t sm = mix64(site_seed);
  std::vector<double> xyz(static_cast<size_t>(n_sites) * 3);
  std::vector<std::pair<uint64_t, int32_t>> order(static_cast<size_t>(n_sites));
  for (int32_t s = 0; s < n_sites; ++s) {
    uint32_t q[3];
    for (int a = 0; a < 3; ++a) {
      const double x = box * u01(sm, static_cast<uint32_t>(s), static_cast<uint32_t>(a));
      xyz[3 * s + a] = x;
      int64_t qi = static_cast<int64_t>(x / box * 1024.0);
      q[a] = static_cast<uint32_t>(std::min<int64_t>(std::max<int64_t>(qi, 0), 1023));
    }
    order[s] = {(spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]), s};
  }
  std::sort(order.begin(), order.end());
  std::vector<double> sorted(xyz.size());
  for (int32_t r = 0; r < n_sites; ++r)
    for (int a = 0; a < 3; ++a) sorted[3 * r + a] = xyz[3 * order[r].second + a];
  if (box_out) *box_out = box;
  return sorted;
}

__host__ __device__ inline double site_distance(const double* p, const double* q) {
#ifdef __CUDA_ARCH__
  const double dx = __dadd_rn(p[0], -q[0]), dy = __dadd_rn(p[1], -q[1]),
               dz = __dadd_rn(p[2], -q[2]);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
#else
  volatile double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
  volatile double xx = dx * dx, yy = dy * dy, zz = dz * dz;
  volatile double s = xx + yy;
  s = s + zz;
  return std::sqrt(static_cast<double>(s));
#endif
}

// Enumerate leaf blocks of the logical grid in Morton order (block rows
// [row_begin, row_end) only, when given).
std::vector<uint64_t> morton_blocks(int32_t nb_logical, int depth, int32_t row_begin = 0,
                                    int32_t row_end = -1) {
  if (row_end < 0) row_end = nb_logical;
  std::vector<uint64_t> keys;
  keys.reserve(static_cast<size_t>(std::max(row_end - row_begin, 0)) * nb_logical);
  const uint64_t total = uint64_t(1) << (2 * depth);
  for (uint64_t key = 0; key < total; ++key) {
    const uint32_t r = morton_row(key);
    if (r >= static_cast<uint32_t>(row_begin) && r < static_cast<uint32_t>(row_end) &&
        morton_col(key) < static_cast<uint32_t>(nb_logical))
      keys.push_back(key);
  }
  return keys;
}

template <typename ValueFn>
int64_t emit_host_blocks(int32_t n, int32_t L, int depth, double drop, ValueFn&& value,
                         int64_t capacity, int32_t* rows, int32_t* cols, double* payload,
                         const std::function<bool(int32_t, int32_t)>& maybe_nonzero) {
  const int32_t nb = (n + L - 1) / L;
  const int64_t LL = static_cast<int64_t>(L) * L;
  std::vector<double> blk(static_cast<size_t>(LL));
  int64_t count = 0;
  for (uint64_t key : morton_blocks(nb, depth)) {
    const int32_t br = static_cast<int32_t>(morton_row(key));
    const int32_t bc = static_cast<int32_t>(morton_col(key));
    if (!maybe_nonzero(br, bc)) continue;
    bool any = false;
    for (int32_t j = 0; j < L; ++j)
      for (int32_t i = 0; i < L; ++i) {
        const int32_t gi = br * L + i, gj = bc * L + j;
        double v = 0.0;
        if (gi < n && gj < n) {
          v = value(gi, gj);
          if (std::fabs(v) < drop) v = 0.0;
        }
        blk[i + static_cast<size_t>(j) * L] = v;
        any = any || v != 0.0;
      }
    if (!any) continue;
    if (payload && count < capacity) {
      rows[count] = br;
      cols[count] = bc;
      std::memcpy(payload + count * LL, blk.data(), sizeof(double) * LL);
    }
    ++count;
  }
  return count;
}

// ---------------------------------------------------------------- device
__global__ void chain_blocks_kernel(const uint64_t* __restrict__ keys, int64_t n_blocks, int32_t n,
                                    int32_t L, double ell, uint64_t seed_mixed, double drop,
                                    double* __restrict__ payload) {
  const int64_t LL = static_cast<int64_t>(L) * L;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const uint64_t key = keys[blk];
    const int32_t br = static_cast<int32_t>(morton_row(key)), bc = static_cast<int32_t>(morton_col(key));
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) {
      const int32_t gi = br * L + static_cast<int32_t>(e % L);
      const int32_t gj = bc * L + static_cast<int32_t>(e / L);
      double v = 0.0;
      if (gi < n && gj < n) {
        const double d = static_cast<double>(gi > gj ? gi - gj : gj - gi);
        v = __dmul_rn(signed_u(seed_mixed, gi, gj), exp(-__ddiv_rn(d, ell)));
        if (fabs(v) < drop) v = 0.0;
      }
      payload[blk * LL + e] = v;
    }
  }
}

__global__ void cluster_rowsum_kernel(const double* __restrict__ sites, int32_t n, double ell,
                                      uint64_t seed_mixed, double* __restrict__ rowsum) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int32_t i = warp;
  const double* pi = sites + 3 * (i >> 2);
  double s = 0.0;
  for (int32_t j = lane; j < n; j += 32) {
    const double d = site_distance(pi, sites + 3 * (j >> 2));
    const double v = __dmul_rn(signed_u(seed_mixed, i, j), exp(-__ddiv_rn(d, ell)));
    s = __dadd_rn(s, fabs(v));
  }
  for (int off = 16; off; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
  if (lane == 0) rowsum[i] = s;
}

__global__ void max_kernel(const double* __restrict__ x, int32_t n, double* __restrict__ out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, x[i]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void cluster_blocks_kernel(const uint64_t* __restrict__ keys, int64_t n_blocks,
                                      const double* __restrict__ sites, int32_t n, int32_t L,
                                      double ell, uint64_t seed_mixed, const double* scale,
                                      double drop, double* __restrict__ payload) {
  const int64_t LL = static_cast<int64_t>(L) * L;
  const double sc = *scale;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const uint64_t key = keys[blk];
    const int32_t br = static_cast<int32_t>(morton_row(key)), bc = static_cast<int32_t>(morton_col(key));
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) {
      const int32_t gi = br * L + static_cast<int32_t>(e % L);
      const int32_t gj = bc * L + static_cast<int32_t>(e / L);
      double v = 0.0;
      if (gi < n && gj < n) {
        const double d = site_distance(sites + 3 * (gi >> 2), sites + 3 * (gj >> 2));
        v = __ddiv_rn(__dmul_rn(signed_u(seed_mixed, gi, gj), exp(-__ddiv_rn(d, ell))), sc);
        if (fabs(v) < drop) v = 0.0;
      }
      payload[blk * LL + e] = v;
    }
  }
}

__global__ void keys_to_rc(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ r,
                           int32_t* __restrict__ c) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  r[t] = static_cast<int32_t>(morton_row(keys[t]));
  c[t] = static_cast<int32_t>(morton_col(keys[t]));
}

spg_matrix* device_blocks_to_matrix(spg_context* ctx, int32_t n, int32_t L,
                                    const std::vector<uint64_t>& hkeys, double* payload,
                                    DevBuf<uint64_t>& dkeys) {
  const int64_t nblk = static_cast<int64_t>(hkeys.size());
  DevBuf<int32_t> r(std::max<int64_t>(nblk, 1), ctx), c(std::max<int64_t>(nblk, 1), ctx);
  if (nblk) {
    keys_to_rc<<<grid_for(nblk, 256), 256, 0, ctx->stream>>>(dkeys.get(), nblk, r.get(), c.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  return matrix_from_device_leaves(ctx, n, L, nblk, r.get(), c.get(), payload);
}

}  // namespace
}  // namespace spg

namespace spg {
namespace {
// The cluster generator's sites and (if scale_in < 0) its global scale, the
// largest absolute row sum, on the device.
void cluster_setup(spg_context* ctx, int32_t n, double ell, double density, uint64_t site_seed,
                   uint64_t value_seed, double scale_in, spg::DevBuf<double>* dsites,
                   spg::DevBuf<double>* scale) {
  using namespace spg;
  if (n % 4 != 0) fail(SPG_EINVAL, "cluster dimension must be a multiple of 4");
  if (!(ell > 0.0) || !(density > 0.0)) fail(SPG_EINVAL, "ell and density must be positive");
  const std::vector<double> sites = cluster_sites(n / 4, density, site_seed, nullptr);
  *dsites = DevBuf<double>(sites.size(), ctx);
  SPG_CUDA(cudaMemcpyAsync(dsites->get(), sites.data(), sites.size() * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
  *scale = DevBuf<double>(1, ctx);
  if (scale_in >= 0.0) {
    SPG_CUDA(cudaMemcpyAsync(scale->get(), &scale_in, sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));  // scale_in is a host local
    return;
  }
  DevBuf<double> rowsum(n, ctx);
  cluster_rowsum_kernel<<<grid_for(int64_t(n) * 32, 256), 256, 0, ctx->stream>>>(
      dsites->get(), n, ell, mix64(value_seed), rowsum.get());
  SPG_CHECK_LAUNCH(ctx);
  max_kernel<<<1, 256, 0, ctx->stream>>>(rowsum.get(), n, scale->get());
  SPG_CHECK_LAUNCH(ctx);
}

spg_matrix* cluster_rows(spg_context* ctx, int32_t n, int32_t L, double ell, double density,
                         uint64_t site_seed, uint64_t value_seed, double drop, double scale_in,
                         int32_t row_begin, int32_t row_end) {
  using namespace spg;
  int32_t padded, depth;
  check_shape(n, L, &padded, &depth);
  if (row_begin < 0 || row_end < row_begin || row_end > (n + L - 1) / L)
    fail(SPG_EINVAL, "synth: bad block row range");
  DevBuf<double> dsites, scale;
  cluster_setup(ctx, n, ell, density, site_seed, value_seed, scale_in, &dsites, &scale);
  const uint64_t sm = mix64(value_seed);
  const int32_t nb = (n + L - 1) / L;
  const std::vector<uint64_t> hkeys = morton_blocks(nb, depth, row_begin, row_end);
  const int64_t nblk = static_cast<int64_t>(hkeys.size());
  const int64_t LL = static_cast<int64_t>(L) * L;
  DevBuf<uint64_t> dkeys(std::max<int64_t>(nblk, 1), ctx);
  SPG_CUDA(cudaMemcpyAsync(dkeys.get(), hkeys.data(), nblk * sizeof(uint64_t),
                           cudaMemcpyHostToDevice, ctx->stream));
  double* payload = dev_alloc<double>(std::max<int64_t>(nblk * LL, 1), ctx);
  if (nblk) {
    cluster_blocks_kernel<<<static_cast<unsigned>(std::min<int64_t>(nblk, 1 << 20)), 256, 0,
                            ctx->stream>>>(dkeys.get(), nblk, dsites.get(), n, L, ell, sm,
                                           scale.get(), drop, payload);
    SPG_CHECK_LAUNCH(ctx);
  }
  return device_blocks_to_matrix(ctx, n, L, hkeys, payload, dkeys);
}
}  // namespace
}  // namespace spg

using namespace spg;

extern "C" {

int spg_synth_chain_host(int32_t n, int32_t L, double ell, uint64_t seed, double drop,
                         int64_t capacity, int32_t* rows, int32_t* cols, double* payload,
                         int64_t* n_leaves) {
  SPG_API_BEGIN
  if (!n_leaves) fail(SPG_EINVAL, "null output");
  if (!(ell > 0.0)) fail(SPG_EINVAL, "ell must be positive");
  int32_t padded, depth;
  check_shape(n, L, &padded, &depth);
  const uint64_t sm = mix64(seed);
  auto value = [&](int32_t i, int32_t j) {
    const double d = static_cast<double>(i > j ? i - j : j - i);
    volatile double e = std::exp(-(d / ell));
    volatile double v = signed_u(sm, i, j) * e;
    return static_cast<double>(v);
  };
  auto maybe = [&](int32_t br, int32_t bc) {
    const int64_t gap = std::max<int64_t>(0, std::llabs(int64_t(br) - bc) * L - (L - 1));
    return drop <= 0.0 || std::exp(-(static_cast<double>(gap) / ell)) >= drop * 0.5;
  };
  *n_leaves = emit_host_blocks(n, L, depth, drop, value, capacity, rows, cols, payload, maybe);
  SPG_API_END
}

int spg_synth_cluster_host(int32_t n, int32_t L, double ell, double density, uint64_t site_seed,
                           uint64_t value_seed, double drop, int64_t capacity, int32_t* rows,
                           int32_t* cols, double* payload, int64_t* n_leaves) {
  SPG_API_BEGIN
  if (!n_leaves) fail(SPG_EINVAL, "null output");
  if (n % 4 != 0) fail(SPG_EINVAL, "cluster dimension must be a multiple of 4");
  if (!(ell > 0.0) || !(density > 0.0)) fail(SPG_EINVAL, "ell and density must be positive");
  int32_t padded, depth;
  check_shape(n, L, &padded, &depth);
  const std::vector<double> sites = cluster_sites(n / 4, density, site_seed, nullptr);
  const uint64_t sm = mix64(value_seed);
  auto raw = [&](int32_t i, int32_t j) {
    const double d = site_distance(&sites[3 * (i >> 2)], &sites[3 * (j >> 2)]);
    volatile double e = std::exp(-(d / ell));
    volatile double v = signed_u(sm, i, j) * e;
    return static_cast<double>(v);
  };
  double scale = 0.0;
  for (int32_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int32_t j = 0; j < n; ++j) s += std::fabs(raw(i, j));
    scale = std::max(scale, s);
  }
  auto value = [&](int32_t i, int32_t j) {
    volatile double v = raw(i, j) / scale;
    return static_cast<double>(v);
  };
  auto maybe = [](int32_t, int32_t) { return true; };
  *n_leaves = emit_host_blocks(n, L, depth, drop, value, capacity, rows, cols, payload, maybe);
  SPG_API_END
}

int spg_synth_chain_device(spg_context* ctx, int32_t n, int32_t L, double ell, uint64_t seed,
                           double drop, spg_matrix** out) {
  return spg_synth_chain_device_rows(ctx, n, L, ell, seed, drop, 0, (n + L - 1) / std::max(L, 1),
                                     out);
}

int spg_synth_chain_device_rows(spg_context* ctx, int32_t n, int32_t L, double ell, uint64_t seed,
                                double drop, int32_t row_begin, int32_t row_end,
                                spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (!(ell > 0.0)) fail(SPG_EINVAL, "ell must be positive");
  int32_t padded, depth;
  check_shape(n, L, &padded, &depth);
  const int32_t nb = (n + L - 1) / L;
  if (row_begin < 0 || row_end < row_begin || row_end > nb)
    fail(SPG_EINVAL, "synth: bad block row range");
  CtxGuard g(ctx);
  std::vector<uint64_t> hkeys;
  for (uint64_t key : morton_blocks(nb, depth, row_begin, row_end)) {
    const int64_t gap =
        std::max<int64_t>(0, std::llabs(int64_t(morton_row(key)) - morton_col(key)) * L - (L - 1));
    if (drop <= 0.0 || std::exp(-(static_cast<double>(gap) / ell)) >= drop * 0.5)
      hkeys.push_back(key);
  }
  const int64_t nblk = static_cast<int64_t>(hkeys.size());
  const int64_t LL = static_cast<int64_t>(L) * L;
  DevBuf<uint64_t> dkeys(std::max<int64_t>(nblk, 1), ctx);
  SPG_CUDA(cudaMemcpyAsync(dkeys.get(), hkeys.data(), nblk * sizeof(uint64_t),
                           cudaMemcpyHostToDevice, ctx->stream));
  double* payload = dev_alloc<double>(std::max<int64_t>(nblk * LL, 1), ctx);
  if (nblk) {
    chain_blocks_kernel<<<static_cast<unsigned>(std::min<int64_t>(nblk, 65535)), 256, 0,
                          ctx->stream>>>(dkeys.get(), nblk, n, L, ell, mix64(seed), drop, payload);
    SPG_CHECK_LAUNCH(ctx);
  }
  *out = device_blocks_to_matrix(ctx, n, L, hkeys, payload, dkeys);
  SPG_API_END
}

int spg_synth_cluster_device(spg_context* ctx, int32_t n, int32_t L, double ell, double density,
                             uint64_t site_seed, uint64_t value_seed, double drop,
                             spg_matrix** out) {
  return spg_synth_cluster_device_rows(ctx, n, L, ell, density, site_seed, value_seed, drop, 0,
                                       (n + L - 1) / std::max(L, 1), out);
}

int spg_synth_cluster_device_rows(spg_context* ctx, int32_t n, int32_t L, double ell,
                                  double density, uint64_t site_seed, uint64_t value_seed,
                                  double drop, int32_t row_begin, int32_t row_end,
                                  spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  CtxGuard g(ctx);
  *out = cluster_rows(ctx, n, L, ell, density, site_seed, value_seed, drop, -1.0, row_begin,
                      row_end);
  SPG_API_END
}

int spg_synth_cluster_scale(spg_context* ctx, int32_t n, double ell, double density,
                            uint64_t site_seed, uint64_t value_seed, double* scale) {
  SPG_API_BEGIN
  if (!ctx || !scale) fail(SPG_EINVAL, "null argument");
  CtxGuard g(ctx);
  DevBuf<double> dsites, dscale;
  cluster_setup(ctx, n, ell, density, site_seed, value_seed, -1.0, &dsites, &dscale);
  SPG_CUDA(cudaMemcpyAsync(scale, dscale.get(), sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  SPG_API_END
}

int spg_synth_cluster_device_rows_scaled(spg_context* ctx, int32_t n, int32_t L, double ell,
                                         double density, uint64_t site_seed, uint64_t value_seed,
                                         double drop, double scale, int32_t row_begin,
                                         int32_t row_end, spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (!(scale >= 0.0)) fail(SPG_EINVAL, "synth: scale must be non-negative");
  CtxGuard g(ctx);
  *out = cluster_rows(ctx, n, L, ell, density, site_seed, value_seed, drop, scale, row_begin,
                      row_end);
  SPG_API_END
}

}  // extern "C"
