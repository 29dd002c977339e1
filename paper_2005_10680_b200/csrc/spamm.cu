// spamm.cu -- K4 task-list builder, K5 dispatch, C finalisation, and the
// product entry points of the C ABI.
//
// K4: the surviving leaf products are exactly the leaves the
// reference recursion spamm_node (multiply.cpp:70-92) reaches: the skip test
// !(fl(nA*nB) < tau) is applied top-down at EVERY level (root included) on
// the dense norm pyramids, so even the underflow corner where an inner norm is
// below a child's (sqrt(fl(x*x)) < x for subnormal squares) skips exactly what
// the reference skips.  K5 takes, per output block in Morton order, the
// [begin, end) range of its (A slot, B slot) pairs with k ascending: for
// trees of depth 3 .. 14 a dense walk per output tile produces them directly
// in that order (below: tl_valid / tl_tile / tl_super); otherwise the tree is
// expanded level by level, the leaf level writes sort keys
// (Morton(i,j) << depth) | k, a deterministic radix sort groups them and run
// heads give the ranges.
//
// C (multiply.cpp:16-20, quadtree.cpp:24-36): one leaf per output block with
// >= 1 survivor; its norm follows block_norm (K1); all-zero sums collapse to
// null (make_leaf); inner norms follow combine_child_norms (K2).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "gemm.cuh"
#include "triples.cuh"

namespace spg {

namespace {

__global__ void head_flags(const uint64_t* __restrict__ keys, int64_t n, int kbits,
                           uint8_t* __restrict__ flags) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  flags[t] = (t == 0) || ((keys[t] >> kbits) != (keys[t - 1] >> kbits));
}

__global__ void run_outputs(const uint64_t* __restrict__ keys, const int64_t* __restrict__ heads,
                            int64_t n_out, int64_t n_surv, int kbits,
                            uint64_t* __restrict__ out_keys, int64_t* __restrict__ out_offset) {
  const int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o > n_out) return;
  if (o == n_out) {
    out_offset[o] = n_surv;
    return;
  }
  const int64_t h = heads[o];
  out_offset[o] = h;
  out_keys[o] = keys[h] >> kbits;
}

__global__ void make_pairs(const uint64_t* __restrict__ keys, int64_t n, int kbits,
                           const int32_t* __restrict__ gridA, const int32_t* __restrict__ gridB,
                           int2* __restrict__ pairs, int* __restrict__ missing = nullptr) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint64_t key = keys[t];
  const uint32_t k = static_cast<uint32_t>(key & ((uint64_t(1) << kbits) - 1));
  const uint64_t ij = key >> kbits;
  const uint32_t i = morton_row(ij), j = morton_col(ij);
  const int2 p = make_int2(gridA[morton2(i, k)], gridB[morton2(k, j)]);
  pairs[t] = p;
  if (missing && (p.x < 0 || p.y < 0)) *missing = 1;
}

// leaves of a matrix per block column (use_col) or row; with use_col, only
// leaves whose block row lies in [row_lo, row_hi) count (a row shard's A)
__global__ void count_by_index(const uint64_t* __restrict__ keys, int64_t n, bool use_col,
                               uint32_t row_lo, uint32_t row_hi, int32_t* __restrict__ counts) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t r = morton_row(keys[t]);
  if (use_col && (r < row_lo || r >= row_hi)) return;
  const uint32_t idx = use_col ? morton_col(keys[t]) : r;
  atomicAdd(counts + idx, 1);
}

__global__ void count_products(const int32_t* __restrict__ colA, const int32_t* __restrict__ rowB,
                               int n, int64_t* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  out[k] = static_cast<int64_t>(colA[k]) * rowB[k];
}

// Parity audit (SURVEY.md 8a "Audit"): candidate leaf products whose norm
// product lies within `ulps` units in the last place of tau -- the pairs
// whose skip decision a 1-ulp difference in a norm could flip.
__global__ void near_tie_count(const int32_t* __restrict__ I, const int32_t* __restrict__ K,
                               const int32_t* __restrict__ J, int64_t n,
                               const double* __restrict__ pa, const double* __restrict__ pb,
                               double tau, double window, unsigned long long* __restrict__ ties,
                               unsigned long long* __restrict__ cands) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long t = 0, c = 0;
  if (p < n) {
    const uint32_t i0 = 2u * I[p], k0 = 2u * K[p], j0 = 2u * J[p];
#pragma unroll
    for (int code = 0; code < 8; ++code) {
      const uint32_t r = code >> 2, cc = (code >> 1) & 1, h = code & 1;
      const double na = pa[morton2(i0 + r, k0 + h)];
      const double nb = pb[morton2(k0 + h, j0 + cc)];
      if (na < 0.0 || nb < 0.0) continue;
      ++c;
      const double prod = __dmul_rn(na, nb);
      if (fabs(prod - tau) <= window) ++t;
    }
  }
  for (int off = 16; off; off >>= 1) {
    t += __shfl_down_sync(0xffffffffu, t, off);
    c += __shfl_down_sync(0xffffffffu, c, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (t) atomicAdd(ties, t);
    if (c) atomicAdd(cands, c);
  }
}

struct TaskList {
  DevBuf<uint64_t> keys;       // sorted survivor keys
  int64_t n_surv = 0;
  int kbits = 0;
};

__global__ void triples_to_keys(const int32_t* __restrict__ I, const int32_t* __restrict__ K,
                                const int32_t* __restrict__ J, int64_t n, int kbits,
                                uint64_t* __restrict__ keys) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  keys[t] = (morton2(static_cast<uint32_t>(I[t]), static_cast<uint32_t>(J[t])) << kbits) |
            static_cast<uint32_t>(K[t]);
}

// ---- K4 without a sort: dense enumeration by output tile -------------------
// The surviving products grouped by output block (Morton order) with k
// ascending is exactly what a warp produces when it owns one 8 x 8 tile of
// output blocks, T = (I, J) at level s = depth - 3, and walks K = 0 .. 2^s - 1
// in order: a product (i, k, j) survives iff every ancestor pair of it passes
// the rule (multiply.cpp:70-76: spamm_node returns at the first null or
// skipped pair), so
//   1. tl_valid: one flag per (T, K) of the shard's tile rows, the pair
//      (I, K, J) and its ancestors of levels 0 .. s pass;
//   2. tl_tile<count>: for every flagged K the warp stages the two tiles' norms
//      of levels d-2, d-1, d in shared memory, and each lane runs the three
//      remaining tests for its two output blocks, k ascending (k2, k1, k0
//      loops); survivors per output block -> counts;
//   3. an exclusive scan of the 4^d counts; 4. tl_tile<write>: the same walk
//      writes each block's keys (Morton(i,j) << d | k) and (A slot, B slot)
//      pairs at its offset -- already in the order the top-down expansion + a
//      64-bit radix sort of all survivors produced (cfg2: 9.2e7 keys, 6.2 ms of
//      expansion, sort, head flags and slot lookups per step -> see DESIGN).
// The decisions are the same keep_pair tests on the same norms, so the set is
// the expansion's bit for bit (tests: every survivor-set parity case, and the
// old path stays behind SPG_TASKLIST=lists and for depth < 3).
constexpr int kTlWarps = 8;

template <KeepRule R>
__global__ void tl_valid(int s, const double* __restrict__ pyrA, const double* __restrict__ pyrB,
                         double tau, uint32_t row_lo, uint32_t row_hi,
                         uint8_t* __restrict__ valid) {
  // x = ((I - row_lo) * 2^s + J) * 2^s + K over the shard's tile rows
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= (static_cast<int64_t>(row_hi - row_lo) << (2 * s))) return;
  const uint32_t K = static_cast<uint32_t>(x) & ((1u << s) - 1u);
  const uint32_t J = static_cast<uint32_t>(x >> s) & ((1u << s) - 1u);
  const uint32_t I = row_lo + static_cast<uint32_t>(x >> (2 * s));
  constexpr int kMaxS = 12;  // levels 0 .. s, s <= 11
  double na[kMaxS], nb[kMaxS];
#pragma unroll
  for (int l = 0; l < kMaxS; ++l) {
    if (l > s) break;
    const int sh = s - l;
    const int64_t off = level_offset(l);
    na[l] = pyrA[off + morton2(I >> sh, K >> sh)];
    nb[l] = pyrB[off + morton2(K >> sh, J >> sh)];
  }
  bool ok = true;
#pragma unroll
  for (int l = 0; l < kMaxS; ++l) {
    if (l > s) break;
    ok = keep_pair<R>(na[l], nb[l], tau) && ok;
  }
  valid[x] = ok;
}

// WRITE = false: counts[T * 64 + m] = survivors of output block m of tile T.
// WRITE = true: keys / pairs (each optional) at offsets[T * 64 + m] + rank.
template <KeepRule R, bool WRITE>
__global__ void __launch_bounds__(kTlWarps * 32)
    tl_tile(int s, int d, int pl, const double* __restrict__ pyrA,
            const double* __restrict__ pyrB, double tau, uint32_t row_lo, uint32_t row_hi,
            const uint8_t* __restrict__ valid, int64_t* __restrict__ counts,
            const int64_t* __restrict__ offsets, uint64_t* __restrict__ keys,
            const int32_t* __restrict__ gridA, const int32_t* __restrict__ gridB,
            int2* __restrict__ pairs, int* __restrict__ missing) {
  __shared__ double sm[kTlWarps][2][84];  // per warp: A then B; levels d-2 (4), d-1 (16), d (64)
  __shared__ int64_t sm_at[kTlWarps][64];  // WRITE: next position of each output block
  __shared__ uint8_t sm_mask[kTlWarps][64];  // WRITE: surviving k (3 bits) of each block at this K
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the shard's tiles in (tile row, J) order, 2^pl warps per tile, each with
  // its own stretch of K (small problems have too few tiles to fill the
  // machine); T = the tile's Morton index
  const int64_t W = static_cast<int64_t>(blockIdx.x) * kTlWarps + warp;
  const int64_t Tl = W >> pl;
  const int part = static_cast<int>(W & ((int64_t(1) << pl) - 1));
  if (Tl >= (static_cast<int64_t>(row_hi - row_lo) << s)) return;
  const uint32_t I = row_lo + static_cast<uint32_t>(Tl >> s);
  const uint32_t J = static_cast<uint32_t>(Tl) & ((1u << s) - 1u);
  const int64_t T = static_cast<int64_t>(morton2(I, J));
  const double* A2 = pyrA + level_offset(d - 2);
  const double* A1 = pyrA + level_offset(d - 1);
  const double* A0 = pyrA + level_offset(d);
  const double* B2 = pyrB + level_offset(d - 2);
  const double* B1 = pyrB + level_offset(d - 1);
  const double* B0 = pyrB + level_offset(d);
  double* sa = sm[warp][0];
  double* sb = sm[warp][1];
  // the lane's two output blocks m = lane, lane + 32 of the tile (local Morton
  // index, digits 2 i_l + j_l from the top level down)
  uint32_t i2[2], j2[2], i1[2], j1[2], i0[2], j0[2];
  int64_t at[2];
  int cnt[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t m = lane + 32 * h;
    i2[h] = (m >> 5) & 1u; j2[h] = (m >> 4) & 1u;
    i1[h] = (m >> 3) & 1u; j1[h] = (m >> 2) & 1u;
    i0[h] = (m >> 1) & 1u; j0[h] = m & 1u;
    at[h] = WRITE ? offsets[((T * 64 + m) << pl) + part] : 0;
  }
  const int k_len = (1 << s) >> pl, k_end = (part + 1) * k_len;
  for (int Kb = part * k_len; Kb < k_end; Kb += 32) {
    const bool flag = Kb + lane < k_end && valid[(Tl << s) + Kb + lane] != 0;
    uint32_t todo = __ballot_sync(0xffffffffu, flag);
    while (todo) {
      const uint32_t K = Kb + __ffs(todo) - 1;
      todo &= todo - 1u;
      const int64_t mA = static_cast<int64_t>(morton2(I, K)), mB = static_cast<int64_t>(morton2(K, J));
      __syncwarp();
      sa[20 + lane] = A0[mA * 64 + lane];
      sa[20 + 32 + lane] = A0[mA * 64 + 32 + lane];
      sb[20 + lane] = B0[mB * 64 + lane];
      sb[20 + 32 + lane] = B0[mB * 64 + 32 + lane];
      if (lane < 16) {
        sa[4 + lane] = A1[mA * 16 + lane];
        sb[4 + lane] = B1[mB * 16 + lane];
      } else if (lane < 20) {
        sa[lane - 16] = A2[mA * 4 + lane - 16];
        sb[lane - 16] = B2[mB * 4 + lane - 16];
      }
      __syncwarp();
      // the surviving k of the lane's blocks at this K: bit 4 k2 + 2 k1 + k0
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t mask = 0;
#pragma unroll
        for (uint32_t k2 = 0; k2 < 2; ++k2) {
          const uint32_t a2 = 2 * i2[h] + k2, b2 = 2 * k2 + j2[h];
          if (!keep_pair<R>(sa[a2], sb[b2], tau)) continue;
#pragma unroll
          for (uint32_t k1 = 0; k1 < 2; ++k1) {
            const uint32_t a1 = 4 * a2 + 2 * i1[h] + k1, b1 = 4 * b2 + 2 * k1 + j1[h];
            if (!keep_pair<R>(sa[4 + a1], sb[4 + b1], tau)) continue;
#pragma unroll
            for (uint32_t k0 = 0; k0 < 2; ++k0) {
              const uint32_t a0 = 4 * a1 + 2 * i0[h] + k0, b0 = 4 * b1 + 2 * k0 + j0[h];
              if (keep_pair<R>(sa[20 + a0], sb[20 + b0], tau)) mask |= 1u << (4 * k2 + 2 * k1 + k0);
            }
          }
        }
        if (WRITE) {
          sm_mask[warp][lane + 32 * h] = static_cast<uint8_t>(mask);
          sm_at[warp][lane + 32 * h] = at[h] + cnt[h];
        }
        cnt[h] += __popc(mask);
      }
      if (WRITE) {
        // 8 lanes per output block (lane & 7 = the k bits), 4 blocks a round:
        // a block's survivors go out as one contiguous run
        __syncwarp();
        const uint32_t kb = lane & 7u, k2 = kb >> 2, k1 = (kb >> 1) & 1u, k0 = kb & 1u;
#pragma unroll 4
        for (uint32_t r = 0; r < 16; ++r) {
          const uint32_t blk = 4 * r + (lane >> 3);
          const uint32_t mask = sm_mask[warp][blk];
          if (!((mask >> kb) & 1u)) continue;
          const int64_t pos = sm_at[warp][blk] + __popc(mask & ((1u << kb) - 1u));
          if (keys)
            keys[pos] = ((static_cast<uint64_t>(T) * 64 + blk) << d) | (8 * K + kb);
          if (pairs) {
            const uint32_t bi2 = (blk >> 5) & 1u, bj2 = (blk >> 4) & 1u, bi1 = (blk >> 3) & 1u,
                           bj1 = (blk >> 2) & 1u, bi0 = (blk >> 1) & 1u, bj0 = blk & 1u;
            const uint32_t a0 = 16 * (2 * bi2 + k2) + 4 * (2 * bi1 + k1) + 2 * bi0 + k0;
            const uint32_t b0 = 16 * (2 * k2 + bj2) + 4 * (2 * k1 + bj1) + 2 * k0 + bj0;
            const int2 pr = make_int2(gridA[mA * 64 + a0], gridB[mB * 64 + b0]);
            pairs[pos] = pr;
            if (missing && (pr.x < 0 || pr.y < 0)) *missing = 1;
          }
        }
      }
    }
  }
  if (!WRITE) {
    counts[((T * 64 + lane) << pl) + part] = cnt[0];
    counts[((T * 64 + 32 + lane) << pl) + part] = cnt[1];
  }
}

// The same walk for the L = 32 super-block GEMM (leaf_gemm_super32): one entry
// per (2x2 super block, k) with the 4-bit mask of the sub blocks present and
// the A slots of rows 2I', 2I'+1 / B slots of columns 2J', 2J'+1 at that k,
// super blocks in Morton order, k ascending -- what re-keying and key-value
// sorting the survivor list produced (build_super32).  A tile holds 4 x 4 super
// blocks; the four sub blocks of super block q are the tile's blocks 4q .. 4q+3
// (four adjacent lanes).  WRITE = false: sb_counts[T * 16 + q] = entries.
template <KeepRule R, bool WRITE>
__global__ void __launch_bounds__(kTlWarps * 32)
    tl_super(int s, int d, int pl, const double* __restrict__ pyrA,
             const double* __restrict__ pyrB, double tau, uint32_t row_lo, uint32_t row_hi,
             const uint8_t* __restrict__ valid, int64_t* __restrict__ sb_counts,
             const int64_t* __restrict__ sb_offsets, const int32_t* __restrict__ gridA,
             const int32_t* __restrict__ gridB, SuperEntry* __restrict__ ent,
             uint32_t* __restrict__ emask, uint32_t* __restrict__ ek, int* __restrict__ missing) {
  __shared__ double sm[kTlWarps][2][84];
  __shared__ int64_t sm_at[kTlWarps][16];
  __shared__ __align__(4) uint8_t sm_mask[kTlWarps][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the shard's tiles in (tile row, J) order, 2^pl warps per tile, each with
  // its own stretch of K (small problems have too few tiles to fill the
  // machine); T = the tile's Morton index
  const int64_t W = static_cast<int64_t>(blockIdx.x) * kTlWarps + warp;
  const int64_t Tl = W >> pl;
  const int part = static_cast<int>(W & ((int64_t(1) << pl) - 1));
  if (Tl >= (static_cast<int64_t>(row_hi - row_lo) << s)) return;
  const uint32_t I = row_lo + static_cast<uint32_t>(Tl >> s);
  const uint32_t J = static_cast<uint32_t>(Tl) & ((1u << s) - 1u);
  const int64_t T = static_cast<int64_t>(morton2(I, J));
  const double* A2 = pyrA + level_offset(d - 2);
  const double* A1 = pyrA + level_offset(d - 1);
  const double* A0 = pyrA + level_offset(d);
  const double* B2 = pyrB + level_offset(d - 2);
  const double* B1 = pyrB + level_offset(d - 1);
  const double* B0 = pyrB + level_offset(d);
  double* sa = sm[warp][0];
  double* sb = sm[warp][1];
  uint32_t i2[2], j2[2], i1[2], j1[2], i0[2], j0[2];
  int64_t at[2];  // lanes 4q: next entry of super blocks q = lane / 4 and 8 + lane / 4
  int cnt[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t m = lane + 32 * h;
    i2[h] = (m >> 5) & 1u; j2[h] = (m >> 4) & 1u;
    i1[h] = (m >> 3) & 1u; j1[h] = (m >> 2) & 1u;
    i0[h] = (m >> 1) & 1u; j0[h] = m & 1u;
    at[h] = WRITE ? sb_offsets[((T * 16 + (m >> 2)) << pl) + part] : 0;
  }
  const int k_len = (1 << s) >> pl, k_end = (part + 1) * k_len;
  for (int Kb = part * k_len; Kb < k_end; Kb += 32) {
    const bool flag = Kb + lane < k_end && valid[(Tl << s) + Kb + lane] != 0;
    uint32_t todo = __ballot_sync(0xffffffffu, flag);
    while (todo) {
      const uint32_t K = Kb + __ffs(todo) - 1;
      todo &= todo - 1u;
      const int64_t mA = static_cast<int64_t>(morton2(I, K)), mB = static_cast<int64_t>(morton2(K, J));
      __syncwarp();
      sa[20 + lane] = A0[mA * 64 + lane];
      sa[20 + 32 + lane] = A0[mA * 64 + 32 + lane];
      sb[20 + lane] = B0[mB * 64 + lane];
      sb[20 + 32 + lane] = B0[mB * 64 + 32 + lane];
      if (lane < 16) {
        sa[4 + lane] = A1[mA * 16 + lane];
        sb[4 + lane] = B1[mB * 16 + lane];
      } else if (lane < 20) {
        sa[lane - 16] = A2[mA * 4 + lane - 16];
        sb[lane - 16] = B2[mB * 4 + lane - 16];
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t mask = 0;
#pragma unroll
        for (uint32_t k2 = 0; k2 < 2; ++k2) {
          const uint32_t a2 = 2 * i2[h] + k2, b2 = 2 * k2 + j2[h];
          if (!keep_pair<R>(sa[a2], sb[b2], tau)) continue;
#pragma unroll
          for (uint32_t k1 = 0; k1 < 2; ++k1) {
            const uint32_t a1 = 4 * a2 + 2 * i1[h] + k1, b1 = 4 * b2 + 2 * k1 + j1[h];
            if (!keep_pair<R>(sa[4 + a1], sb[4 + b1], tau)) continue;
#pragma unroll
            for (uint32_t k0 = 0; k0 < 2; ++k0) {
              const uint32_t a0 = 4 * a1 + 2 * i0[h] + k0, b0 = 4 * b1 + 2 * k0 + j0[h];
              if (keep_pair<R>(sa[20 + a0], sb[20 + b0], tau)) mask |= 1u << (4 * k2 + 2 * k1 + k0);
            }
          }
        }
        // k with any of the super block's four sub blocks present
        uint32_t any = mask | __shfl_xor_sync(0xffffffffu, mask, 1);
        any |= __shfl_xor_sync(0xffffffffu, any, 2);
        if (WRITE) {
          sm_mask[warp][lane + 32 * h] = static_cast<uint8_t>(mask);
          if ((lane & 3) == 0) sm_at[warp][(lane >> 2) + 8 * h] = at[h] + cnt[h];
        }
        cnt[h] += __popc(any);
      }
      if (WRITE) {
        // 8 lanes per super block (lane & 7 = the k bits), 4 super blocks a round
        __syncwarp();
        const uint32_t kb = lane & 7u, k2 = kb >> 2, k1 = (kb >> 1) & 1u, k0 = kb & 1u;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) {
          const uint32_t q = 4 * r + (lane >> 3);
          const uint32_t m4 = *reinterpret_cast<const uint32_t*>(&sm_mask[warp][4 * q]);
          const uint32_t em = ((m4 >> kb) & 1u) | (((m4 >> (8 + kb)) & 1u) << 1) |
                              (((m4 >> (16 + kb)) & 1u) << 2) | (((m4 >> (24 + kb)) & 1u) << 3);
          if (!em) continue;
          const uint32_t any = (m4 | (m4 >> 8) | (m4 >> 16) | (m4 >> 24)) & 0xffu;
          const int64_t pos = sm_at[warp][q] + __popc(any & ((1u << kb) - 1u));
          // super block q = local Morton (i2 j2 i1 j1); sub block = 2 r + c
          const uint32_t qi2 = (q >> 3) & 1u, qj2 = (q >> 2) & 1u, qi1 = (q >> 1) & 1u, qj1 = q & 1u;
          const uint32_t arow = 16 * (2 * qi2 + k2) + 4 * (2 * qi1 + k1) + k0;  // + 2 r
          const uint32_t bcol = 16 * (2 * k2 + qj2) + 4 * (2 * k1 + qj1) + 2 * k0;  // + c
          SuperEntry e{0, 0, 0, 0};
          if (em & 0x3u) e.a0 = gridA[mA * 64 + arow];
          if (em & 0xcu) e.a1 = gridA[mA * 64 + arow + 2];
          if (em & 0x5u) e.b0 = gridB[mB * 64 + bcol];
          if (em & 0xau) e.b1 = gridB[mB * 64 + bcol + 1];
          if (missing && (e.a0 < 0 || e.a1 < 0 || e.b0 < 0 || e.b1 < 0)) *missing = 1;
          ent[pos] = e;
          emask[pos] = em;
          ek[pos] = 8 * K + kb;
        }
      }
    }
  }
  if (!WRITE && (lane & 3) == 0) {
    sb_counts[((T * 16 + (lane >> 2)) << pl) + part] = cnt[0];
    sb_counts[((T * 16 + 8 + (lane >> 2)) << pl) + part] = cnt[1];
  }
}

// offsets hold 2^pl K-parts per block: a block's range starts at its first part
__global__ void tl_outputs(const int64_t* __restrict__ blocks, const int64_t* __restrict__ offsets,
                           int pl, int64_t n_out, int64_t n_surv, uint64_t* __restrict__ out_keys,
                           int64_t* __restrict__ out_offset) {
  const int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o > n_out) return;
  if (o == n_out) {
    out_offset[o] = n_surv;
    return;
  }
  out_keys[o] = static_cast<uint64_t>(blocks[o]);
  out_offset[o] = offsets[blocks[o] << pl];
}

// survivors per block over its 2^pl K-parts (the flags of the block select)
__global__ void tl_block_totals(const int64_t* __restrict__ offsets, int64_t n_blocks, int pl,
                                int64_t* __restrict__ totals) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b < n_blocks) totals[b] = offsets[(b + 1) << pl] - offsets[b << pl];
}

// 2^pl warps per tile so that a small problem still fills the machine
int tile_parts_log(const spg_context* ctx, int64_t n_tiles, int s) {
  const int64_t want = static_cast<int64_t>(ctx->sm_count) * 64;
  int pl = 0;
  while (pl < s && (n_tiles << pl) < want) ++pl;
  return pl;
}

// The dense walk covers trees of depth 3 .. 14 (every depth the Morton grids
// allow) while the flags of a shard's tiles, one byte per (tile, K), stay
// below 8 GB: depth 14 unsharded is 8^11 of them.
bool dense_walk_fits(int depth, int shard_level) {
  const int s = depth - 3;
  if (s < 0 || s > 11 || shard_level > s) return false;
  return (3 * s - shard_level) <= 33;
}

// developer switch SPG_TASKLIST=lists: the top-down expansion + radix sort
bool dense_tasklist_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPG_TASKLIST");
    return !(e && std::strcmp(e, "lists") == 0);
  }();
  return on;
}

struct DenseTasks {
  int64_t n_surv = 0, n_out = 0;
  DevBuf<uint64_t> keys, out_keys;
  DevBuf<int64_t> out_offset;
  DevBuf<int2> pairs;
};

// The dense path applies to trees of depth 3 .. 14 (dense_walk_fits) and
// shards of whole tile rows; false = use the expansion.  want_keys / want_pairs choose the outputs
// (pairs with their per-block ranges out_keys / out_offset).
template <KeepRule R>
bool dense_tasklist(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                    Shard sh, bool want_keys, bool want_pairs, const spg_matrix* a_slots,
                    DenseTasks* out, bool want_blocks = false) {
  want_blocks = want_blocks || want_pairs;
  const int d = a->depth, s = d - 3;
  if (!dense_tasklist_enabled() || !dense_walk_fits(d, sh.level)) return false;
  PhaseTrace tr(ctx, "tasklist.dense");
  const uint32_t tile_rows = (1u << s) >> sh.level;
  const uint32_t row_lo = tile_rows * static_cast<uint32_t>(sh.index), row_hi = row_lo + tile_rows;
  // flags and warps cover the shard's tile rows only; the per-block counts
  // stay indexed by global Morton order (zero outside the shard)
  const int64_t n_tiles = static_cast<int64_t>(tile_rows) << s, n_flags = n_tiles << s;
  const int64_t n_blocks = int64_t(64) << (2 * s);
  DevBuf<uint8_t> valid(n_flags, ctx);
  tl_valid<R><<<grid_for(n_flags, 256), 256, 0, ctx->stream>>>(s, a->pyramid, b->pyramid, tau,
                                                               row_lo, row_hi, valid.get());
  SPG_CHECK_LAUNCH(ctx);
  const int pl = tile_parts_log(ctx, n_tiles, s);
  const int64_t n_cnt = n_blocks << pl;
  DevBuf<int64_t> counts(n_cnt + 1, ctx), offsets(n_cnt + 1, ctx);
  if (sh.level > 0)
    SPG_CUDA(cudaMemsetAsync(counts.get(), 0, (n_cnt + 1) * sizeof(int64_t), ctx->stream));
  else
    SPG_CUDA(cudaMemsetAsync(counts.get() + n_cnt, 0, sizeof(int64_t), ctx->stream));
  const unsigned grid = static_cast<unsigned>(((n_tiles << pl) + kTlWarps - 1) / kTlWarps);
  tl_tile<R, false><<<grid, kTlWarps * 32, 0, ctx->stream>>>(
      s, d, pl, a->pyramid, b->pyramid, tau, row_lo, row_hi, valid.get(), counts.get(), nullptr,
      nullptr, nullptr, nullptr, nullptr, nullptr);
  SPG_CHECK_LAUNCH(ctx);
  out->n_surv = scan_counts(ctx, counts.get(), n_cnt, offsets.get());
  out->n_out = 0;
  if (out->n_surv == 0) return true;
  if (want_keys) out->keys = DevBuf<uint64_t>(out->n_surv, ctx);
  const bool split = want_pairs && a_slots != a;
  DevBuf<int> missing(split ? 1 : 0, ctx);
  if (split) SPG_CUDA(cudaMemsetAsync(missing.get(), 0, sizeof(int), ctx->stream));
  if (want_pairs) out->pairs = DevBuf<int2>(out->n_surv, ctx);
  if (want_keys || want_pairs) {
    tl_tile<R, true><<<grid, kTlWarps * 32, 0, ctx->stream>>>(
        s, d, pl, a->pyramid, b->pyramid, tau, row_lo, row_hi, valid.get(), nullptr,
        offsets.get(),
        want_keys ? out->keys.get() : nullptr, want_pairs ? a_slots->grid_slot : nullptr,
        want_pairs ? b->grid_slot : nullptr, want_pairs ? out->pairs.get() : nullptr,
        split ? missing.get() : nullptr);
    SPG_CHECK_LAUNCH(ctx);
  }
  if (want_blocks) {
    // the non-empty output blocks, ascending, with their pair ranges
    DevBuf<int64_t> blocks(n_blocks, ctx), n_sel(1, ctx), totals(pl ? n_blocks : 0, ctx);
    const int64_t* per_block = counts.get();
    if (pl) {
      tl_block_totals<<<grid_for(n_blocks, 256), 256, 0, ctx->stream>>>(offsets.get(), n_blocks,
                                                                        pl, totals.get());
      SPG_CHECK_LAUNCH(ctx);
      per_block = totals.get();
    }
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    SPG_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, per_block, blocks.get(),
                                        n_sel.get(), n_blocks, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx);
    SPG_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, per_block, blocks.get(),
                                        n_sel.get(), n_blocks, ctx->stream));
    ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
    out->n_out = copy_scalar_to_host_i64(ctx, n_sel.get());
    out->out_keys = DevBuf<uint64_t>(out->n_out, ctx);
    out->out_offset = DevBuf<int64_t>(out->n_out + 1, ctx);
    tl_outputs<<<grid_for(out->n_out + 1, 256), 256, 0, ctx->stream>>>(
        blocks.get(), offsets.get(), pl, out->n_out, out->n_surv, out->out_keys.get(),
        out->out_offset.get());
    SPG_CHECK_LAUNCH(ctx);
    if (split) {
      int h = 0;
      SPG_CUDA(cudaMemcpyAsync(&h, missing.get(), sizeof(int), cudaMemcpyDeviceToHost,
                               ctx->stream));
      SPG_CUDA(cudaStreamSynchronize(ctx->stream));
      if (h)
        fail(SPG_EINVAL, "plan: a_norms lists a leaf in the shard rows that the local A does "
                         "not hold (the shard rows of a and a_norms must have the same leaves)");
    }
  }
  return true;
}

// Surviving (i,k,j) leaf products, sorted by (Morton(i,j), k); with a shard,
// only the leaf products of its block-rows (ancestors above the shard level
// are tested on the host, shard_list).
template <KeepRule R>
TaskList build_tasklist(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                        Shard sh) {
  const int d = a->depth;
  TaskList tl;
  tl.kbits = d;
  PhaseTrace tr_all(ctx, "tasklist.total");
  {
    DenseTasks dt;
    if (dense_tasklist<R>(ctx, a, b, tau, sh, true, false, nullptr, &dt)) {
      tl.n_surv = dt.n_surv;
      tl.keys = dt.n_surv ? std::move(dt.keys) : DevBuf<uint64_t>(1, ctx);
      return tl;
    }
  }
  TripleList cur = sh.level == 0 ? root_list<R>(ctx, a, b, tau)
                                 : shard_list<R>(ctx, a, b, sh.level, sh.index, tau, true);
  DevBuf<uint64_t> keys;
  if (sh.level == d) {
    tl.n_surv = cur.n;
    keys = DevBuf<uint64_t>(std::max<int64_t>(cur.n, 1), ctx);
    if (cur.n) {
      triples_to_keys<<<grid_for(cur.n, 256), 256, 0, ctx->stream>>>(
          cur.I.get(), cur.K.get(), cur.J.get(), cur.n, d, keys.get());
      SPG_CHECK_LAUNCH(ctx);
    }
  } else {
    PhaseTrace tr(ctx, "tasklist.expand");
    for (int l = sh.level; l < d - 1 && cur.n > 0; ++l) {
      TripleList next = expand_level<R>(ctx, cur, a->pyramid + level_offset(l + 1),
                                        b->pyramid + level_offset(l + 1), tau);
      cur = std::move(next);
    }
    // last level: write sort keys directly
    const int64_t n = cur.n;
    DevBuf<uint8_t> masks(std::max<int64_t>(n, 1), ctx);
    DevBuf<int64_t> counts(n + 1, ctx);
    DevBuf<int64_t> offsets(n + 1, ctx);
    SPG_CUDA(cudaMemsetAsync(counts.get() + n, 0, sizeof(int64_t), ctx->stream));
    if (n) {
      expand_count<R><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
          cur.I.get(), cur.K.get(), cur.J.get(), n, a->pyramid + level_offset(d),
          b->pyramid + level_offset(d), tau, masks.get(), counts.get());
      SPG_CHECK_LAUNCH(ctx);
    }
    tl.n_surv = scan_counts(ctx, counts.get(), n, offsets.get());
    keys = DevBuf<uint64_t>(std::max<int64_t>(tl.n_surv, 1), ctx);
    if (tl.n_surv) {
      expand_write_keys<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
          cur.I.get(), cur.K.get(), cur.J.get(), n, masks.get(), offsets.get(), d, keys.get());
      SPG_CHECK_LAUNCH(ctx);
    }
  }
  if (tl.n_surv > 1) {
    PhaseTrace tr(ctx, "tasklist.sort");
    DevBuf<uint64_t> sorted(tl.n_surv, ctx);
    size_t bytes = 0;
    const int end_bit = std::max(1, 3 * d);
    SPG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.get(), sorted.get(), tl.n_surv,
                                            0, end_bit, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx);
    SPG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, keys.get(), sorted.get(),
                                            tl.n_surv, 0, end_bit, ctx->stream));
    ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
    keys = std::move(sorted);
  }
  tl.keys = std::move(keys);
  return tl;
}

int64_t count_candidates(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                         Shard sh = {}) {
  const int nb = 1 << a->depth;
  const uint32_t rows_per = static_cast<uint32_t>(nb >> sh.level);
  const uint32_t row_lo = rows_per * sh.index, row_hi = row_lo + rows_per;
  DevBuf<int32_t> colA(nb, ctx), rowB(nb, ctx);
  DevBuf<int64_t> prod(nb, ctx), total(1, ctx);
  SPG_CUDA(cudaMemsetAsync(colA.get(), 0, nb * sizeof(int32_t), ctx->stream));
  SPG_CUDA(cudaMemsetAsync(rowB.get(), 0, nb * sizeof(int32_t), ctx->stream));
  if (a->nnzb) {
    count_by_index<<<grid_for(a->nnzb, 256), 256, 0, ctx->stream>>>(a->keys, a->nnzb, true,
                                                                    row_lo, row_hi, colA.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  if (b->nnzb) {
    count_by_index<<<grid_for(b->nnzb, 256), 256, 0, ctx->stream>>>(b->keys, b->nnzb, false, 0,
                                                                    0, rowB.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  count_products<<<grid_for(nb, 256), 256, 0, ctx->stream>>>(colA.get(), rowB.get(), nb,
                                                             prod.get());
  SPG_CHECK_LAUNCH(ctx);
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, prod.get(), total.get(), nb, ctx->stream));
  DevBuf<uint8_t> tmp(bytes, ctx);
  SPG_CUDA(cub::DeviceReduce::Sum(tmp.get(), bytes, prod.get(), total.get(), nb, ctx->stream));
  ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
  return copy_scalar_to_host_i64(ctx, total.get());
}

template <int L, int KC, int WM, int WN, int NSTAGE>
void launch_dmma(spg_context* ctx, const double* A, const double* B, const int2* pairs,
                 const int64_t* out_offset, int64_t n_out, double* C, cudaStream_t st,
                 const int64_t* out_end, int accumulate, const double* const* btab,
                 const int32_t* order = nullptr) {
  using Cfg = DmmaGemmCfg<L, KC, WM, WN, NSTAGE>;
  auto kern = btab ? leaf_gemm_dmma<L, KC, WM, WN, NSTAGE, true>
                   : leaf_gemm_dmma<L, KC, WM, WN, NSTAGE, false>;
  SPG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(Cfg::kSmemBytes)));
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n_out, int64_t(1) << 30));
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, st>>>(A, B, pairs, out_offset, n_out, C, out_end,
                                                     accumulate, btab, order);
  SPG_CHECK_LAUNCH(ctx);
}

void run_gemm(spg_context* ctx, int L, const double* A, const double* B, const int2* pairs,
              const int64_t* out_offset, int64_t n_out, double* C, cudaStream_t st = nullptr,
              const int64_t* out_end = nullptr, int accumulate = 0,
              const double* const* btab = nullptr, const int32_t* order = nullptr) {
  if (n_out == 0) return;
  if (!st) st = ctx->stream;
  switch (L) {
    case 32: {
      // per-block L = 32 tiling (the super-block kernel is the default where
      // it applies; SPG_GEMM32=6 forces this one)
      launch_dmma<32, 32, 32, 16, 2>(ctx, A, B, pairs, out_offset, n_out, C, st, out_end,
                                     accumulate, btab, order);
      break;
    }
    case 64:  // 4 warps x 32x32 tiles, 2 stages, 3 CTAs/SM
      launch_dmma<64, 32, 32, 32, 2>(ctx, A, B, pairs, out_offset, n_out, C, st, out_end,
                                     accumulate, btab, order);
      break;
    case 128: {
      // L = 128 kernel (the L = 64 sub-products are the default where they
      // apply; SPG_GEMM128=3 forces this one)
      launch_dmma<128, 32, 64, 32, 2>(ctx, A, B, pairs, out_offset, n_out, C, st, out_end,
                                      accumulate, btab, order);
      break;
    }
    default: {
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n_out, int64_t(1) << 30));
      leaf_gemm_generic<<<grid, 256, 0, st>>>(A, B, pairs, out_offset, n_out, L, C, out_end,
                                              accumulate, btab, order);
      SPG_CHECK_LAUNCH(ctx);
    }
  }
}

// Task list grouped by output block: C block o = Morton key out_keys[o] sums
// the products pairs[out_offset[o], out_offset[o+1]) (k ascending); with
// keep_keys the sorted (Morton(i,j) << depth | k) keys stay for B panels.
// ---- L = 32 super-block task list (leaf_gemm_super32): survivors re-keyed
// (super block, k, sub block), sorted; one entry per (super block, k).
__global__ void super_keys(const uint64_t* __restrict__ keys, int64_t n, int kbits,
                           uint64_t* __restrict__ key2, int64_t* __restrict__ val) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint64_t m = keys[t] >> kbits, k = keys[t] & ((uint64_t(1) << kbits) - 1);
  key2[t] = ((m >> 2) << (kbits + 2)) | (k << 2) | (m & 3u);
  val[t] = t;
}

__global__ void super_heads(const uint64_t* __restrict__ key2, int64_t n,
                            int64_t* __restrict__ head) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  head[t] = (t == 0 || (key2[t] >> 2) != (key2[t - 1] >> 2)) ? 1 : 0;
}

// eidx: inclusive scan of the heads (entry of survivor t' = eidx - 1)
__global__ void super_fill(const uint64_t* __restrict__ key2, const int64_t* __restrict__ val,
                           const int64_t* __restrict__ eidx, int64_t n, int kbits,
                           const int2* __restrict__ pairs, SuperEntry* __restrict__ ent,
                           uint32_t* __restrict__ emask, uint64_t* __restrict__ ekey,
                           uint32_t* __restrict__ ek) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t e = eidx[t] - 1;
  const uint32_t sub = static_cast<uint32_t>(key2[t] & 3u);
  const int2 pr = pairs[val[t]];
  // the A slot of row ri (and the B slot of column cj) at this k is the same
  // leaf for every sub block that shares it: concurrent writes agree
  if (sub >> 1) ent[e].a1 = pr.x;
  else ent[e].a0 = pr.x;
  if (sub & 1u) ent[e].b1 = pr.y;
  else ent[e].b0 = pr.y;
  atomicOr(&emask[e], 1u << sub);
  if (t == 0 || (key2[t] >> 2) != (key2[t - 1] >> 2)) {
    ekey[e] = key2[t] >> (kbits + 2);
    ek[e] = static_cast<uint32_t>((key2[t] >> 2) & ((uint64_t(1) << kbits) - 1));
  }
}

// per super block, the entry range whose k lies in [k0, k1) (a B panel)
__global__ void super_panel_ranges(const uint32_t* __restrict__ ek,
                                   const int64_t* __restrict__ sb_offset, int64_t n_sb,
                                   uint32_t k0, uint32_t k1, int64_t* __restrict__ beg,
                                   int64_t* __restrict__ end) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= n_sb) return;
  auto lower = [&](uint32_t k) {
    int64_t lo = sb_offset[b], hi = sb_offset[b + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ek[mid] < k) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  beg[b] = lower(k0);
  end[b] = lower(k1);
}

__global__ void super_sb_heads(const uint64_t* __restrict__ ekey, int64_t n_ent,
                               uint8_t* __restrict__ flag) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n_ent) return;
  flag[e] = (e == 0 || ekey[e] != ekey[e - 1]) ? 1 : 0;
}

__global__ void super_sb_finish(const uint64_t* __restrict__ ekey, const int64_t* __restrict__ heads,
                                int64_t n_sb, int64_t n_ent, int64_t* __restrict__ sb_offset,
                                uint64_t* __restrict__ sb_keys) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b > n_sb) return;
  sb_offset[b] = b < n_sb ? heads[b] : n_ent;
  if (b < n_sb) sb_keys[b] = ekey[heads[b]];
}

// output block o -> (super block, sub block) slot of sb_out
__global__ void super_out(const uint64_t* __restrict__ out_keys, int64_t n_out,
                          const uint64_t* __restrict__ sb_keys, int64_t n_sb,
                          int32_t* __restrict__ sb_out) {
  const int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o >= n_out) return;
  const uint64_t sup = out_keys[o] >> 2;
  int64_t lo = 0, hi = n_sb;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sb_keys[mid] < sup) lo = mid + 1;
    else hi = mid;
  }
  sb_out[4 * lo + static_cast<int64_t>(out_keys[o] & 3u)] = static_cast<int32_t>(o);
}

// ---- L = 128 leaves as 2x2 x 2 L = 64 sub-products (leaf_gemm_dmma<64, ..., 128>):
// output o -> sub outputs 4o + (2a + b); product (x, y) -> for k-half h the
// sub pair (4x + 2h + a, 4y + 2h + b); per sub output the original pairs in
// order, h = 0 then 1 (the L = 128 kernel's k order).
__global__ void expand_sub128(const int2* __restrict__ pairs,
                              const int64_t* __restrict__ out_offset,
                              const uint64_t* __restrict__ out_keys, int64_t n_out,
                              int2* __restrict__ sub_pairs, int64_t* __restrict__ sub_offset,
                              uint64_t* __restrict__ sub_keys) {
  for (int64_t o = blockIdx.x; o < n_out; o += gridDim.x) {
    const int64_t beg = out_offset[o], cnt = out_offset[o + 1] - beg;
    if (threadIdx.x < 4) {
      sub_offset[4 * o + threadIdx.x] = 8 * beg + threadIdx.x * 2 * cnt;
      sub_keys[4 * o + threadIdx.x] = (out_keys[o] << 2) | threadIdx.x;
    }
    if (o == n_out - 1 && threadIdx.x == 0) sub_offset[4 * n_out] = 8 * (beg + cnt);
    for (int64_t q = threadIdx.x; q < 8 * cnt; q += blockDim.x) {
      const int64_t p = q >> 3;
      const int s = static_cast<int>((q >> 1) & 3), h = static_cast<int>(q & 1);
      const int a = s >> 1, b = s & 1;
      const int2 pr = pairs[beg + p];
      sub_pairs[8 * beg + s * 2 * cnt + 2 * p + h] =
          make_int2(4 * pr.x + 2 * h + a, 4 * pr.y + 2 * h + b);
    }
  }
}

struct Plan {
  int64_t n_surv = 0, n_out = 0;
  int kbits = 0;
  DevBuf<uint64_t> keys, out_keys;
  DevBuf<int64_t> out_offset;
  DevBuf<int2> pairs;
  // built by the dense walk for the L = 32 super-block GEMM: no keys or pairs,
  // build_super32 repeats the walk per super block from this recipe
  bool dense_super = false;
  const spg_matrix *src_a = nullptr, *src_b = nullptr, *src_slots = nullptr;
  double tau = 0.0;
  bool skip_test = true;
  Shard shard;
};

// keep_keys: the sorted survivor keys stay (B panels, super-block re-keying);
// for_super: the product runs through leaf_gemm_super32 -- with the dense walk
// only the output blocks are produced here (implies keep_keys otherwise)
Plan plan_product(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                  bool skip_test, Shard shard, bool keep_keys,
                  const spg_matrix* a_slots = nullptr, bool for_super = false) {
  if (!a_slots) a_slots = a;  // a: norms for the skip tests; a_slots: A's payload slots
  keep_keys = keep_keys || for_super;
  {
    DenseTasks dt;
    const bool wk = keep_keys && !for_super, wp = !for_super;
    const bool dense =
        skip_test ? dense_tasklist<KeepRule::kSkip>(ctx, a, b, tau, shard, wk, wp, a_slots, &dt,
                                                    true)
                  : dense_tasklist<KeepRule::kExact>(ctx, a, b, tau, shard, wk, wp, a_slots, &dt,
                                                     true);
    if (dense) {
      Plan pl;
      pl.n_surv = dt.n_surv;
      pl.n_out = dt.n_out;
      pl.kbits = a->depth;
      pl.dense_super = for_super;
      pl.src_a = a;
      pl.src_b = b;
      pl.src_slots = a_slots;
      pl.tau = tau;
      pl.skip_test = skip_test;
      pl.shard = shard;
      pl.keys = std::move(dt.keys);
      pl.out_keys = std::move(dt.out_keys);
      pl.out_offset = std::move(dt.out_offset);
      pl.pairs = std::move(dt.pairs);
      return pl;
    }
  }
  TaskList tl = skip_test ? build_tasklist<KeepRule::kSkip>(ctx, a, b, tau, shard)
                          : build_tasklist<KeepRule::kExact>(ctx, a, b, tau, shard);
  Plan pl;
  pl.n_surv = tl.n_surv;
  pl.kbits = tl.kbits;
  const int64_t n_surv = tl.n_surv;
  if (n_surv) {
    PhaseTrace tr(ctx, "tasklist.group+pairs");
    DevBuf<uint8_t> flags(n_surv, ctx);
    head_flags<<<grid_for(n_surv, 256), 256, 0, ctx->stream>>>(tl.keys.get(), n_surv, tl.kbits,
                                                              flags.get());
    SPG_CHECK_LAUNCH(ctx);
    DevBuf<int64_t> heads(n_surv, ctx);
    DevBuf<int64_t> n_sel(1, ctx);
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    SPG_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags.get(), heads.get(), n_sel.get(),
                                        n_surv, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx);
    SPG_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flags.get(), heads.get(),
                                        n_sel.get(), n_surv, ctx->stream));
    ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
    pl.n_out = copy_scalar_to_host_i64(ctx, n_sel.get());
    pl.out_keys = DevBuf<uint64_t>(pl.n_out, ctx);
    pl.out_offset = DevBuf<int64_t>(pl.n_out + 1, ctx);
    run_outputs<<<grid_for(pl.n_out + 1, 256), 256, 0, ctx->stream>>>(
        tl.keys.get(), heads.get(), pl.n_out, n_surv, tl.kbits, pl.out_keys.get(),
        pl.out_offset.get());
    SPG_CHECK_LAUNCH(ctx);
    pl.pairs = DevBuf<int2>(n_surv, ctx);
    // norms and payload slots from different matrices (a_norms plans): a
    // survivor whose A leaf the slot matrix lacks would read A + (-1) L^2
    const bool split = a_slots != a;
    DevBuf<int> missing(split ? 1 : 0, ctx);
    if (split) SPG_CUDA(cudaMemsetAsync(missing.get(), 0, sizeof(int), ctx->stream));
    make_pairs<<<grid_for(n_surv, 256), 256, 0, ctx->stream>>>(tl.keys.get(), n_surv, tl.kbits,
                                                              a_slots->grid_slot, b->grid_slot,
                                                              pl.pairs.get(),
                                                              split ? missing.get() : nullptr);
    SPG_CHECK_LAUNCH(ctx);
    if (split) {
      int h = 0;
      SPG_CUDA(cudaMemcpyAsync(&h, missing.get(), sizeof(int), cudaMemcpyDeviceToHost,
                               ctx->stream));
      SPG_CUDA(cudaStreamSynchronize(ctx->stream));
      if (h)
        fail(SPG_EINVAL, "plan: a_norms lists a leaf in the shard rows that the local A does "
                         "not hold (the shard rows of a and a_norms must have the same leaves)");
    }
  }
  if (keep_keys) pl.keys = std::move(tl.keys);
  return pl;
}


// CTA order of the output blocks for the GEMM: row-major (within each chunk
// of `chunk` consecutive Morton-ordered blocks).  The C blocks stay in
// Morton order; only which CTA computes which block changes.  Concurrent CTAs
// then share the A row panel A(i, :) (16 MB on cfg2: L2-resident), which cut
// DRAM traffic and measured +1.5 % over Morton order on cfg2 (35.4 vs 34.9).
// strip_log > 0: strips of 2^strip_log block rows, column-major inside a
// strip, so the CTAs in flight also share each B leaf B(k, j) between the
// strip's rows.
__global__ void order_keys_kernel(const uint64_t* __restrict__ mkeys, int64_t n, int64_t chunk,
                                  int strip_log, uint64_t* __restrict__ skeys,
                                  int32_t* __restrict__ idx) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint64_t r = morton_row(mkeys[t]), c = morton_col(mkeys[t]);
  const uint64_t rs = r >> strip_log, ri = r & ((uint64_t(1) << strip_log) - 1);
  skeys[t] = (static_cast<uint64_t>(t / chunk) << 48) | (rs << 30) | (c << 15) | ri;
  idx[t] = static_cast<int32_t>(t % chunk);
}

// developer switch SPG_ORDER: 0 = Morton CTA order, 1 = row-major (default),
// 2 + s = strips of 2^s block rows
int block_order_mode() {
  static const int v = [] {
    const char* e = std::getenv("SPG_ORDER");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
bool block_order_enabled() { return block_order_mode() != 0; }

DevBuf<int32_t> make_block_order(spg_context* ctx, const uint64_t* mkeys, int64_t n,
                                 int64_t chunk) {
  if (n < 2 || !block_order_enabled()) return DevBuf<int32_t>();
  DevBuf<uint64_t> k1(n, ctx), k2(n, ctx);
  DevBuf<int32_t> i1(n, ctx), i2(n, ctx);
  const int strip_log = block_order_mode() >= 2 ? block_order_mode() - 2 : 0;
  order_keys_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(mkeys, n, chunk, strip_log,
                                                               k1.get(), i1.get());
  SPG_CHECK_LAUNCH(ctx);
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.get(), k2.get(), i1.get(), i2.get(),
                                           n, 0, 64, ctx->stream));
  DevBuf<uint8_t> tmp(bytes, ctx);
  SPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, k1.get(), k2.get(), i1.get(),
                                           i2.get(), n, 0, 64, ctx->stream));
  ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
  return i2;
}

// L = 32 resident product through leaf_gemm_super32 (the default; another
// SPG_GEMM32 value selects a per-block tiling): the (super block, k) entry
// list from the sorted survivor keys, then one CTA per 2x2 super block.
// Config-5-style L = 32 product (tools/profile_leaf.py 32): 29.1 -> 32.3
// TFLOP/s, C~ bitwise unchanged.
bool super32_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPG_GEMM32");
    return !e || std::atoi(e) == 9;
  }();
  return on;
}

struct Super32 {
  int64_t n_sb = 0, n_ent = 0;
  DevBuf<SuperEntry> ent;
  DevBuf<uint32_t> emask, ek;
  DevBuf<int64_t> sb_offset;
  DevBuf<int32_t> sb_out, order;
};

// build_super32 by the dense walk (tl_super): entries straight from the norm
// pyramids, no survivor keys, no sort.
template <KeepRule R>
Super32 dense_super32(spg_context* ctx, const Plan& pl) {
  Super32 sp;
  const spg_matrix *a = pl.src_a, *b = pl.src_b;
  const int d = a->depth, s = d - 3;
  PhaseTrace tr(ctx, "tasklist.dense_super");
  const uint32_t tile_rows = (1u << s) >> pl.shard.level;
  const uint32_t row_lo = tile_rows * static_cast<uint32_t>(pl.shard.index);
  const uint32_t row_hi = row_lo + tile_rows;
  const int64_t n_tiles = static_cast<int64_t>(tile_rows) << s, n_flags = n_tiles << s;
  const int64_t n_sup = int64_t(16) << (2 * s);
  DevBuf<uint8_t> valid(n_flags, ctx);
  tl_valid<R><<<grid_for(n_flags, 256), 256, 0, ctx->stream>>>(
      s, a->pyramid, b->pyramid, pl.tau, row_lo, row_hi, valid.get());
  SPG_CHECK_LAUNCH(ctx);
  const int kp = tile_parts_log(ctx, n_tiles, s);
  const int64_t n_cnt = n_sup << kp;
  DevBuf<int64_t> counts(n_cnt + 1, ctx), offsets(n_cnt + 1, ctx);
  if (pl.shard.level > 0)
    SPG_CUDA(cudaMemsetAsync(counts.get(), 0, (n_cnt + 1) * sizeof(int64_t), ctx->stream));
  else
    SPG_CUDA(cudaMemsetAsync(counts.get() + n_cnt, 0, sizeof(int64_t), ctx->stream));
  const unsigned grid = static_cast<unsigned>(((n_tiles << kp) + kTlWarps - 1) / kTlWarps);
  tl_super<R, false><<<grid, kTlWarps * 32, 0, ctx->stream>>>(
      s, d, kp, a->pyramid, b->pyramid, pl.tau, row_lo, row_hi, valid.get(), counts.get(),
      nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  SPG_CHECK_LAUNCH(ctx);
  const int64_t n_ent = scan_counts(ctx, counts.get(), n_cnt, offsets.get());
  sp.n_ent = n_ent;
  if (n_ent == 0) return sp;
  sp.ent = DevBuf<SuperEntry>(n_ent, ctx);
  sp.emask = DevBuf<uint32_t>(n_ent, ctx);
  sp.ek = DevBuf<uint32_t>(n_ent, ctx);
  const bool split = pl.src_slots != a;
  DevBuf<int> missing(split ? 1 : 0, ctx);
  if (split) SPG_CUDA(cudaMemsetAsync(missing.get(), 0, sizeof(int), ctx->stream));
  tl_super<R, true><<<grid, kTlWarps * 32, 0, ctx->stream>>>(
      s, d, kp, a->pyramid, b->pyramid, pl.tau, row_lo, row_hi, valid.get(), nullptr,
      offsets.get(),
      pl.src_slots->grid_slot, b->grid_slot, sp.ent.get(), sp.emask.get(), sp.ek.get(),
      split ? missing.get() : nullptr);
  SPG_CHECK_LAUNCH(ctx);
  // the non-empty super blocks, ascending (Morton), with their entry ranges
  DevBuf<int64_t> sbl(n_sup, ctx), n_sel(1, ctx), totals(kp ? n_sup : 0, ctx);
  const int64_t* per_sb = counts.get();
  if (kp) {
    tl_block_totals<<<grid_for(n_sup, 256), 256, 0, ctx->stream>>>(offsets.get(), n_sup, kp,
                                                                   totals.get());
    SPG_CHECK_LAUNCH(ctx);
    per_sb = totals.get();
  }
  thrust::counting_iterator<int64_t> it(0);
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, per_sb, sbl.get(), n_sel.get(), n_sup,
                                      ctx->stream));
  {
    DevBuf<uint8_t> tmp(bytes, ctx);
    SPG_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, per_sb, sbl.get(), n_sel.get(),
                                        n_sup, ctx->stream));
  }
  ctx->lib_calls += 2;  // CUB device-wide primitives (library kernels)
  const int64_t n_sb = copy_scalar_to_host_i64(ctx, n_sel.get());
  sp.n_sb = n_sb;
  sp.sb_offset = DevBuf<int64_t>(n_sb + 1, ctx);
  DevBuf<uint64_t> sb_keys(n_sb, ctx);
  tl_outputs<<<grid_for(n_sb + 1, 256), 256, 0, ctx->stream>>>(
      sbl.get(), offsets.get(), kp, n_sb, n_ent, sb_keys.get(), sp.sb_offset.get());
  SPG_CHECK_LAUNCH(ctx);
  sp.sb_out = DevBuf<int32_t>(4 * n_sb, ctx);
  SPG_CUDA(cudaMemsetAsync(sp.sb_out.get(), 0xff, 4 * n_sb * sizeof(int32_t), ctx->stream));
  super_out<<<grid_for(pl.n_out, 256), 256, 0, ctx->stream>>>(pl.out_keys.get(), pl.n_out,
                                                              sb_keys.get(), n_sb,
                                                              sp.sb_out.get());
  SPG_CHECK_LAUNCH(ctx);
  sp.order = make_block_order(ctx, sb_keys.get(), n_sb, n_sb);
  if (split) {
    int h = 0;
    SPG_CUDA(cudaMemcpyAsync(&h, missing.get(), sizeof(int), cudaMemcpyDeviceToHost,
                             ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h)
      fail(SPG_EINVAL, "plan: a_norms lists a leaf in the shard rows that the local A does "
                       "not hold (the shard rows of a and a_norms must have the same leaves)");
  }
  return sp;
}

Super32 build_super32(spg_context* ctx, int depth, const Plan& pl) {
  if (pl.dense_super)
    return pl.skip_test ? dense_super32<KeepRule::kSkip>(ctx, pl)
                        : dense_super32<KeepRule::kExact>(ctx, pl);
  Super32 sp;
  const int64_t n = pl.n_surv;
  if (n == 0) return sp;
  const int kbits = pl.kbits;
  DevBuf<uint64_t> k2(n, ctx), k2s(n, ctx);
  DevBuf<int64_t> v(n, ctx), vs(n, ctx);
  super_keys<<<grid_for(n, 256), 256, 0, ctx->stream>>>(pl.keys.get(), n, kbits, k2.get(),
                                                         v.get());
  SPG_CHECK_LAUNCH(ctx);
  size_t bytes = 0;
  const int end_bit = 2 * depth + kbits;
  SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k2.get(), k2s.get(), v.get(), vs.get(),
                                           n, 0, end_bit, ctx->stream));
  {
    DevBuf<uint8_t> tmp(bytes, ctx);
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, k2.get(), k2s.get(), v.get(),
                                             vs.get(), n, 0, end_bit, ctx->stream));
  }
  k2.reset();
  v.reset();
  DevBuf<int64_t> head(n, ctx), eidx(n, ctx);
  super_heads<<<grid_for(n, 256), 256, 0, ctx->stream>>>(k2s.get(), n, head.get());
  SPG_CHECK_LAUNCH(ctx);
  bytes = 0;
  SPG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, head.get(), eidx.get(), n, ctx->stream));
  {
    DevBuf<uint8_t> tmp(bytes, ctx);
    SPG_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, head.get(), eidx.get(), n,
                                           ctx->stream));
  }
  const int64_t n_ent = copy_scalar_to_host_i64(ctx, eidx.get() + n - 1);
  sp.n_ent = n_ent;
  sp.ent = DevBuf<SuperEntry>(n_ent, ctx);
  sp.emask = DevBuf<uint32_t>(n_ent, ctx);
  sp.ek = DevBuf<uint32_t>(n_ent, ctx);
  DevBuf<uint64_t> ekey(n_ent, ctx);
  SPG_CUDA(cudaMemsetAsync(sp.ent.get(), 0, n_ent * sizeof(SuperEntry), ctx->stream));
  SPG_CUDA(cudaMemsetAsync(sp.emask.get(), 0, n_ent * sizeof(uint32_t), ctx->stream));
  super_fill<<<grid_for(n, 256), 256, 0, ctx->stream>>>(k2s.get(), vs.get(), eidx.get(), n, kbits,
                                                         pl.pairs.get(), sp.ent.get(),
                                                         sp.emask.get(), ekey.get(), sp.ek.get());
  SPG_CHECK_LAUNCH(ctx);
  head.reset();
  eidx.reset();
  k2s.reset();
  vs.reset();
  DevBuf<uint8_t> flag(n_ent, ctx);
  super_sb_heads<<<grid_for(n_ent, 256), 256, 0, ctx->stream>>>(ekey.get(), n_ent, flag.get());
  SPG_CHECK_LAUNCH(ctx);
  DevBuf<int64_t> heads(n_ent, ctx), n_sel(1, ctx);
  thrust::counting_iterator<int64_t> it(0);
  bytes = 0;
  SPG_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flag.get(), heads.get(), n_sel.get(),
                                      n_ent, ctx->stream));
  {
    DevBuf<uint8_t> tmp(bytes, ctx);
    SPG_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flag.get(), heads.get(),
                                        n_sel.get(), n_ent, ctx->stream));
  }
  ctx->lib_calls += 4;  // CUB device-wide primitives (library kernels)
  const int64_t n_sb = copy_scalar_to_host_i64(ctx, n_sel.get());
  sp.n_sb = n_sb;
  sp.sb_offset = DevBuf<int64_t>(n_sb + 1, ctx);
  DevBuf<uint64_t> sb_keys(n_sb, ctx);
  super_sb_finish<<<grid_for(n_sb + 1, 256), 256, 0, ctx->stream>>>(
      ekey.get(), heads.get(), n_sb, n_ent, sp.sb_offset.get(), sb_keys.get());
  SPG_CHECK_LAUNCH(ctx);
  sp.sb_out = DevBuf<int32_t>(4 * n_sb, ctx);
  SPG_CUDA(cudaMemsetAsync(sp.sb_out.get(), 0xff, 4 * n_sb * sizeof(int32_t), ctx->stream));
  super_out<<<grid_for(pl.n_out, 256), 256, 0, ctx->stream>>>(pl.out_keys.get(), pl.n_out,
                                                              sb_keys.get(), n_sb,
                                                              sp.sb_out.get());
  SPG_CHECK_LAUNCH(ctx);
  sp.order = make_block_order(ctx, sb_keys.get(), n_sb, n_sb);
  return sp;
}

// beg/end: per super block entry range (nullptr: all of its entries);
// accumulate: continue the sub blocks' accumulators stored in C
void launch_super32(spg_context* ctx, const Super32& sp, const double* A,
                    const double* const* btab, double* C, const int64_t* beg = nullptr,
                    const int64_t* end = nullptr, int accumulate = 0) {
  if (sp.n_sb == 0) return;
  constexpr size_t smem = 2 * 4 * 32 * 36 * sizeof(double);
  auto go = [&](auto kern) {
    SPG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(sp.n_sb, int64_t(1) << 30));
    kern<<<grid, 128, smem, ctx->stream>>>(
        A, btab, sp.ent.get(), sp.emask.get(), beg ? beg : sp.sb_offset.get(),
        end ? end : sp.sb_offset.get() + 1, sp.sb_out.get(), sp.n_sb, C, sp.order.get(),
        accumulate);
    SPG_CHECK_LAUNCH(ctx);
  };
  // developer switch SPG_SUPER32_QUAD=0: one warp per block (the round-1 kernel)
  static const bool quad = [] {
    const char* e = std::getenv("SPG_SUPER32_QUAD");
    return !e || std::atoi(e) != 0;
  }();
  if (quad) go(leaf_gemm_super32<true>);
  else go(leaf_gemm_super32<false>);
}

void run_super32(spg_context* ctx, int depth, const Plan& pl, const double* A,
                 const double* const* btab, double* C) {
  const Super32 sp = build_super32(ctx, depth, pl);
  launch_super32(ctx, sp, A, btab, C);
}

// L = 128 products as L = 64 sub-products (the default; another SPG_GEMM128
// value selects an L = 128 tiling): one L = 64 CTA per output sub-block,
// three per SM, where the L = 128 kernel fits one (registers) and idles the
// DMMA pipe between blocks.  Config-5 style L = 128 product
// (tools/profile_leaf.py 128): 32.7 -> 34.8 TFLOP/s, C~ bitwise unchanged.
bool sub128_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPG_GEMM128");
    return !e || std::atoi(e) == 9;
  }();
  return on;
}

struct Sub128 {
  int64_t n_sub = 0;
  DevBuf<int2> pairs;
  DevBuf<int64_t> offset;  // 4 n_out + 1
  DevBuf<int32_t> order;
};

Sub128 build_sub128(spg_context* ctx, const Plan& pl) {
  Sub128 sb;
  const int64_t n_out = pl.n_out;
  if (n_out == 0) return sb;
  sb.n_sub = 4 * n_out;
  sb.pairs = DevBuf<int2>(std::max<int64_t>(8 * pl.n_surv, 1), ctx);
  sb.offset = DevBuf<int64_t>(4 * n_out + 1, ctx);
  DevBuf<uint64_t> sk(4 * n_out, ctx);
  expand_sub128<<<static_cast<unsigned>(std::min<int64_t>(n_out, 1 << 20)), 256, 0,
                  ctx->stream>>>(pl.pairs.get(), pl.out_offset.get(), pl.out_keys.get(), n_out,
                                 sb.pairs.get(), sb.offset.get(), sk.get());
  SPG_CHECK_LAUNCH(ctx);
  sb.order = make_block_order(ctx, sk.get(), 4 * n_out, 4 * n_out);
  return sb;
}

// beg/end: per sub output pair range (beg = offset, end = nullptr: all)
void launch_sub128(spg_context* ctx, const Sub128& sb, const double* A, const double* const* btab,
                   double* C, const int64_t* beg = nullptr, const int64_t* end = nullptr,
                   int accumulate = 0) {
  if (sb.n_sub == 0) return;
  using Cfg = DmmaGemmCfg<64, 32, 32, 32, 2>;
  auto kern = leaf_gemm_dmma<64, 32, 32, 32, 2, true, 128>;
  SPG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(Cfg::kSmemBytes)));
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(sb.n_sub, int64_t(1) << 30));
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, ctx->stream>>>(
      A, nullptr, sb.pairs.get(), beg ? beg : sb.offset.get(), sb.n_sub, C, end, accumulate,
      btab, sb.order.get());
  SPG_CHECK_LAUNCH(ctx);
}

// a B panel's per-block pair ranges [bbeg, bend) -> the sub outputs' ranges
__global__ void sub128_ranges(const int64_t* __restrict__ out_offset,
                              const int64_t* __restrict__ bbeg, const int64_t* __restrict__ bend,
                              int64_t n_out, int64_t* __restrict__ sbeg,
                              int64_t* __restrict__ send) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= 4 * n_out) return;
  const int64_t o = q >> 2, s = q & 3;
  const int64_t b0 = out_offset[o], cnt = out_offset[o + 1] - b0;
  const int64_t base = 8 * b0 + s * 2 * cnt;
  sbeg[q] = base + 2 * (bbeg[o] - b0);
  send[q] = base + 2 * (bend[o] - b0);
}

void run_sub128(spg_context* ctx, const Plan& pl, const double* A, const double* const* btab,
                double* C) {
  const Sub128 sb = build_sub128(ctx, pl);
  launch_sub128(ctx, sb, A, btab, C);
}

// The product streamed to host buffers: the GEMM runs in chunks of output
// blocks (Morton order); after each chunk its leaf norms are computed (K1)
// and the chunk is copied D2H on the copy stream while the next chunk
// computes.  Result identical to building C on the device and downloading it
// (same blocks, order, payload and norms; all-zero blocks dropped).
void stream_product_to_host(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                            DevBuf<int2>& pairs, DevBuf<int64_t>& out_offset,
                            DevBuf<uint64_t>& out_keys, int64_t n_out, HostOut* host) {
  const double* const* btab = leaf_table(ctx, b);  // before the aux stream forks
  const int L = a->leaf;
  const int64_t LL = static_cast<int64_t>(L) * L;
  if (n_out > host->capacity) fail(SPG_EINVAL, "output capacity smaller than the product");
  host->count = 0;
  if (n_out == 0) return;
  std::vector<uint64_t> hkeys(static_cast<size_t>(n_out));
  std::vector<uint8_t> hnz(static_cast<size_t>(n_out));
  SPG_CUDA(cudaMemcpyAsync(hkeys.data(), out_keys.get(), n_out * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, ctx->stream));
  DevBuf<double> c_payload(n_out * LL, ctx);
  DevBuf<double> norms(n_out, ctx);
  DevBuf<uint8_t> nz(n_out, ctx);
  const int32_t nb = (a->dimension + L - 1) / L;
  // developer switch SPG_STREAM_CHUNKS: upper bound of the chunk count
  static const int64_t max_chunks = [] {
    const char* e = std::getenv("SPG_STREAM_CHUNKS");
    return e && std::atoi(e) > 0 ? static_cast<int64_t>(std::atoi(e)) : int64_t(32);
  }();
  const int64_t n_chunks = std::min<int64_t>(max_chunks, std::max<int64_t>(1, n_out / 4096));
  const int64_t cs = (n_out + n_chunks - 1) / n_chunks;
  // row-major CTA order inside each chunk (indices local to the chunk)
  DevBuf<int32_t> order = make_block_order(ctx, out_keys.get(), n_out, cs);
  std::vector<cudaEvent_t> done(static_cast<size_t>(n_chunks));
  for (auto& e : done) SPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct EventGuard {
    std::vector<cudaEvent_t>& v;
    ~EventGuard() {
      for (auto& e : v) cudaEventDestroy(e);
    }
  } guard{done};
  {
    PhaseTrace tr(ctx, "gemm+stream");
    // chunks alternate between two compute streams so one chunk's tail
    // (uneven survivor counts per block) overlaps the next chunk's head
    cudaStream_t cs_[2] = {ctx->stream, ctx->aux_stream};
    cudaEvent_t ready;
    SPG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    SPG_CUDA(cudaEventRecord(ready, ctx->stream));
    SPG_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ready, 0));
    cudaEventDestroy(ready);
    static const int dbg = [] {
      const char* e = std::getenv("SPG_STREAM_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    const auto tq0 = std::chrono::steady_clock::now();
    for (int64_t c = 0; c < n_chunks; ++c) {
      const int64_t o0 = c * cs, o1 = std::min(n_out, o0 + cs);
      if (o0 >= o1) break;
      cudaStream_t st = cs_[c & 1];
      if (dbg == 2) {  // no copies at all
        run_gemm(ctx, L, a->payload, b->payload, pairs.get(), out_offset.get() + o0, o1 - o0,
                 c_payload.get() + o0 * LL, st, nullptr, 0, btab,
                 order.get() ? order.get() + o0 : nullptr);
        continue;
      }
      run_gemm(ctx, L, a->payload, b->payload, pairs.get(), out_offset.get() + o0, o1 - o0,
               c_payload.get() + o0 * LL, st, nullptr, 0, btab,
               order.get() ? order.get() + o0 : nullptr);
      leaf_norms(ctx, c_payload.get() + o0 * LL, o1 - o0, L, a->dimension, nb, nullptr, nullptr,
                 norms.get() + o0, nz.get() + o0, nullptr, st);
      SPG_CUDA(cudaEventRecord(done[c], st));
      SPG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, done[c], 0));
      SPG_CUDA(cudaMemcpyAsync(host->payload + o0 * LL, c_payload.get() + o0 * LL,
                               (o1 - o0) * LL * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx->copy_stream));
      SPG_CUDA(cudaMemcpyAsync(host->norms + o0, norms.get() + o0, (o1 - o0) * sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->copy_stream));
    }
    // the all-zero flags go to pageable host memory: one copy after the loop
    // (a pageable cudaMemcpyAsync blocks the host and would serialise the chunks)
    if (dbg)
      std::fprintf(stderr, "[spg] enqueue loop %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count());
    // join: the pool's stream order requires the main stream to see all work
    SPG_CUDA(cudaEventRecord(done[0], ctx->copy_stream));
    SPG_CUDA(cudaStreamWaitEvent(ctx->stream, done[0], 0));
    SPG_CUDA(cudaEventRecord(done[0], ctx->aux_stream));
    SPG_CUDA(cudaStreamWaitEvent(ctx->stream, done[0], 0));
    SPG_CUDA(cudaMemcpyAsync(hnz.data(), nz.get(), n_out, cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->aux_stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  // keys -> coordinates; drop the (rare) all-zero sums like make_leaf
  int64_t kept = 0;
  for (int64_t o = 0; o < n_out; ++o) {
    if (!hnz[o]) continue;
    if (kept != o) {
      std::memmove(host->payload + kept * LL, host->payload + o * LL, LL * sizeof(double));
      host->norms[kept] = host->norms[o];
    }
    const uint64_t key = hkeys[o];
    if (host->rows) host->rows[kept] = static_cast<int32_t>(morton_row(key));
    if (host->cols) host->cols[kept] = static_cast<int32_t>(morton_col(key));
    ++kept;
  }
  host->count = kept;
}

}  // namespace

// Row chunks of a product whose task list would not fit (include/spamm_gpu.h
// spg_context_set_task_budget): 2^c sub-shards of `sh`, one task list at a
// time.  Peak device bytes per candidate leaf product of a plan, against half
// of the free memory (plus this context's cached blocks) left after `reserve`
// bytes for the output, whose chunks accumulate:
//  * dense walk (depth 3 .. 14, chunks of whole tile rows): 16 B -- a key and
//    a slot pair per survivor; 24 B for the L = 32 super-block entries (slots,
//    mask and k per entry, at most one entry per survivor);
//  * expansion + radix sort (other depths, or chunks thinner than a tile row):
//    about 40 B (triples, masks, keys and their sorted copy, sort temp, pairs),
//    96 B when the super-block re-keying (its own key-value sort) follows.
int chunk_bits(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, Shard sh,
               int max_bits, bool super32, int64_t reserve) {
  if (max_bits <= 0) return 0;
  int64_t budget = ctx->task_budget;
  if (budget <= 0) {
    size_t fr = 0, tot = 0;
    SPG_CUDA(cudaMemGetInfo(&fr, &tot));
    size_t cached = 0;
    for (const auto& kv : ctx->pool.free_blocks) cached += kv.first;
    const int64_t avail = static_cast<int64_t>(fr + cached) - std::max<int64_t>(reserve, 0);
    budget = std::max<int64_t>(avail / 2, static_cast<int64_t>(fr / 8));
  }
  const double cand = static_cast<double>(count_candidates(ctx, a, b, sh));
  auto bits_for = [&](double per_cand, int limit) {
    int c = 0;
    while (c < limit && per_cand * cand / static_cast<double>(int64_t(1) << c) >
                            static_cast<double>(budget))
      ++c;
    return per_cand * cand / static_cast<double>(int64_t(1) << c) <= static_cast<double>(budget)
               ? c : -1;
  };
  static const bool trace = [] {
    const char* e = std::getenv("SPG_TRACE");
    return e && e[0] == '1';
  }();
  const int s = a->depth - 3;
  int c = -1;
  if (dense_tasklist_enabled() && dense_walk_fits(a->depth, sh.level))
    c = bits_for(super32 ? 24.0 : 16.0, std::min(max_bits, s - sh.level));
  if (c < 0) {
    c = bits_for(super32 ? 96.0 : 40.0, max_bits);
    if (c < 0) c = max_bits;
  }
  if (trace)
    std::fprintf(stderr, "[spg] row chunks 2^%d: %.3g candidates, budget %.3g B (reserve %.3g B)\n",
                 c, cand, static_cast<double>(budget), static_cast<double>(reserve));
  return c;
}

// upper bound of an output's payload bytes: the shard's block rows x all
// block columns
int64_t output_bytes_bound(const spg_matrix* a, Shard sh) {
  const int64_t nb = (a->dimension + a->leaf - 1) / a->leaf;
  const int64_t rows = std::max<int64_t>(1, ((int64_t(1) << a->depth) >> sh.level));
  const int64_t LL = static_cast<int64_t>(a->leaf) * a->leaf;
  return std::min(rows, nb) * nb * LL * static_cast<int64_t>(sizeof(double));
}

void gemm_plan(spg_context* ctx, int depth, int L, const Plan& plan, bool super32,
               const double* A, const double* B, const double* const* btab, double* C) {
  if (super32) {
    PhaseTrace tr(ctx, "gemm(super32)");
    run_super32(ctx, depth, plan, A, btab, C);
  } else if (L == 128 && sub128_enabled()) {
    PhaseTrace tr(ctx, "gemm(sub128)");
    run_sub128(ctx, plan, A, btab, C);
  } else {
    DevBuf<int32_t> order = make_block_order(ctx, plan.out_keys.get(), plan.n_out, plan.n_out);
    PhaseTrace tr(ctx, "gemm");
    run_gemm(ctx, L, A, B, plan.pairs.get(), plan.out_offset.get(), plan.n_out, C, nullptr,
             nullptr, 0, btab, order.get());
  }
}

// The product in 2^c row chunks: pass 1 sizes every chunk's output (its task
// list, then freed), pass 2 rebuilds each chunk's task list and runs its GEMM
// into its rows' place in one C payload.  Per block the same pairs in the
// same k order: C is bitwise the unchunked product.
spg_matrix* spamm_device_chunked(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                                 double tau, bool skip_test, spg_spamm_stats* stats, Shard sh,
                                 int c, bool super32) {
  const int L = a->leaf;
  const int64_t LL = static_cast<int64_t>(L) * L;
  const int nch = 1 << c;
  auto sub = [&](int q) { return Shard{sh.level + c, (sh.index << c) + q}; };
  std::vector<int64_t> n_out(static_cast<size_t>(nch));
  int64_t total_out = 0;
  for (int q = 0; q < nch; ++q) {
    // sizing only: with the dense walk, for_super stops after the count pass
    const Plan pl = plan_product(ctx, a, b, tau, skip_test, sub(q), false, nullptr, true);
    n_out[q] = pl.n_out;
    total_out += pl.n_out;
  }
  double* c_payload = dev_alloc<double>(std::max<int64_t>(total_out * LL, 1), ctx);
  uint64_t* keys = nullptr;
  try {
    keys = dev_alloc<uint64_t>(std::max<int64_t>(total_out, 1), ctx);
  } catch (...) {
    dev_free(c_payload, ctx);
    throw;
  }
  const double* const* btab = leaf_table(ctx, b);
  float ms_task = 0.0f, ms_gemm = 0.0f;
  int64_t n_surv = 0, off = 0;
  try {
    for (int q = 0; q < nch; ++q) {
      SPG_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
      Plan pl = plan_product(ctx, a, b, tau, skip_test, sub(q), false, nullptr, super32);
      SPG_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
      if (pl.n_out != n_out[q]) fail(SPG_EINTERNAL, "chunked product: chunk size changed");
      if (pl.n_out) {
        gemm_plan(ctx, a->depth, L, pl, super32, a->payload, b->payload, btab,
                  c_payload + off * LL);
        SPG_CUDA(cudaMemcpyAsync(keys + off, pl.out_keys.get(), pl.n_out * sizeof(uint64_t),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
      }
      SPG_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
      SPG_CUDA(cudaEventSynchronize(ctx->ev[4]));
      float t1 = 0.0f, t2 = 0.0f;
      SPG_CUDA(cudaEventElapsedTime(&t1, ctx->ev[2], ctx->ev[3]));
      SPG_CUDA(cudaEventElapsedTime(&t2, ctx->ev[3], ctx->ev[4]));
      ms_task += t1;
      ms_gemm += t2;
      n_surv += pl.n_surv;
      off += pl.n_out;
    }
  } catch (...) {
    dev_free(keys, ctx);
    dev_free(c_payload, ctx);
    throw;
  }
  SPG_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
  // chunk keys are not globally in Morton order: the matrix scatters them
  spg_matrix* out = matrix_from_morton_blocks(ctx, a->dimension, L, total_out, keys, c_payload);
  SPG_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
  SPG_CUDA(cudaEventSynchronize(ctx->ev[5]));
  if (stats) {
    stats->survivors = n_surv;
    stats->output_blocks = total_out;
    stats->flops = 2.0 * static_cast<double>(L) * L * L * static_cast<double>(n_surv);
    stats->ms_tasklist = ms_task;
    stats->ms_gemm = ms_gemm;
    SPG_CUDA(cudaEventElapsedTime(&stats->ms_finalize, ctx->ev[4], ctx->ev[5]));
    stats->candidates = count_candidates(ctx, a, b, sh);
  }
  return out;
}

spg_matrix* spamm_device(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                         bool skip_test, spg_spamm_stats* stats, Shard shard, HostOut* host) {
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "multiply: dimension or leaf size mismatch");
  if (tau < 0.0) fail(SPG_EINVAL, "spamm: tau must be nonnegative");
  require_payload(a);
  require_payload(b);
  if (shard.level < 0 || shard.level > a->depth || shard.index < 0 ||
      shard.index >= (1 << shard.level))
    fail(SPG_EINVAL, "spamm: shard outside the quadtree");
  const int L = a->leaf;
  const int64_t LL = static_cast<int64_t>(L) * L;
  const bool super32 = L == 32 && !host && super32_enabled();
  if (!host) {  // super blocks pair rows 2I, 2I+1: a chunk keeps >= 2 rows for them
    const int c = chunk_bits(ctx, a, b, shard, a->depth - shard.level - (super32 ? 1 : 0),
                             super32, output_bytes_bound(a, shard));
    if (c > 0) return spamm_device_chunked(ctx, a, b, tau, skip_test, stats, shard, c, super32);
  }
  SPG_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  Plan plan = plan_product(ctx, a, b, tau, skip_test, shard, false, nullptr, super32);
  const int64_t n_surv = plan.n_surv, n_out = plan.n_out;
  DevBuf<uint64_t>& out_keys = plan.out_keys;
  DevBuf<int64_t>& out_offset = plan.out_offset;
  DevBuf<int2>& pairs = plan.pairs;
  SPG_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
  spg_matrix* c = nullptr;
  if (host) {
    stream_product_to_host(ctx, a, b, pairs, out_offset, out_keys, n_out, host);
    SPG_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
    SPG_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
    SPG_CUDA(cudaEventSynchronize(ctx->ev[5]));
  } else {
    double* c_payload = dev_alloc<double>(std::max<int64_t>(n_out * LL, 1), ctx);
    const double* const* btab = leaf_table(ctx, b);
    gemm_plan(ctx, a->depth, L, plan, super32, a->payload, b->payload, btab, c_payload);
    SPG_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
    pairs.reset();
    out_offset.reset();
    {
      PhaseTrace tr(ctx, "finalize");
      c = matrix_from_morton_blocks(ctx, a->dimension, L, n_out, out_keys.release(), c_payload);
    }
    SPG_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
    SPG_CUDA(cudaEventSynchronize(ctx->ev[5]));
  }
  if (stats) {
    stats->survivors = n_surv;
    stats->output_blocks = n_out;
    stats->flops = 2.0 * static_cast<double>(L) * L * L * static_cast<double>(n_surv);
    SPG_CUDA(cudaEventElapsedTime(&stats->ms_tasklist, ctx->ev[2], ctx->ev[3]));
    SPG_CUDA(cudaEventElapsedTime(&stats->ms_gemm, ctx->ev[3], ctx->ev[4]));
    SPG_CUDA(cudaEventElapsedTime(&stats->ms_finalize, ctx->ev[4], ctx->ev[5]));
    stats->candidates = count_candidates(ctx, a, b, shard);
  }
  return c;
}

namespace {
// per output block, the pair range whose k lies in [k0, k1) (keys of a block
// are sorted by k)
__global__ void panel_ranges(const uint64_t* __restrict__ keys,
                             const int64_t* __restrict__ out_offset, int64_t n_out, int kbits,
                             uint32_t k0, uint32_t k1, int64_t* __restrict__ beg,
                             int64_t* __restrict__ end) {
  const int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o >= n_out) return;
  const uint64_t kmask = (uint64_t(1) << kbits) - 1;
  auto lower = [&](int64_t lo, int64_t hi, uint32_t k) {
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((keys[mid] & kmask) < k) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  const int64_t hi = out_offset[o + 1];
  const int64_t b = lower(out_offset[o], hi, k0);
  beg[o] = b;
  end[o] = lower(b, hi, k1);
}

struct EventSet {
  cudaEvent_t e[4] = {};
  EventSet() {
    for (auto& x : e) SPG_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  }
  ~EventSet() {
    for (auto& x : e) cudaEventDestroy(x);
  }
};
}  // namespace
}  // namespace spg

// A product whose B arrives in panels of block rows: B from
// host memory (spg_bstream) or from the GPU that owns those rows (NCCL
// broadcast, sharded.py).  The task list comes from the norm pyramids alone;
// C starts at zero and every panel continues each output block's accumulator
// over the products whose k lies in the panel.  Panels must tile the block
// rows in ascending order, so each C element sees the same FP64 operation
// sequence as the resident product and C is bitwise identical to it.
struct spg_plan {
  bool external_c = false;  // c is a slice of the caller's payload (not owned)
  spg_context* ctx = nullptr;
  const spg_matrix* a = nullptr;
  const spg_matrix* b = nullptr;  // norm-only, slots sorted by block row
  spg::Plan pl;
  spg::DevBuf<double> c;
  spg::DevBuf<int64_t> beg, end;
  spg::DevBuf<const double*> btab;  // B leaf addresses of the panels seen so far
  spg::DevBuf<int32_t> order;        // CTA order of the output blocks (row-major)
  // L = 32: the 2x2 super-block entry list and its per-panel ranges
  std::unique_ptr<spg::Super32> sup;
  spg::DevBuf<int64_t> sb_beg, sb_end;
  // L = 128: the L = 64 sub-product list and its per-panel ranges
  std::unique_ptr<spg::Sub128> sub;
  spg::DevBuf<int64_t> sub_beg, sub_end;
  int32_t next_row = 0;
  bool finished = false;
  spg_spamm_stats stats{};
  cudaEvent_t ev[2] = {};
  cudaEvent_t t_first = nullptr, t_last = nullptr;  // GEMM phase: first panel .. finish
  // per panel launch: (start, stop) around its kernels; ms_gemm = their sum
  // (the phase span above also holds the waits for the panels themselves)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> panel_ev;
  bool started = false;
  ~spg_plan() {
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);
    if (t_first) cudaEventDestroy(t_first);
    if (t_last) cudaEventDestroy(t_last);
    for (auto& pe : panel_ev) {
      cudaEventDestroy(pe.first);
      cudaEventDestroy(pe.second);
    }
  }
};

namespace spg {

// a_norms (optional): the norms of the whole A when `a` holds only the
// shard's block rows (skip tests above the shard level need the global
// ancestors); the shard's rows of a_norms must be a's.
// external_c: the plan's output blocks live in the caller's payload (row
// chunks of one product written in place, plan_finish_into) instead of a
// buffer of its own
spg_plan* plan_create(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                      Shard shard, const spg_matrix* a_norms = nullptr,
                      double* external_c = nullptr) {
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "multiply: dimension or leaf size mismatch");
  if (a_norms && (a_norms->dimension != a->dimension || a_norms->leaf != a->leaf))
    fail(SPG_EINVAL, "plan: A norms do not match A's shape");
  if (tau < 0.0) fail(SPG_EINVAL, "spamm: tau must be nonnegative");
  require_payload(a);
  if (!b->norms_only || b->row_slot_begin.empty())
    fail(SPG_EINVAL, "plan: B must be a norm-only matrix (spg_matrix_from_leaf_norms, "
                     "spg_bstream)");
  if (shard.level < 0 || shard.level > a->depth || shard.index < 0 ||
      shard.index >= (1 << shard.level))
    fail(SPG_EINVAL, "spamm: shard outside the quadtree");
  auto plan = std::make_unique<spg_plan>();
  plan->ctx = ctx;
  plan->a = a;
  plan->b = b;
  for (auto& x : plan->ev) SPG_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  SPG_CUDA(cudaEventCreate(&plan->t_first));
  SPG_CUDA(cudaEventCreate(&plan->t_last));
  const int64_t LL = static_cast<int64_t>(a->leaf) * a->leaf;
  SPG_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  plan->pl = plan_product(ctx, a_norms ? a_norms : a, b, tau, true, shard, true, a,
                          a->leaf == 32 && super32_enabled());
  SPG_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
  const int64_t n_out = plan->pl.n_out;
  plan->c = external_c ? DevBuf<double>::adopt(external_c, std::max<int64_t>(n_out * LL, 1), ctx)
                       : DevBuf<double>(std::max<int64_t>(n_out * LL, 1), ctx);
  plan->external_c = external_c != nullptr;
  if (n_out) SPG_CUDA(cudaMemsetAsync(plan->c.get(), 0, n_out * LL * sizeof(double), ctx->stream));
  plan->beg = DevBuf<int64_t>(std::max<int64_t>(n_out, 1), ctx);
  plan->end = DevBuf<int64_t>(std::max<int64_t>(n_out, 1), ctx);
  plan->btab = DevBuf<const double*>(std::max<int64_t>(b->n_slots, 1), ctx);
  if (a->leaf == 128 && sub128_enabled() && plan->pl.n_surv) {
    plan->sub = std::make_unique<Sub128>(build_sub128(ctx, plan->pl));
    plan->sub_beg = DevBuf<int64_t>(std::max<int64_t>(plan->sub->n_sub, 1), ctx);
    plan->sub_end = DevBuf<int64_t>(std::max<int64_t>(plan->sub->n_sub, 1), ctx);
  } else if (a->leaf == 32 && super32_enabled() && plan->pl.n_surv) {
    plan->sup = std::make_unique<Super32>(build_super32(ctx, a->depth, plan->pl));
    plan->sb_beg = DevBuf<int64_t>(std::max<int64_t>(plan->sup->n_sb, 1), ctx);
    plan->sb_end = DevBuf<int64_t>(std::max<int64_t>(plan->sup->n_sb, 1), ctx);
  } else {
    plan->order = make_block_order(ctx, plan->pl.out_keys.get(), n_out, n_out);
  }
  SPG_CUDA(cudaEventSynchronize(ctx->ev[3]));
  spg_spamm_stats& st = plan->stats;
  st.survivors = plan->pl.n_surv;
  st.output_blocks = n_out;
  st.flops = 2.0 * static_cast<double>(a->leaf) * a->leaf * a->leaf *
             static_cast<double>(plan->pl.n_surv);
  SPG_CUDA(cudaEventElapsedTime(&st.ms_tasklist, ctx->ev[2], ctx->ev[3]));
  st.candidates = count_candidates(ctx, a, b, shard);
  return plan.release();
}

// B slots [row_slot_begin[r0], row_slot_begin[r1]) at d_panel, enqueued on
// ctx->stream
void plan_accumulate(spg_plan* plan, int32_t r0, int32_t r1, const double* d_panel) {
  spg_context* ctx = plan->ctx;
  const spg_matrix* b = plan->b;
  const int32_t nbp = 1 << b->depth;
  if (plan->finished) fail(SPG_EINVAL, "plan: already finished");
  if (r0 != plan->next_row)
    fail(SPG_EINVAL, "plan: panels must tile the block rows in ascending order (expected row " +
                         std::to_string(plan->next_row) + ")");
  if (r1 <= r0 || r1 > nbp) fail(SPG_EINVAL, "plan: bad panel row range");
  const int64_t lo = b->row_slot_begin[r0], cnt = b->row_slot_begin[r1] - lo;
  if (cnt > 0 && !d_panel) fail(SPG_EINVAL, "plan: panel holds leaves but no buffer was given");
  plan->next_row = r1;
  const int64_t n_out = plan->pl.n_out;
  if (n_out == 0 || cnt == 0) return;
  if (!plan->started) {
    SPG_CUDA(cudaEventRecord(plan->t_first, ctx->stream));
    plan->started = true;
  }
  const int L = b->leaf;
  const int64_t LL = static_cast<int64_t>(L) * L;
  std::pair<cudaEvent_t, cudaEvent_t> pe{};
  SPG_CUDA(cudaEventCreate(&pe.first));
  SPG_CUDA(cudaEventCreate(&pe.second));
  plan->panel_ev.push_back(pe);
  SPG_CUDA(cudaEventRecord(pe.first, ctx->stream));
  // pairs hold B slots; the panel buffer starts at slot lo
  leaf_ptr_kernel<<<grid_for(cnt, 256), 256, 0, ctx->stream>>>(d_panel, cnt, LL,
                                                              plan->btab.get() + lo);
  SPG_CHECK_LAUNCH(ctx);
  if (plan->sup) {
    const Super32& sp = *plan->sup;
    super_panel_ranges<<<grid_for(std::max<int64_t>(sp.n_sb, 1), 256), 256, 0, ctx->stream>>>(
        sp.ek.get(), sp.sb_offset.get(), sp.n_sb, static_cast<uint32_t>(r0),
        static_cast<uint32_t>(r1), plan->sb_beg.get(), plan->sb_end.get());
    SPG_CHECK_LAUNCH(ctx);
    launch_super32(ctx, sp, plan->a->payload, plan->btab.get(), plan->c.get(),
                   plan->sb_beg.get(), plan->sb_end.get(), 1);
  } else if (plan->sub) {
    panel_ranges<<<grid_for(n_out, 256), 256, 0, ctx->stream>>>(
        plan->pl.keys.get(), plan->pl.out_offset.get(), n_out, plan->pl.kbits,
        static_cast<uint32_t>(r0), static_cast<uint32_t>(r1), plan->beg.get(), plan->end.get());
    SPG_CHECK_LAUNCH(ctx);
    sub128_ranges<<<grid_for(4 * n_out, 256), 256, 0, ctx->stream>>>(
        plan->pl.out_offset.get(), plan->beg.get(), plan->end.get(), n_out,
        plan->sub_beg.get(), plan->sub_end.get());
    SPG_CHECK_LAUNCH(ctx);
    launch_sub128(ctx, *plan->sub, plan->a->payload, plan->btab.get(), plan->c.get(),
                  plan->sub_beg.get(), plan->sub_end.get(), 1);
  } else {
    panel_ranges<<<grid_for(n_out, 256), 256, 0, ctx->stream>>>(
        plan->pl.keys.get(), plan->pl.out_offset.get(), n_out, plan->pl.kbits,
        static_cast<uint32_t>(r0), static_cast<uint32_t>(r1), plan->beg.get(), plan->end.get());
    SPG_CHECK_LAUNCH(ctx);
    run_gemm(ctx, L, plan->a->payload, nullptr, plan->pl.pairs.get(), plan->beg.get(), n_out,
             plan->c.get(), ctx->stream, plan->end.get(), 1, plan->btab.get(),
             plan->order.get());
  }
  SPG_CUDA(cudaEventRecord(pe.second, ctx->stream));
}

// Every product at once, B leaf t read from btab[t] (one GEMM launch; the
// leaves may live in other GPUs' memory mapped over NVLink).
void plan_run_table(spg_plan* plan, const double* const* h_table, int64_t n_table) {
  spg_context* ctx = plan->ctx;
  if (plan->finished) fail(SPG_EINVAL, "plan: already finished");
  if (plan->next_row != 0) fail(SPG_EINVAL, "plan: panels already accumulated");
  if (n_table != plan->b->n_slots) fail(SPG_EINVAL, "plan: leaf table size != B leaf count");
  const int32_t nbp = 1 << plan->b->depth;
  plan->next_row = nbp;
  const int64_t n_out = plan->pl.n_out;
  if (n_out == 0) return;
  DevBuf<const double*> d_tab(std::max<int64_t>(n_table, 1), ctx);
  SPG_CUDA(cudaMemcpyAsync(d_tab.get(), h_table, n_table * sizeof(const double*),
                           cudaMemcpyHostToDevice, ctx->stream));
  SPG_CUDA(cudaEventRecord(plan->t_first, ctx->stream));
  plan->started = true;
  if (plan->sup)
    launch_super32(ctx, *plan->sup, plan->a->payload, d_tab.get(), plan->c.get());
  else if (plan->sub)
    launch_sub128(ctx, *plan->sub, plan->a->payload, d_tab.get(), plan->c.get());
  else
    run_gemm(ctx, plan->a->leaf, plan->a->payload, nullptr, plan->pl.pairs.get(),
             plan->pl.out_offset.get(), n_out, plan->c.get(), ctx->stream, nullptr, 0,
             d_tab.get(), plan->order.get());
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));  // the table buffer returns to the pool
}

spg_matrix* plan_finish(spg_plan* plan, uint64_t* keys_out = nullptr) {
  spg_context* ctx = plan->ctx;
  const spg_matrix* a = plan->a;
  const int32_t nb_logical = (a->dimension + a->leaf - 1) / a->leaf;
  if (plan->finished) fail(SPG_EINVAL, "plan: already finished");
  if (plan->next_row < nb_logical)
    fail(SPG_EINVAL, "plan: panels cover block rows [0, " + std::to_string(plan->next_row) +
                         ") only");
  plan->finished = true;
  SPG_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
  SPG_CUDA(cudaEventRecord(plan->t_last, ctx->stream));
  plan->pl.pairs.reset();
  plan->pl.out_offset.reset();
  plan->pl.keys.reset();
  plan->beg.reset();
  plan->end.reset();
  spg_matrix* c = nullptr;
  if (plan->external_c) {  // blocks already in place: hand their keys over
    if (!keys_out) fail(SPG_EINTERNAL, "plan: external output without a key array");
    if (plan->pl.n_out)
      SPG_CUDA(cudaMemcpyAsync(keys_out, plan->pl.out_keys.get(),
                               plan->pl.n_out * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                               ctx->stream));
    plan->c.release();
  } else {
    c = matrix_from_morton_blocks(ctx, a->dimension, a->leaf, plan->pl.n_out,
                                  plan->pl.out_keys.release(), plan->c.release());
  }
  SPG_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
  SPG_CUDA(cudaEventSynchronize(ctx->ev[5]));
  SPG_CUDA(cudaEventElapsedTime(&plan->stats.ms_finalize, ctx->ev[4], ctx->ev[5]));
  if (!plan->panel_ev.empty()) {  // panels: the sum of the panel launches' kernel time
    float sum = 0.0f;
    for (auto& pe : plan->panel_ev) {
      float ms = 0.0f;
      SPG_CUDA(cudaEventElapsedTime(&ms, pe.first, pe.second));
      sum += ms;
    }
    plan->stats.ms_gemm = sum;
  } else if (plan->started) {  // one table-addressed launch
    SPG_CUDA(cudaEventElapsedTime(&plan->stats.ms_gemm, plan->t_first, plan->t_last));
  }
  return c;
}

// B in host memory (spg_bstream): panels copied into two device buffers on
// the copy stream, panel q+1 in flight while panel q's GEMM runs.
spg_matrix* spamm_streamed_device(spg_context* ctx, const spg_matrix* a, const spg_bstream* bs,
                                  double tau, spg_spamm_stats* stats) {
  std::unique_ptr<spg_plan> plan(plan_create(ctx, a, bs->norms, tau, Shard{}));
  const int64_t LL = static_cast<int64_t>(a->leaf) * a->leaf;
  SPG_CUDA(cudaEventRecord(ctx->ev[6], ctx->stream));
  const int n_panels = static_cast<int>(bs->panel_row.size()) - 1;
  if (plan->pl.n_out == 0) {
    plan->next_row = bs->panel_row.back();
  } else {
    const int64_t cap = bs->max_panel_leaves;
    DevBuf<double> buf[2] = {DevBuf<double>(cap * LL, ctx), DevBuf<double>(cap * LL, ctx)};
    EventSet ev;  // e[0..1]: panel in buffer i copied; e[2..3]: buffer i free again
    // the pool hands out blocks in ctx->stream order: the copy stream starts
    // after everything queued so far
    SPG_CUDA(cudaEventRecord(ev.e[2], ctx->stream));
    SPG_CUDA(cudaEventRecord(ev.e[3], ctx->stream));
    std::vector<int> live;
    for (int p = 0; p < n_panels; ++p)
      if (bs->panel_leaf[p + 1] > bs->panel_leaf[p]) live.push_back(p);
    auto issue_copy = [&](size_t q) {
      const int p = live[q], i = static_cast<int>(q & 1);
      const int64_t lo = bs->panel_leaf[p], cnt = bs->panel_leaf[p + 1] - lo;
      SPG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ev.e[2 + i], 0));
      SPG_CUDA(cudaMemcpyAsync(buf[i].get(), bs->host_payload + lo * LL,
                               cnt * LL * sizeof(double), cudaMemcpyHostToDevice,
                               ctx->copy_stream));
      SPG_CUDA(cudaEventRecord(ev.e[i], ctx->copy_stream));
    };
    if (!live.empty()) issue_copy(0);
    size_t q = 0;
    for (int p = 0; p < n_panels; ++p) {
      const bool has = q < live.size() && live[q] == p;
      if (!has) {  // no leaves in these rows
        plan_accumulate(plan.get(), bs->panel_row[p], bs->panel_row[p + 1], nullptr);
        continue;
      }
      if (q + 1 < live.size()) issue_copy(q + 1);
      const int i = static_cast<int>(q & 1);
      SPG_CUDA(cudaStreamWaitEvent(ctx->stream, ev.e[i], 0));
      plan_accumulate(plan.get(), bs->panel_row[p], bs->panel_row[p + 1], buf[i].get());
      SPG_CUDA(cudaEventRecord(ev.e[2 + i], ctx->stream));
      ++q;
    }
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  SPG_CUDA(cudaEventRecord(ctx->ev[7], ctx->stream));
  spg_matrix* c = plan_finish(plan.get());
  if (stats) {
    *stats = plan->stats;
    SPG_CUDA(cudaEventElapsedTime(&stats->ms_gemm, ctx->ev[6], ctx->ev[7]));
  }
  return c;
}


// A (shard of a) product whose B arrives in panels from the caller's fetch
// callback (host memory, NCCL broadcast by the owning GPU, a generator ...),
// two panels in flight, in 2^c row chunks when the task list would exceed
// the task budget; each chunk receives every panel again.  The chunks' rows
// are disjoint, so their C's merge leaf for leaf; bitwise the resident product.
// The context lock is released while the callback runs (it may call back in).
spg_matrix* spamm_panels_device(spg_context* ctx, std::unique_lock<std::mutex>& lock,
                                const spg_matrix* a, const spg_matrix* a_norms,
                                const spg_matrix* b, double tau, Shard sh, int32_t panel_rows,
                                int32_t owner_rows, spg_panel_fetch_fn fetch, void* user,
                                spg_spamm_stats* stats) {
  if (!b->norms_only || b->row_slot_begin.empty())
    fail(SPG_EINVAL, "panels: B must be a norm-only matrix (spg_matrix_from_leaf_norms)");
  if (panel_rows < 1) fail(SPG_EINVAL, "panels: panel_rows must be positive");
  const int64_t LL = static_cast<int64_t>(a->leaf) * a->leaf;
  const int32_t nb = (a->dimension + a->leaf - 1) / a->leaf;
  // panels tile [0, nb) and never cross an owner boundary
  std::vector<std::pair<int32_t, int32_t>> panels;
  for (int32_t r = 0; r < nb;) {
    int32_t r1 = std::min(r + panel_rows, nb);
    if (owner_rows > 0) r1 = std::min(r1, (r / owner_rows + 1) * owner_rows);
    panels.push_back({r, r1});
    r = r1;
  }
  const auto& rs = b->row_slot_begin;
  int64_t cap = 0;
  for (const auto& pr : panels) cap = std::max(cap, rs[pr.second] - rs[pr.first]);
  const spg_matrix* an = a_norms ? a_norms : a;
  // super blocks pair rows 2I, 2I+1: a chunk keeps >= 2 rows for them
  const bool super32 = a->leaf == 32 && super32_enabled();
  // reserved before the task lists are sized: the output's bound and the two
  // panel buffers allocated below
  const int c = chunk_bits(ctx, an, b, sh, a->depth - sh.level - (super32 ? 1 : 0), super32,
                           output_bytes_bound(a, sh) +
                               2 * std::max<int64_t>(cap * LL, 1) * int64_t(sizeof(double)));
  std::vector<spg_matrix*> parts;
  struct Parts {
    std::vector<spg_matrix*>& v;
    ~Parts() {
      for (spg_matrix* m : v) matrix_destroy(m);
    }
  } guard{parts};
  // Several row chunks: every chunk's blocks go straight into one payload
  // (sized by a pass over the chunks' output counts), so the product never
  // holds C twice -- a config-4 rank keeps 52 GB of A rows and 69 GB of C.
  const int nch = 1 << c;
  auto sub = [&](int q) { return Shard{sh.level + c, (sh.index << c) + q}; };
  std::vector<int64_t> n_out_q(static_cast<size_t>(nch), 0);
  int64_t total_out = 0;
  double* c_payload = nullptr;
  uint64_t* c_keys = nullptr;
  struct InPlace {
    spg_context* ctx;
    double*& pay;
    uint64_t*& keys;
    ~InPlace() {
      if (pay) dev_free(pay, ctx);
      if (keys) dev_free(keys, ctx);
    }
  } in_place{ctx, c_payload, c_keys};
  if (nch > 1) {
    for (int q = 0; q < nch; ++q) {
      // sizing only: with the dense walk, for_super stops after the count pass
      const Plan pl = plan_product(ctx, an, b, tau, true, sub(q), false, a, true);
      n_out_q[q] = pl.n_out;
      total_out += pl.n_out;
    }
    c_payload = dev_alloc<double>(std::max<int64_t>(total_out * LL, 1), ctx);
    c_keys = dev_alloc<uint64_t>(std::max<int64_t>(total_out, 1), ctx);
  }
  int64_t out_off = 0;
  spg_spamm_stats total{};
  DevBuf<double> buf[2] = {DevBuf<double>(std::max<int64_t>(cap * LL, 1), ctx),
                           DevBuf<double>(std::max<int64_t>(cap * LL, 1), ctx)};
  cudaStream_t fs[2] = {ctx->copy_stream, ctx->h2d_stream};
  EventSet ev;  // e[0..1]: buffer i filled; e[2..3]: buffer i free again
  for (int q = 0; q < nch; ++q) {
    std::unique_ptr<spg_plan> plan(plan_create(
        ctx, a, b, tau, sub(q), a_norms, nch > 1 ? c_payload + out_off * LL : nullptr));
    if (nch > 1 && plan->pl.n_out != n_out_q[q])
      fail(SPG_EINTERNAL, "panels: chunk size changed");
    SPG_CUDA(cudaEventRecord(ev.e[2], ctx->stream));
    SPG_CUDA(cudaEventRecord(ev.e[3], ctx->stream));
    std::vector<size_t> live;
    for (size_t p = 0; p < panels.size(); ++p)
      if (plan->pl.n_out && rs[panels[p].second] > rs[panels[p].first]) live.push_back(p);
    auto issue = [&](size_t k) {
      const size_t p = live[k];
      const int i = static_cast<int>(k & 1);
      SPG_CUDA(cudaStreamWaitEvent(fs[i], ev.e[2 + i], 0));
      const int64_t cnt = rs[panels[p].second] - rs[panels[p].first];
      lock.unlock();
      const int rc = fetch(user, panels[p].first, panels[p].second, buf[i].get(), cnt, fs[i]);
      lock.lock();
      if (rc != 0) fail(SPG_EINVAL, "panels: fetch callback failed for block rows [" +
                                        std::to_string(panels[p].first) + ", " +
                                        std::to_string(panels[p].second) + ")");
      SPG_CUDA(cudaEventRecord(ev.e[i], fs[i]));
    };
    if (!live.empty()) issue(0);
    size_t k = 0;
    for (size_t p = 0; p < panels.size(); ++p) {
      if (k < live.size() && live[k] == p) {
        if (k + 1 < live.size()) issue(k + 1);
        const int i = static_cast<int>(k & 1);
        SPG_CUDA(cudaStreamWaitEvent(ctx->stream, ev.e[i], 0));
        plan_accumulate(plan.get(), panels[p].first, panels[p].second, buf[i].get());
        SPG_CUDA(cudaEventRecord(ev.e[2 + i], ctx->stream));
        ++k;
      } else {
        plan_accumulate(plan.get(), panels[p].first, panels[p].second, nullptr);
      }
    }
    if (nch > 1) {
      plan_finish(plan.get(), c_keys + out_off);
      out_off += n_out_q[q];
    } else {
      parts.push_back(plan_finish(plan.get()));
    }
    const spg_spamm_stats& st = plan->stats;
    total.candidates += st.candidates;
    total.survivors += st.survivors;
    total.output_blocks += st.output_blocks;
    total.flops += st.flops;
    total.ms_tasklist += st.ms_tasklist;
    total.ms_gemm += st.ms_gemm;
    total.ms_finalize += st.ms_finalize;
  }
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  spg_matrix* out = nullptr;
  if (nch == 1) {
    out = parts[0];
    parts.clear();
  } else {
    // chunk keys are not globally in Morton order: the matrix scatters them
    double* pay = c_payload;
    uint64_t* keys = c_keys;
    c_payload = nullptr;  // owned by the matrix from here on
    c_keys = nullptr;
    out = matrix_from_morton_blocks(ctx, a->dimension, a->leaf, total_out, keys, pay);
  }
  if (stats) *stats = total;
  return out;
}

namespace {
using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}
}  // namespace

// spamm_with_error_control (error_control.cpp:203-220) with the context lock
// held: cse -> select (first k with bound < delta) -> spamm_multiply.
spg_matrix* controlled_product(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                               double delta, const double* taus, int n_taus, double* bounds,
                               spg_controlled_stats* stats) {
  std::vector<double> local(static_cast<size_t>(n_taus));
  double* bv = bounds ? bounds : local.data();
  float cse_ms = 0.0f;
  const auto t0 = Clock::now();
  cse_device(ctx, a, b, taus, n_taus, bv, &cse_ms);
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
  spg_matrix* c = spamm_device(ctx, a, b, tau, true, stats ? &ss : nullptr);
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

}  // namespace spg

using namespace spg;

extern "C" {

int spg_spamm(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
              spg_matrix** c, spg_spamm_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  CtxGuard g(ctx);
  *c = spamm_device(ctx, a, b, tau, true, stats);
  SPG_API_END
}

int spg_multiply_exact(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                       spg_matrix** c, spg_spamm_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  CtxGuard g(ctx);
  *c = spamm_device(ctx, a, b, 0.0, false, stats);
  SPG_API_END
}

int spg_spamm_with_error_control(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                                 double delta, const double* taus, int32_t n_taus,
                                 spg_matrix** c, double* bounds, spg_controlled_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  // error_control.cpp:205
  if (!(delta > 0.0)) fail(SPG_EINVAL, "spamm_with_error_control: delta must be positive");
  int rc = spg_tolerance_grid_check(taus, n_taus);
  if (rc != SPG_OK) return rc;
  CtxGuard g(ctx);
  *c = controlled_product(ctx, a, b, delta, taus, n_taus, bounds, stats);
  SPG_API_END
}

int spg_spamm_shard(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                    int32_t level, int32_t shard, spg_matrix** c, spg_spamm_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  CtxGuard g(ctx);
  *c = spamm_device(ctx, a, b, tau, true, stats, Shard{level, shard});
  SPG_API_END
}

int spg_spamm_with_error_control_to_host(spg_context* ctx, const spg_matrix* a,
                                         const spg_matrix* b, double delta, const double* taus,
                                         int32_t n_taus, int64_t capacity, int32_t* c_rows,
                                         int32_t* c_cols, double* c_payload, double* c_norms,
                                         int64_t* c_count, double* bounds,
                                         spg_controlled_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !c_payload || !c_norms || !c_count) fail(SPG_EINVAL, "null argument");
  if (!(delta > 0.0)) fail(SPG_EINVAL, "spamm_with_error_control: delta must be positive");
  int rc = spg_tolerance_grid_check(taus, n_taus);
  if (rc != SPG_OK) return rc;
  CtxGuard g(ctx);
  std::vector<double> local(static_cast<size_t>(n_taus));
  double* bv = bounds ? bounds : local.data();
  float cse_ms = 0.0f;
  const auto t0 = Clock::now();
  cse_device(ctx, a, b, taus, n_taus, bv, &cse_ms);
  const double cse_seconds = seconds_since(t0);
  int32_t k = -1;
  for (int32_t i = 0; i < n_taus; ++i)
    if (bv[i] < delta) {
      k = i;
      break;
    }
  const double tau = k >= 0 ? taus[k] : 0.0;
  HostOut out;
  out.capacity = capacity;
  out.rows = c_rows;
  out.cols = c_cols;
  out.payload = c_payload;
  out.norms = c_norms;
  spg_spamm_stats ss{};
  const auto t1 = Clock::now();
  spamm_device(ctx, a, b, tau, true, stats ? &ss : nullptr, Shard{}, &out);
  *c_count = out.count;
  if (stats) {
    stats->tau = tau;
    stats->tau_index = k;
    stats->bound = k >= 0 ? bv[k] : 0.0;
    stats->cse_seconds = cse_seconds;
    stats->spamm_seconds = seconds_since(t1);
    stats->ms_cse = cse_ms;
    stats->spamm = ss;
  }
  SPG_API_END
}

namespace spg {
namespace {
__device__ __forceinline__ uint64_t digest_mix(uint64_t z) {  // SplitMix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// sum over the task list of mix64(i << 42 | k << 21 | j), mod 2^64 (order-free)
__global__ void survivor_digest_kernel(const uint64_t* __restrict__ keys, int64_t n, int kbits,
                                       unsigned long long* __restrict__ sum) {
  unsigned long long local = 0;
  const uint64_t kmask = (uint64_t(1) << kbits) - 1;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[t], ij = key >> kbits;
    const uint64_t i = morton_row(ij), j = morton_col(ij), k = key & kmask;
    local += digest_mix((i << 42) | (k << 21) | j);
  }
  for (int off = 16; off; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(sum, local);
}
}  // namespace
}  // namespace spg

int spg_survivor_digest(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                        int32_t level, int32_t shard, int64_t* count, uint64_t* digest) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !count || !digest) fail(SPG_EINVAL, "null argument");
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "multiply: dimension or leaf size mismatch");
  if (tau < 0.0) fail(SPG_EINVAL, "spamm: tau must be nonnegative");
  if (level < 0 || level > a->depth || shard < 0 || shard >= (1 << level))
    fail(SPG_EINVAL, "shard outside the tree");
  CtxGuard g(ctx);
  TaskList tl = build_tasklist<KeepRule::kSkip>(ctx, a, b, tau, Shard{level, shard});
  DevBuf<unsigned long long> sum(1, ctx);
  SPG_CUDA(cudaMemsetAsync(sum.get(), 0, sizeof(unsigned long long), ctx->stream));
  if (tl.n_surv) {
    survivor_digest_kernel<<<grid_for(tl.n_surv, 256, int64_t(ctx->sm_count) * 8), 256, 0,
                             ctx->stream>>>(tl.keys.get(), tl.n_surv, tl.kbits, sum.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  unsigned long long h = 0;
  SPG_CUDA(cudaMemcpyAsync(&h, sum.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  *count = tl.n_surv;
  *digest = h;
  SPG_API_END
}

int spg_parity_audit(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                     int32_t ulps, int64_t* near_ties, int64_t* candidates) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !near_ties || !candidates) fail(SPG_EINVAL, "null argument");
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "multiply: dimension or leaf size mismatch");
  CtxGuard g(ctx);
  *near_ties = 0;
  *candidates = 0;
  const int d = a->depth;
  const double window = ulps * (std::nextafter(tau, 2.0 * tau + 1.0) - tau);
  if (d == 0) {
    double na = -1, nb = -1;
    SPG_CUDA(cudaMemcpy(&na, a->pyramid, 8, cudaMemcpyDeviceToHost));
    SPG_CUDA(cudaMemcpy(&nb, b->pyramid, 8, cudaMemcpyDeviceToHost));
    if (na >= 0 && nb >= 0) {
      *candidates = 1;
      volatile double p = na * nb;
      *near_ties = std::fabs(p - tau) <= window;
    }
    return SPG_OK;
  }
  TripleList cur = root_list<KeepRule::kExact>(ctx, a, b, 0.0);
  for (int l = 0; l < d - 1 && cur.n > 0; ++l) {
    TripleList next = expand_level<KeepRule::kExact>(ctx, cur, a->pyramid + level_offset(l + 1),
                                                     b->pyramid + level_offset(l + 1), 0.0);
    cur = std::move(next);
  }
  DevBuf<unsigned long long> cnt(2, ctx);
  SPG_CUDA(cudaMemsetAsync(cnt.get(), 0, 16, ctx->stream));
  if (cur.n) {
    near_tie_count<<<grid_for(cur.n, 256), 256, 0, ctx->stream>>>(
        cur.I.get(), cur.K.get(), cur.J.get(), cur.n, a->pyramid + level_offset(d),
        b->pyramid + level_offset(d), tau, window, cnt.get(), cnt.get() + 1);
    SPG_CHECK_LAUNCH(ctx);
  }
  unsigned long long h[2] = {0, 0};
  SPG_CUDA(cudaMemcpyAsync(h, cnt.get(), 16, cudaMemcpyDeviceToHost, ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  *near_ties = static_cast<int64_t>(h[0]);
  *candidates = static_cast<int64_t>(h[1]);
  SPG_API_END
}

int spg_survivors(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                  int64_t* count, int32_t* triples, int64_t capacity) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !count) fail(SPG_EINVAL, "null argument");
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "multiply: dimension or leaf size mismatch");
  if (tau < 0.0) fail(SPG_EINVAL, "spamm: tau must be nonnegative");
  CtxGuard g(ctx);
  TaskList tl = build_tasklist<KeepRule::kSkip>(ctx, a, b, tau, Shard{});
  *count = tl.n_surv;
  if (triples && capacity > 0 && tl.n_surv > 0) {
    const int64_t n = std::min(capacity, tl.n_surv);
    std::vector<uint64_t> keys(static_cast<size_t>(n));
    SPG_CUDA(cudaMemcpyAsync(keys.data(), tl.keys.get(), n * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint64_t kmask = (uint64_t(1) << tl.kbits) - 1;
    for (int64_t t = 0; t < n; ++t) {
      const uint64_t ij = keys[t] >> tl.kbits;
      triples[3 * t + 0] = static_cast<int32_t>(morton_row(ij));
      triples[3 * t + 1] = static_cast<int32_t>(keys[t] & kmask);
      triples[3 * t + 2] = static_cast<int32_t>(morton_col(ij));
    }
  }
  SPG_API_END
}

// ---- panel plans (B arriving in block-row panels) -------------------------
namespace {
// make ctx->stream wait for `foreign` (the caller's stream) and, after the
// enqueued work, `foreign` wait for ctx->stream: stream-ordered hand-off
struct ForeignOrder {
  spg_context* ctx;
  cudaStream_t foreign;
  cudaEvent_t ev;
  ForeignOrder(spg_context* c, void* s, cudaEvent_t e)
      : ctx(c), foreign(static_cast<cudaStream_t>(s)), ev(e) {
    if (foreign && foreign != ctx->stream) {
      SPG_CUDA(cudaEventRecord(ev, foreign));
      SPG_CUDA(cudaStreamWaitEvent(ctx->stream, ev, 0));
    }
  }
  void done() {
    if (foreign && foreign != ctx->stream) {
      SPG_CUDA(cudaEventRecord(ev, ctx->stream));
      SPG_CUDA(cudaStreamWaitEvent(foreign, ev, 0));
    }
  }
};
}  // namespace

int spg_plan_create(spg_context* ctx, const spg_matrix* a, const spg_matrix* a_norms,
                    const spg_matrix* b, double tau, int32_t level, int32_t shard,
                    spg_plan** plan) {
  SPG_API_BEGIN
  if (!ctx || !a || !b || !plan) fail(SPG_EINVAL, "null argument");
  *plan = nullptr;
  if (a->ctx != ctx || b->ctx != ctx || (a_norms && a_norms->ctx != ctx))
    fail(SPG_EINVAL, "operands belong to another context");
  CtxGuard g(ctx);
  *plan = plan_create(ctx, a, b, tau, Shard{level, shard}, a_norms);
  SPG_API_END
}

int spg_plan_panel_slots(const spg_plan* plan, int32_t row_begin, int32_t row_end,
                         int64_t* slot_begin, int64_t* count) {
  SPG_API_BEGIN
  if (!plan) fail(SPG_EINVAL, "null argument");
  const auto& rs = plan->b->row_slot_begin;
  const int32_t nbp = static_cast<int32_t>(rs.size()) - 1;
  if (row_begin < 0 || row_end < row_begin || row_end > nbp)
    fail(SPG_EINVAL, "plan: bad panel row range");
  if (slot_begin) *slot_begin = rs[row_begin];
  if (count) *count = rs[row_end] - rs[row_begin];
  SPG_API_END
}

int spg_plan_accumulate(spg_plan* plan, int32_t row_begin, int32_t row_end,
                        const double* d_panel, void* stream) {
  SPG_API_BEGIN
  if (!plan) fail(SPG_EINVAL, "null argument");
  CtxGuard g(plan->ctx);
  ForeignOrder fo(plan->ctx, stream, plan->ev[0]);
  plan_accumulate(plan, row_begin, row_end, d_panel);
  fo.done();
  SPG_API_END
}

int spg_plan_finish(spg_plan* plan, spg_matrix** c, spg_spamm_stats* stats) {
  SPG_API_BEGIN
  if (!plan || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  CtxGuard g(plan->ctx);
  *c = plan_finish(plan);
  if (stats) *stats = plan->stats;
  SPG_API_END
}

int spg_plan_run_table(spg_plan* plan, int32_t n_owners, const double* const* owner_base,
                       const int32_t* slot_owner, const int32_t* slot_local, void* stream) {
  SPG_API_BEGIN
  if (!plan || (n_owners > 0 && !owner_base)) fail(SPG_EINVAL, "null argument");
  const int64_t n = plan->b->n_slots;
  if (n > 0 && (!slot_owner || !slot_local)) fail(SPG_EINVAL, "null argument");
  const int64_t LL = static_cast<int64_t>(plan->b->leaf) * plan->b->leaf;
  std::vector<const double*> tab(static_cast<size_t>(n));
  for (int64_t t = 0; t < n; ++t) {
    const int32_t o = slot_owner[t];
    if (o < 0 || o >= n_owners || slot_local[t] < 0)
      fail(SPG_EINVAL, "plan: leaf table entry outside the owners");
    tab[t] = owner_base[o] + static_cast<int64_t>(slot_local[t]) * LL;
  }
  CtxGuard g(plan->ctx);
  ForeignOrder fo(plan->ctx, stream, plan->ev[0]);
  plan_run_table(plan, tab.data(), n);
  fo.done();
  SPG_API_END
}

int spg_spamm_panels(spg_context* ctx, const spg_matrix* a, const spg_matrix* a_norms,
                     const spg_matrix* b_norms, double tau, int32_t level, int32_t shard,
                     int32_t panel_rows, int32_t owner_rows, spg_panel_fetch_fn fetch,
                     void* user, spg_matrix** c, spg_spamm_stats* stats) {
  SPG_API_BEGIN
  if (!ctx || !a || !b_norms || !fetch || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  if (a->ctx != ctx || b_norms->ctx != ctx || (a_norms && a_norms->ctx != ctx))
    fail(SPG_EINVAL, "operands belong to another context");
  if (level < 0 || level > a->depth || shard < 0 || shard >= (1 << level))
    fail(SPG_EINVAL, "spamm: shard outside the quadtree");
  std::unique_lock<std::mutex> lock(ctx->mu);
  SPG_CUDA(cudaSetDevice(ctx->device));
  *c = spamm_panels_device(ctx, lock, a, a_norms, b_norms, tau, Shard{level, shard}, panel_rows,
                           owner_rows, fetch, user, stats);
  SPG_API_END
}

void spg_plan_free(spg_plan* plan) {
  if (!plan) return;
  try {
    CtxGuard g(plan->ctx);
    delete plan;
  } catch (...) {
  }
}

}  // extern "C"
