// norms.cu -- K1 leaf Frobenius norms and K2 level-norm pyramid.
//
// Bit-exactness contract: a leaf norm is the reference's
// block_norm (node_ops.hpp:24-28): s = 0; for t in storage order:
// s = fl(s + fl(b[t]*b[t])); norm = fl(sqrt(s)).  Inner norms are
// combine_child_norms (node_ops.hpp:30-36): children 0..3, null skipped.
// Every multiply/add below is an explicit round-to-nearest intrinsic, so no
// FMA contraction can change the bits, and the summation order is sequential
// per leaf (a tree/shuffle reduction would change 91.5% of leaf norms, F3).
//
// K1 layout: one warp owns 32 leaves (one lane per leaf).  Each 32-element
// chunk is loaded coalesced -- for every leaf the warp reads 32 consecutive
// doubles (256 B) -- squared by the loading lane (the square is elementwise,
// so who computes it does not matter), transposed through shared memory, and
// each lane then adds its own leaf's 32 squares in storage order.  HBM-bound:
// 8 B read per element; the dependent DADD chain is hidden by 32 leaves per
// warp and many warps per SM.
#include "common.cuh"

namespace spg {

namespace {

constexpr int kNormWarps = 4;

template <bool kCheckPadding>
__global__ void __launch_bounds__(kNormWarps * 32)
    leaf_norm_kernel(const double* __restrict__ payload, int64_t n_slots, int leaf,
                     int32_t dimension, int32_t nb_logical, const int32_t* __restrict__ rows,
                     const int32_t* __restrict__ cols, double* __restrict__ norms,
                     uint8_t* __restrict__ nonzero, int* __restrict__ bad_padding) {
  __shared__ double sq[kNormWarps][32][33];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t base = (static_cast<int64_t>(blockIdx.x) * kNormWarps + warp) * 32;
  if (base >= n_slots) return;
  const int nleaf = (n_slots - base < 32) ? static_cast<int>(n_slots - base) : 32;
  const int64_t elems = static_cast<int64_t>(leaf) * leaf;

  // Padding bookkeeping: which leaves sit on the last logical block row/col.
  int32_t my_r = 0, my_c = 0;
  if (kCheckPadding && lane < nleaf) {
    my_r = rows[base + lane];
    my_c = cols[base + lane];
  }

  // Software-pipelined: the next chunk's 32 loads are in flight while this
  // chunk's squares are summed; nonzero flags accumulate per lane and are
  // OR-reduced once at the end (no per-element ballot).
  double sum = 0.0;
  unsigned my_nz = 0;  // bit j: this lane saw a nonzero entry of leaf j
  double cur[32];
  auto load_chunk = [&](int64_t e0) {
    const int cnt = (elems - e0 < 32) ? static_cast<int>(elems - e0) : 32;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      cur[j] = (j < nleaf && lane < cnt) ? __ldg(payload + (base + j) * elems + e0 + lane) : 0.0;
  };
  load_chunk(0);
  for (int64_t e0 = 0; e0 < elems; e0 += 32) {
    const int cnt = (elems - e0 < 32) ? static_cast<int>(elems - e0) : 32;
    const int64_t e = e0 + lane;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double v = cur[j];
      my_nz |= static_cast<unsigned>(v != 0.0) << j;
      if (kCheckPadding) {
        const int32_t r = __shfl_sync(0xffffffffu, my_r, j);
        const int32_t c = __shfl_sync(0xffffffffu, my_c, j);
        if (v != 0.0) {
          const int64_t i_in = e % leaf, j_in = e / leaf;
          if (static_cast<int64_t>(r) * leaf + i_in >= dimension ||
              static_cast<int64_t>(c) * leaf + j_in >= dimension)
            atomicOr(bad_padding, 1);
        }
      }
      sq[warp][j][lane] = __dmul_rn(v, v);
    }
    __syncwarp();
    if (e0 + 32 < elems) load_chunk(e0 + 32);
    if (lane < nleaf) {
      const double* row = sq[warp][lane];
      for (int i = 0; i < cnt; ++i) sum = __dadd_rn(sum, row[i]);
    }
    __syncwarp();
  }
  const unsigned nz_mask = __reduce_or_sync(0xffffffffu, my_nz);
  if (lane < nleaf) {
    norms[base + lane] = __dsqrt_rn(sum);
    nonzero[base + lane] = (nz_mask >> lane) & 1u;
  }
  (void)nb_logical;
}

// Level `depth` of the pyramid: leaf norm, or -1 for null; all-zero leaves
// collapse to null (node_ops.hpp:40-53) and are removed from grid_slot.
__global__ void pyramid_leaf_level(int32_t* __restrict__ grid_slot, int64_t count,
                                   const double* __restrict__ slot_norms,
                                   const uint8_t* __restrict__ slot_nonzero,
                                   double* __restrict__ level) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= count) return;
  const int32_t s = grid_slot[p];
  double v = -1.0;
  if (s >= 0) {
    if (slot_nonzero[s]) {
      v = slot_norms[s];
    } else {
      grid_slot[p] = -1;
    }
  }
  level[p] = v;
}

// combine_child_norms (node_ops.hpp:30-36) for every node of one level.
__global__ void pyramid_inner_level(const double* __restrict__ child_level,
                                    double* __restrict__ level, int64_t count) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (m >= count) return;
  const double ch[4] = {child_level[4 * m], child_level[4 * m + 1], child_level[4 * m + 2],
                        child_level[4 * m + 3]};
  double s = 0.0;
  bool any = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!(ch[q] < 0.0)) {  // non-null (a NaN norm is non-null too)
      any = true;
      s = __dadd_rn(s, __dmul_rn(ch[q], ch[q]));
    }
  }
  level[m] = any ? __dsqrt_rn(s) : -1.0;
}

}  // namespace

void leaf_norms(spg_context* ctx, const double* payload, int64_t n_slots, int leaf,
                int32_t dimension, int32_t nb_logical, const int32_t* slot_rows,
                const int32_t* slot_cols, double* norms, uint8_t* nonzero, int* bad_padding,
                cudaStream_t st) {
  if (n_slots == 0) return;
  if (!st) st = ctx->stream;
  const int64_t warps = (n_slots + 31) / 32;
  const unsigned grid = grid_for(warps, kNormWarps);
  const bool check = slot_rows != nullptr && (dimension % leaf) != 0;
  if (check)
    leaf_norm_kernel<true><<<grid, kNormWarps * 32, 0, st>>>(
        payload, n_slots, leaf, dimension, nb_logical, slot_rows, slot_cols, norms, nonzero,
        bad_padding);
  else
    leaf_norm_kernel<false><<<grid, kNormWarps * 32, 0, st>>>(
        payload, n_slots, leaf, dimension, nb_logical, slot_rows, slot_cols, norms, nonzero,
        bad_padding);
  SPG_CHECK_LAUNCH(ctx);
}

void build_pyramid(spg_context* ctx, spg_matrix* m, const double* slot_norms,
                   const uint8_t* slot_nonzero) {
  const int d = m->depth;
  const int64_t leaves = int64_t(1) << (2 * d);
  pyramid_leaf_level<<<grid_for(leaves, 256), 256, 0, ctx->stream>>>(
      m->grid_slot, leaves, slot_norms, slot_nonzero, m->pyramid + level_offset(d));
  SPG_CHECK_LAUNCH(ctx);
  for (int l = d - 1; l >= 0; --l) {
    const int64_t count = int64_t(1) << (2 * l);
    pyramid_inner_level<<<grid_for(count, 256), 256, 0, ctx->stream>>>(
        m->pyramid + level_offset(l + 1), m->pyramid + level_offset(l), count);
    SPG_CHECK_LAUNCH(ctx);
  }
}

}  // namespace spg
