// gemm.cuh -- K5: batched FP64 leaf GEMM on the DMMA tensor pipe (sm_100a).
//
// C(i,j) = sum over surviving k of A(i,k) * B(k,j), one output leaf block per
// CTA, accumulated in registers in ascending k (the reference sums the same
// products as a binary tree over k with unfused multiply-add, quadtree.cpp:
// 24-49; P5 allows 1e-12 relative Frobenius for this reordering).
//
// sm_100a has no FP64 tcgen05/UMMA kind; the FP64 tensor path is warp-level
// mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4, measured at
// 37.1 TFLOP/s over 148 SMs (profiles/r01_fp64_peak.txt).
//
// Data movement: each pipeline stage holds a KC-wide k-chunk of one surviving
// product -- A(:, kc:kc+KC) (contiguous in the column-major leaf) and
// B(kc:kc+KC, :) (KC doubles per column) -- copied with cp.async 16-byte
// chunks into padded shared memory.  Fragment loads are 64-bit (LDS.64, two
// 128-byte shared wavefronts minimum per warp).  Column strides == 4 (mod 16
// doubles) for both operands plus the tile permutation perm8(g) of the eight
// rows (A) / columns (B) a fragment touches make each 16-lane phase of a
// fragment load hit 16 distinct 8-byte bank pairs -- under both the
// lanes-0-15/16-31 and the {0-7,16-23}/{8-15,24-31} phase splits -- so the
// loads run at the 2-wavefront minimum (round 1 measured 4 with stride 72).
// The permutation is undone in the epilogue (C rows/cols use the same perm8).
#pragma once

#include "common.cuh"

namespace spg {

__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ constexpr int perm8(int g) { return g ^ ((g >> 2) << 1); }

template <int L, int KC, int WM, int WN, int NSTAGE>
struct DmmaGemmCfg {
  static constexpr int kWarps = (L / WM) * (L / WN);
  static constexpr int kThreads = 32 * kWarps;
  static constexpr int AS = L + 4;   // == 4 (mod 16)
  static constexpr int BS = KC + 4;  // == 4 (mod 16)
  static constexpr int A_STAGE = KC * AS;
  static constexpr int B_STAGE = L * BS;
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int CHUNKS = L / KC;
  static constexpr int WARPS_M = L / WM;
  static constexpr int TM = WM / 8;
  static constexpr int TN = WN / 8;
  static constexpr size_t kSmemBytes = sizeof(double) * NSTAGE * STAGE;
  static_assert(kWarps == 1 || kWarps == 2 || kWarps == 4 || kWarps == 8 || kWarps == 16,
                "1-16 warps per CTA");
  static_assert(AS % 16 == 4 && BS % 16 == 4, "bank-conflict-free strides");
  static_assert(L % KC == 0 && KC % 4 == 0, "k chunking");
};

// kTable: B leaf pr.y lives at btab[pr.y] (leaves spread over several
// allocations, e.g. peer GPUs' memory mapped over NVLink, or a matrix's own
// leaf table: the table form also measured 3.6 % faster on cfg2 -- the loaded
// pointer spares the per-copy 64-bit address rematerialisation of B + y L^2).
// LD > L: the operands and outputs are L x L sub-blocks of LD x LD leaves
// (column-major, leading dimension LD).  Pair (ax, by) then names A sub-block
// (ax/4, k-half (ax/2)&1, row half ax&1) and B sub-block (by/4, k-half
// (by/2)&1, column half by&1), and output o is sub-block (o/4, row half
// (o/2)&1, column half o&1) -- so L = 128 leaves run as L = 64 products with
// the same per-element DMMA sequence (leaf_gemm_dmma<64, ..., 128>).
template <int L, int KC, int WM, int WN, int NSTAGE, bool kTable = false, int LD = L>
__global__ void __launch_bounds__(32 * (L / WM) * (L / WN),
                                  (L > 64) ? 1 : ((L / WM) * (L / WN) <= 4 ? 3 : 2))
    leaf_gemm_dmma(const double* __restrict__ A, const double* __restrict__ B,
                   const int2* __restrict__ pairs, const int64_t* __restrict__ out_offset,
                   int64_t n_out, double* __restrict__ C, const int64_t* __restrict__ out_end,
                   int accumulate, const double* const* __restrict__ btab,
                   const int32_t* __restrict__ order = nullptr) {
  using Cfg = DmmaGemmCfg<L, KC, WM, WN, NSTAGE>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int pg = perm8(g);
  const int m0 = (warp % Cfg::WARPS_M) * WM;
  const int n0 = (warp / Cfg::WARPS_M) * WN;
  constexpr int64_t LL = static_cast<int64_t>(LD) * LD;  // leaf stride
  static_assert(LD == L || LD == 2 * L, "sub-blocks: halves of the leaf");
  // offset of sub-block (row half r, column half c) inside a leaf
  auto sub_off = [](int64_t idx, int r, int c) -> int64_t {
    return LD == L ? 0 : static_cast<int64_t>(c) * L * LD + static_cast<int64_t>(r) * L;
  };

  for (int64_t ob = blockIdx.x; ob < n_out; ob += gridDim.x) {
    const int64_t o = order ? order[ob] : ob;
    // products of block o: pairs[beg, end); a B-panel launch passes its own
    // end[] and continues the accumulator stored by the previous panel
    const int64_t beg = out_offset[o];
    const int64_t nsteps = ((out_end ? out_end[o] : out_offset[o + 1]) - beg) * Cfg::CHUNKS;
    if (nsteps == 0) continue;  // uniform per CTA

    // a stage's source: A slot and the B leaf's address
    struct Src {
      int ax;
      const double* b;
    };
    auto load_stage = [&](Src pr, int64_t step, int stage) {
      const int c = static_cast<int>(step % Cfg::CHUNKS);
      const double* Ablk = A + static_cast<int64_t>(LD == L ? pr.ax : (pr.ax >> 2)) * LL +
                           (LD == L ? 0 : sub_off(0, pr.ax & 1, (pr.ax >> 1) & 1)) +
                           static_cast<int64_t>(c) * KC * LD;
      const double* Bblk = pr.b + c * KC;
      double* As = smem + stage * Cfg::STAGE;
      double* Bs = As + Cfg::A_STAGE;
      constexpr int A_PIECES = KC * L / 2;
#pragma unroll
      for (int p = tid; p < A_PIECES; p += Cfg::kThreads) {
        const int kk = p / (L / 2), off = (p % (L / 2)) * 2;
        cp_async16(As + kk * Cfg::AS + off, Ablk + kk * LD + off);
      }
      constexpr int B_PIECES = L * KC / 2;
#pragma unroll
      for (int p = tid; p < B_PIECES; p += Cfg::kThreads) {
        const int j = p / (KC / 2), off = (p % (KC / 2)) * 2;
        cp_async16(Bs + j * Cfg::BS + off, Bblk + static_cast<int64_t>(j) * LD + off);
      }
    };
    auto pair_of = [&](int64_t step) -> Src {
      const int2 pr = step < nsteps ? __ldg(pairs + beg + step / Cfg::CHUNKS) : make_int2(0, 0);
      if constexpr (LD != L) {
        // B sub-block: leaf pr.y/4, k-half (pr.y/2)&1 (rows), column half pr.y&1
        const double* leaf = step < nsteps ? btab[pr.y >> 2] : B;
        return Src{pr.x, leaf + sub_off(0, (pr.y >> 1) & 1, pr.y & 1)};
      }
      if constexpr (kTable) return Src{pr.x, step < nsteps ? btab[pr.y] : B};
      return Src{pr.x, B + static_cast<int64_t>(pr.y) * LL};
    };

    double acc[Cfg::TM][Cfg::TN][2];
#pragma unroll
    for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::TN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          acc[i][j][e] = accumulate ? C[(LD == L ? o * LL : (o >> 2) * LL + sub_off(0, (o >> 1) & 1, o & 1)) +
                                        static_cast<int64_t>(n0 + 8 * j + perm8(2 * t + e)) * LD +
                                        m0 + 8 * i + pg]
                                    : 0.0;

#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
      if (s < nsteps) load_stage(pair_of(s), s, s);
      cp_async_commit();
    }
    // the (A slot, B slot) pair of the next stage to load is fetched one
    // iteration ahead so its global latency hides behind a compute step
    Src pr_next = pair_of(NSTAGE - 1);
    for (int64_t step = 0; step < nsteps; ++step) {
      cp_async_wait<NSTAGE - 2>();
      __syncthreads();
      const int64_t nxt = step + NSTAGE - 1;
      if (nxt < nsteps) load_stage(pr_next, nxt, static_cast<int>(nxt % NSTAGE));
      cp_async_commit();
      pr_next = pair_of(nxt + 1);
      const double* As = smem + static_cast<int>(step % NSTAGE) * Cfg::STAGE;
      const double* Bs = As + Cfg::A_STAGE;
#pragma unroll
      for (int ks = 0; ks < KC / 4; ++ks) {
        double a[Cfg::TM], b[Cfg::TN];
#pragma unroll
        for (int i = 0; i < Cfg::TM; ++i) a[i] = As[(4 * ks + t) * Cfg::AS + m0 + 8 * i + pg];
#pragma unroll
        for (int j = 0; j < Cfg::TN; ++j) b[j] = Bs[(n0 + 8 * j + pg) * Cfg::BS + 4 * ks + t];
#pragma unroll
        for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::TN; ++j) dmma_884(acc[i][j], a[i], b[j]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();

    double* Cblk = C + (LD == L ? o * LL : (o >> 2) * LL + sub_off(0, (o >> 1) & 1, o & 1));
#pragma unroll
    for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::TN; ++j) {
        const int row = m0 + 8 * i + pg;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = n0 + 8 * j + perm8(2 * t + e);
          Cblk[static_cast<int64_t>(col) * LD + row] = acc[i][j][e];
        }
      }
  }
}

// Any leaf size (small test leaves): plain FP64 FMA, one CTA per output block.
static __global__ void leaf_gemm_generic(const double* __restrict__ A, const double* __restrict__ B,
                                  const int2* __restrict__ pairs,
                                  const int64_t* __restrict__ out_offset, int64_t n_out, int L,
                                  double* __restrict__ C, const int64_t* __restrict__ out_end,
                                  int accumulate, const double* const* __restrict__ btab,
                                  const int32_t* __restrict__ order) {
  const int64_t LL = static_cast<int64_t>(L) * L;
  for (int64_t ob = blockIdx.x; ob < n_out; ob += gridDim.x) {
    const int64_t o = order ? order[ob] : ob;
    const int64_t beg = out_offset[o], end = out_end ? out_end[o] : out_offset[o + 1];
    if (beg == end) continue;
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) {
      const int64_t i = e % L, j = e / L;
      double acc = accumulate ? C[o * LL + e] : 0.0;
      for (int64_t s = beg; s < end; ++s) {
        const int2 pr = pairs[s];
        const double* a = A + pr.x * LL + i;
        const double* b = (btab ? btab[pr.y] : B + pr.y * LL) + j * L;
        for (int k = 0; k < L; ++k) acc = fma(a[static_cast<int64_t>(k) * L], b[k], acc);
      }
      C[o * LL + e] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// L = 32 super-block GEMM: one CTA per 2x2 group of output blocks
// (rows 2I, 2I+1 x cols 2J, 2J+1), warp s = 2 ri + cj owning block
// (2I+ri, 2J+cj) as a 32x32 tile (16 DMMA per 8 fragment loads).  Each
// pipeline stage holds, for one k, the A leaves A(2I+ri, k) and B leaves
// B(k, 2J+cj) any of the four blocks needs (entry mask bit s = product
// (2I+ri, k, 2J+cj) survives), so a stage feeds up to four products: the
// operand bytes per flop of an L = 64 product.  Every block still sees its
// products in ascending k, each as the same 8 DMMA k-steps as in
// leaf_gemm_dmma<32, ...>, so C~ is bitwise that kernel's.
// ---------------------------------------------------------------------------
struct SuperEntry {
  int32_t a0, a1, b0, b1;  // A slots of rows 2I, 2I+1 at k; B slots of cols 2J, 2J+1
};

// kQuad: warp w owns the 16x16 quadrant (w >> 1, w & 1) of EACH of the four
// blocks instead of one whole block, so every warp has the same work whatever
// the entry mask (a warp owning a block the entry skips used to wait at the
// barrier: 18 % of stall samples, DMMA pipe 86 % active at 55 % skipped).
// A full mask shares each block row's A and block column's B fragments
// between the two blocks using them (16 DMMA per 8 fragment loads); a partial
// mask runs the present blocks one by one (4 DMMA per 4 loads).  Every output
// element sees the same DMMA k-steps in the same order: bitwise the one-warp-
// per-block variant (kQuad = false).
template <bool kQuad>
__global__ void __launch_bounds__(128, 3)
    leaf_gemm_super32(const double* __restrict__ A, const double* const* __restrict__ btab,
                      const SuperEntry* __restrict__ ent, const uint32_t* __restrict__ emask,
                      const int64_t* __restrict__ sb_beg, const int64_t* __restrict__ sb_end,
                      const int32_t* __restrict__ sb_out, int64_t n_sb, double* __restrict__ C,
                      const int32_t* __restrict__ order, int accumulate) {
  constexpr int L = 32, S = 36;  // leaf, padded stride (== 4 mod 16)
  constexpr int TILE = L * S;
  constexpr int STAGE = 4 * TILE;  // A row 0, A row 1, B col 0, B col 1
  constexpr int64_t LL = L * L;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3, pg = perm8(g);
  const int ri = warp >> 1, cj = warp & 1;  // whole-block mode: the warp's block
  const int qr = warp >> 1, qc = warp & 1;  // quadrant mode: the warp's quadrant

  for (int64_t sbi = blockIdx.x; sbi < n_sb; sbi += gridDim.x) {
    const int64_t sb = order ? order[sbi] : sbi;
    // entries [sb_beg[sb], sb_end[sb]): all of the super block's, or those
    // of one B panel (sb_end = sb_beg + 1 pointer for the whole list)
    const int64_t beg = sb_beg[sb];
    const int64_t n = sb_end[sb] - beg;
    if (n == 0) continue;  // uniform per CTA

    auto load_stage = [&](const SuperEntry& en, uint32_t m, int stage) {
      double* st = smem + stage * STAGE;
      // tile q: 0 = A row 2I, 1 = A row 2I+1, 2 = B col 2J, 3 = B col 2J+1
      const bool need[4] = {(m & 3u) != 0, (m & 12u) != 0, (m & 5u) != 0, (m & 10u) != 0};
      const double* src[4] = {A + static_cast<int64_t>(en.a0) * LL,
                              A + static_cast<int64_t>(en.a1) * LL, btab[need[2] ? en.b0 : 0],
                              btab[need[3] ? en.b1 : 0]};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!need[q]) continue;  // uniform per CTA
        double* dst = st + q * TILE;
#pragma unroll
        for (int p = tid; p < L * L / 2; p += 128) {
          // A: column kk of the leaf (L rows) -> dst[kk * S + row];
          // B: column j of the leaf (L k-entries) -> dst[j * S + kk]; same copy
          const int c = p / (L / 2), off = (p % (L / 2)) * 2;
          cp_async16(dst + c * S + off, src[q] + c * L + off);
        }
      }
    };

    // whole-block mode: acc[i][j] = the warp's block; quadrant mode: acc[b][2 i + j]
    // with b the block, i, j < 2 the 8x8 tiles of the warp's quadrant
    double acc[4][4][2];
    if constexpr (kQuad) {
#pragma unroll
      for (int bl = 0; bl < 4; ++bl) {
        const int32_t ob = sb_out[4 * sb + bl];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              acc[bl][2 * i + j][e] =
                  (accumulate && ob >= 0)
                      ? C[static_cast<int64_t>(ob) * LL +
                          static_cast<int64_t>(16 * qc + 8 * j + perm8(2 * t + e)) * L +
                          16 * qr + 8 * i + pg]
                      : 0.0;
      }
    } else {
      const int32_t o = sb_out[4 * sb + warp];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            acc[i][j][e] = (accumulate && o >= 0)
                               ? C[static_cast<int64_t>(o) * LL +
                                   static_cast<int64_t>(8 * j + perm8(2 * t + e)) * L + 8 * i + pg]
                               : 0.0;
    }

    // entries are fetched one step ahead, so their global latency hides
    // behind a compute step (as pr_next in leaf_gemm_dmma)
    SuperEntry en_next{};
    uint32_t m_cur = 0, m_next = 0;
    if (n > 0) {
      m_cur = emask[beg];
      load_stage(ent[beg], m_cur, 0);
    }
    cp_async_commit();
    if (n > 1) {
      en_next = ent[beg + 1];
      m_next = emask[beg + 1];
    }
    for (int64_t step = 0; step < n; ++step) {
      cp_async_wait<0>();
      __syncthreads();
      if (step + 1 < n) load_stage(en_next, m_next, static_cast<int>((step + 1) & 1));
      cp_async_commit();
      const uint32_t m_step = m_cur;
      m_cur = m_next;
      if (step + 2 < n) {
        en_next = ent[beg + step + 2];
        m_next = emask[beg + step + 2];
      }
      const double* st = smem + static_cast<int>(step & 1) * STAGE;
      if constexpr (kQuad) {
        if (m_step == 15u) {
          // all four products: each block row's A fragments and each block
          // column's B fragments loaded once for the two blocks sharing them
          // (16 DMMA per 8 fragment loads, as the one-warp-per-block kernel)
#pragma unroll
          for (int ks = 0; ks < L / 4; ++ks) {
            double a[2][2], b[2][2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              a[0][i] = st[(4 * ks + t) * S + 16 * qr + 8 * i + pg];
              a[1][i] = st[TILE + (4 * ks + t) * S + 16 * qr + 8 * i + pg];
              b[0][i] = st[2 * TILE + (16 * qc + 8 * i + pg) * S + 4 * ks + t];
              b[1][i] = st[3 * TILE + (16 * qc + 8 * i + pg) * S + 4 * ks + t];
            }
#pragma unroll
            for (int bl = 0; bl < 4; ++bl)
#pragma unroll
              for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                  dmma_884(acc[bl][2 * i + j], a[bl >> 1][i], b[bl & 1][j]);
          }
        } else {
        // a partial mask: one branch per block (a predicated DMMA would still
        // occupy the pipe)
#pragma unroll
        for (int bl = 0; bl < 4; ++bl) {
          if (!((m_step >> bl) & 1u)) continue;  // uniform per CTA
          const double* As = st + (bl >> 1) * TILE;
          const double* Bs = st + (2 + (bl & 1)) * TILE;
#pragma unroll
          for (int ks = 0; ks < L / 4; ++ks) {
            double a[2], b[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              a[i] = As[(4 * ks + t) * S + 16 * qr + 8 * i + pg];
              b[i] = Bs[(16 * qc + 8 * i + pg) * S + 4 * ks + t];
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int j = 0; j < 2; ++j) dmma_884(acc[bl][2 * i + j], a[i], b[j]);
          }
        }
        }
      } else if ((m_step >> warp) & 1u) {
        const double* As = st + ri * TILE;
        const double* Bs = st + (2 + cj) * TILE;
#pragma unroll
        for (int ks = 0; ks < L / 4; ++ks) {
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = As[(4 * ks + t) * S + 8 * i + pg];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = Bs[(8 * j + pg) * S + 4 * ks + t];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_884(acc[i][j], a[i], b[j]);
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    if constexpr (kQuad) {
#pragma unroll
      for (int bl = 0; bl < 4; ++bl) {
        const int32_t ob = sb_out[4 * sb + bl];
        if (ob < 0) continue;
        double* Cblk = C + static_cast<int64_t>(ob) * LL;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int row = 16 * qr + 8 * i + pg;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = 16 * qc + 8 * j + perm8(2 * t + e);
              Cblk[static_cast<int64_t>(col) * L + row] = acc[bl][2 * i + j][e];
            }
          }
      }
    } else {
      const int32_t o = sb_out[4 * sb + warp];
      if (o >= 0) {
        double* Cblk = C + static_cast<int64_t>(o) * LL;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int row = 8 * i + pg;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = 8 * j + perm8(2 * t + e);
              Cblk[static_cast<int64_t>(col) * L + row] = acc[i][j][e];
            }
          }
      }
    }
  }
}

}  // namespace spg
