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
  static constexpr int kThreads = 256;
  static constexpr int kWarps = 8;
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
  static_assert((L / WM) * (L / WN) == kWarps, "warp tiling must cover the leaf with 8 warps");
  static_assert(AS % 16 == 4 && BS % 16 == 4, "bank-conflict-free strides");
  static_assert(L % KC == 0 && KC % 4 == 0, "k chunking");
};

template <int L, int KC, int WM, int WN, int NSTAGE>
__global__ void __launch_bounds__(256, (NSTAGE <= 3 && L <= 64) ? 2 : 1)
    leaf_gemm_dmma(const double* __restrict__ A, const double* __restrict__ B,
                   const int2* __restrict__ pairs, const int64_t* __restrict__ out_offset,
                   int64_t n_out, double* __restrict__ C) {
  using Cfg = DmmaGemmCfg<L, KC, WM, WN, NSTAGE>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int pg = perm8(g);
  const int m0 = (warp % Cfg::WARPS_M) * WM;
  const int n0 = (warp / Cfg::WARPS_M) * WN;
  constexpr int64_t LL = static_cast<int64_t>(L) * L;

  for (int64_t o = blockIdx.x; o < n_out; o += gridDim.x) {
    const int64_t beg = out_offset[o];
    const int64_t nsteps = (out_offset[o + 1] - beg) * Cfg::CHUNKS;

    auto load_stage = [&](int2 pr, int64_t step, int stage) {
      const int c = static_cast<int>(step % Cfg::CHUNKS);
      const double* Ablk = A + static_cast<int64_t>(pr.x) * LL + static_cast<int64_t>(c) * KC * L;
      const double* Bblk = B + static_cast<int64_t>(pr.y) * LL + c * KC;
      double* As = smem + stage * Cfg::STAGE;
      double* Bs = As + Cfg::A_STAGE;
      constexpr int A_PIECES = KC * L / 2;
#pragma unroll
      for (int p = tid; p < A_PIECES; p += Cfg::kThreads) {
        const int kk = p / (L / 2), off = (p % (L / 2)) * 2;
        cp_async16(As + kk * Cfg::AS + off, Ablk + kk * L + off);
      }
      constexpr int B_PIECES = L * KC / 2;
#pragma unroll
      for (int p = tid; p < B_PIECES; p += Cfg::kThreads) {
        const int j = p / (KC / 2), off = (p % (KC / 2)) * 2;
        cp_async16(Bs + j * Cfg::BS + off, Bblk + static_cast<int64_t>(j) * L + off);
      }
    };
    auto pair_of = [&](int64_t step) {
      return step < nsteps ? __ldg(pairs + beg + step / Cfg::CHUNKS) : make_int2(0, 0);
    };

    double acc[Cfg::TM][Cfg::TN][2];
#pragma unroll
    for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
      if (s < nsteps) load_stage(pair_of(s), s, s);
      cp_async_commit();
    }
    // the (A slot, B slot) pair of the next stage to load is fetched one
    // iteration ahead so its global latency hides behind a compute step
    int2 pr_next = pair_of(NSTAGE - 1);
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

    double* Cblk = C + o * LL;
#pragma unroll
    for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::TN; ++j) {
        const int row = m0 + 8 * i + pg;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = n0 + 8 * j + perm8(2 * t + e);
          Cblk[static_cast<int64_t>(col) * L + row] = acc[i][j][e];
        }
      }
  }
}

// Any leaf size (small test leaves): plain FP64 FMA, one CTA per output block.
static __global__ void leaf_gemm_generic(const double* __restrict__ A, const double* __restrict__ B,
                                  const int2* __restrict__ pairs,
                                  const int64_t* __restrict__ out_offset, int64_t n_out, int L,
                                  double* __restrict__ C) {
  const int64_t LL = static_cast<int64_t>(L) * L;
  for (int64_t o = blockIdx.x; o < n_out; o += gridDim.x) {
    const int64_t beg = out_offset[o], end = out_offset[o + 1];
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) {
      const int64_t i = e % L, j = e / L;
      double acc = 0.0;
      for (int64_t s = beg; s < end; ++s) {
        const int2 pr = pairs[s];
        const double* a = A + pr.x * LL + i;
        const double* b = B + pr.y * LL + j * L;
        for (int k = 0; k < L; ++k) acc = fma(a[static_cast<int64_t>(k) * L], b[k], acc);
      }
      C[o * LL + e] = acc;
    }
  }
}

}  // namespace spg
