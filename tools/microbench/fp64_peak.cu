// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Establishes the roofline denominator for the SpAMM leaf GEMM (K5).
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_m8n8k4_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16_loop(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

// dependent DADD chain latency + DSQRT throughput (for the τ-sweep and norms)
__global__ void dadd_chain(double* out, int iters) {
  double s = threadIdx.x;
  double v = 1e-3;
  for (int it = 0; it < iters; ++it) { s = __dadd_rn(s, v); }
  if (s == 12345.0) out[0] = s;
}
__global__ void dsqrt_loop(double* out, int iters) {
  double s[8];
  for (int i = 0; i < 8; ++i) s[i] = threadIdx.x + i + 2.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] = __dsqrt_rn(s[i]) + 1.5;
  }
  double t = 0; for (int i = 0; i < 8; ++i) t += s[i];
  if (t == 12345.0) out[0] = t;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int blocks_per_sm : {1, 2, 4}) {
      int grid = sms * blocks_per_sm, threads = 32 * wpb;
      float ms = time_it([&] { dmma_m8n8k4_loop<8><<<grid, threads>>>(out, iters); });
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * grid * wpb;
      printf("DMMA m8n8k4   wpb=%2d bps=%d : %.2f TFLOP/s (%.3f ms)\n", wpb, blocks_per_sm, flops / ms / 1e9, ms);
      ms = time_it([&] { dmma_m16n8k16_loop<4><<<grid, threads>>>(out, iters / 4); });
      flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * grid * wpb;
      printf("DMMA m16n8k16 wpb=%2d bps=%d : %.2f TFLOP/s (%.3f ms)\n", wpb, blocks_per_sm, flops / ms / 1e9, ms);
      ms = time_it([&] { dfma_loop<8><<<grid, threads>>>(out, iters); });
      flops = 2.0 * 8.0 * iters * grid * threads;
      printf("DFMA          wpb=%2d bps=%d : %.2f TFLOP/s (%.3f ms)\n", wpb, blocks_per_sm, flops / ms / 1e9, ms);
    }
  }
  float ms = time_it([&] { dadd_chain<<<1, 32>>>(out, iters); });
  printf("DADD dependent latency: %.2f ns/op\n", ms * 1e6 / iters);
  ms = time_it([&] { dsqrt_loop<<<sms * 4, 256>>>(out, 2000); });
  printf("DSQRT(+add) throughput: %.2f Gop/s\n", 8.0 * 2000 * sms * 4 * 256 / ms / 1e6);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock=%d kHz\n", sms, clk);
  return 0;
}
