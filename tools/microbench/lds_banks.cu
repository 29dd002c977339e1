// LDS.64 bank behaviour of the DMMA fragment patterns (lane g = lane>>2,
// t = lane&3): cycles per warp-wide 64-bit shared load for candidate layouts.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int perm(int g) { return g ^ ((g >> 2) << 1); }

template <int MODE>
__global__ void lds_kernel(long long* out, double* sink, int iters) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  int addr;
  switch (MODE) {
    case 0: addr = lane; break;                 // ideal: consecutive
    case 1: addr = t * 72 + g; break;           // A, stride 72 (round 1)
    case 2: addr = t * 68 + perm(g); break;     // A, stride 68 + perm
    case 3: addr = g * 36 + t; break;           // B, stride 36 (round 1)
    case 4: addr = perm(g) * 36 + t; break;     // B, stride 36 + perm
    case 5: addr = t * 68 + g; break;           // A, stride 68, no perm
    default: addr = lane * 16; break;           // worst: all one bank pair
  }
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += s[(addr + u * 256 + (it & 1) * 2048) & 4095];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
  if (acc == 1234.5) sink[0] = acc;
}

int main() {
  long long* d; double* sink;
  cudaMalloc(&d, 8 * 1024); cudaMalloc(&sink, 8);
  const char* names[] = {"ideal", "A s72", "A s68+perm", "B s36", "B s36+perm", "A s68", "worst"};
  for (int m = 0; m < 7; ++m) {
    const int iters = 2000, warps = 8;
    auto run = [&](auto kern) { kern<<<1, 32 * warps>>>(d, sink, iters); };
    switch (m) {
      case 0: run(lds_kernel<0>); break; case 1: run(lds_kernel<1>); break;
      case 2: run(lds_kernel<2>); break; case 3: run(lds_kernel<3>); break;
      case 4: run(lds_kernel<4>); break; case 5: run(lds_kernel<5>); break;
      default: run(lds_kernel<6>); break;
    }
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-12s %.2f cycles per warp-LDS.64 (8 warps on one SM)\n", names[m], (double)h / (iters * 16.0 * warps));
  }
  return 0;
}
