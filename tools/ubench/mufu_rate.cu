// MUFU sin/cos throughput per SM (one CTA per SM, W warps, independent chains)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
__global__ void k(int iters, float* out, long long* cyc) {
  float a[8], acc = 0.f;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i * 0.1f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float s, c;
      __sincosf(a[i], &s, &c);
      a[i] = s + c;   // dependent chain per slot; 8 independent chains
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < 8; ++i) acc += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMallocManaged(&c, 8);
  for (int w : {4, 8, 12, 16, 32}) {
    const int iters = 2000;
    k<<<148, w * 32>>>(iters, o, c);
    cudaDeviceSynchronize();
    const double mufu = (double)iters * 8 * 2 * w * 32;   // MUFU lane-ops per SM
    printf("warps=%2d: %.2f MUFU lane-ops/clk/SM\n", w, mufu / *c);
  }
}
