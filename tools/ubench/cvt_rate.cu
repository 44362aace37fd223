// throughput of the f16 split ops: F2FP (float2 -> half2 pack), HADD2.F32 (half -> float), FADD2
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdint.h>
template <int OP>
__global__ void k(int iters, uint32_t* out, long long* cyc) {
  float a[8];
  uint32_t acc = 0, accs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i * 0.1f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (OP == 0) {   // F2FP pack: 1 per pair
        __half2 h = __floats2half2_rn(a[i], a[i + 1]);
        uint32_t u = *reinterpret_cast<uint32_t*>(&h);
        accs[i] += u;
        a[i] = __uint_as_float(__float_as_uint(a[i]) + 1u); a[i + 1] = __uint_as_float(__float_as_uint(a[i + 1]) + 1u);
      } else if (OP == 1) {   // half2 -> float2 unpack
        __half2 h = *reinterpret_cast<__half2*>(&accs[i + 1]);
        float2 f = __half22float2(h);
        accs[i] += __float_as_uint(f.x) + __float_as_uint(f.y);
        accs[i + 1] += 0x00010001u;
      } else {   // MUFU sin for reference
        float s, c;
        __sincosf(a[i], &s, &c);
        a[i] = s + c; a[i + 1] += 1e-3f;
      }
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < 8; ++i) acc += __float_as_uint(a[i]) + accs[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  uint32_t* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMallocManaged(&c, 8);
  const char* nm[3] = {"F2FP pack (per pair)", "HADD2.F32 unpack x2 (per pair)", "MUFU sin+cos (per item)"};
  for (int op = 0; op < 3; ++op) {
    const int iters = 2000, w = 16;
    if (op == 0) k<0><<<148, w * 32>>>(iters, o, c);
    if (op == 1) k<1><<<148, w * 32>>>(iters, o, c);
    if (op == 2) k<2><<<148, w * 32>>>(iters, o, c);
    cudaDeviceSynchronize();
    printf("%-32s: %.1f ops/clk/SM (4 per lane-iteration)\n", nm[op], (double)iters * 4 * w * 32 / *c);
  }
}
