// standalone throughput of the generator math (integer phase -> sin/cos -> FP16 hi/lo) for
// W warps per SM, no TMEM / barriers: MUFU utilisation ceiling of the instruction mix
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdint.h>
__device__ __forceinline__ float turns_m(uint32_t tu) { return __uint_as_float((tu >> 9) + 0x3F800000u); }
__device__ __forceinline__ void fixed_sincos2(uint32_t t0, uint32_t t1, float& s0, float& c0, float& s1, float& c1) {
  constexpr float TWO_PI = 6.28318530717958647692f;
  const float2 x = __ffma2_rn(make_float2(turns_m(t0), turns_m(t1)), make_float2(TWO_PI, TWO_PI), make_float2(-TWO_PI, -TWO_PI));
  __sincosf(x.x, &s0, &c0);
  __sincosf(x.y, &s1, &c1);
}
__device__ __forceinline__ void f16_split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  const float2 r = __fadd2_rn(make_float2(x, y), make_float2(-hf.x, -hf.y));
  const __half2 l = __floats2half2_rn(r.x, r.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
template <int NI, int MODE>
__global__ void k(int iters, uint32_t* out, long long* cyc) {
  uint32_t t[NI], acc = 0;
  for (int i = 0; i < NI; ++i) t[i] = (threadIdx.x * 2654435761u) ^ (i * 40503u);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
    for (int sl = 0; sl < NI; sl += 8) {
      uint32_t hl[16];
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        float s0, c0, s1, c1;
        fixed_sincos2(t[sl + i], t[sl + i + 1], s0, c0, s1, c1);
        f16_split2(c0, s0, hl[i], hl[8 + i]);
        f16_split2(c1, s1, hl[i + 1], hl[8 + i + 1]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += hl[i];
    }
    } else {
#pragma unroll
    for (int sl = 0; sl < NI; sl += 16) {
      float sn[16], cs[16];
#pragma unroll
      for (int i = 0; i < 16; i += 2) fixed_sincos2(t[sl + i], t[sl + i + 1], sn[i], cs[i], sn[i + 1], cs[i + 1]);
      uint32_t hl[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) f16_split2(cs[i], sn[i], hl[i], hl[16 + i]);
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += hl[i];
    }
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) t[i] += 0x9E3779B9u;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  uint32_t* o; long long* c; cudaMalloc(&o, 148 * 2048 * 4); cudaMallocManaged(&c, 8);
  for (int mode = 0; mode < 2; ++mode)
  for (int w = 4; w <= 16; w *= 2) {
    const int iters = 500;
    if (mode == 0) k<32, 0><<<148, w * 32>>>(iters, o, c); else k<32, 1><<<148, w * 32>>>(iters, o, c);
    cudaDeviceSynchronize();
    const double mufu = (double)iters * 32 * 2 * w * 32;
    printf("mode %d warps/SM=%2d: %.2f MUFU lane-ops/clk/SM (peak 16) -> %.0f%%\n", mode, w, mufu / *c, 100 * mufu / *c / 16);
  }
}
