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
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NI, int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, uint32_t* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (MODE >= 2) {
    if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  }
  const uint32_t tb = MODE >= 2 ? slot + ((uint32_t)((warp & 3) * 32) << 16) : 0;
  uint32_t t[NI], acc = 0, pv[32];
  for (int i = 0; i < NI; ++i) t[i] = (threadIdx.x * 2654435761u) ^ (i * 40503u);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE >= 2) {
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
      if (MODE >= 2 && MODE != 6) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" :: "r"(tb + 384 + ((warp >> 2) & 1) * 64 + (sl / 8 % 4) * 16),
          "r"(hl[0]),"r"(hl[1]),"r"(hl[2]),"r"(hl[3]),"r"(hl[4]),"r"(hl[5]),"r"(hl[6]),"r"(hl[7]),"r"(hl[8]),"r"(hl[9]),"r"(hl[10]),"r"(hl[11]),"r"(hl[12]),"r"(hl[13]),"r"(hl[14]),"r"(hl[15]) : "memory");
      }
      if (MODE == 6) {
        for (int i = 0; i < 16; ++i) acc += hl[i];
      }
      if (MODE >= 2) {
        if (MODE == 4 || MODE == 6) {   // pipelined: wait for the load issued one slice earlier, then issue the next
          if (sl > 0) {
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 8; ++i) t[sl - 8 + i] += pv[4 * i] + (pv[4 * i + 1] << 8) + (pv[4 * i + 2] << 16) + (pv[4 * i + 3] << 24);
          }
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(pv[0]),"=r"(pv[1]),"=r"(pv[2]),"=r"(pv[3]),"=r"(pv[4]),"=r"(pv[5]),"=r"(pv[6]),"=r"(pv[7]),"=r"(pv[8]),"=r"(pv[9]),"=r"(pv[10]),"=r"(pv[11]),"=r"(pv[12]),"=r"(pv[13]),"=r"(pv[14]),"=r"(pv[15]),"=r"(pv[16]),"=r"(pv[17]),"=r"(pv[18]),"=r"(pv[19]),"=r"(pv[20]),"=r"(pv[21]),"=r"(pv[22]),"=r"(pv[23]),"=r"(pv[24]),"=r"(pv[25]),"=r"(pv[26]),"=r"(pv[27]),"=r"(pv[28]),"=r"(pv[29]),"=r"(pv[30]),"=r"(pv[31])
            : "r"(tb + 128 + ((warp >> 2) & 1) * 128 + (sl / 8 % 4) * 32) : "memory");
        }
        if (MODE == 7 || MODE == 8) {
          if (sl > 0) {
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < (MODE == 7 ? 8 : 4); ++i) t[sl - 8 + i] += pv[4 * i] + (pv[4 * i + 1] << 8) + (pv[4 * i + 2] << 16) + (pv[4 * i + 3] << 24);
          }
          if (MODE == 7) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(pv[0]),"=r"(pv[1]),"=r"(pv[2]),"=r"(pv[3]),"=r"(pv[4]),"=r"(pv[5]),"=r"(pv[6]),"=r"(pv[7]),"=r"(pv[8]),"=r"(pv[9]),"=r"(pv[10]),"=r"(pv[11]),"=r"(pv[12]),"=r"(pv[13]),"=r"(pv[14]),"=r"(pv[15])
              : "r"(tb + 128 + ((warp >> 2) & 1) * 128 + (sl / 8 % 4) * 32) : "memory");
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(pv[16]),"=r"(pv[17]),"=r"(pv[18]),"=r"(pv[19]),"=r"(pv[20]),"=r"(pv[21]),"=r"(pv[22]),"=r"(pv[23]),"=r"(pv[24]),"=r"(pv[25]),"=r"(pv[26]),"=r"(pv[27]),"=r"(pv[28]),"=r"(pv[29]),"=r"(pv[30]),"=r"(pv[31])
              : "r"(tb + 128 + ((warp >> 2) & 1) * 128 + (sl / 8 % 4) * 32 + 16) : "memory");
          } else {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(pv[0]),"=r"(pv[1]),"=r"(pv[2]),"=r"(pv[3]),"=r"(pv[4]),"=r"(pv[5]),"=r"(pv[6]),"=r"(pv[7]),"=r"(pv[8]),"=r"(pv[9]),"=r"(pv[10]),"=r"(pv[11]),"=r"(pv[12]),"=r"(pv[13]),"=r"(pv[14]),"=r"(pv[15])
              : "r"(tb + 128 + ((warp >> 2) & 1) * 128 + (sl / 8 % 4) * 32) : "memory");
          }
        }
        if (MODE == 3) {
          uint32_t v[32];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
            : "r"(tb + 128 + ((warp >> 2) & 1) * 128 + (sl / 8 % 4) * 32) : "memory");
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; ++i) t[sl + i] += v[4 * i] + (v[4 * i + 1] << 8) + (v[4 * i + 2] << 16) + (v[4 * i + 3] << 24);
        }
      } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += hl[i];
      }
    }
    if (MODE == 4 || MODE == 6 || MODE == 7 || MODE == 8) {
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 8; ++i) t[NI - 8 + i] += pv[4 * i] + (pv[4 * i + 1] << 8) + (pv[4 * i + 2] << 16) + (pv[4 * i + 3] << 24);
    }
    if (MODE >= 2) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
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
  if (MODE >= 2) {
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot));
  }
}
int main() {
  uint32_t* o; long long* c; cudaMalloc(&o, 148 * 2048 * 4); cudaMallocManaged(&c, 8);
  for (int mode = 0; mode < 9; ++mode)
  for (int w : {4, 8, 12, 16}) {
    const int iters = 500;
    if (mode == 0) k<32, 0><<<148, w * 32>>>(iters, o, c);
    if (mode == 1) k<32, 1><<<148, w * 32>>>(iters, o, c);
    if (mode == 2) k<32, 2><<<148, w * 32>>>(iters, o, c);
    if (mode == 3) k<32, 3><<<148, w * 32>>>(iters, o, c);
    if (mode == 4) k<32, 4><<<148, w * 32>>>(iters, o, c);
    if (mode == 5) k<16, 4><<<148, w * 32>>>(iters, o, c);
    if (mode == 6) k<32, 6><<<148, w * 32>>>(iters, o, c);
    if (mode == 7) k<32, 7><<<148, w * 32>>>(iters, o, c);
    if (mode == 8) k<32, 8><<<148, w * 32>>>(iters, o, c);
    cudaDeviceSynchronize();
    const double mufu = (double)iters * (mode == 5 ? 16 : 32) * 2 * w * 32;
    printf("mode %d warps/SM=%2d: %.2f MUFU lane-ops/clk/SM (peak 16) -> %.0f%%\n", mode, w, mufu / *c, 100 * mufu / *c / 16);
  }
}
