// TMEM load/store throughput per SM: W warps (warp w -> lane quadrant w%4) repeatedly move
// 32 columns (32x32b.x32) between TMEM and registers.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
template <int MODE>   // 0 ld x32, 1 st x32, 2 ld x16 pack::16b
__global__ void bw(int iters, long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32 % 512;
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = tid * i;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
        : "r"(t));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += v[0] ^ v[9] ^ v[17] ^ v[31];
    } else if (MODE == 1) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        :: "r"(t), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),"r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
      v[0] += 1;
    } else {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15])
        : "r"(t));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += v[0] ^ v[9] ^ v[15];
    }
  }
  long long dt = clock64() - t0;
  __syncthreads();
  if (tid == 0) *cyc = dt;
  sink[blockIdx.x * blockDim.x + tid] = acc + v[3];
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot));
}
int main() {
  long long* cyc; uint32_t* sink; cudaMallocManaged(&cyc, 8); cudaMalloc(&sink, 1 << 20);
  const char* names[3] = {"ld x32", "st x32", "ld x32 pack16"};
  for (int mode = 0; mode < 3; ++mode)
    for (int w = 4; w <= 16; w *= 2) {
      const int iters = 2000;
      if (mode == 0) bw<0><<<1, w * 32>>>(iters, cyc, sink);
      if (mode == 1) bw<1><<<1, w * 32>>>(iters, cyc, sink);
      if (mode == 2) bw<2><<<1, w * 32>>>(iters, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      const double bytes = (double)iters * w * 32 * 32 * 4;   // TMEM cells touched (32 cols x 32 lanes x 4 B)
      printf("%-14s warps=%2d: %.1f B/clk per SM (cells), %.1f cycles per warp-op  (%s)\n", names[mode], w, bytes / *cyc,
             (double)*cyc / iters, cudaGetErrorString(e));
    }
}
