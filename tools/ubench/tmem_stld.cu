// latency of the generator TMEM pattern: tcgen05.st.x16 (A slice) then tcgen05.ld.x32 (next
// phase slice) + wait::ld, per warp, W warps per SM; with and without a wait::st per slice
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>   // 0: st16 + ld32 + wait::ld ; 1: + wait::st each iteration ; 2: ld only ; 3: st + wait::st only
__global__ void k(int iters, long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t ph = base + 128 + (warp >> 2) * 128 % 256, aa = base + 384 + ((warp >> 2) % 2) * 64;
  uint32_t hl[16], acc = 0;
  for (int i = 0; i < 16; ++i) hl[i] = tid * i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[32];
    if (MODE != 2) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" :: "r"(aa + (it & 3) * 16),
        "r"(hl[0]),"r"(hl[1]),"r"(hl[2]),"r"(hl[3]),"r"(hl[4]),"r"(hl[5]),"r"(hl[6]),"r"(hl[7]),"r"(hl[8]),"r"(hl[9]),"r"(hl[10]),"r"(hl[11]),"r"(hl[12]),"r"(hl[13]),"r"(hl[14]),"r"(hl[15]) : "memory");
      if (MODE == 1 || MODE == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (MODE != 3) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
        : "r"(ph + (it & 3) * 32) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 32; i += 4) acc += v[i] + (v[i + 1] << 8) + (v[i + 2] << 16) + (v[i + 3] << 24);
      hl[it & 15] ^= acc;
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  long long dt = clock64() - t0;
  sink[blockIdx.x * blockDim.x + tid] = acc + hl[3];
  if ((tid & 31) == 0) atomicAdd((unsigned long long*)out, (unsigned long long)dt);
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot));
}
int main() {
  long long* o; uint32_t* sink; cudaMallocManaged(&o, 8); cudaMalloc(&sink, 1 << 22);
  const char* nm[4] = {"st16 + ld32 + wait::ld", "st16 + wait::st + ld32 + wait::ld", "ld32 + wait::ld", "st16 + wait::st"};
  for (int m = 0; m < 4; ++m)
    for (int w = 4; w <= 16; w *= 2) {
      *o = 0;
      if (m == 0) k<0><<<148, w * 32>>>(1000, o, sink);
      if (m == 1) k<1><<<148, w * 32>>>(1000, o, sink);
      if (m == 2) k<2><<<148, w * 32>>>(1000, o, sink);
      if (m == 3) k<3><<<148, w * 32>>>(1000, o, sink);
      cudaError_t e = cudaDeviceSynchronize();
      printf("%-36s warps=%2d: %.1f cycles/iter per warp (%s)\n", nm[m], w, (double)*o / w / 1000, cudaGetErrorString(e));
    }
}
