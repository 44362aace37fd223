// latency of tcgen05.ld x32 + wait::ld per warp, W concurrent warps, with/without fences
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int FENCE>
__global__ void k(int iters, long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) * 32) % 448;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[32];
    if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
      : "r"(t + (acc & 0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) acc += v[i];
    if (FENCE) { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); __syncwarp(); }
  }
  long long dt = clock64() - t0;
  sink[blockIdx.x * blockDim.x + tid] = acc;
  if ((tid & 31) == 0) atomicAdd((unsigned long long*)out, (unsigned long long)dt);
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot));
}
int main() {
  long long* o; uint32_t* sink; cudaMallocManaged(&o, 8); cudaMalloc(&sink, 1 << 20);
  for (int f = 0; f < 2; ++f)
    for (int w = 1; w <= 32; w *= 2) {
      if (w == 32) w = 31;
      *o = 0;
      if (f) k<1><<<1, w * 32>>>(1000, o, sink); else k<0><<<1, w * 32>>>(1000, o, sink);
      cudaError_t e = cudaDeviceSynchronize();
      printf("fence=%d warps=%2d: %.1f cycles per ld32+wait+use (avg per warp)  %s\n", f, w, (double)*o / w / 1000, cudaGetErrorString(e));
    }
}
