// latency: issue n MMAs (f16 TS M128 N64 K16) + commit -> mbarrier observed by the same warp
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__global__ void k(int nmma, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = tid; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | (8u << 24);
  if (warp == 0) {
    long long best = 1 << 30, sum = 0;
    for (int rep = 0; rep < 20; ++rep) {
      long long t0 = clock64();
      for (int j = 0; j < nmma; ++j)
        asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n}" :: "r"(t), "r"(t + 256 + 8 * (j & 7)), "l"(desc(su32(sm) + (j & 7) * 2048, 1024, 128)), "r"(idesc));
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" :: "r"(su32(&mbar)));
      uint32_t done = 0;
      while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)), "r"((uint32_t)(rep & 1)));
      long long dt = clock64() - t0;
      if (rep >= 2) { sum += dt; if (dt < best) best = dt; }
    }
    if (tid == 0) { out[0] = best; out[1] = sum / 18; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}
int main() {
  long long* o; cudaMallocManaged(&o, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  int ns[] = {0, 1, 2, 3, 9, 18, 36};
  for (int n : ns) {
    k<<<1, 128, 32 * 1024>>>(n, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("n_mma=%2d: issue->commit->wait observed: best %lld avg %lld cycles (%s)\n", n, o[0], o[1], cudaGetErrorString(e));
  }
}
