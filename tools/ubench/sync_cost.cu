// issue cost of tcgen05.commit, mbarrier.arrive and try_wait (already complete) from one thread
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(long long* out) {
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  if (tid < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (tid == 0) {
    const int N = 1024;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar[i & 7])) : "memory");
    long long t1 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&bar[i & 7])) : "memory");
    long long t2 = clock64();
    // bar[0] has completed many phases; wait for the parity of a completed phase
    uint32_t acc = 0;
    for (int i = 0; i < N; ++i) {
      uint32_t done;
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(su32(&bar[i & 7])), "r"(1u) : "memory");
      acc += done;
    }
    long long t3 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    long long t4 = clock64();
    out[0] = (t1 - t0) / N; out[1] = (t2 - t1) / N; out[2] = (t3 - t2) / N; out[3] = acc; out[4] = (t4 - t3) / N;
  }
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(slot));
}
int main() {
  long long* o; cudaMallocManaged(&o, 64);
  k<<<1, 128>>>(o); cudaError_t e = cudaDeviceSynchronize();
  printf("commit %lld  arrive %lld  try_wait(done) %lld (ok=%lld)  fence_after %lld cycles  (%s)\n", o[0], o[1], o[2], o[3], o[4], cudaGetErrorString(e));
}
