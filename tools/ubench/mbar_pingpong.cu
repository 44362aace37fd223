// mbarrier hand-off latency on sm_100a: warp 0 <-> warp 1 ping-pong, plain arrive vs
// tcgen05.commit (empty commit) on the return path, and try_wait with/without suspend hint.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <bool HINT>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  while (!done) {
    if (HINT)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(b)), "r"(par), "r"(1000000) : "memory");
    else
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(b)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }

template <bool HINT, bool COMMIT>
__global__ void pingpong(int iters, long long* out) {
  __shared__ uint64_t X, Y;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&X)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&Y)));
  }
  if (COMMIT && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t par = i & 1;
    if (warp == 0) {
      if (lane == 0) arrive(&X);
      wait<HINT>(&Y, par);
    } else if (warp == 1) {
      wait<HINT>(&X, par);
      if (lane == 0) {
        if (COMMIT) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&Y)) : "memory");
        else arrive(&Y);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *out = (t1 - t0) / iters;
  __syncthreads();
  if (COMMIT && warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(slot));
}

int main() {
  long long* d; cudaMallocManaged(&d, 8);
  const int it = 20000;
  pingpong<false, false><<<1, 64>>>(it, d); cudaDeviceSynchronize(); printf("arrive, spin      : %lld cycles/round trip (%s)\n", *d, cudaGetErrorString(cudaGetLastError()));
  pingpong<true, false><<<1, 64>>>(it, d); cudaDeviceSynchronize(); printf("arrive, hint      : %lld cycles/round trip\n", *d);
  pingpong<false, true><<<1, 64>>>(it, d); cudaDeviceSynchronize(); printf("commit, spin      : %lld cycles/round trip (%s)\n", *d, cudaGetErrorString(cudaGetLastError()));
  pingpong<true, true><<<1, 64>>>(it, d); cudaDeviceSynchronize(); printf("commit, hint      : %lld cycles/round trip\n", *d);
  return 0;
}
