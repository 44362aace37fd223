// tcgen05.mma issue-rate sweep (timing only): kind::i8 / kind::f16, SS and TS, M=128, N varied.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <int KIND, bool TS, int N, int NACC = 1, int DATA = 1>   // KIND 0 = i8 (K=32 bytes), 1 = f16 (K=16)
__global__ void rate(int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<uint32_t*>(sm)[i] = DATA == 0 ? 0u : (DATA == 1 ? (h & 0x3bff3bffu) : 0x3c003c00u);   // 0, random |x|<1 f16 pairs, ones
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  {  // A operand region in TMEM (cols 256..511) filled with the same data class
    uint32_t h = tid * 2654435761u;
    for (int cb = 256; cb < 512; cb += 1) {
      h ^= h << 13; h ^= h >> 17; h ^= h << 5;
      const uint32_t v = DATA == 0 ? 0u : (DATA == 1 ? (h & 0x3bff3bffu) : 0x3c003c00u);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(t + ((uint32_t)((tid >> 5) * 32) << 16) + cb), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (tid == 0) {
    const uint32_t idesc = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24))
                                     : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24));
    const uint32_t a = su32(sm), b = su32(sm + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint64_t db = desc(b + j * 256, (N / 8) * 128, 128);
        const uint32_t acc = (it > 0 || j >= NACC) ? 1u : 0u;
        if (TS) {
          if (KIND == 0) asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" :: "r"(t + (j % NACC) * 64), "r"(t + 256 + 8 * j), "l"(db), "r"(idesc), "r"(acc));
          else asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" :: "r"(t + (j % NACC) * 64), "r"(t + 256 + 8 * j), "l"(db), "r"(idesc), "r"(acc));
        } else {
          const uint64_t da = desc(a + j * 256, 16 * 128, 128);
          if (KIND == 0) asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" :: "r"(t), "l"(da), "l"(db), "r"(idesc), "r"(acc));
          else asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(t), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&mbar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
    *cyc = (clock64() - t0) * 100 / ((long long)iters * 8);
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}
template <int KIND, bool TS, int N, int NACC = 1, int DATA = 1> void run(long long* cyc) {
  cudaFuncSetAttribute(rate<KIND, TS, N, NACC, DATA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  rate<KIND, TS, N, NACC, DATA><<<1, 128, 48 * 1024>>>(400, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  printf("data=%d %s %s N=%3d nacc=%d: %6.2f cycles/MMA  (%s)\n", DATA, KIND ? "f16" : "i8 ", TS ? "TS" : "SS", N, NACC, *cyc / 100.0, cudaGetErrorString(e));
}
int main() {
  long long* cyc; cudaMallocManaged(&cyc, 8);
  run<1, true, 64, 1, 0>(cyc); run<1, true, 64, 1, 1>(cyc); run<1, true, 64, 1, 2>(cyc);
  run<1, true, 128, 1, 0>(cyc); run<1, true, 128, 1, 1>(cyc); run<1, true, 128, 1, 2>(cyc);
  run<1, true, 256, 1, 0>(cyc); run<1, true, 256, 1, 1>(cyc); run<1, true, 256, 1, 2>(cyc);
  run<1, false, 64, 1, 1>(cyc); run<1, false, 128, 1, 1>(cyc); run<1, false, 256, 1, 1>(cyc);
  run<0, true, 128, 1, 0>(cyc); run<0, true, 128, 1, 1>(cyc); run<0, true, 128, 1, 2>(cyc);
  run<0, false, 128, 1, 1>(cyc); run<0, false, 256, 1, 1>(cyc);
}
