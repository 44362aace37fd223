// tcgen05.mma issue-rate: lane-0 region (compiler waterfall per MMA) vs whole-warp elect.sync
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <int VARIANT, int N, int HAMMER = 0>
__global__ void k(int iters, long long* cyc) {
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
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  const uint32_t b = su32(sm);
  long long t0 = clock64();
  if (VARIANT == 0) {
    if (tid == 0) {
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" :: "r"(t), "r"(t + 256 + 8 * j), "l"(desc(b + j * 2048, 1024, 128)), "r"(idesc), "r"(1u));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&mbar)));
    }
  } else if (VARIANT == 1) {
    if (warp == 0) {
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" :: "r"(t), "r"(t + 256 + 8 * j), "l"(desc(b + j * 2048, 1024, 128)), "r"(idesc), "r"(1u));
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" :: "r"(su32(&mbar)));
    }
  } else if (VARIANT == 3) {   // SS: A from smem too (elected issue)
    if (warp == 0) {
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(t), "l"(desc(b + 16384 + j * 256, 2048, 128)), "l"(desc(b + j * 2048, 1024, 128)), "r"(idesc), "r"(1u));
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" :: "r"(su32(&mbar)));
    }
  } else {
    if (warp == 0) {
      const uint64_t d0 = desc(b, 1024, 128);
      for (int it = 0; it < iters; ++it)
        asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %5, %3, 1;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %7, %3, 1;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %9, %3, 1;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %5, %3, 1;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %7, %3, 1;\n"
                     "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %9, %3, 1;\n}"
                     :: "r"(t), "r"(t + 256), "l"(d0), "r"(idesc), "r"(t + 264), "l"(d0 + 128), "r"(t + 272), "l"(d0 + 256), "r"(t + 280), "l"(d0 + 384));
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" :: "r"(su32(&mbar)));
    }
  }
  if (HAMMER && warp > 0) {   // other warps stream shared memory (LDS.128 + STS.128)
    float4* p = reinterpret_cast<float4*>(sm + 32768);
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters * 4; ++it) {
      float4 v = p[(tid + it * 32) & 1023];
      acc.x += v.x; acc.y += v.y;
      if (HAMMER == 2) p[(tid + it * 64) & 1023] = acc;
    }
    if (acc.x == 12345.f) *cyc = 1;
  }
  if (tid == 0) {
    uint32_t done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
    *cyc = (clock64() - t0) * 100 / ((long long)iters * 8);
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}
template <int V, int N, int H = 0> void run(long long* c) {
  cudaFuncSetAttribute(k<V, N, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<V, N, H><<<1, H ? 512 : 128, 64 * 1024>>>(500, c);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d N=%3d hammer=%d: %.2f cycles/MMA (%s)\n", V, N, H, *c / 100.0, cudaGetErrorString(e));
}
int main() {
  long long* c; cudaMallocManaged(&c, 8);
  run<1, 64>(c); run<3, 64>(c); run<1, 128>(c); run<3, 128>(c); run<3, 256>(c);
  run<1, 64, 1>(c); run<3, 64, 1>(c); run<1, 64, 2>(c); run<3, 64, 2>(c);
}
