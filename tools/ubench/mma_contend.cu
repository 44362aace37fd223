// Does concurrent tcgen05.ld / st traffic from other warps slow tcgen05.mma (TS, f16, N=64)?
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
#define R16 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}"
__global__ void k(int mode, int n_mma, long long* out, uint32_t* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { stop = 0; asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = tid; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (warp < 16) {
    const uint32_t my = t + ((uint32_t)((warp & 3) * 32) << 16) + 256 + (warp >> 2) * 64;
    uint32_t v[16], acc = 0;
    for (int i = 0; i < 16; ++i) v[i] = i;
    long long n = 0;
    while (!stop && mode != 0) {
      if (mode == 1) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 " R16 ", [%16];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]) : "r"(my));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        acc += v[0] ^ v[15];
      } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" :: "r"(my), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        v[0] += 1;
      }
      ++n;
    }
    sink[tid] = acc + (uint32_t)n;
    if (lane == 0) atomicAdd((unsigned long long*)&out[2], (unsigned long long)n);
  } else if (tid == 16 * 32) {
    // wait a bit so loaders are running
    long long w0 = clock64(); while (clock64() - w0 < 20000) {}
    const uint32_t idesc = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | (8u << 24);
    const uint32_t b = su32(sm);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int j = i & 7;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" :: "r"(t), "r"(t + 128 + 8 * j), "l"(desc(b + j * 256, 8 * 128, 128)), "r"(idesc), "r"(i > 0 ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&mbar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
    long long t1 = clock64();
    out[0] = (t1 - t0) * 100 / n_mma;
    out[1] = t1 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}
int main() {
  long long* o; uint32_t* sink; cudaMallocManaged(&o, 64); cudaMalloc(&sink, 4096 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  const char* nm[3] = {"alone", "16 warps tcgen05.ld", "16 warps tcgen05.st"};
  for (int mode = 0; mode < 3; ++mode) {
    o[2] = 0;
    k<<<1, 17 * 32, 32 * 1024>>>(mode, 4000, o, sink);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-22s: %.2f cycles/MMA (f16 TS N=64); other-warp ops %lld over %lld cycles -> %.1f B/clk  (%s)\n", nm[mode], o[0] / 100.0, o[2], o[1],
           o[2] * 2048.0 / o[1], cudaGetErrorString(e));
  }
}
