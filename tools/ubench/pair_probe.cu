// cta_group::2 semantics probe: which CTA's shared memory supplies which B rows, whether A
// comes from each CTA's own shared memory / TMEM, where D lands, and multicast commits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o pair_probe pair_probe.cu && ./pair_probe
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// K-major canonical image offset (bytes) of (row r, k) for R rows, 2-byte elements
__device__ __forceinline__ uint32_t koff(int r, int k, int R) {
  return (uint32_t)(((k / 8) * (R / 8) + r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int N = 64;
// MODE 0: SS (A and B in shared memory); MODE 1: TS (A in TMEM)
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out, int* flag) {
  __shared__ __align__(1024) unsigned char sA[128 * 16 * 2];
  __shared__ __align__(1024) unsigned char sB[N * 16 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t r = cluster_rank();
  // A_r[m][k] = 1 + r if k == 0 else 0; B_r[n][k] = (k == 0) ? 1000 r + n : 0
  for (int i = tid; i < 128 * 16; i += 128) {
    const int m = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sA + koff(m, k, 128)) = __float2half(k == 0 ? (float)(1 + r) : 0.f);
  }
  for (int i = tid; i < N * 16; i += 128) {
    const int n = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sB + koff(n, k, N)) = __float2half(k == 0 ? (float)(100 * r + n) : 0.f);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (MODE == 1) {   // A rows of this CTA into its TMEM columns 64.. (f16 pairs per 32-bit column)
    uint32_t v[8];
    const int m = warp * 32 + lane;
    for (int c = 0; c < 8; ++c) {
      const __half2 h = __floats2half2_rn(2 * c == 0 ? (float)(1 + r) : 0.f, 0.f);
      v[c] = *reinterpret_cast<const uint32_t*>(&h);
    }
    (void)m;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t + ((warp * 32) << 16) + 64),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // M = 256 (idesc M field 256 >> 4 = 16), N = 64
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (16u << 24);
  if (r == 0 && warp == 0) {
    const uint64_t bd = desc(su32(sB), (N / 8) * 128, 128);
    if (MODE == 0) {
      const uint64_t ad = desc(su32(sA), (128 / 8) * 128, 128);
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                   "@q tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 0;\n}" ::"r"(t), "l"(ad), "l"(bd), "r"(idesc));
    } else {
      asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                   "@q tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 0;\n}" ::"r"(t), "r"(t + 64), "l"(bd), "r"(idesc));
    }
    asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                 "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(su32(&bar)),
                 "h"((unsigned short)3));
  }
  // both CTAs wait for the multicast commit on their own barrier
  {
    uint32_t done = 0;
    long long spins = 0;
    while (!done && spins < 20000000) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(su32(&bar)), "r"(0u) : "memory");
      ++spins;
    }
    if (!done && tid == 0) atomicAdd(flag, 1 + (int)r * 10);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t d[N];
  for (int c = 0; c < N; c += 16)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(d[c]), "=r"(d[c + 1]), "=r"(d[c + 2]), "=r"(d[c + 3]), "=r"(d[c + 4]), "=r"(d[c + 5]),
                   "=r"(d[c + 6]), "=r"(d[c + 7]), "=r"(d[c + 8]), "=r"(d[c + 9]), "=r"(d[c + 10]), "=r"(d[c + 11]),
                   "=r"(d[c + 12]), "=r"(d[c + 13]), "=r"(d[c + 14]), "=r"(d[c + 15])
                 : "r"(t + ((warp * 32) << 16) + c));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int m = warp * 32 + lane;
  for (int c = 0; c < N; ++c) out[((size_t)r * 128 + m) * N + c] = __uint_as_float(d[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(t));
}

template <int MODE>
static void run(const char* name) {
  float* d_out;
  int* d_flag;
  cudaMalloc(&d_out, 2 * 128 * N * sizeof(float));
  cudaMalloc(&d_flag, sizeof(int));
  cudaMemset(d_out, 0xff, 2 * 128 * N * sizeof(float));
  cudaMemset(d_flag, 0, sizeof(int));
  probe<MODE><<<2, 128>>>(d_out, d_flag);
  cudaError_t e = cudaDeviceSynchronize();
  float h[2 * 128 * N];
  int flag = 0;
  cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
  cudaMemcpy(&flag, d_flag, sizeof flag, cudaMemcpyDeviceToHost);
  printf("== %s: %s, wait-timeout flag %d\n", name, cudaGetErrorString(e), flag);
  for (int r = 0; r < 2; ++r)
    for (int m : {0, 1, 127}) {
      printf("CTA %d row %3d:", r, m);
      for (int c : {0, 1, 2, 31, 32, 33, 63}) printf(" [%d]=%g", c, h[((size_t)r * 128 + m) * N + c]);
      printf("\n");
    }
  cudaFree(d_out);
  cudaFree(d_flag);
}

int main() {
  run<0>("SS f16 M=256 N=64");
  run<1>("TS f16 M=256 N=64 (A from each CTA's TMEM)");
  return 0;
}
