// MMA issue-rate / correctness probe: kind::i8 SS (M=128,N=32,K=32) and kind::f16 TS
// (M=128,N=64,K=16), K-major operands with SWIZZLE_NONE vs SWIZZLE_128B layouts.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | ((uint64_t)layout << 61);
}
// image offsets: K-major, rows R, row bytes KB (multiple of 128 for SW128)
__host__ __device__ uint32_t off_none(int r, int kb, int R) { return ((kb / 16) * (R / 8) + r / 8) * 128 + (r % 8) * 16 + (kb % 16); }
__host__ __device__ uint32_t off_sw128(int r, int kb, int R) {
  const int atom = kb / 128, c = kb % 128;
  return atom * (R * 128) + r * 128 + (((c / 16) ^ (r % 8)) * 16) + (c % 16);
}
template <bool SW>
__global__ void i8_rate(const int8_t* A, const int8_t* B, int* D, int iters, long long* cyc) {
  constexpr int M = 128, N = 32, KT = 256;   // 256 bytes of K per row = 2 SW128 atoms
  __shared__ __align__(1024) int8_t sA[M * KT];
  __shared__ __align__(1024) int8_t sB[N * KT];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = tid; i < M * KT; i += blockDim.x) { int r = i / KT, k = i % KT; sA[SW ? off_sw128(r, k, M) : off_none(r, k, M)] = A[i]; }
  for (int i = tid; i < N * KT; i += blockDim.x) { int r = i / KT, k = i % KT; sB[SW ? off_sw128(r, k, N) : off_none(r, k, N)] = B[i]; }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < KT / 32; ++j) {
        uint64_t da, db;
        if (SW) {
          da = desc(su32(sA) + (j / 4) * M * 128 + (j % 4) * 32, 16, 1024, 2);
          db = desc(su32(sB) + (j / 4) * N * 128 + (j % 4) * 32, 16, 1024, 2);
        } else {
          da = desc(su32(sA) + j * 2 * (M / 8) * 128, (M / 8) * 128, 128, 0);
          db = desc(su32(sB) + j * 2 * (N / 8) * 128, (N / 8) * 128, 128, 0);
        }
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" :: "r"(t), "l"(da), "l"(db), "r"(idesc), "r"((it | j) ? 1u : 0u));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&mbar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
    *cyc = (clock64() - t0) / ((long long)iters * (KT / 32));
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
    : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
    : "r"(t + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) D[tid * N + n] = (int)v[n];
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(t));
}

__global__ void i8_ts_rate(const int8_t* A, const int8_t* B, int* D, int iters, long long* cyc) {
  constexpr int M = 128, N = 32, KT = 256;
  __shared__ __align__(1024) int8_t sB[N * KT];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = tid; i < N * KT; i += blockDim.x) { int r = i / KT, k = i % KT; sB[off_none(r, k, N)] = B[i]; }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  // A row tid -> TMEM lane tid, columns 64.. (64 cols = 256 bytes), 4 bytes per column little endian
  {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(A + tid * KT);
    for (int cb = 0; cb < 64; cb += 8) {
      uint32_t v0=row[cb],v1=row[cb+1],v2=row[cb+2],v3=row[cb+3],v4=row[cb+4],v5=row[cb+5],v6=row[cb+6],v7=row[cb+7];
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "r"(t + ((uint32_t)(warp*32) << 16) + 64 + cb), "r"(v0),"r"(v1),"r"(v2),"r"(v3),"r"(v4),"r"(v5),"r"(v6),"r"(v7));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < KT / 32; ++j) {
        uint64_t db = desc(su32(sB) + j * 2 * (N / 8) * 128, (N / 8) * 128, 128, 0);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" :: "r"(t), "r"(t + 64 + 8 * j), "l"(db), "r"(idesc), "r"((it | j) ? 1u : 0u));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&mbar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
    *cyc = (clock64() - t0) / ((long long)iters * (KT / 32));
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(su32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
    : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
    : "r"(t + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) D[tid * N + n] = (int)v[n];
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(t));
}
int main() {
  const int M = 128, N = 32, KT = 256;
  int8_t *A, *B; int* D; long long* cyc;
  cudaMallocManaged(&A, M * KT); cudaMallocManaged(&B, N * KT); cudaMallocManaged(&D, M * N * 4); cudaMallocManaged(&cyc, 8);
  srand(5);
  for (int i = 0; i < M * KT; ++i) A[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < N * KT; ++i) B[i] = (int8_t)(rand() % 256 - 128);
  for (int sw = 0; sw < 2; ++sw) {
    const int iters = 200;
    if (sw) i8_rate<true><<<1, 128>>>(A, B, D, iters, cyc); else i8_rate<false><<<1, 128>>>(A, B, D, iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    int bad = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
      long long ref = 0; for (int k = 0; k < KT; ++k) ref += (int)A[m * KT + k] * (int)B[n * KT + k];
      if (ref * iters != D[m * N + n]) ++bad;
    }
    if (sw == 1) {
      i8_ts_rate<<<1, 128>>>(A, B, D, iters, cyc); cudaError_t e2 = cudaDeviceSynchronize(); int bad2 = 0;
      for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { long long ref = 0; for (int k = 0; k < KT; ++k) ref += (int)A[m * KT + k] * (int)B[n * KT + k]; if (ref * iters != D[m * N + n]) ++bad2; }
      printf("i8 TS M128 N32 K32: %lld cycles/MMA, %s, %d mismatches\n", *cyc, cudaGetErrorString(e2), bad2);
    }
    printf("i8 SS M128 N32 K32 %s: %lld cycles/MMA, %s, %d mismatches\n", sw ? "SW128" : "NONE ", *cyc, cudaGetErrorString(e), bad);
  }
}
