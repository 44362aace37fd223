// Probe: tcgen05.mma kind::i8 (s8 x s8 -> s32), SS form, M=128, N=32, K=64 (2 MMAs of K=32),
// K-major SWIZZLE_NONE layouts (16-byte core-matrix rows = 16 K values).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#define M 128
#define N 32
#define KT 64
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// byte offset of (row r, k) in a K-major interleaved image with R rows: unit (k/16, r/8), row r%8
__host__ __device__ uint32_t off(int r, int k, int R) { return ((k / 16) * (R / 8) + r / 8) * 128 + (r % 8) * 16 + (k % 16); }
__global__ void probe(const int8_t* A, const int8_t* B, int* D) {
  __shared__ __align__(1024) int8_t sA[M * KT];
  __shared__ __align__(1024) int8_t sB[N * KT];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = tid; i < M * KT; i += blockDim.x) { int r = i / KT, k = i % KT; sA[off(r, k, M)] = A[i]; }
  for (int i = tid; i < N * KT; i += blockDim.x) { int r = i / KT, k = i % KT; sB[off(r, k, N)] = B[i]; }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (tid == 0) {
    // c_format S32 = 2, a/b format signed 8-bit = 1, K-major, N>>3, M>>4
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < KT / 32; ++j) {
      uint64_t da = desc(su32(sA) + j * 2 * (M / 8) * 128, (M / 8) * 128, 128);
      uint64_t db = desc(su32(sB) + j * 2 * (N / 8) * 128, (N / 8) * 128, 128);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" :: "r"(t), "l"(da), "l"(db), "r"(idesc), "r"(j > 0 ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&mbar)));
  }
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
int main() {
  int8_t *A, *B; int* D;
  cudaMallocManaged(&A, M * KT); cudaMallocManaged(&B, N * KT); cudaMallocManaged(&D, M * N * 4);
  srand(3);
  for (int i = 0; i < M * KT; ++i) A[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < N * KT; ++i) B[i] = (int8_t)(rand() % 256 - 128);
  probe<<<1, 128>>>(A, B, D);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  int bad = 0;
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
    long long ref = 0; for (int k = 0; k < KT; ++k) ref += (int)A[m * KT + k] * (int)B[n * KT + k];
    if (ref != D[m * N + n]) { if (bad < 5) printf("m=%d n=%d ref=%lld got=%d\n", m, n, ref, D[m * N + n]); ++bad; }
  }
  printf("%s (%d mismatches)\n", bad ? "I8_PROBE_FAIL" : "I8_PROBE_OK", bad);
}
