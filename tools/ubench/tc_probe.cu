// tc_probe.cu -- validate the tcgen05 building blocks used by the tensor-core operator:
// TMEM alloc, tcgen05.st of A (TS form), K-major SWIZZLE_NONE B descriptor in smem,
// kind::tf32 MMA M=128 N=64, commit -> mbarrier, tcgen05.ld of D.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>

#define M 128
#define N 64
#define KT 32   // total K (4 MMAs of K=8)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (sm100)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__global__ void probe(const float* A, const float* B, float* D, int mode) {
  __shared__ __align__(1024) float sB[KT * N];     // canonical K-major interleave layout
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // B[k][n] (row-major K x N in global) -> smem: unit (g = n/8, r = n%8, u = k/4) at
  // u*1024 + g*128 + r*16 bytes, 4 consecutive k inside the unit.
  for (int i = tid; i < KT * N; i += blockDim.x) {
    const int k = i / N, n = i % N;
    const int u = k >> 2, e = k & 3, g = n >> 3, r = n & 7;
    sB[(u * 1024 + g * 128 + r * 16) / 4 + e] = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  const uint32_t d_col = 0, a_col = 64;

  // A row `tid` -> TMEM lane tid, columns a_col .. a_col+31
  {
    uint32_t v[32];
    for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(A[tid * KT + k]);
    const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + a_col;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < KT / 8; ++j) {
      const uint64_t bdesc = make_desc(smem_u32(sB) + j * 2048, 1024, 128);
      const uint32_t acc = j > 0 ? 1u : 0u;
      if (mode == 0) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tbase + d_col),
            "r"(tbase + a_col + 8 * j), "l"(bdesc), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  __syncwarp();
  // wait for MMA completion (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t v[64];
    const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + d_col;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,"
        "%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
          "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]),
          "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]),
          "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
          "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 64; ++n) D[tid * N + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128));
}

static float tf32(float x) {   // round-to-nearest-even to 10 mantissa bits (approx cvt.rna)
  uint32_t u; memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;
  float y; memcpy(&y, &u, 4);
  return y;
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, M * KT * 4); cudaMallocManaged(&B, KT * N * 4); cudaMallocManaged(&D, M * N * 4);
  srand(1);
  for (int i = 0; i < M * KT; ++i) A[i] = tf32((rand() / (float)RAND_MAX) - 0.5f);
  for (int i = 0; i < KT * N; ++i) B[i] = tf32((rand() / (float)RAND_MAX) - 0.5f);
  probe<<<1, 128>>>(A, B, D, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < KT; ++k) ref += (double)A[m * KT + k] * B[k * N + n];
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("max |D - ref| = %.3e (max |ref| %.3e)  D[0]=%f D[1]=%f D[64]=%f\n", maxerr, maxref, D[0], D[1], D[64]);
  printf("%s\n", maxerr < 1e-4 ? "TC_PROBE_OK" : "TC_PROBE_FAIL");
  return 0;
}
