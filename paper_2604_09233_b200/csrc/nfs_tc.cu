// nfs_tc.cu -- tensor-core (tcgen05, 3xTF32) generated-phase operator, NFS_PREC_TF32X3.
//
// The complex contraction of one operator (nfs/engine.py:98-108) is real-ified into a GEMM
//   D[o, n] = sum_j A[o, j] B[j, n],   o = owner (128 per CTA = TMEM lanes), n < 2*NC,
//   j = 2*item + {0: cos, 1: sin}, A = generated phasors, B = [[Xr, Xi], [-Xi, Xr]] per item,
// so D[o, c] = Re(sum e^{+-i phi} X), D[o, NC + c] = Im(...).  A is generated on the CUDA
// cores (same FP32 phase + MUFU sincos as the CUDA-core path, bit for bit), split into
// TF32 hi + lo and written straight into TMEM with tcgen05.st; B (hi/lo) is built once per
// operator call by a prep kernel in the UMMA K-major canonical layout and streamed into
// shared memory with cp.async.bulk (TMA bulk copies) on an mbarrier pipeline.  One elected
// thread issues tcgen05.mma.kind::tf32 in the TS form (A from TMEM, B from SMEM),
// D += Ahi Bhi + Ahi Blo + Alo Bhi  (3xTF32, FP32 accumulation in TMEM).
//
// Warp roles (320 threads): warps 0-7 generate A (warp w: TMEM lane quadrant w%4, half w/4
// of each chunk's items) and run the epilogue (warps 0-3); warp 8 = bulk-copy producer;
// warp 9 = MMA issuer.  Two CTAs per SM, 256 TMEM columns each (D 64 + 3 A stages x 64).
#include <stdio.h>

#include <string>

#include "nfs_common.cuh"
#include "nfs_phase.cuh"
#include "nfs_tc.cuh"
#include "nfs_vec.cuh"

namespace nfs {

static thread_local std::string g_tc_err;
const char* tc_last_error() { return g_tc_err.c_str(); }

namespace tc {

constexpr int IC = 16;          // streamed items per chunk (K = 32 real per chunk)
constexpr int KC = 2 * IC;      // real K per chunk
constexpr int SB = 4;           // shared-memory stages of B (+ table rows)
constexpr int SA = 2;           // TMEM stages of generated A
constexpr int SEG = 16;         // chunks accumulated in one TMEM D buffer before it is drained
constexpr int THREADS = 320;
constexpr int TMEM_COLS = 256;  // D0 [0,64) D1 [64,128) A stages [128,256)
constexpr int A_STAGE_COLS = 2 * KC;   // hi + lo

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) break;
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version for sm_100; SWIZZLE_NONE, base offset 0
  return d;
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// byte offset of real-K index j, column n inside one K-major interleaved B image (N columns)
__host__ __device__ __forceinline__ uint32_t bimg_off(int j, int n, int N) {
  return (uint32_t)(((j >> 2) * (N >> 3) + (n >> 3)) * 128 + (n & 7) * 16 + (j & 3) * 4);
}

struct Args {
  int nc;                 // coils per group (8, 16, 32); N = 2 * nc
  int nt;
  int n_groups, ldc;
  int64_t n_own, n_str;
  int n_chunks_total;     // ceil(n_str / IC)
  int n_split;
  const float* own_tab;   // [n_own][nt]
  const float* tab_img;   // [chunk][IC/2][nt][2]
  const float* b_img;     // [group][chunk][2 (hi, lo)][KC x N]
  const float2* sens;     // S' [L][ldc] (adjoint epilogue)
  float2* out;            // fwd: partial y [split][K][ldc]; adj: partial q [group*split+split][L]
  const int* stop;
};

// ------------------------------------------------------------------ main kernel
template <int NC, int NT, bool FWD>
__global__ void __launch_bounds__(THREADS, 2) tc_contract_kernel(Args a) {
  constexpr int N = 2 * NC;
  constexpr uint32_t B_IMG_BYTES = KC * N * 4;            // one of hi / lo
  constexpr uint32_t B_STAGE_BYTES = 2 * B_IMG_BYTES;
  constexpr uint32_t T_STAGE_BYTES = IC * NT * 4;
  if (a.stop != nullptr && *a.stop) return;

  // shared memory: B stages | table stages | FP32 accumulator [N][128] | mbarriers | tmem slot
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sB = smem;
  float* sT = reinterpret_cast<float*>(smem + SB * B_STAGE_BYTES);
  float* sAcc = reinterpret_cast<float*>(smem + SB * (B_STAGE_BYTES + T_STAGE_BYTES));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAcc + N * 128);
  uint64_t* full_b = bars;              // [SB] producer -> generators, MMA (tx bytes)
  uint64_t* empty_b = bars + SB;        // [SB] MMA commit -> producer
  uint64_t* full_a = empty_b + SB;      // [SA] generators (8 warps) -> MMA
  uint64_t* empty_a = full_a + SA;      // [SA] MMA commit -> generators
  uint64_t* dfull = empty_a + SA;       // [2]  MMA commit -> drain warps
  uint64_t* dempty = dfull + 2;         // [2]  drain warps (4) -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int group = blockIdx.y / a.n_split;
  const int split = blockIdx.y - group * a.n_split;
  const int per = (a.n_chunks_total + a.n_split - 1) / a.n_split;
  const int chunk0 = split * per;
  const int n_chunks = max(0, min(a.n_chunks_total, chunk0 + per) - chunk0);
  const int n_segs = (n_chunks + SEG - 1) / SEG;
  const int64_t own0 = (int64_t)blockIdx.x * 128;

  if (tid == 0) {
    for (int s = 0; s < SB; ++s) { mbar_init(&full_b[s], 1); mbar_init(&empty_b[s], 1); }
    for (int s = 0; s < SA; ++s) { mbar_init(&full_a[s], 8); mbar_init(&empty_a[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&dfull[s], 1); mbar_init(&dempty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < N * 128; i += THREADS) sAcc[i] = 0.f;
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;
  constexpr uint32_t A_COL0 = 128;

  if (warp < 8) {
    // ======================= A generators (+ D drain, warps 0-3) =======================
    const int q = warp & 3, h = warp >> 2;
    const int64_t o = own0 + q * 32 + lane;
    float own[NT];
#pragma unroll
    for (int p = 0; p < NT; ++p) own[p] = (o < a.n_own) ? a.own_tab[o * NT + p] : 0.f;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    int next_drain = 0;
    // TMEM D buffer of segment d -> smem accumulator (FP32, round-to-nearest adds)
    auto drain = [&](int d) {
      const int db = d & 1;
      mbar_wait(&dfull[db], (d >> 1) & 1);
      fence_after();
#pragma unroll
      for (int cb = 0; cb < N; cb += 16) {
        uint32_t v[16];
        tmem_ld16(tbase + lane_addr + db * 64 + cb, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) sAcc[(cb + i) * 128 + q * 32 + lane] += __uint_as_float(v[i]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[db]);
    };
    for (int c = 0; c < n_chunks; ++c) {
      const int sb = c % SB, sa = c % SA;
      mbar_wait(&full_b[sb], (c / SB) & 1);
      const float* tb = sT + sb * (T_STAGE_BYTES / 4);
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {           // 4 item pairs = 8 items of this half
        const float* row = tb + (h * 4 + pp) * NT * 2;
        float2 t;
        {
          const float4 v = *reinterpret_cast<const float4*>(row);
          t = __fmul2_rn(make_float2(own[0], own[0]), make_float2(v.x, v.y));
          t = __ffma2_rn(make_float2(own[1], own[1]), make_float2(v.z, v.w), t);
        }
#pragma unroll
        for (int p = 2; p < NT; p += 2) {
          const float4 v = *reinterpret_cast<const float4*>(row + 2 * p);
          t = __ffma2_rn(make_float2(own[p], own[p]), make_float2(v.x, v.y), t);
          t = __ffma2_rn(make_float2(own[p + 1], own[p + 1]), make_float2(v.z, v.w), t);
        }
        float s0, c0, s1, c1;
        turns_sincos_generic(t.x, s0, c0);
        turns_sincos_generic(t.y, s1, c1);
        if (!FWD) { s0 = -s0; s1 = -s1; }
        const float vals[4] = {c0, s0, c1, s1};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float vh = tf32_rna(vals[e]);
          hi[pp * 4 + e] = __float_as_uint(vh);
          lo[pp * 4 + e] = __float_as_uint(tf32_rna(vals[e] - vh));
        }
      }
      mbar_wait(&empty_a[sa], ((c / SA) & 1) ^ 1);   // MMAs of chunk c - SA drained A stage sa
      fence_after();
      const uint32_t col = A_COL0 + sa * (2 * KC) + h * 16;
      tmem_st16(tbase + lane_addr + col, hi);
      tmem_st16(tbase + lane_addr + col + KC, lo);
      tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_a[sa]);
      // drain segment d half-way through segment d+1 (the MMA is then on the other buffer)
      if (warp < 4 && next_drain < c / SEG && (c % SEG) >= SEG / 2) drain(next_drain++);
    }
    if (warp < 4) {
      while (next_drain < n_segs) drain(next_drain++);
      __syncwarp();
      if (o < a.n_own) {
        const int c0 = group * NC;
        const float* acc = sAcc + q * 32 + lane;   // acc[n * 128]
        if constexpr (FWD) {
          float2* out = a.out + (int64_t)split * a.n_own * a.ldc + o * a.ldc + c0;
#pragma unroll
          for (int c = 0; c < NC; ++c) out[c] = make_float2(acc[c * 128], acc[(NC + c) * 128]);
        } else {
          float qx = 0.f, qy = 0.f;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const float2 sv = a.sens[o * a.ldc + c0 + c];   // conj(S') * acc
            const float ar = acc[c * 128], ai = acc[(NC + c) * 128];
            qx = fmaf(sv.x, ar, qx);
            qx = fmaf(sv.y, ai, qx);
            qy = fmaf(sv.x, ai, qy);
            qy = fmaf(-sv.y, ar, qy);
          }
          a.out[(int64_t)blockIdx.y * a.n_own + o] = make_float2(qx, qy);
        }
      }
    }
  } else if (warp == 8) {
    // ======================= bulk-copy producer =======================
    if (lane == 0) {
      for (int c = 0; c < n_chunks; ++c) {
        const int sb = c % SB;
        mbar_wait(&empty_b[sb], ((c / SB) & 1) ^ 1);
        const int gc = chunk0 + c;
        mbar_expect_tx(&full_b[sb], B_STAGE_BYTES + T_STAGE_BYTES);
        const unsigned char* bsrc = reinterpret_cast<const unsigned char*>(a.b_img) +
                                    ((size_t)group * a.n_chunks_total + gc) * B_STAGE_BYTES;
        bulk_g2s(sB + sb * B_STAGE_BYTES, bsrc, B_STAGE_BYTES, &full_b[sb]);
        bulk_g2s(sT + sb * (T_STAGE_BYTES / 4), a.tab_img + (size_t)gc * (IC * NT), T_STAGE_BYTES, &full_b[sb]);
      }
    }
  } else {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
      constexpr uint32_t LBO = (N / 8) * 128, SBO = 128;
      for (int c = 0; c < n_chunks; ++c) {
        const int sb = c % SB, sa = c % SA, seg = c / SEG, db = seg & 1;
        if (c % SEG == 0) {
          mbar_wait(&dempty[db], ((seg >> 1) & 1) ^ 1);   // segment seg-2 drained from buffer db
          fence_after();
        }
        mbar_wait(&full_b[sb], (c / SB) & 1);
        mbar_wait(&full_a[sa], (c / SA) & 1);
        fence_after();
        const uint32_t d_tmem = tbase + db * 64;
        const uint32_t bhi = smem_u32(sB + sb * B_STAGE_BYTES), blo = bhi + B_IMG_BYTES;
        const uint32_t ahi = tbase + A_COL0 + sa * (2 * KC), alo = ahi + KC;
#pragma unroll
        for (int t = 0; t < KC / 8; ++t) {
          const uint32_t boff = (uint32_t)(2 * t) * LBO;
          const uint32_t acc = (c % SEG != 0 || t > 0) ? 1u : 0u;
          mma_tf32_ts(d_tmem, ahi + 8 * t, smem_desc(bhi + boff, LBO, SBO), idesc, acc);
          mma_tf32_ts(d_tmem, ahi + 8 * t, smem_desc(blo + boff, LBO, SBO), idesc, 1u);
          mma_tf32_ts(d_tmem, alo + 8 * t, smem_desc(bhi + boff, LBO, SBO), idesc, 1u);
        }
        mma_commit(&empty_b[sb]);
        mma_commit(&empty_a[sa]);
        if (c % SEG == SEG - 1 || c == n_chunks - 1) mma_commit(&dfull[db]);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ B image prep
// item i of chunk ch, coil c of group g:  x = X[i][g*NC + c] (forward: S' * p on the fly)
// rows n = c: (j=2il: xr, j=2il+1: -xi);  n = NC + c: (j=2il: xi, j=2il+1: xr); hi/lo split.
template <int NC, bool FWD>
__global__ void prep_b_kernel(const float2* __restrict__ x, const float2* __restrict__ sens,
                              const double2* __restrict__ p, int64_t n_str, int ldc, int n_groups,
                              int n_chunks, float* __restrict__ img, const int* stop) {
  if (stop && *stop) return;
  constexpr int N = 2 * NC;
  const int64_t total = (int64_t)n_groups * n_chunks * IC * NC;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx % NC);
    const int64_t r = idx / NC;
    const int il = (int)(r % IC);
    const int64_t gc = r / IC;                    // group * n_chunks + chunk
    const int g = (int)(gc / n_chunks);
    const int64_t item = (gc - (int64_t)g * n_chunks) * IC + il;
    float xr = 0.f, xi = 0.f;
    if (item < n_str) {
      const float2 v = (FWD ? sens : x)[item * ldc + g * NC + c];
      if (FWD) {
        const double2 pv = p[item];
        const float pr = (float)pv.x, pi = (float)pv.y;
        xr = v.x * pr - v.y * pi;
        xi = v.x * pi + v.y * pr;
      } else {
        xr = v.x;
        xi = v.y;
      }
    }
    float* hi = img + gc * (2 * KC * N);
    float* lo = hi + KC * N;
    const float vals[4] = {xr, -xi, xi, xr};   // (j0,n=c) (j1,n=c) (j0,n=NC+c) (j1,n=NC+c)
    const int js[4] = {2 * il, 2 * il + 1, 2 * il, 2 * il + 1};
    const int ns[4] = {c, c, NC + c, NC + c};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float vh = tf32_rna(vals[e]);
      const uint32_t off = bimg_off(js[e], ns[e], N) / 4;
      hi[off] = vh;
      lo[off] = tf32_rna(vals[e] - vh);
    }
  }
}

// streamed table rows -> chunk images [chunk][IC/2 pairs][nt][2]
__global__ void prep_tab_kernel(const float* __restrict__ tab, int64_t n_str, int nt, int n_chunks,
                                float* __restrict__ img) {
  const int64_t total = (int64_t)n_chunks * IC * nt;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(idx % nt);
    const int64_t item = idx / nt;
    const int64_t ch = item / IC;
    const int il = (int)(item % IC);
    const float v = item < n_str ? tab[item * nt + p] : 0.f;
    img[ch * IC * nt + ((il >> 1) * nt + p) * 2 + (il & 1)] = v;
  }
}

}  // namespace tc

// ------------------------------------------------------------------ host plan
struct TcPlan {
  int64_t K = 0, L = 0;
  int G = 0, nt = 0, nc = 0, n_groups = 0, ldc = 0, sms = 148;
  int chunks_f = 0, chunks_a = 0, split_f = 1, split_a = 1;
  const float* d_T = nullptr;   // [K][nt]
  const float* d_R = nullptr;   // [L][nt]
  const float2* d_S = nullptr;  // [L][ldc]
  float *img_f = nullptr, *img_a = nullptr, *tab_f = nullptr, *tab_a = nullptr;
  float2 *part_y = nullptr, *part_q = nullptr;
  size_t smem = 0;
  std::string desc;
};

static int tc_fail(const std::string& m) {
  g_tc_err = m;
  return 1;
}

int tc_coil_width(int G) { return G <= 8 ? 8 : (G <= 16 ? 16 : 32); }

template <int NC, int NT, bool FWD>
static void* tc_kernel_ptr() { return (void*)tc::tc_contract_kernel<NC, NT, FWD>; }

template <int NC, bool FWD>
static void* tc_kernel_nt(int nt) {
  switch (nt) {
    case 4: return tc_kernel_ptr<NC, 4, FWD>();
    case 8: return tc_kernel_ptr<NC, 8, FWD>();
    case 16: return tc_kernel_ptr<NC, 16, FWD>();
    case 20: return tc_kernel_ptr<NC, 20, FWD>();
    case 32: return tc_kernel_ptr<NC, 32, FWD>();
  }
  return nullptr;
}

static void* tc_kernel(int nc, int nt, bool fwd) {
  switch (nc) {
    case 8: return fwd ? tc_kernel_nt<8, true>(nt) : tc_kernel_nt<8, false>(nt);
    case 16: return fwd ? tc_kernel_nt<16, true>(nt) : tc_kernel_nt<16, false>(nt);
    case 32: return fwd ? tc_kernel_nt<32, true>(nt) : tc_kernel_nt<32, false>(nt);
  }
  return nullptr;
}

static size_t tc_smem_bytes(int nc, int nt) {
  const size_t b = 2ull * tc::KC * (2 * nc) * 4, t = (size_t)tc::IC * nt * 4;
  return tc::SB * (b + t) + (size_t)(2 * nc) * 128 * 4 + (2 * tc::SB + 2 * tc::SA + 4) * 8 + 16;
}

static int pick_split(int64_t tiles, int chunks, int resident) {
  const int cap = std::max(1, std::min(64, chunks / 4));
  int best = 1;
  double best_eff = -1;
  for (int s = 1; s <= cap; ++s) {
    const double waves = (double)(tiles * s) / resident;
    if (waves < 1.0 && s < cap) continue;
    const double eff = waves / std::ceil(waves);
    if (eff >= 0.97 && waves >= 2.0) return s;
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return best;
}

TcPlan* tc_create(int64_t K, int64_t L, int G, int nt, int sms, std::string* why) {
  TcPlan* t = new TcPlan();
  t->K = K; t->L = L; t->G = G; t->nt = nt; t->sms = sms;
  t->nc = tc_coil_width(G);
  t->n_groups = (G + t->nc - 1) / t->nc;
  t->ldc = t->nc * t->n_groups;
  t->chunks_f = (int)((L + tc::IC - 1) / tc::IC);
  t->chunks_a = (int)((std::max<int64_t>(K, 1) + tc::IC - 1) / tc::IC);
  t->smem = tc_smem_bytes(t->nc, nt);
  // keep two CTAs per SM (TMEM: 2 x 256 columns); pad smem so a third cannot co-reside
  const size_t smem_req = std::max<size_t>(t->smem, 80 * 1024);
  if (smem_req > 110 * 1024) { *why = "shared memory budget"; delete t; return nullptr; }
  for (int fwd = 0; fwd < 2; ++fwd) {
    void* k = tc_kernel(t->nc, nt, fwd != 0);
    if (!k) { *why = "unsupported term count"; delete t; return nullptr; }
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_req) != cudaSuccess) {
      *why = "cannot set dynamic shared memory";
      delete t;
      return nullptr;
    }
  }
  t->smem = smem_req;
  const int resident = sms * 2;
  const int64_t tiles_f = (std::max<int64_t>(K, 1) + 127) / 128 * t->n_groups;
  const int64_t tiles_a = (L + 127) / 128 * t->n_groups;
  t->split_f = pick_split(tiles_f, t->chunks_f, resident);
  t->split_a = pick_split(tiles_a, t->chunks_a, resident);
  const size_t img_chunk = 2ull * tc::KC * (2 * t->nc);   // floats per chunk (hi + lo)
  auto al = [&](void** p, size_t bytes) { return cudaMalloc(p, std::max<size_t>(bytes, 256)) == cudaSuccess; };
  bool ok = al((void**)&t->img_f, img_chunk * t->chunks_f * t->n_groups * 4) &&
            al((void**)&t->img_a, img_chunk * t->chunks_a * t->n_groups * 4) &&
            al((void**)&t->tab_f, (size_t)t->chunks_f * tc::IC * nt * 4) &&
            al((void**)&t->tab_a, (size_t)t->chunks_a * tc::IC * nt * 4) &&
            al((void**)&t->part_y, (size_t)t->split_f * std::max<int64_t>(K, 1) * t->ldc * 8) &&
            al((void**)&t->part_q, (size_t)t->split_a * t->n_groups * L * 8);
  if (!ok) { *why = "device memory"; tc_destroy(t); return nullptr; }
  char buf[256];
  snprintf(buf, sizeof buf, " tc[nc=%d groups=%d chunks f/a=%d/%d split f/a=%d/%d smem=%zu]", t->nc,
           t->n_groups, t->chunks_f, t->chunks_a, t->split_f, t->split_a, t->smem);
  t->desc = buf;
  return t;
}

void tc_destroy(TcPlan* t) {
  if (!t) return;
  void* bufs[] = {t->img_f, t->img_a, t->tab_f, t->tab_a, t->part_y, t->part_q};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete t;
}

const char* tc_describe(TcPlan* t) { return t ? t->desc.c_str() : ""; }

static int grid_for(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 16); }

int tc_set_tables(TcPlan* t, const void* d_T, const void* d_R, cudaStream_t st) {
  t->d_T = (const float*)d_T;
  t->d_R = (const float*)d_R;
  tc::prep_tab_kernel<<<grid_for((int64_t)t->chunks_f * tc::IC * t->nt), 256, 0, st>>>(t->d_R, t->L, t->nt,
                                                                                        t->chunks_f, t->tab_f);
  tc::prep_tab_kernel<<<grid_for((int64_t)t->chunks_a * tc::IC * t->nt), 256, 0, st>>>(t->d_T, t->K, t->nt,
                                                                                        t->chunks_a, t->tab_a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return tc_fail(cudaGetErrorString(e));
  return 0;
}

int tc_set_sens(TcPlan* t, const void* d_S, int ldc, cudaStream_t) {
  if (ldc != t->ldc) return tc_fail("coil stride mismatch between plan and tensor-core path");
  t->d_S = (const float2*)d_S;
  return 0;
}

template <bool FWD>
static cudaError_t launch_prep(TcPlan* t, const float2* x, const double2* p, const int* stop, cudaStream_t st) {
  const int chunks = FWD ? t->chunks_f : t->chunks_a;
  const int64_t n_str = FWD ? t->L : t->K;
  float* img = FWD ? t->img_f : t->img_a;
  const int64_t total = (int64_t)t->n_groups * chunks * tc::IC * t->nc;
  const int gb = grid_for(total);
  switch (t->nc) {
    case 8: tc::prep_b_kernel<8, FWD><<<gb, 256, 0, st>>>(x, t->d_S, p, n_str, t->ldc, t->n_groups, chunks, img, stop); break;
    case 16: tc::prep_b_kernel<16, FWD><<<gb, 256, 0, st>>>(x, t->d_S, p, n_str, t->ldc, t->n_groups, chunks, img, stop); break;
    default: tc::prep_b_kernel<32, FWD><<<gb, 256, 0, st>>>(x, t->d_S, p, n_str, t->ldc, t->n_groups, chunks, img, stop); break;
  }
  return cudaGetLastError();
}

static cudaError_t launch_main(TcPlan* t, bool fwd, const int* stop, cudaStream_t st) {
  tc::Args a{};
  a.nc = t->nc;
  a.nt = t->nt;
  a.n_groups = t->n_groups;
  a.ldc = t->ldc;
  a.n_own = fwd ? t->K : t->L;
  a.n_str = fwd ? t->L : t->K;
  a.n_chunks_total = fwd ? t->chunks_f : t->chunks_a;
  a.n_split = fwd ? t->split_f : t->split_a;
  a.own_tab = fwd ? t->d_T : t->d_R;
  a.tab_img = fwd ? t->tab_f : t->tab_a;
  a.b_img = fwd ? t->img_f : t->img_a;
  a.sens = t->d_S;
  a.out = fwd ? t->part_y : t->part_q;
  a.stop = stop;
  if (a.n_own <= 0) return cudaSuccess;
  void* k = tc_kernel(t->nc, t->nt, fwd);
  dim3 grid((unsigned)((a.n_own + 127) / 128), (unsigned)(a.n_split * t->n_groups));
  void* args[] = {&a};
  return cudaLaunchKernel(k, grid, dim3(tc::THREADS), args, t->smem, st);
}

int tc_forward_parts(TcPlan* t, const double2* p, void* y, const int* stop, cudaStream_t st, int part) {
  cudaError_t e = cudaSuccess;
  if (part == 0) {
    e = launch_prep<true>(t, nullptr, p, stop, st);
    if (e == cudaSuccess) e = launch_main(t, true, stop, st);
  } else {
    e = launch_reduce_parts(0, t->part_y, y, t->K * t->ldc, t->split_f, stop, st);
  }
  if (e != cudaSuccess) return tc_fail(std::string("tc forward: ") + cudaGetErrorString(e));
  return 0;
}

int tc_adjoint_parts(TcPlan* t, const void* y, double2* q, const int* stop, cudaStream_t st, int part) {
  cudaError_t e = cudaSuccess;
  if (part == 0) {
    e = launch_prep<false>(t, (const float2*)y, nullptr, stop, st);
    if (e == cudaSuccess) e = launch_main(t, false, stop, st);
  } else {
    e = launch_reduce_image(0, t->part_q, q, t->L, t->split_a * t->n_groups, stop, st);
  }
  if (e != cudaSuccess) return tc_fail(std::string("tc adjoint: ") + cudaGetErrorString(e));
  return 0;
}

int tc_forward(TcPlan* t, const double2* p, void* y, const int* stop, cudaStream_t st) {
  if (t->K == 0) return 0;
  if (tc_forward_parts(t, p, y, stop, st, 0)) return 1;
  return tc_forward_parts(t, p, y, stop, st, 1);
}

int tc_adjoint(TcPlan* t, const void* y, double2* q, const int* stop, cudaStream_t st) {
  if (t->K == 0) {
    cudaMemsetAsync(q, 0, t->L * sizeof(double2), st);
    return 0;
  }
  if (tc_adjoint_parts(t, y, q, stop, st, 0)) return 1;
  return tc_adjoint_parts(t, y, q, stop, st, 1);
}

int tc_launches_per_apply(TcPlan*) { return 6; }

}  // namespace nfs
