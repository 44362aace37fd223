// nfs_tc.cu -- tensor-core (tcgen05) generated-phase operator, split-precision MMA.
//
// The complex contraction of one operator (nfs/engine.py:98-108) is real-ified into a GEMM
//   D[o, n] = sum_j A[o, j] B[j, n],   o = owner (128 per CTA = TMEM lanes), n < 2*NC,
//   j = 2*item + {0: cos, 1: sin}, A = generated phasors e^{+i phi},
//   forward B rows per item: j0 = [Xr, Xi], j1 = [-Xi, Xr]   (e^{+i phi} X)
//   adjoint B rows per item: j0 = [Xr, Xi], j1 = [ Xi, -Xr]  (e^{-i phi} X, conj folded into B)
// so D[o, c] = Re(sum ...), D[o, NC + c] = Im(sum ...).
//
// A is generated on the CUDA cores (the FP32 phase FMA chain of the CUDA-core path, bit for
// bit, + MUFU sincos), split hi + lo and written straight into TMEM with tcgen05.st; B (hi/lo)
// is built once per operator call by a prep kernel in the UMMA K-major canonical layout and
// streamed into shared memory with cp.async.bulk on an mbarrier pipeline.  One elected thread
// issues tcgen05.mma in the TS form (A from TMEM, B from SMEM): D += Ah Bh + Ah Bl + Al Bh.
//   KIND_TF32: kind::tf32, hi/lo are TF32 (FP32 containers)
//   KIND_F16 : kind::f16, hi/lo are FP16 (B scaled by a power of two per call so its largest
//              entry is ~2^14); half the TMEM / SMEM bytes and twice the MMA rate of TF32.
// The TMEM accumulator is double-buffered and drained into an FP32 shared-memory accumulator
// every SEG chunks, the small split products of a chunk issued before its large one: the
// tensor core's accumulation truncates (biased error ~ steps x 2^-24 of |D|).  Measured on the
// masked config A (CG iterate vs the reference at iteration 10, SURVEY 8d bound 1e-5): SEG = 8
// 3.2e-5, 4: 1.5e-5, 2: 3.2e-6, 1: 1.1e-6; per-operator time 5.2 / 5.5 / 6.2 / 7.3 ms (config
// B).  SEG = 2 (32 items between drains) meets the bound.
//
// Warp roles (320 threads): warps 0-7 generate A (warp w: TMEM lane quadrant w%4, half w/4
// of each chunk's items); warps 0-3 also drain D and run the epilogue; warp 8 = bulk-copy
// producer; warp 9 = MMA issuer.  Two CTAs per SM, 256 TMEM columns each.
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
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
#ifndef NFS_TC_SEG
#define NFS_TC_SEG 2
#endif
constexpr int SEG = NFS_TC_SEG; // chunks accumulated in one TMEM D buffer before it is drained
constexpr int GPQ = 2;          // generator warps per TMEM lane quadrant (chunk c -> warp c % GPQ)
constexpr int GEN_WARPS = 4 * GPQ;
constexpr int THREADS = (GEN_WARPS + 2) * 32;
#ifndef NFS_TC_DEBUG
#define NFS_TC_DEBUG 0
#endif
// profiling builds only (-DNFS_TC_DEBUG=m): bit0 skip the phasor math, bit1 skip the MMAs,
// bit2 skip the TMEM stores, bit3 skip the bulk copies; compile-time so the product kernel
// carries no runtime branch in its inner loops
constexpr int TC_DEBUG = NFS_TC_DEBUG;
constexpr int CTAS_PER_SM = 2;
constexpr int TMEM_COLS = 512 / CTAS_PER_SM;  // D0 [0,64) D1 [64,128) A stages [128, TMEM_COLS)
constexpr int A_COL0 = 128;

template <bool F16> struct Kind {
  static constexpr int ebytes = F16 ? 2 : 4;               // bytes per operand element
  static constexpr int kstep = F16 ? 16 : 8;               // K per MMA instruction
  static constexpr int a_img_cols = KC * ebytes / 4;       // TMEM columns per A image (hi or lo)
  static constexpr int sa = (TMEM_COLS - A_COL0) / (2 * a_img_cols);   // A stages
  static constexpr uint32_t fmt = F16 ? 0u : 2u;           // F16 = 0, TF32 = 2
  static constexpr int sb = sa;                            // B stages tied to A stages
};

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
#ifndef NFS_TC_JITTER
#define NFS_TC_JITTER 0
#endif
// Race-detection builds only (tests/test_gpu_race_jitter.py, -DNFS_TC_JITTER=1): pseudo-random
// sleeps of up to ~2 us at one in four hand-offs of every warp role; compiled out otherwise.
__device__ __forceinline__ void jitter(uint32_t key) {
#if NFS_TC_JITTER
  uint32_t h = key * 2654435761u ^ (blockIdx.x * 40503u + blockIdx.y * 977u + 0x9e3779b9u);
  h ^= h >> 15;
  h *= 2246822519u;
  h ^= h >> 13;
  if ((h & 3u) == 0u) __nanosleep(h >> 21);
#else
  (void)key;
#endif
}

// wait for a single-thread role (producer, MMA issuer, drain): let the hardware suspend the
// warp instead of spinning, so it does not steal issue slots from the generator warps
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity), "r"(1000000)
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

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (canonical ((8,n),2):((1,SBO),LBO))
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version for sm_100; base offset 0
  return d;
}

template <bool F16>
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  if constexpr (F16)
    asm volatile(
        "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
        "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|q, 0xffffffff;\n"
        "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// issued by a converged warp: elect.sync inside the asm avoids ptxas' per-MMA waterfall loop
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
      : "memory");
}

// TF32 split: hi = round-half-away TF32 (finite x), lo = x - hi exact; the MMA truncates lo's
// low mantissa bits, |lo| <= 2^-12 |x| so the split error is <= 2^-22 |x|.
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  const uint32_t h = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  hi = h;
  lo = __float_as_uint(__fsub_rn(x, __uint_as_float(h)));
}

// FP16 split of a pair (x, y) into packed hi (x in the low half) and lo = (x, y) - hi
__device__ __forceinline__ void f16_split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  const float2 r = __fadd2_rn(make_float2(x, y), make_float2(-hf.x, -hf.y));
  const __half2 l = __floats2half2_rn(r.x, r.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// sin/cos of 2 pi t (t in turns): rint via the 1.5*2^23 magic constant (exact, |t| < 2^22,
// same value as rintf) keeps the range reduction on the FMA pipe, MUFU for sin/cos.
__device__ __forceinline__ void turns_sincos_fma(float t, float& s, float& c) {
  const float magic = 12582912.0f;
  const float r = __fsub_rn(__fadd_rn(t, magic), magic);
  const float f = __fsub_rn(t, r);
  __sincosf(f * 6.28318530717958647692f, &s, &c);
}

// packed range reduction of an item pair (FADD2 / FMUL2 on the FMA pipe), MUFU per item
__device__ __forceinline__ void turns_sincos_pair(float2 t, float& s0, float& c0, float& s1, float& c1) {
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  const float2 r = __fadd2_rn(__fadd2_rn(t, magic), make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __fadd2_rn(t, make_float2(-r.x, -r.y));
  const float2 a = __fmul2_rn(f, make_float2(6.28318530717958647692f, 6.28318530717958647692f));
  __sincosf(a.x, &s0, &c0);
  __sincosf(a.y, &s1, &c1);
}

template <int NCOL>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&v)[NCOL]) {
  static_assert(NCOL == 8 || NCOL == 16, "x8 / x16 only");
  if constexpr (NCOL == 16)
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
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

// byte offset of real-K index j, column n inside one K-major interleaved B image (N columns);
// a 16-byte core-matrix row holds 16/ebytes consecutive K values
template <int EB>
__host__ __device__ __forceinline__ uint32_t bimg_off(int j, int n, int N) {
  constexpr int KU = 16 / EB;   // K values per 16-byte unit
  return (uint32_t)(((j / KU) * (N >> 3) + (n >> 3)) * 128 + (n & 7) * 16 + (j % KU) * EB);
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
  const void* b_img;      // [group][chunk][2 (hi, lo)][KC x N]
  const float2* sens;     // S' [L][ldc] (adjoint epilogue)
  const float* scale;     // [1] B scale of this call (F16), device
  float2* out;            // fwd: partial y [split][K][ldc]
  double2* out_q;         // adj: partial q [group*split+split][L] (FP64)
  const int* stop;
  int unused_debug;       // (profiling switches are compile-time: NFS_TC_DEBUG)
  long long* trace;       // profiling only: per-chunk timestamps of CTA (0,0), or null
};

// ------------------------------------------------------------------ main kernel
template <int NC, int NT, bool FWD, bool F16>
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM) tc_contract_kernel(Args a) {
  using K_ = Kind<F16>;
  constexpr int N = 2 * NC;
  constexpr int SA = K_::sa;
  constexpr int SB = K_::sb;
  constexpr int ACOLS = K_::a_img_cols;                    // columns per A image (hi or lo)
  constexpr uint32_t B_IMG_BYTES = KC * N * K_::ebytes;    // one of hi / lo
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
  uint64_t* full_a = empty_b + SB;      // [SA] generator warps (one per quadrant) -> MMA
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
    for (int s = 0; s < SA; ++s) { mbar_init(&full_a[s], 4); mbar_init(&empty_a[s], 1); }
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

  if (warp < GEN_WARPS) {
    // ======================= A generators (+ D drain, warps 0-3) =======================
    const int q = warp & 3, h = warp >> 2;   // lane quadrant, chunk phase (c % GPQ)
    const int64_t o = own0 + q * 32 + lane;
    float own[NT];
#pragma unroll
    for (int p = 0; p < NT; ++p) own[p] = (o < a.n_own) ? a.own_tab[o * NT + p] : 0.f;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    float* acc_row = sAcc + q * 32 + lane;   // acc[n * 128]
    int next_drain = 0;
    // TMEM D buffer of segment d -> smem accumulator (FP32 round-to-nearest adds)
    auto drain = [&](int d) {
      const int db = d & 1;
      jitter((uint32_t)d * 64u + 60u + (uint32_t)q);
      mbar_wait_sleep(&dfull[db], (d >> 1) & 1);
      fence_after();
#pragma unroll
      for (int cb = 0; cb < N; cb += 16) {
        uint32_t v[16];
        tmem_ld16(tbase + lane_addr + db * 64 + cb, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc_row[(cb + i) * 128] += __uint_as_float(v[i]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[db]);
    };
    constexpr int NV = F16 ? 8 : 16;   // TMEM columns per image per 8 items (cos/sin)
    // warp (q, h) owns chunks c = h, h + GPQ, ... for its lane quadrant: the warps of a
    // quadrant work on different chunks, so their barrier waits do not line up
    for (int c = h; c < n_chunks; c += GPQ) {
      jitter((uint32_t)c * 64u + (uint32_t)warp);
      const int sb = c % SB, sa = c % SA;
      mbar_wait(&full_b[sb], (c / SB) & 1);
      const float* tb = sT + sb * (T_STAGE_BYTES / 4);
      const uint32_t col = A_COL0 + sa * (2 * ACOLS);
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint32_t hi[NV], lo[NV];
        if (TC_DEBUG & 1) {
#pragma unroll
          for (int i = 0; i < NV; ++i) { hi[i] = __float_as_uint(own[i % NT]); lo[i] = 0u; }
        } else {
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) {           // 4 item pairs = 8 items of this half
            const float* row = tb + (half * 4 + pp) * NT * 2;
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
            turns_sincos_pair(t, s0, c0, s1, c1);
            if constexpr (F16) {   // one 32-bit column = (cos, sin) of one item
              f16_split2(c0, s0, hi[pp * 2 + 0], lo[pp * 2 + 0]);
              f16_split2(c1, s1, hi[pp * 2 + 1], lo[pp * 2 + 1]);
            } else {
              tf32_split(c0, hi[pp * 4 + 0], lo[pp * 4 + 0]);
              tf32_split(s0, hi[pp * 4 + 1], lo[pp * 4 + 1]);
              tf32_split(c1, hi[pp * 4 + 2], lo[pp * 4 + 2]);
              tf32_split(s1, hi[pp * 4 + 3], lo[pp * 4 + 3]);
            }
          }
        }
        if (half == 0) {
          mbar_wait(&empty_a[sa], ((c / SA) & 1) ^ 1);   // MMAs of chunk c - SA drained stage sa
          fence_after();
        }
        if (!(TC_DEBUG & 4)) {
          tmem_st<NV>(tbase + lane_addr + col + half * NV, hi);
          tmem_st<NV>(tbase + lane_addr + col + ACOLS + half * NV, lo);
        }
      }
      if (!(TC_DEBUG & 4)) tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_a[sa]);
      if (a.trace && lane == 0 && q == 0 && blockIdx.x == 0 && blockIdx.y == 0 && c < 64) a.trace[c * 4 + 1] = clock64();
      // drain segment d half-way through segment d+1 (the MMA is then on the other buffer)
      // (after producing chunk c >= (d+1)*SEG + SEG/2; the MMA needs it before chunk (d+2)*SEG)
      while (h == 0 && next_drain < n_segs && (next_drain + 1) * SEG + SEG / 2 <= c) drain(next_drain++);
    }
    if (warp < 4) {
      while (next_drain < n_segs) drain(next_drain++);
      __syncwarp();
      if (o < a.n_own) {
        const int c0 = group * NC;
        const float inv = F16 ? 1.0f / *a.scale : 1.0f;
        if constexpr (FWD) {
          float2* out = a.out + (int64_t)split * a.n_own * a.ldc + o * a.ldc + c0;
#pragma unroll
          for (int c = 0; c < NC; ++c) out[c] = make_float2(acc_row[c * 128] * inv, acc_row[(NC + c) * 128] * inv);
        } else {
          double qx = 0.0, qy = 0.0;   // FP64 coil combine and partial (nfs_tci.cu)
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const float2 sv = a.sens[o * a.ldc + c0 + c];   // conj(S') * acc
            const double ar = acc_row[c * 128], ai = acc_row[(NC + c) * 128];
            qx = fma((double)sv.x, ar, qx);
            qx = fma((double)sv.y, ai, qx);
            qy = fma((double)sv.x, ai, qy);
            qy = fma(-(double)sv.y, ar, qy);
          }
          a.out_q[(int64_t)blockIdx.y * a.n_own + o] = make_double2(qx * (double)inv, qy * (double)inv);
        }
      }
    }
  } else if (warp == GEN_WARPS) {
    // ======================= bulk-copy producer =======================
    if (lane == 0) {
      for (int c = 0; c < n_chunks; ++c) {
        const int sb = c % SB;
        mbar_wait_sleep(&empty_a[sb], ((c / SB) & 1) ^ 1);
        jitter((uint32_t)c * 64u + 50u);
        const int gc = chunk0 + c;
        if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && c < 64) a.trace[c * 4 + 0] = clock64();
        if (TC_DEBUG & 8) { mbar_arrive(&full_b[sb]); continue; }
        mbar_expect_tx(&full_b[sb], B_STAGE_BYTES + T_STAGE_BYTES);
        const unsigned char* bsrc = reinterpret_cast<const unsigned char*>(a.b_img) +
                                    ((size_t)group * a.n_chunks_total + gc) * B_STAGE_BYTES;
        bulk_g2s(sB + sb * B_STAGE_BYTES, bsrc, B_STAGE_BYTES, &full_b[sb]);
        bulk_g2s(sT + sb * (T_STAGE_BYTES / 4), a.tab_img + (size_t)gc * (IC * NT), T_STAGE_BYTES, &full_b[sb]);
      }
    }
  } else {
    // ======================= MMA issuer (whole warp, elected issue) =======================
    {
      constexpr uint32_t idesc =
          (1u << 4) | (K_::fmt << 7) | (K_::fmt << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
      constexpr uint32_t LBO = (N / 8) * 128, SBO = 128;
      constexpr int KSTEPS = KC / K_::kstep;
      constexpr int COLS_PER_STEP = K_::kstep * K_::ebytes / 4;
      for (int c = 0; c < n_chunks; ++c) {
        const int sb = c % SB, sa = c % SA, seg = c / SEG, db = seg & 1;
        jitter((uint32_t)c * 64u + 41u);
        if (c % SEG == 0) {
          mbar_wait_sleep(&dempty[db], ((seg >> 1) & 1) ^ 1);   // segment seg-2 drained from buffer db
          fence_after();
        }
        // every generator warp waited full_b[sb] before arriving on full_a[sa], so full_a
        // completing implies the staged B chunk is visible (release/acquire chain)
        mbar_wait(&full_a[sa], (c / SA) & 1);
        fence_after();
        if (a.trace && lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && c < 64) a.trace[c * 4 + 2] = clock64();
        const uint32_t d_tmem = tbase + db * 64;
        const uint32_t bhi = smem_u32(sB + sb * B_STAGE_BYTES), blo = bhi + B_IMG_BYTES;
        const uint32_t ahi = tbase + A_COL0 + sa * (2 * ACOLS), alo = ahi + ACOLS;
        // small split products first (while |D| is small), then the large Ah Bh: the truncating
        // accumulation then adds the large terms KSTEPS times per chunk only (nfs_tci.cu)
#pragma unroll
        for (int t = 0; t < KSTEPS; ++t) {
          if (TC_DEBUG & 2) break;
          const uint32_t boff = (uint32_t)(2 * t) * LBO;
          const uint32_t acc = (c % SEG != 0 || t > 0) ? 1u : 0u;
          mma_ts<F16>(d_tmem, ahi + COLS_PER_STEP * t, smem_desc(blo + boff, LBO, SBO), idesc, acc);
          mma_ts<F16>(d_tmem, alo + COLS_PER_STEP * t, smem_desc(bhi + boff, LBO, SBO), idesc, 1u);
        }
#pragma unroll
        for (int t = 0; t < KSTEPS; ++t) {
          if (TC_DEBUG & 2) break;
          mma_ts<F16>(d_tmem, ahi + COLS_PER_STEP * t, smem_desc(bhi + (uint32_t)(2 * t) * LBO, LBO, SBO), idesc, 1u);
        }
        mma_commit(&empty_a[sa]);   // A stage and B stage share the index (SB == SA)
        if (a.trace && lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && c < 64) a.trace[c * 4 + 3] = clock64();
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

// ------------------------------------------------------------------ B operand prep
__device__ __forceinline__ float2 b_source(const float2* __restrict__ x, const float2* __restrict__ sens,
                                          const double2* __restrict__ p, bool fwd, int64_t item, int64_t col,
                                          int ldc) {
  const float2 v = (fwd ? sens : x)[item * ldc + col];
  if (!fwd) return v;
  const double2 pv = p[item];
  const float pr = (float)pv.x, pi = (float)pv.y;
  return make_float2(v.x * pr - v.y * pi, v.x * pi + v.y * pr);
}

// max |component| of the B source (F16 scaling), one atomicMax on the float bits per block
__global__ void amax_kernel(const float2* __restrict__ x, const float2* __restrict__ sens,
                            const double2* __restrict__ p, bool fwd, int64_t n_str, int ldc,
                            unsigned int* out_bits, const int* stop) {
  if (stop && *stop) return;
  float m = 0.f;
  const int64_t n = n_str * ldc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = b_source(x, sens, p, fwd, i / ldc, i % ldc, ldc);
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, wm[w]);
    atomicMax(out_bits, __float_as_uint(m));   // non-negative floats order like their bits
  }
}

// scale = 2^(14 - ceil(log2 amax)) so the largest |B| entry is <= 2^14 (FP16 max 65504)
__global__ void scale_kernel(const unsigned int* amax_bits, float* scale, const int* stop) {
  if (stop && *stop) return;
  const float amax = __uint_as_float(*amax_bits);
  float s = 1.f;
  if (amax > 0.f && isfinite(amax)) {
    int e;
    frexpf(amax, &e);          // amax in [2^(e-1), 2^e)
    s = ldexpf(1.f, 14 - e);
  }
  *scale = s;
}

// item i of chunk ch, coil c of group g -> its 4 B entries (hi/lo) of the chunk image
template <int NC, bool FWD, bool F16>
__global__ void prep_b_kernel(const float2* __restrict__ x, const float2* __restrict__ sens,
                              const double2* __restrict__ p, int64_t n_str, int ldc, int n_groups,
                              int n_chunks, void* __restrict__ img, const float* scale_ptr, const int* stop) {
  if (stop && *stop) return;
  constexpr int N = 2 * NC;
  constexpr int EB = F16 ? 2 : 4;
  const float scale = F16 ? *scale_ptr : 1.f;
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
      const float2 v = b_source(x, sens, p, FWD, item, g * NC + c, ldc);
      xr = v.x * scale;
      xi = v.y * scale;
    }
    unsigned char* hi = reinterpret_cast<unsigned char*>(img) + gc * (2 * KC * N * EB);
    unsigned char* lo = hi + KC * N * EB;
    // listed as (j0,n=c) (j1,n=c) (j0,n=NC+c) (j1,n=NC+c)
    const float vals[4] = {xr, FWD ? -xi : xi, xi, FWD ? xr : -xr};
    const int js[4] = {2 * il, 2 * il + 1, 2 * il, 2 * il + 1};
    const int ns[4] = {c, c, NC + c, NC + c};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t off = bimg_off<EB>(js[e], ns[e], N);
      if constexpr (F16) {
        const __half vh = __float2half_rn(vals[e]);
        const __half vl = __float2half_rn(__fsub_rn(vals[e], __half2float(vh)));
        *reinterpret_cast<__half*>(hi + off) = vh;
        *reinterpret_cast<__half*>(lo + off) = vl;
      } else {
        uint32_t vh, vl;
        tf32_split(vals[e], vh, vl);
        *reinterpret_cast<uint32_t*>(hi + off) = vh;
        *reinterpret_cast<uint32_t*>(lo + off) = vl;
      }
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
  bool f16 = true;
  int chunks_f = 0, chunks_a = 0, split_f = 1, split_a = 1;
  const float* d_T = nullptr;   // [K][nt]
  const float* d_R = nullptr;   // [L][nt]
  const float2* d_S = nullptr;  // [L][ldc]
  void *img_f = nullptr, *img_a = nullptr;
  float *tab_f = nullptr, *tab_a = nullptr;
  float2* part_y = nullptr;
  double2* part_q = nullptr;
  unsigned int* d_amax = nullptr;   // [2]
  float* d_scale = nullptr;         // [2]
  size_t smem = 0;
  std::string desc;
};



static long long* g_tc_trace = nullptr;
extern "C" long long* nfs_tc_trace_enable() {   // profiling hook (not part of the C ABI)
  if (!g_tc_trace) { cudaMallocManaged(&g_tc_trace, 64 * 4 * sizeof(long long)); }
  return g_tc_trace;
}

static int tc_fail(const std::string& m) {
  g_tc_err = m;
  return 1;
}

int tc_coil_width(int G) { return G <= 8 ? 8 : (G <= 16 ? 16 : 32); }

template <int NC, int NT, bool FWD, bool F16>
static void* tc_kernel_ptr() { return (void*)tc::tc_contract_kernel<NC, NT, FWD, F16>; }

template <int NC, bool FWD, bool F16>
static void* tc_kernel_nt(int nt) {
  switch (nt) {
    case 4: return tc_kernel_ptr<NC, 4, FWD, F16>();
    case 8: return tc_kernel_ptr<NC, 8, FWD, F16>();
    case 16: return tc_kernel_ptr<NC, 16, FWD, F16>();
    case 20: return tc_kernel_ptr<NC, 20, FWD, F16>();
    case 32: return tc_kernel_ptr<NC, 32, FWD, F16>();
  }
  return nullptr;
}

template <bool F16>
static void* tc_kernel_k(int nc, int nt, bool fwd) {
  switch (nc) {
    case 8: return fwd ? tc_kernel_nt<8, true, F16>(nt) : tc_kernel_nt<8, false, F16>(nt);
    case 16: return fwd ? tc_kernel_nt<16, true, F16>(nt) : tc_kernel_nt<16, false, F16>(nt);
    case 32: return fwd ? tc_kernel_nt<32, true, F16>(nt) : tc_kernel_nt<32, false, F16>(nt);
  }
  return nullptr;
}

static void* tc_kernel(bool f16, int nc, int nt, bool fwd) {
  return f16 ? tc_kernel_k<true>(nc, nt, fwd) : tc_kernel_k<false>(nc, nt, fwd);
}

static size_t tc_smem_bytes(bool f16, int nc, int nt) {
  const int eb = f16 ? 2 : 4;
  const int sa = f16 ? tc::Kind<true>::sa : tc::Kind<false>::sa;
  const int sb = f16 ? tc::Kind<true>::sb : tc::Kind<false>::sb;
  const size_t b = 2ull * tc::KC * (2 * nc) * eb, t = (size_t)tc::IC * nt * 4;
  return sb * (b + t) + (size_t)(2 * nc) * 128 * 4 + (2 * sb + 2 * sa + 4) * 8 + 16;
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

TcPlan* tc_create(int64_t K, int64_t L, int G, int nt, int sms, bool f16, std::string* why) {
  TcPlan* t = new TcPlan();
  t->K = K; t->L = L; t->G = G; t->nt = nt; t->sms = sms; t->f16 = f16;
  t->nc = tc_coil_width(G);
  t->n_groups = (G + t->nc - 1) / t->nc;
  t->ldc = t->nc * t->n_groups;
  t->chunks_f = (int)((L + tc::IC - 1) / tc::IC);
  t->chunks_a = (int)((std::max<int64_t>(K, 1) + tc::IC - 1) / tc::IC);
  t->smem = tc_smem_bytes(f16, t->nc, nt);
  // CTAS_PER_SM CTAs share the 512 TMEM columns; pad smem so no further CTA can co-reside
  const size_t smem_req = std::max<size_t>(t->smem, tc::CTAS_PER_SM == 1 ? 120 * 1024 : 80 * 1024);
  if (smem_req > (tc::CTAS_PER_SM == 1 ? 220 : 110) * 1024) { *why = "shared memory budget"; delete t; return nullptr; }
  for (int fwd = 0; fwd < 2; ++fwd) {
    void* k = tc_kernel(f16, t->nc, nt, fwd != 0);
    if (!k) { *why = "unsupported term count"; delete t; return nullptr; }
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_req) != cudaSuccess) {
      *why = "cannot set dynamic shared memory";
      delete t;
      return nullptr;
    }
  }
  t->smem = smem_req;
  const int resident = sms * tc::CTAS_PER_SM;
  const int64_t tiles_f = (std::max<int64_t>(K, 1) + 127) / 128 * t->n_groups;
  const int64_t tiles_a = (L + 127) / 128 * t->n_groups;
  t->split_f = pick_split(tiles_f, t->chunks_f, resident);
  t->split_a = pick_split(tiles_a, t->chunks_a, resident);
  const size_t img_chunk = 2ull * tc::KC * (2 * t->nc) * (f16 ? 2 : 4);   // bytes per chunk (hi + lo)
  auto al = [&](void** p, size_t bytes) { return nfs::dev_alloc(p, std::max<size_t>(bytes, 256)) == cudaSuccess; };
  bool ok = al(&t->img_f, img_chunk * t->chunks_f * t->n_groups) &&
            al(&t->img_a, img_chunk * t->chunks_a * t->n_groups) &&
            al((void**)&t->tab_f, (size_t)t->chunks_f * tc::IC * nt * 4) &&
            al((void**)&t->tab_a, (size_t)t->chunks_a * tc::IC * nt * 4) &&
            al((void**)&t->part_y, (size_t)t->split_f * std::max<int64_t>(K, 1) * t->ldc * 8) &&
            al((void**)&t->part_q, (size_t)t->split_a * t->n_groups * L * 16) &&
            al((void**)&t->d_amax, 2 * sizeof(unsigned int)) && al((void**)&t->d_scale, 2 * sizeof(float));
  if (!ok) { *why = "device memory"; tc_destroy(t); return nullptr; }
  const float one[2] = {1.f, 1.f};
  cudaMemcpy(t->d_scale, one, sizeof one, cudaMemcpyHostToDevice);
  char buf[256];
  snprintf(buf, sizeof buf, " tc[%s nc=%d groups=%d chunks f/a=%d/%d split f/a=%d/%d smem=%zu]",
           f16 ? "f16x3" : "tf32x3", t->nc, t->n_groups, t->chunks_f, t->chunks_a, t->split_f, t->split_a,
           t->smem);
  t->desc = buf;
  return t;
}

void tc_destroy(TcPlan* t) {
  if (!t) return;
  void* bufs[] = {t->img_f, t->img_a, t->tab_f, t->tab_a, t->part_y, t->part_q, t->d_amax, t->d_scale};
  for (void* b : bufs)
    if (b) nfs::dev_free(b);
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

template <bool FWD, bool F16>
static cudaError_t launch_prep_k(TcPlan* t, const float2* x, const double2* p, const int* stop, cudaStream_t st) {
  const int chunks = FWD ? t->chunks_f : t->chunks_a;
  const int64_t n_str = FWD ? t->L : t->K;
  void* img = FWD ? t->img_f : t->img_a;
  float* scale = t->d_scale + (FWD ? 0 : 1);
  if (F16) {
    unsigned int* amax = t->d_amax + (FWD ? 0 : 1);
    cudaMemsetAsync(amax, 0, sizeof(unsigned int), st);
    tc::amax_kernel<<<std::min(grid_for(n_str * t->ldc), 148 * 4), 256, 0, st>>>(x, t->d_S, p, FWD, n_str, t->ldc,
                                                                                   amax, stop);
    tc::scale_kernel<<<1, 1, 0, st>>>(amax, scale, stop);
  }
  const int64_t total = (int64_t)t->n_groups * chunks * tc::IC * t->nc;
  const int gb = grid_for(total);
  switch (t->nc) {
    case 8: tc::prep_b_kernel<8, FWD, F16><<<gb, 256, 0, st>>>(x, t->d_S, p, n_str, t->ldc, t->n_groups, chunks, img, scale, stop); break;
    case 16: tc::prep_b_kernel<16, FWD, F16><<<gb, 256, 0, st>>>(x, t->d_S, p, n_str, t->ldc, t->n_groups, chunks, img, scale, stop); break;
    default: tc::prep_b_kernel<32, FWD, F16><<<gb, 256, 0, st>>>(x, t->d_S, p, n_str, t->ldc, t->n_groups, chunks, img, scale, stop); break;
  }
  return cudaGetLastError();
}

template <bool FWD>
static cudaError_t launch_prep(TcPlan* t, const float2* x, const double2* p, const int* stop, cudaStream_t st) {
  return t->f16 ? launch_prep_k<FWD, true>(t, x, p, stop, st) : launch_prep_k<FWD, false>(t, x, p, stop, st);
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
  a.scale = t->d_scale + (fwd ? 0 : 1);
  a.out = t->part_y;
  a.out_q = t->part_q;
  a.stop = stop;
  a.trace = g_tc_trace;
  if (a.n_own <= 0) return cudaSuccess;
  void* k = tc_kernel(t->f16, t->nc, t->nt, fwd);
  dim3 grid((unsigned)((a.n_own + 127) / 128), (unsigned)(a.n_split * t->n_groups));
  void* args[] = {&a};
  kev_record(fwd ? 0 : 2, st);
  const cudaError_t e = cudaLaunchKernel(k, grid, dim3(tc::THREADS), args, t->smem, st);
  kev_record(fwd ? 1 : 3, st);
  return e;
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
    e = launch_reduce_image(1, t->part_q, q, t->L, t->split_a * t->n_groups, stop, st);
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

int tc_launches_per_apply(TcPlan* t) { return t->f16 ? 10 : 6; }

}  // namespace nfs
