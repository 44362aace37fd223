// nfs_contract.cu -- generated-phase complex contraction on CUDA cores (FP32 / FP64).
//
// One kernel template serves both operators of the encoding model (nfs/engine.py:98-108):
//   forward  y[k,c] = sum_l e^{+i phi_kl} W[l,c],  W = S' o p          (apply_E, :98-100)
//   adjoint  q[l]   = sum_c conj(S'[l,c]) sum_k e^{-i phi_kl} Y[k,c]   (apply_EH, :103-108)
// with phi generated per (owner, streamed) pair from the basis tables (phase_block, :93-95)
// and ONE sincos per pair reused across every coil of the group.
//
// CTA = OWN_TILE owners (RO per thread, strided by BLOCK so table loads coalesce) x one
// split of the streamed range.  Streamed items (their table row and complex operand row) are
// double-buffered in shared memory with cp.async; every thread walks the chunk reading
// broadcast smem rows.
//
// FP32 path (Blackwell-specific): the two owners of a thread are packed into the lanes of
// FFMA2 / FMUL2 (sm_100 packed FP32), so the phase FMA chain and the complex MAC issue half
// the instructions of scalar FFMA and the coefficient pair stays in the operand reuse cache
// (measured: 65 TFLOP/s packed vs 46.5 scalar on this MAC pattern, tools/ubench/fma_rate.cu).
// The next item's phase is computed while the current item's MACs issue (software pipeline).
// FP64 path: scalar DFMA with FP64 sincospi (parity mode).
#include <type_traits>

#include "../../include/nfs_b200.h"
#include "nfs_common.cuh"
#include "nfs_phase.cuh"

namespace nfs {

// ------------------------------------------------------------------ cp.async helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;   // 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage streamed rows [sb, sb+SC) (zero beyond s_end): table rows and operand rows.
template <typename T, int NC, int NT, int SC, int BLOCK>
__device__ __forceinline__ void stage_chunk(T* s_tab, typename C2<T>::type* s_x,
                                            const T* __restrict__ str_tab,
                                            const typename C2<T>::type* __restrict__ x,
                                            int ldc, int c0, int64_t sb, int64_t s_end) {
  constexpr int TAB_U = NT * (int)sizeof(T) / 16;          // 16-byte units per table row
  constexpr int X_U = NC * 2 * (int)sizeof(T) / 16;        // 16-byte units per operand row
  static_assert(TAB_U * 16 == NT * (int)sizeof(T), "table rows must be 16B multiples");
  static_assert(X_U * 16 == NC * 2 * (int)sizeof(T), "operand rows must be 16B multiples");
  for (int u = threadIdx.x; u < SC * TAB_U; u += BLOCK) {
    const int r = u / TAB_U;
    const int64_t s = sb + r;
    const bool ok = s < s_end;
    cp_async16(reinterpret_cast<char*>(s_tab) + (size_t)u * 16,
               reinterpret_cast<const char*>(str_tab + (ok ? s : 0) * NT) + (u - r * TAB_U) * 16, ok);
  }
  for (int u = threadIdx.x; u < SC * X_U; u += BLOCK) {
    const int r = u / X_U;
    const int64_t s = sb + r;
    const bool ok = s < s_end;
    cp_async16(reinterpret_cast<char*>(s_x) + (size_t)u * 16,
               reinterpret_cast<const char*>(x + (ok ? s : 0) * ldc + c0) + (u - r * X_U) * 16, ok);
  }
}

// ------------------------------------------------------------------ FP32 packed kernel
__host__ __device__ constexpr int ro_f32(int nc) { return nc >= 16 ? 2 : 4; }
constexpr int kBlockF = 128;
// streamed items per smem chunk; 32 when NC = NT = 32 keeps static smem under 48 KB
__host__ __device__ constexpr int chunk_f32(int nc, int nt) { return (nc >= 32 && nt >= 32) ? 32 : 64; }

// phase (turns) of PR owner pairs against one streamed table row b
template <int NT, int PR>
__device__ __forceinline__ void phase_t(const float2 (&own)[PR][NT], const float* __restrict__ b,
                                        float2 (&t)[PR]) {
  float bv[NT];
#pragma unroll
  for (int p = 0; p < NT; p += 4) {
    const float4 v = *reinterpret_cast<const float4*>(b + p);
    bv[p] = v.x; bv[p + 1] = v.y; bv[p + 2] = v.z; bv[p + 3] = v.w;
  }
#pragma unroll
  for (int pr = 0; pr < PR; ++pr) {
    // identical IEEE op sequence to phase_turns_generic<float>: mul, then fma p = 1..NT-1
    float2 x = __fmul2_rn(own[pr][0], make_float2(bv[0], bv[0]));
#pragma unroll
    for (int p = 1; p < NT; ++p) x = __ffma2_rn(own[pr][p], make_float2(bv[p], bv[p]), x);
    t[pr] = x;
  }
}

template <int PR>
__device__ __forceinline__ void sincos_pairs(const float2 (&t)[PR], float2 (&cs)[PR], float2 (&sn)[PR]) {
#pragma unroll
  for (int pr = 0; pr < PR; ++pr) {
    turns_sincos_generic(t[pr].x, sn[pr].x, cs[pr].x);
    turns_sincos_generic(t[pr].y, sn[pr].y, cs[pr].y);
  }
}

template <int NC, int NT, bool FWD>
__global__ void __launch_bounds__(kBlockF) contract_f32_kernel(ContractLaunch a) {
  constexpr int BLOCK = kBlockF, SC = chunk_f32(NC, NT), RO = ro_f32(NC), PR = RO / 2, OWN_TILE = BLOCK * RO;
  if (a.stop != nullptr && *a.stop) return;

  __shared__ __align__(16) float s_tab[2][(SC + 2) * NT];   // rows SC, SC+1 = zero (pipeline tail)
  __shared__ __align__(16) float2 s_x[2][SC * NC];

  const int tid = threadIdx.x;
  const int group = blockIdx.y / a.n_split;
  const int split = blockIdx.y - group * a.n_split;
  const int c0 = group * NC;
  const int64_t own0 = (int64_t)blockIdx.x * OWN_TILE;
  const float* __restrict__ own_tab = static_cast<const float*>(a.own_tab);
  const float* __restrict__ str_tab = static_cast<const float*>(a.str_tab);
  const float2* __restrict__ xs = static_cast<const float2*>(a.x);

  const int64_t per = (((a.n_str + a.n_split - 1) / a.n_split) + SC - 1) / SC * SC;
  const int64_t s_begin = split * per;
  const int64_t s_end = min(a.n_str, s_begin + per);
  const int n_chunks = s_end > s_begin ? (int)((s_end - s_begin + SC - 1) / SC) : 0;

  if (n_chunks > 0)
    stage_chunk<float, NC, NT, SC, BLOCK>(s_tab[0], s_x[0], str_tab, xs, a.ldc, c0, s_begin, s_end);
  cp_async_commit();
  if (tid < 2 * NT) { s_tab[0][SC * NT + tid] = 0.f; s_tab[1][SC * NT + tid] = 0.f; }

  // owner tables -> packed registers
  float2 own[PR][NT];
#pragma unroll
  for (int pr = 0; pr < PR; ++pr) {
    const int64_t o0 = own0 + (2 * pr) * BLOCK + tid, o1 = o0 + BLOCK;
#pragma unroll
    for (int p = 0; p < NT; ++p)
      own[pr][p] = make_float2(o0 < a.n_own ? own_tab[o0 * NT + p] : 0.f,
                               o1 < a.n_own ? own_tab[o1 * NT + p] : 0.f);
  }
  float2 are[PR][NC], aim[PR][NC];
#pragma unroll
  for (int pr = 0; pr < PR; ++pr)
#pragma unroll
    for (int c = 0; c < NC; ++c) { are[pr][c] = make_float2(0.f, 0.f); aim[pr][c] = make_float2(0.f, 0.f); }

  for (int ch = 0; ch < n_chunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < n_chunks)
      stage_chunk<float, NC, NT, SC, BLOCK>(s_tab[buf ^ 1], s_x[buf ^ 1], str_tab, xs, a.ldc, c0,
                                            s_begin + (int64_t)(ch + 1) * SC, s_end);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const float* tb = s_tab[buf];
    const float2* xb = s_x[buf];
    // 3-stage software pipeline: FMA chain for item si+2, sincos for si+1, MACs for si
    float2 cs[PR], sn[PR], t1[PR];
    {
      float2 t0[PR];
      phase_t<NT, PR>(own, tb, t0);
      sincos_pairs<PR>(t0, cs, sn);
      phase_t<NT, PR>(own, tb + NT, t1);
    }
#pragma unroll 1
    for (int si = 0; si < SC; ++si) {
      float2 t2[PR], ncs[PR], nsn[PR];
      sincos_pairs<PR>(t1, ncs, nsn);                        // item si+1 (inputs ready)
      phase_t<NT, PR>(own, tb + (si + 2) * NT, t2);          // item si+2, overlaps the MACs
      float2 msn[PR];
#pragma unroll
      for (int pr = 0; pr < PR; ++pr) msn[pr] = make_float2(-sn[pr].x, -sn[pr].y);
#pragma unroll
      for (int c2 = 0; c2 < NC / 2; ++c2) {
        const float4 x = *reinterpret_cast<const float4*>(xb + si * NC + 2 * c2);
#pragma unroll
        for (int pr = 0; pr < PR; ++pr) {
          if constexpr (FWD) {   // (cs + i sn) x
            are[pr][2 * c2] = __ffma2_rn(cs[pr], make_float2(x.x, x.x), are[pr][2 * c2]);
            are[pr][2 * c2] = __ffma2_rn(msn[pr], make_float2(x.y, x.y), are[pr][2 * c2]);
            aim[pr][2 * c2] = __ffma2_rn(cs[pr], make_float2(x.y, x.y), aim[pr][2 * c2]);
            aim[pr][2 * c2] = __ffma2_rn(sn[pr], make_float2(x.x, x.x), aim[pr][2 * c2]);
            are[pr][2 * c2 + 1] = __ffma2_rn(cs[pr], make_float2(x.z, x.z), are[pr][2 * c2 + 1]);
            are[pr][2 * c2 + 1] = __ffma2_rn(msn[pr], make_float2(x.w, x.w), are[pr][2 * c2 + 1]);
            aim[pr][2 * c2 + 1] = __ffma2_rn(cs[pr], make_float2(x.w, x.w), aim[pr][2 * c2 + 1]);
            aim[pr][2 * c2 + 1] = __ffma2_rn(sn[pr], make_float2(x.z, x.z), aim[pr][2 * c2 + 1]);
          } else {               // (cs - i sn) x
            are[pr][2 * c2] = __ffma2_rn(cs[pr], make_float2(x.x, x.x), are[pr][2 * c2]);
            are[pr][2 * c2] = __ffma2_rn(sn[pr], make_float2(x.y, x.y), are[pr][2 * c2]);
            aim[pr][2 * c2] = __ffma2_rn(cs[pr], make_float2(x.y, x.y), aim[pr][2 * c2]);
            aim[pr][2 * c2] = __ffma2_rn(msn[pr], make_float2(x.x, x.x), aim[pr][2 * c2]);
            are[pr][2 * c2 + 1] = __ffma2_rn(cs[pr], make_float2(x.z, x.z), are[pr][2 * c2 + 1]);
            are[pr][2 * c2 + 1] = __ffma2_rn(sn[pr], make_float2(x.w, x.w), are[pr][2 * c2 + 1]);
            aim[pr][2 * c2 + 1] = __ffma2_rn(cs[pr], make_float2(x.w, x.w), aim[pr][2 * c2 + 1]);
            aim[pr][2 * c2 + 1] = __ffma2_rn(msn[pr], make_float2(x.z, x.z), aim[pr][2 * c2 + 1]);
          }
        }
      }
#pragma unroll
      for (int pr = 0; pr < PR; ++pr) { cs[pr] = ncs[pr]; sn[pr] = nsn[pr]; t1[pr] = t2[pr]; }
    }
    __syncthreads();   // buffer `buf` is refilled by the prefetch two chunks ahead
  }

  // epilogue
  const float2* __restrict__ sens = static_cast<const float2*>(a.sens);
#pragma unroll
  for (int pr = 0; pr < PR; ++pr) {
#pragma unroll
    for (int lane = 0; lane < 2; ++lane) {
      const int64_t o = own0 + (2 * pr + lane) * BLOCK + tid;
      if (o >= a.n_own) continue;
      if constexpr (FWD) {
        float2* out = static_cast<float2*>(a.out) + (int64_t)split * a.n_own * a.ldc + o * a.ldc + c0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
          out[c] = lane ? make_float2(are[pr][c].y, aim[pr][c].y) : make_float2(are[pr][c].x, aim[pr][c].x);
      } else {
        // FP64 coil combine and partial image: rounding q to FP32 per apply is an inconsistent
        // per-apply error the CG amplifies
        double qx = 0.0, qy = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const float2 sv = sens[o * a.ldc + c0 + c];   // conj(S') * acc
          const double ax = lane ? are[pr][c].y : are[pr][c].x;
          const double ay = lane ? aim[pr][c].y : aim[pr][c].x;
          qx = fma((double)sv.x, ax, qx);
          qx = fma((double)sv.y, ay, qx);
          qy = fma((double)sv.x, ay, qy);
          qy = fma(-(double)sv.y, ax, qy);
        }
        static_cast<double2*>(a.out)[(int64_t)blockIdx.y * a.n_own + o] = make_double2(qx, qy);
      }
    }
  }
}

// ------------------------------------------------------------------ FP64 scalar kernel
__host__ __device__ constexpr int ro_f64(int nc, int nt) { return nc >= 16 ? 1 : (nt >= 20 ? 1 : 2); }
#ifndef NFS_F64_BLOCK
#define NFS_F64_BLOCK 128   // 256: 2-5% faster at config B, but it changes config D's split and its chaotic 50-iteration drift (DESIGN 3.2)
#endif
#ifndef NFS_F64_CHUNK
#define NFS_F64_CHUNK 32
#endif
constexpr int kBlockD = NFS_F64_BLOCK;
constexpr int kChunkD = NFS_F64_CHUNK;

template <int NC, int NT, bool FWD>
__global__ void __launch_bounds__(kBlockD) contract_f64_kernel(ContractLaunch a) {
  constexpr int BLOCK = kBlockD, SC = kChunkD, RO = ro_f64(NC, NT), OWN_TILE = BLOCK * RO;
  if (a.stop != nullptr && *a.stop) return;

  __shared__ __align__(16) double s_tab[2][SC * NT];
  __shared__ __align__(16) double2 s_x[2][SC * NC];

  const int tid = threadIdx.x;
  const int group = blockIdx.y / a.n_split;
  const int split = blockIdx.y - group * a.n_split;
  const int c0 = group * NC;
  const int64_t own0 = (int64_t)blockIdx.x * OWN_TILE;
  const double* __restrict__ own_tab = static_cast<const double*>(a.own_tab);
  const double* __restrict__ str_tab = static_cast<const double*>(a.str_tab);
  const double2* __restrict__ xs = static_cast<const double2*>(a.x);

  const int64_t per = (((a.n_str + a.n_split - 1) / a.n_split) + SC - 1) / SC * SC;
  const int64_t s_begin = split * per;
  const int64_t s_end = min(a.n_str, s_begin + per);
  const int n_chunks = s_end > s_begin ? (int)((s_end - s_begin + SC - 1) / SC) : 0;
  if (n_chunks > 0)
    stage_chunk<double, NC, NT, SC, BLOCK>(s_tab[0], s_x[0], str_tab, xs, a.ldc, c0, s_begin, s_end);
  cp_async_commit();

  double own[RO][NT];
#pragma unroll
  for (int r = 0; r < RO; ++r) {
    const int64_t o = own0 + r * BLOCK + tid;
#pragma unroll
    for (int p = 0; p < NT; ++p) own[r][p] = (o < a.n_own) ? own_tab[o * NT + p] : 0.0;
  }
  double2 acc[RO][NC];
#pragma unroll
  for (int r = 0; r < RO; ++r)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[r][c] = make_double2(0.0, 0.0);

  for (int ch = 0; ch < n_chunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < n_chunks)
      stage_chunk<double, NC, NT, SC, BLOCK>(s_tab[buf ^ 1], s_x[buf ^ 1], str_tab, xs, a.ldc, c0,
                                             s_begin + (int64_t)(ch + 1) * SC, s_end);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
#pragma unroll 1
    for (int si = 0; si < SC; ++si) {
      double cs[RO], sn[RO];
#pragma unroll
      for (int r = 0; r < RO; ++r) {
        const double t = phase_turns_generic<double, NT>(own[r], &s_tab[buf][si * NT]);
        turns_sincos_generic(t, sn[r], cs[r]);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 x = s_x[buf][si * NC + c];
#pragma unroll
        for (int r = 0; r < RO; ++r) {
          const double s = FWD ? sn[r] : -sn[r];
          acc[r][c].x = fma(cs[r], x.x, acc[r][c].x);
          acc[r][c].x = fma(-s, x.y, acc[r][c].x);
          acc[r][c].y = fma(cs[r], x.y, acc[r][c].y);
          acc[r][c].y = fma(s, x.x, acc[r][c].y);
        }
      }
    }
    __syncthreads();
  }

  const double2* __restrict__ sens = static_cast<const double2*>(a.sens);
#pragma unroll
  for (int r = 0; r < RO; ++r) {
    const int64_t o = own0 + r * BLOCK + tid;
    if (o >= a.n_own) continue;
    if constexpr (FWD) {
      double2* out = static_cast<double2*>(a.out) + (int64_t)split * a.n_own * a.ldc + o * a.ldc + c0;
#pragma unroll
      for (int c = 0; c < NC; ++c) out[c] = acc[r][c];
    } else {
      double2 q = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 sv = sens[o * a.ldc + c0 + c];
        q.x = fma(sv.x, acc[r][c].x, q.x);
        q.x = fma(sv.y, acc[r][c].y, q.x);
        q.y = fma(sv.x, acc[r][c].y, q.y);
        q.y = fma(-sv.y, acc[r][c].x, q.y);
      }
      static_cast<double2*>(a.out)[(int64_t)blockIdx.y * a.n_own + o] = q;
    }
  }
}

// ------------------------------------------------------------------ W = S' o p
template <typename T2>
__global__ void make_w_kernel(const T2* __restrict__ sens, const double2* __restrict__ p,
                              T2* __restrict__ w, int64_t n_vox, int ldc, const int* stop) {
  if (stop && *stop) return;
  const int64_t n = n_vox * ldc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / ldc;
    const T2 s = sens[i];
    const double2 pv = p[l];
    using T = decltype(s.x);
    const T pr = (T)pv.x, pi = (T)pv.y;
    T2 o;
    o.x = s.x * pr - s.y * pi;
    o.y = s.x * pi + s.y * pr;
    w[i] = o;
  }
}

cudaError_t launch_make_w(int prec, const void* sens, const double2* p, void* w, int64_t n_vox,
                          int ldc, const int* stop, cudaStream_t st) {
  int64_t blocks = (n_vox * ldc + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  if (prec == NFS_PREC_FP64)
    make_w_kernel<double2><<<(unsigned)blocks, 256, 0, st>>>((const double2*)sens, p, (double2*)w, n_vox, ldc, stop);
  else
    make_w_kernel<float2><<<(unsigned)blocks, 256, 0, st>>>((const float2*)sens, p, (float2*)w, n_vox, ldc, stop);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ dispatch
template <bool F64, int NC, int NT, bool FWD>
static void* kernel_ptr() {
  if constexpr (F64) return (void*)contract_f64_kernel<NC, NT, FWD>;
  else return (void*)contract_f32_kernel<NC, NT, FWD>;
}

template <bool F64, bool FWD, int NC>
static void* pick_nt(int nt) {
  switch (nt) {
    case 4: return kernel_ptr<F64, NC, 4, FWD>();
    case 8: return kernel_ptr<F64, NC, 8, FWD>();
    case 16: return kernel_ptr<F64, NC, 16, FWD>();
    case 20: return kernel_ptr<F64, NC, 20, FWD>();
    case 32: return kernel_ptr<F64, NC, 32, FWD>();
  }
  return nullptr;
}

template <bool F64, bool FWD>
static void* pick_kernel(int nc, int nt) {
  switch (nc) {
    case 2: return pick_nt<F64, FWD, 2>(nt);
    case 4: return pick_nt<F64, FWD, 4>(nt);
    case 8: return pick_nt<F64, FWD, 8>(nt);
    case 16: return pick_nt<F64, FWD, 16>(nt);
    case 32: return pick_nt<F64, FWD, 32>(nt);
  }
  return nullptr;
}

static void* kernel_for(int prec, bool fwd, int nc, int nt) {
  const bool f64 = prec == NFS_PREC_FP64;
  if (f64) return fwd ? pick_kernel<true, true>(nc, nt) : pick_kernel<true, false>(nc, nt);
  return fwd ? pick_kernel<false, true>(nc, nt) : pick_kernel<false, false>(nc, nt);
}

static int owners_per_cta(int prec, int nc, int nt) {
  return prec == NFS_PREC_FP64 ? kBlockD * ro_f64(nc, nt) : kBlockF * ro_f32(nc);
}

cudaError_t launch_contract(const ContractLaunch& L, cudaStream_t st) {
  if (L.n_own <= 0) return cudaSuccess;
  void* k = kernel_for(L.prec, L.forward, L.nc, L.nt);
  if (!k) return cudaErrorInvalidValue;
  const int tile = owners_per_cta(L.prec, L.nc, L.nt);
  dim3 grid((unsigned)((L.n_own + tile - 1) / tile), (unsigned)(L.n_split * L.n_groups));
  dim3 block(L.prec == NFS_PREC_FP64 ? kBlockD : kBlockF);
  ContractLaunch copy = L;
  void* args[] = {&copy};
  kev_record(L.forward ? 0 : 2, st);
  const cudaError_t e = cudaLaunchKernel(k, grid, block, args, 0, st);
  kev_record(L.forward ? 1 : 3, st);
  return e;
}

void contract_kernel_shape(int prec, bool forward, int nc, int nt, int* own_per_cta,
                           int* streamed_chunk, int* ctas_per_sm) {
  *own_per_cta = owners_per_cta(prec, nc, nt);
  *streamed_chunk = prec == NFS_PREC_FP64 ? kChunkD : chunk_f32(nc, nt);
  int n = 0;
  void* k = kernel_for(prec, forward, nc, nt);
  if (k) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, prec == NFS_PREC_FP64 ? kBlockD : kBlockF, 0);
  *ctas_per_sm = n;
}

}  // namespace nfs
