// nfs_contract.cu -- generated-phase complex contraction on CUDA cores (FP32 / FP64).
//
// One kernel template serves both operators of the encoding model (nfs/engine.py:98-108):
//   forward  y[k,c] = sum_l e^{+i phi_kl} S'[l,c] p[l]           (apply_E, :98-100)
//   adjoint  q[l]   = sum_c conj(S'[l,c]) sum_k e^{-i phi_kl} Y[k,c] (apply_EH, :103-108)
// with phi generated per (owner, streamed) pair from the basis tables (phase_block, :93-95)
// and ONE sincos per pair reused across every coil of the group.
//
// CTA = OWN_TILE owners (RO per thread, strided by BLOCK so table loads coalesce) x one
// split of the streamed range.  Streamed items are staged in shared memory in chunks of SC
// (their table rows and their complex operand X), then every thread walks the chunk reading
// broadcast smem rows.  Per (owner, streamed) pair and coil the inner loop is 4 FFMA; the
// phase costs NT FFMA + rint/sub + 2 MUFU; roofline = FP32 (or FP64) FMA pipe.
#include "nfs_common.cuh"
#include "nfs_phase.cuh"
#include "../../include/nfs_b200.h"

namespace nfs {

// phase generator shared with every other kernel of the path (nfs_phase.cuh)
template <typename T, int NT>
__device__ __forceinline__ T phase_turns(const T (&a)[NT], const T* __restrict__ b) {
  return phase_turns_generic<T, NT>(a, b);
}
template <typename T>
__device__ __forceinline__ void turns_sincos(T t, T& s, T& c) { turns_sincos_generic(t, s, c); }

template <typename T> struct KShape;
// RO owners per thread: keeps RO*NC complex accumulators in registers.
template <> struct KShape<float> {
  static constexpr int block = 128;
  static constexpr int sc = 64;
  __host__ __device__ static constexpr int ro(int nc, int nt) { return nc >= 16 ? 2 : (nt >= 20 ? 2 : 4); }
};
template <> struct KShape<double> {
  static constexpr int block = 128;
  static constexpr int sc = 32;
  __host__ __device__ static constexpr int ro(int nc, int nt) { return nc >= 16 ? 1 : (nt >= 20 ? 1 : 2); }
};

template <typename T, int NC, int NT, bool FWD>
__global__ void __launch_bounds__(KShape<T>::block)
contract_kernel(ContractLaunch a) {
  using T2 = typename C2<T>::type;
  constexpr int BLOCK = KShape<T>::block;
  constexpr int SC = KShape<T>::sc;
  constexpr int RO = KShape<T>::ro(NC, NT);
  constexpr int OWN_TILE = BLOCK * RO;

  if (a.stop != nullptr && *a.stop) return;

  __shared__ __align__(16) T s_tab[SC * NT];
  __shared__ __align__(16) T2 s_x[SC * NC];

  const int tid = threadIdx.x;
  const int group = blockIdx.y / a.n_split;
  const int split = blockIdx.y - group * a.n_split;
  const int c0 = group * NC;
  const int64_t own0 = (int64_t)blockIdx.x * OWN_TILE;

  const T* __restrict__ own_tab = static_cast<const T*>(a.own_tab);
  const T* __restrict__ str_tab = static_cast<const T*>(a.str_tab);
  const T2* __restrict__ sens = static_cast<const T2*>(a.sens);

  // owner tables -> registers
  T own[RO][NT];
#pragma unroll
  for (int r = 0; r < RO; ++r) {
    const int64_t o = own0 + r * BLOCK + tid;
#pragma unroll
    for (int p = 0; p < NT; ++p) own[r][p] = (o < a.n_own) ? own_tab[o * NT + p] : T(0);
  }

  T2 acc[RO][NC];
#pragma unroll
  for (int r = 0; r < RO; ++r)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[r][c] = T2{T(0), T(0)};

  // streamed range of this split, chunk aligned
  const int64_t per = (((a.n_str + a.n_split - 1) / a.n_split) + SC - 1) / SC * SC;
  const int64_t s_begin = split * per;
  const int64_t s_end = min(a.n_str, s_begin + per);

  for (int64_t sb = s_begin; sb < s_end; sb += SC) {
    __syncthreads();
    // stage table rows (zero beyond the end)
    for (int i = tid; i < SC * NT; i += BLOCK) {
      const int64_t s = sb + i / NT;
      s_tab[i] = (s < s_end) ? str_tab[sb * NT + i] : T(0);
    }
    // stage the streamed operand
    for (int i = tid; i < SC * NC; i += BLOCK) {
      const int si = i / NC, c = i - si * NC;
      const int64_t s = sb + si;
      T2 x = T2{T(0), T(0)};
      if (s < s_end) {
        if constexpr (FWD) {
          const T2 sv = sens[s * a.ldc + c0 + c];
          const double2 pv = a.p[s];
          const T pr = (T)pv.x, pi = (T)pv.y;
          x.x = sv.x * pr - sv.y * pi;
          x.y = sv.x * pi + sv.y * pr;
        } else {
          x = static_cast<const T2*>(a.y)[s * a.ldc + c0 + c];
        }
      }
      s_x[i] = x;
    }
    __syncthreads();

#pragma unroll 1
    for (int si = 0; si < SC; ++si) {
      T cs[RO], sn[RO];
#pragma unroll
      for (int r = 0; r < RO; ++r) {
        const T t = phase_turns<T, NT>(own[r], &s_tab[si * NT]);
        turns_sincos(t, sn[r], cs[r]);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const T2 x = s_x[si * NC + c];
#pragma unroll
        for (int r = 0; r < RO; ++r) {
          if constexpr (FWD) {   // (cs + i sn) * x
            acc[r][c].x = fma(cs[r], x.x, acc[r][c].x);
            acc[r][c].x = fma(-sn[r], x.y, acc[r][c].x);
            acc[r][c].y = fma(cs[r], x.y, acc[r][c].y);
            acc[r][c].y = fma(sn[r], x.x, acc[r][c].y);
          } else {               // (cs - i sn) * x
            acc[r][c].x = fma(cs[r], x.x, acc[r][c].x);
            acc[r][c].x = fma(sn[r], x.y, acc[r][c].x);
            acc[r][c].y = fma(cs[r], x.y, acc[r][c].y);
            acc[r][c].y = fma(-sn[r], x.x, acc[r][c].y);
          }
        }
      }
    }
  }

  // epilogue
#pragma unroll
  for (int r = 0; r < RO; ++r) {
    const int64_t o = own0 + r * BLOCK + tid;
    if (o >= a.n_own) continue;
    if constexpr (FWD) {
      T2* out = static_cast<T2*>(a.out) + (int64_t)split * a.n_own * a.ldc + o * a.ldc + c0;
#pragma unroll
      for (int c = 0; c < NC; ++c) out[c] = acc[r][c];
    } else {
      T2 q = T2{T(0), T(0)};
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const T2 sv = sens[o * a.ldc + c0 + c];   // conj(S') * acc
        q.x = fma(sv.x, acc[r][c].x, q.x);
        q.x = fma(sv.y, acc[r][c].y, q.x);
        q.y = fma(sv.x, acc[r][c].y, q.y);
        q.y = fma(-sv.y, acc[r][c].x, q.y);
      }
      static_cast<T2*>(a.out)[(int64_t)blockIdx.y * a.n_own + o] = q;
    }
  }
}

// ---------------------------------------------------------------- dispatch
template <typename T, bool FWD, int NC>
static cudaError_t dispatch_nt(const ContractLaunch& L, dim3 grid, cudaStream_t st) {
  constexpr int B = KShape<T>::block;
  switch (L.nt) {
    case 4: contract_kernel<T, NC, 4, FWD><<<grid, B, 0, st>>>(L); break;
    case 8: contract_kernel<T, NC, 8, FWD><<<grid, B, 0, st>>>(L); break;
    case 16: contract_kernel<T, NC, 16, FWD><<<grid, B, 0, st>>>(L); break;
    case 20: contract_kernel<T, NC, 20, FWD><<<grid, B, 0, st>>>(L); break;
    case 32: contract_kernel<T, NC, 32, FWD><<<grid, B, 0, st>>>(L); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <typename T, bool FWD>
static cudaError_t dispatch_nc(const ContractLaunch& L, cudaStream_t st) {
  const int ro = KShape<T>::ro(L.nc, L.nt);
  const int own_tile = KShape<T>::block * ro;
  dim3 grid((unsigned)((L.n_own + own_tile - 1) / own_tile), (unsigned)(L.n_split * L.n_groups));
  switch (L.nc) {
    case 2: return dispatch_nt<T, FWD, 2>(L, grid, st);
    case 4: return dispatch_nt<T, FWD, 4>(L, grid, st);
    case 8: return dispatch_nt<T, FWD, 8>(L, grid, st);
    case 16: return dispatch_nt<T, FWD, 16>(L, grid, st);
    case 32: return dispatch_nt<T, FWD, 32>(L, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_contract(const ContractLaunch& L, cudaStream_t st) {
  if (L.n_own <= 0) return cudaSuccess;
  if (L.prec == NFS_PREC_FP64)
    return L.forward ? dispatch_nc<double, true>(L, st) : dispatch_nc<double, false>(L, st);
  return L.forward ? dispatch_nc<float, true>(L, st) : dispatch_nc<float, false>(L, st);
}

template <typename T, bool FWD, int NC>
static int occ_nt(int nt) {
  int n = 0;
  constexpr int B = KShape<T>::block;
  switch (nt) {
    case 4: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, contract_kernel<T, NC, 4, FWD>, B, 0); break;
    case 8: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, contract_kernel<T, NC, 8, FWD>, B, 0); break;
    case 16: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, contract_kernel<T, NC, 16, FWD>, B, 0); break;
    case 20: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, contract_kernel<T, NC, 20, FWD>, B, 0); break;
    case 32: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, contract_kernel<T, NC, 32, FWD>, B, 0); break;
  }
  return n;
}

template <typename T, bool FWD>
static int occ_nc(int nc, int nt) {
  switch (nc) {
    case 2: return occ_nt<T, FWD, 2>(nt);
    case 4: return occ_nt<T, FWD, 4>(nt);
    case 8: return occ_nt<T, FWD, 8>(nt);
    case 16: return occ_nt<T, FWD, 16>(nt);
    case 32: return occ_nt<T, FWD, 32>(nt);
  }
  return 0;
}

void contract_kernel_shape(int prec, bool forward, int nc, int nt, int* owners_per_cta,
                           int* streamed_chunk, int* ctas_per_sm) {
  if (prec == NFS_PREC_FP64) {
    *owners_per_cta = KShape<double>::block * KShape<double>::ro(nc, nt);
    *streamed_chunk = KShape<double>::sc;
    *ctas_per_sm = forward ? occ_nc<double, true>(nc, nt) : occ_nc<double, false>(nc, nt);
  } else {
    *owners_per_cta = KShape<float>::block * KShape<float>::ro(nc, nt);
    *streamed_chunk = KShape<float>::sc;
    *ctas_per_sm = forward ? occ_nc<float, true>(nc, nt) : occ_nc<float, false>(nc, nt);
  }
}

}  // namespace nfs
