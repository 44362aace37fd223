// nfs_common.cuh -- shared device/host declarations of the B200 non-Fourier SENSE path.
//
// Data layout in HBM (one plan = one device, sample rows sharded across ranks):
//   T_tab  [K][NT]      temporal basis in TURNS (temporal / 2pi), zero-padded to NT terms
//   R_tab  [L][NT]      spatial basis, transposed so that one voxel's terms are contiguous
//   S      [L][ldc]     S' = S o j, complex, coils padded to ldc = NC * n_groups
//   Y      [K][ldc]     coil samples (sigma or E p), complex
// The phase t[k,l] = sum_p T_tab[k,p] * R_tab[l,p] (turns) is regenerated on the fly by both
// operators with the SAME fma chain (phase_turns below), so E and E^H see bit-identical
// phasors -- the consistent-perturbation property SURVEY.md Appendix A relies on.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace nfs {

// Benchmark hook: when `on`, the main contraction kernel of each operator is bracketed by CUDA
// events on its launch stream (ev[0]/ev[1] forward, ev[2]/ev[3] adjoint), so nfs_bench_applies
// measures the dominant kernel inside the same timed steps as the whole apply.
struct KernelEvents {
  cudaEvent_t ev[4];
  int on;
};
inline KernelEvents& kernel_events() {
  static thread_local KernelEvents k{};
  return k;
}
inline void kev_record(int i, cudaStream_t st) {
  KernelEvents& k = kernel_events();
  if (k.on) cudaEventRecord(k.ev[i], st);
}

// Device buffers come from the device's default stream-ordered memory pool with the release
// threshold raised, so the next plan of a CG solve (or the next recon call) reuses freed
// memory instead of paying cudaMalloc/cudaFree page-mapping costs (tens to hundreds of ms for
// the GB-scale partial buffers).  Allocation is made visible to every stream by synchronising
// the private allocation stream; callers synchronise their own stream before dev_free.
inline cudaStream_t alloc_stream() {
  static cudaStream_t streams[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 0;
  if (!streams[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
  }
  return streams[dev];
}
inline cudaError_t dev_alloc(void** p, size_t bytes) {
  cudaStream_t s = alloc_stream();
  cudaError_t e = cudaMallocAsync(p, bytes, s);
  if (e == cudaErrorMemoryAllocation) {   // give cached pool memory back to the device, retry once
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    cudaStreamSynchronize(s);
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(p, bytes, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e;
}
inline void dev_free(void* p) {
  if (!p) return;
  cudaStream_t s = alloc_stream();
  cudaFreeAsync(p, s);
}


// Host -> device copy of a caller (pageable) array through a pinned staging ring with
// multi-threaded staging (nfs_upload.cu); same semantics as cudaMemcpyAsync from pageable memory.
cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);
cudaError_t h2d_file(void* dst, const char* path, int64_t offset, size_t bytes, cudaStream_t st);

template <typename T> struct C2;
template <> struct C2<float> { using type = float2; };
template <> struct C2<double> { using type = double2; };

// Launch description of one generated-phase contraction (forward or adjoint).
//   forward : owner = sample k (rows of T_tab), streamed = voxel l; X = W [L][ldc], W = S' o p
//             out: partial y [split][K][ldc]
//   adjoint : owner = voxel l (rows of R_tab), streamed = sample k; X[k][c] = Y[k][c]
//             out: partial q [group * n_split + split][L] = sum_c conj(S'[l][c]) acc[l][c]
struct ContractLaunch {
  int prec;        // NFS_PREC_FP32 / NFS_PREC_FP64
  bool forward;
  int nc;          // coil group width (template NC)
  int nt;          // padded term count (template NT)
  int n_groups;    // coil groups of width nc
  int ldc;         // padded coil stride
  int64_t n_own, n_str;
  int n_split;     // split of the streamed range
  const void* own_tab;
  const void* str_tab;
  const void* sens;      // S' [L][ldc] (adjoint epilogue)
  const void* x;         // streamed operand rows [n_str][ldc]: W (forward) or samples (adjoint)
  void* out;             // partial y or partial q (or final if n_split == 1 for forward)
  const int* stop;       // device flag: skip work when the CG has stopped (may be null)
};

// Returns the number of CTAs per SM the contraction kernel for this launch achieves, and
// its CTA owner-tile size (owners per CTA).  Used by the host planner.
void contract_kernel_shape(int prec, bool forward, int nc, int nt, int* owners_per_cta,
                           int* streamed_chunk, int* ctas_per_sm);
cudaError_t launch_contract(const ContractLaunch& L, cudaStream_t st);
// W[l][c] = S'[l][c] * p[l] in the operator precision (forward operand)
cudaError_t launch_make_w(int prec, const void* sens, const double2* p, void* w, int64_t n_vox,
                          int ldc, const int* stop, cudaStream_t st);

}  // namespace nfs
