// nfs_plan.cu -- C ABI (include/nfs_b200.h): device plan, host<->device staging, the E^H E
// apply sequence, the device-resident CG driver (CUDA graph per iteration) and NCCL.
//
// One plan = one GPU = one contiguous shard of the readout samples.  The
// adjoint image is all-reduced (sum) once per CG iteration over NCCL when world > 1; every
// rank then runs the identical, deterministic CG update (nfs/engine.py:154-178).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/nfs_b200.h"
#include "nfs_common.cuh"
#include "nfs_tc.cuh"
#include "nfs_tci.cuh"
#include "nfs_bases.cuh"
#include "nfs_vec.cuh"

using nfs::CGState;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define NFS_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? NFS_ERR_BUDGET : NFS_ERR_CUDA,         \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                      \
  } while (0)

#define NFS_TRY(expr)            \
  do {                           \
    int s_ = (expr);             \
    if (s_ != NFS_OK) return s_; \
  } while (0)

// ------------------------------------------------------------------ NCCL (dlopen)
// Resolved at run time so the process shares the NCCL that torch already loaded.
typedef struct { char internal[128]; } nfsNcclUniqueId;
typedef void* nfsNcclComm;
typedef int (*pf_init_rank)(nfsNcclComm*, int, nfsNcclUniqueId, int);
typedef int (*pf_allreduce)(const void*, void*, size_t, int, int, nfsNcclComm, cudaStream_t);
typedef int (*pf_destroy)(nfsNcclComm);
typedef const char* (*pf_errstr)(int);
static const int kNcclDouble = 8;   // ncclFloat64
static const int kNcclSum = 0;      // ncclSum

struct NcclApi {
  bool ok = false;
  pf_init_rank init_rank = nullptr;
  pf_allreduce allreduce = nullptr;
  pf_destroy destroy = nullptr;
  pf_errstr errstr = nullptr;
  int (*count)(void*, int*) = nullptr;
};

static NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.init_rank = (pf_init_rank)dlsym(h, "ncclCommInitRank");
      api.allreduce = (pf_allreduce)dlsym(h, "ncclAllReduce");
      api.destroy = (pf_destroy)dlsym(h, "ncclCommDestroy");
      api.errstr = (pf_errstr)dlsym(h, "ncclGetErrorString");
      api.count = (int (*)(void*, int*))dlsym(h, "ncclCommCount");
      api.ok = api.init_rank && api.allreduce && api.destroy;
    }
  }
  return api;
}

// ------------------------------------------------------------------ plan
struct nfs_plan {
  int device = 0, prec = NFS_PREC_FP32;
  int64_t K = 0, L = 0;
  int G = 0, P1 = 0, NT = 0, NC = 0, NG = 0, ldc = 0;
  size_t esz = 4;                       // sizeof(T) of the operator arithmetic
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // tables and operands
  void *d_T = nullptr, *d_R = nullptr, *d_S = nullptr, *d_sig = nullptr, *d_y = nullptr;
  void *d_party = nullptr, *d_partq = nullptr, *d_w = nullptr;
  // CG vectors (complex128)
  double2 *d_p = nullptr, *d_q = nullptr, *d_r = nullptr, *d_rho = nullptr, *d_q0 = nullptr;
  double2* d_io = nullptr;
  size_t io_cap = 0;
  double* d_partials = nullptr;
  CGState* d_cg = nullptr;
  double *d_res = nullptr, *d_sol = nullptr;
  int log_cap = 0;
  int split_f = 1, split_a = 1;
  bool have_tables = false, have_sens = false, have_samples = false;
  nfsNcclComm comm = nullptr;
  bool owns_comm = true;   // false: a shared communicator (nfs_plan_use_comm) outlives the plan
  int rank = 0, world = 1;
  nfs::TcPlan* tc = nullptr;            // tensor-core operator, FP32 phase (NFS_PREC_TF32X3)
  nfs::TciPlan* tci = nullptr;          // tensor-core operator, exact int8 phase (NFS_PREC_F16X3)
  std::string desc;
  // device RMSE diagnostic (nfs_set_rmse_reference)
  double2* d_rmse_ref = nullptr;
  double* d_rmse_w = nullptr;
  double* d_rmse_log = nullptr;
  double rmse_outside = 0.0, rmse_ref_sq = 0.0;
  int rmse_cap = 0;
  bool rmse_on = false;
  // device SSIM diagnostic (nfs_set_ssim_reference)
  int64_t* d_ssim_vox = nullptr;
  double *d_ssim_w = nullptr, *d_ssim_img = nullptr, *d_ssim_ref = nullptr, *d_ssim_kern = nullptr, *d_ssim_log = nullptr;
  unsigned char* d_ssim_sel = nullptr;
  int ssim_nx = 0, ssim_ny = 0, ssim_win = 0, ssim_cap = 0;
  double ssim_c1 = 0, ssim_c2 = 0, ssim_nsel = 0;
  bool ssim_on = false;
};

static size_t t2size(const nfs_plan* P) { return 2 * P->esz; }

static int pick_nt(int p1) {
  if (p1 <= 4) return 4;
  if (p1 <= 8) return 8;
  if (p1 <= 16) return 16;
  if (p1 <= 20) return 20;
  if (p1 <= 32) return 32;
  return -1;
}

static int pick_nc(int g) {
  if (g <= 2) return 2;
  if (g <= 4) return 4;
  if (g <= 8) return 8;
  if (g <= 16) return 16;
  return 32;
}

static int choose_split(int64_t tiles, int64_t n_str, int chunk, int resident) {
  // Choose the split of the streamed range so that the CTA count fills whole waves of the
  // resident slots (148 SMs x CTAs/SM): tail waves idle SMs.  Keep >= 4 chunks per CTA.
  const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(64, n_str / (4LL * chunk)));
  int best = 1;
  double best_eff = -1.0;
  for (int64_t s = 1; s <= cap; ++s) {
    const double waves = (double)(tiles * s) / resident;
    if (waves < 1.0 && s < cap) continue;
    const double eff = waves / std::ceil(waves);
    if (eff >= 0.97 && waves >= 2.0) return (int)s;   // smallest split that packs well
    if (eff > best_eff + 1e-9) { best_eff = eff; best = (int)s; }
  }
  return best;
}

static int ensure_io(nfs_plan* P, size_t n_c128) {
  if (P->io_cap >= n_c128) return NFS_OK;
  if (P->d_io) {
    cudaStreamSynchronize(P->stream);   // the old buffer may still be read by queued work
    nfs::dev_free(P->d_io);
  }
  P->d_io = nullptr;
  NFS_CUDA(nfs::dev_alloc((void**)&P->d_io, n_c128 * sizeof(double2)));
  P->io_cap = n_c128;
  return NFS_OK;
}

extern "C" const char* nfs_last_error(void) { return g_err.c_str(); }
extern "C" const char* nfs_version(void) { return "nfs_b200 0.1 (sm_100a)"; }

static int f16x3_fallback(nfs_plan* P, const std::string& reason);

extern "C" int nfs_plan_create(nfs_plan** out, int64_t n_samples, int64_t n_voxels,
                               int32_t n_coils, int32_t n_terms, int32_t precision,
                               int32_t device) {
  if (!out) return fail(NFS_ERR_INVALID, "null plan pointer");
  *out = nullptr;
  if (n_samples < 0 || n_voxels < 1 || n_coils < 1 || n_terms < 1)
    return fail(NFS_ERR_INVALID, "plan sizes must be positive");
  const bool tensor = precision == NFS_PREC_TF32X3 || precision == NFS_PREC_F16X3;
  if (precision != NFS_PREC_FP32 && precision != NFS_PREC_FP64 && !tensor)
    return fail(NFS_ERR_INVALID, "unknown precision");
  const int nt = pick_nt(n_terms);
  if (nt < 0) return fail(NFS_ERR_INVALID, "at most 32 basis terms (P+1 <= 32) are supported");
  int ndev = 0;
  NFS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(NFS_ERR_INVALID, "invalid CUDA device");
  NFS_CUDA(cudaSetDevice(device));

  nfs_plan* P = new nfs_plan();
  P->device = device;
  P->prec = precision;
  P->K = n_samples;
  P->L = n_voxels;
  P->G = n_coils;
  P->P1 = n_terms;
  P->NT = nt;
  P->NC = pick_nc(n_coils);
  if (tensor) P->NC = std::max(P->NC, nfs::tc_coil_width(n_coils));   // 8 / 16 / 32 (same for tci)
  P->NG = (n_coils + P->NC - 1) / P->NC;
  P->ldc = P->NC * P->NG;
  P->esz = (precision == NFS_PREC_FP64) ? 8 : 4;
  auto bail = [&](int code) {
    nfs_plan_destroy(P);
    return code;
  };
  if (cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(NFS_ERR_CUDA, "stream creation failed"));
  P->own_stream = true;

  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int cprec = (precision == NFS_PREC_FP64) ? NFS_PREC_FP64 : NFS_PREC_FP32;
  int own_f, sc_f, occ_f, own_a, sc_a, occ_a;
  nfs::contract_kernel_shape(cprec, true, P->NC, nt, &own_f, &sc_f, &occ_f);
  nfs::contract_kernel_shape(cprec, false, P->NC, nt, &own_a, &sc_a, &occ_a);
  const int64_t K = std::max<int64_t>(P->K, 1), L = P->L;
  P->split_f = choose_split(((K + own_f - 1) / own_f) * P->NG, L, sc_f, sms * std::max(occ_f, 1));
  P->split_a = choose_split(((L + own_a - 1) / own_a) * P->NG, K, sc_a, sms * std::max(occ_a, 1));
  // forward partials are large (K x ldc per split): cap at ~1 GiB
  while (P->split_f > 1 && (size_t)P->split_f * K * P->ldc * t2size(P) > (1ull << 30)) --P->split_f;

  const size_t t2 = t2size(P);
  auto alloc = [&](void** p, size_t bytes) -> int {
    NFS_CUDA(nfs::dev_alloc(p, std::max<size_t>(bytes, 16)));
    NFS_CUDA(cudaMemsetAsync(*p, 0, std::max<size_t>(bytes, 16), P->stream));
    return NFS_OK;
  };
  int s = NFS_OK;
  if ((s = alloc(&P->d_T, (size_t)K * nt * P->esz)) ||
      (s = alloc(&P->d_R, (size_t)L * nt * P->esz)) ||
      (s = alloc(&P->d_S, (size_t)L * P->ldc * t2)) ||
      (s = alloc(&P->d_sig, (size_t)K * P->ldc * t2)) ||
      (s = alloc(&P->d_y, (size_t)K * P->ldc * t2)) ||
      (s = alloc(&P->d_w, (size_t)L * P->ldc * t2)) ||
      (s = alloc(&P->d_partq, (size_t)P->split_a * P->NG * L * sizeof(double2))) ||   // FP64 partial images
      (s = alloc((void**)&P->d_p, L * sizeof(double2))) ||
      (s = alloc((void**)&P->d_q, L * sizeof(double2))) ||
      (s = alloc((void**)&P->d_r, L * sizeof(double2))) ||
      (s = alloc((void**)&P->d_rho, L * sizeof(double2))) ||
      (s = alloc((void**)&P->d_q0, L * sizeof(double2))) ||
      (s = alloc((void**)&P->d_partials, 8 * 2048 * sizeof(double))) ||
      (s = alloc((void**)&P->d_cg, sizeof(CGState))))
    return bail(s);
  if (P->split_f > 1 && (s = alloc(&P->d_party, (size_t)P->split_f * K * P->ldc * t2)))
    return bail(s);
  std::string tci_note;
  if (precision == NFS_PREC_TF32X3) {
    std::string why;
    P->tc = nfs::tc_create(P->K, P->L, P->G, nt, sms, false, &why);
    if (!P->tc) return bail(fail(NFS_ERR_INVALID, "tensor-core path unavailable: " + why));
  } else if (precision == NFS_PREC_F16X3) {
    std::string why;
    P->tci = nfs::tci_create(P->K, P->L, P->G, nt, sms, &why);
    // too many basis terms for the kernel's shared-memory staging: fall back (after the
    // description is written, below)
    if (!P->tci && why.rfind("shared memory budget", 0) == 0) tci_note = std::to_string(P->P1) + " basis terms";
    else if (!P->tci) return bail(fail(NFS_ERR_INVALID, "tensor-core path unavailable: " + why));
  }
  char buf[512];
  snprintf(buf, sizeof buf,
           "prec=%s K=%lld L=%lld G=%d P1=%d NT=%d NC=%d groups=%d split_fwd=%d(occ %d, %d owners/CTA) "
           "split_adj=%d(occ %d, %d owners/CTA)%s",
           precision == NFS_PREC_FP64 ? "fp64" : (precision == NFS_PREC_FP32 ? "fp32" : (precision == NFS_PREC_F16X3 ? "f16x3" : "tf32x3")),
           (long long)P->K, (long long)P->L, P->G, P->P1, nt, P->NC, P->NG, P->split_f, occ_f,
           own_f, P->split_a, occ_a, own_a, P->tc ? nfs::tc_describe(P->tc) : (P->tci ? nfs::tci_describe(P->tci) : ""));
  P->desc = buf;
  if (!tci_note.empty()) {
    const int s = f16x3_fallback(P, tci_note);
    if (s) return bail(s);
  }
  if (cudaStreamSynchronize(P->stream) != cudaSuccess)
    return bail(fail(NFS_ERR_CUDA, "plan init failed"));
  *out = P;
  return NFS_OK;
}

extern "C" void nfs_plan_destroy(nfs_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  if (P->stream) cudaStreamSynchronize(P->stream);
  if (P->tc) nfs::tc_destroy(P->tc);
  if (P->tci) nfs::tci_destroy(P->tci);
  void* bufs[] = {P->d_T, P->d_R, P->d_S, P->d_sig, P->d_y, P->d_w, P->d_party, P->d_partq,
                  P->d_p, P->d_q, P->d_r, P->d_rho, P->d_q0, P->d_io, P->d_partials,
                  P->d_cg, P->d_res, P->d_sol, P->d_rmse_ref, P->d_rmse_w, P->d_rmse_log,
                  P->d_ssim_vox, P->d_ssim_w, P->d_ssim_img, P->d_ssim_ref, P->d_ssim_kern, P->d_ssim_log,
                  P->d_ssim_sel};
  for (void* b : bufs)
    if (b) nfs::dev_free(b);
  if (P->comm && P->owns_comm && nccl_api().ok) nccl_api().destroy(P->comm);
  if (P->own_stream && P->stream) cudaStreamDestroy(P->stream);
  delete P;
}

extern "C" int nfs_plan_set_stream(nfs_plan* P, void* stream) {
  if (!P) return fail(NFS_ERR_INVALID, "null plan");
  NFS_CUDA(cudaSetDevice(P->device));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  if (stream) {
    if (P->own_stream) cudaStreamDestroy(P->stream);
    P->own_stream = false;
    P->stream = (cudaStream_t)stream;
  }
  return NFS_OK;
}

extern "C" int nfs_plan_attach_comm(nfs_plan* P, const void* uid, int32_t rank, int32_t world) {
  if (!P) return fail(NFS_ERR_INVALID, "null plan");
  if (world <= 1 && !uid) { P->world = 1; P->rank = 0; return NFS_OK; }   // no exchange needed
  if (!uid || world < 1 || rank < 0 || rank >= world) return fail(NFS_ERR_INVALID, "bad rank/world");
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(NFS_ERR_NCCL, "libnccl.so.2 could not be loaded");
  NFS_CUDA(cudaSetDevice(P->device));
  nfsNcclUniqueId id;
  memcpy(id.internal, uid, 128);
  int r = api.init_rank(&P->comm, world, id, rank);
  if (r != 0) return fail(NFS_ERR_NCCL, std::string("ncclCommInitRank: ") + (api.errstr ? api.errstr(r) : "?"));
  P->rank = rank;
  P->world = world;
  int n = -1;
  if (api.count) api.count(P->comm, &n);   // the communicator's own rank count, for the logs
  P->desc += " [nccl comm rank " + std::to_string(rank) + " of " + std::to_string(n) + "]";
  return NFS_OK;
}

// A communicator shared by every plan of a process (one per rank, created once): plans borrow
// it with nfs_plan_use_comm, so a recon does not pay ncclCommInitRank again.
extern "C" int nfs_comm_create(const void* uid, int32_t rank, int32_t world, int32_t device, void** comm) {
  if (!uid || !comm || world < 1 || rank < 0 || rank >= world) return fail(NFS_ERR_INVALID, "bad rank/world");
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(NFS_ERR_NCCL, "libnccl.so.2 could not be loaded");
  NFS_CUDA(cudaSetDevice(device));
  nfsNcclUniqueId id;
  memcpy(id.internal, uid, 128);
  nfsNcclComm c = nullptr;
  int r = api.init_rank(&c, world, id, rank);
  if (r != 0) return fail(NFS_ERR_NCCL, std::string("ncclCommInitRank: ") + (api.errstr ? api.errstr(r) : "?"));
  *comm = c;
  return NFS_OK;
}

extern "C" void nfs_comm_destroy(void* comm) {
  if (comm && nccl_api().ok) nccl_api().destroy((nfsNcclComm)comm);
}

extern "C" int nfs_plan_use_comm(nfs_plan* P, void* comm, int32_t rank, int32_t world) {
  if (!P || !comm || world < 1 || rank < 0 || rank >= world) return fail(NFS_ERR_INVALID, "bad communicator");
  if (P->comm && P->owns_comm && nccl_api().ok) nccl_api().destroy(P->comm);
  P->comm = (nfsNcclComm)comm;
  P->owns_comm = false;
  P->rank = rank;
  P->world = world;
  int n = -1;
  if (nccl_api().count) nccl_api().count(P->comm, &n);
  P->desc += " [shared nccl comm rank " + std::to_string(rank) + " of " + std::to_string(n) + "]";
  return NFS_OK;
}

// ------------------------------------------------------------------ inputs
// An f16x3 plan whose basis the exact int8 phase kernel cannot take (phase range, or more terms
// than its shared-memory staging holds) runs on the TF32x3 tensor-core contraction (FP32 phase,
// the same accuracy class), else on the FP32 CUDA-core contraction; the description says which.
static int f16x3_fallback(nfs_plan* P, const std::string& reason) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device);
  std::string why;
  P->tc = nfs::tc_create(P->K, P->L, P->G, P->NT, sms, false, &why);
  if (!P->tc) {
    P->desc += " [f16x3 unavailable for " + reason + ": FP32 CUDA-core contraction]";
    return NFS_OK;
  }
  if (P->have_sens && nfs::tc_set_sens(P->tc, P->d_S, P->ldc, P->stream))
    return fail(NFS_ERR_CUDA, "tc sens: " + std::string(nfs::tc_last_error()));
  if (P->have_tables && nfs::tc_set_tables(P->tc, P->d_T, P->d_R, P->stream))
    return fail(NFS_ERR_CUDA, "tc tables: " + std::string(nfs::tc_last_error()));
  P->desc += " [f16x3 unavailable for " + reason + ": TF32x3 tensor-core contraction" +
             nfs::tc_describe(P->tc) + "]";
  return NFS_OK;
}

// FP64 device tables tt [K][nt] (turns) and rr [L][nt] -> the plan's operator tables, the
// tensor-core images, and the int8-phase fixed-point scales (all on the device)
static int finish_tables(nfs_plan* P, const double* d_tt, const double* d_rr) {
  const int nt = P->NT;
  const int64_t K = P->K, L = P->L;
  if (P->esz == 8) {
    NFS_CUDA(cudaMemcpyAsync(P->d_T, d_tt, (size_t)K * nt * 8, cudaMemcpyDeviceToDevice, P->stream));
    NFS_CUDA(cudaMemcpyAsync(P->d_R, d_rr, (size_t)L * nt * 8, cudaMemcpyDeviceToDevice, P->stream));
  } else {
    NFS_CUDA(nfs::launch_to_float(d_tt, (float*)P->d_T, K * nt, P->stream));
    NFS_CUDA(nfs::launch_to_float(d_rr, (float*)P->d_R, L * nt, P->stream));
  }
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  P->have_tables = true;
  if (P->tc) {
    int st = nfs::tc_set_tables(P->tc, P->d_T, P->d_R, P->stream);
    if (st) return fail(NFS_ERR_CUDA, "tc tables: " + std::string(nfs::tc_last_error()));
  }
  if (P->tci) {
    unsigned long long* d_max = nullptr;
    std::vector<unsigned long long> mx(2 * nt, 0ull);
    NFS_CUDA(nfs::dev_alloc((void**)&d_max, 2 * nt * sizeof(unsigned long long)));
    cudaError_t e = nfs::launch_col_absmax(d_tt, K, nt, d_max, P->stream);
    if (e == cudaSuccess) e = nfs::launch_col_absmax(d_rr, L, nt, d_max + nt, P->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(mx.data(), d_max, 2 * nt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, P->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(P->stream);
    nfs::dev_free(d_max);
    if (e != cudaSuccess) return fail(NFS_ERR_CUDA, std::string("table maxima: ") + cudaGetErrorString(e));
    std::vector<double> amax(2 * nt);
    for (int p = 0; p < 2 * nt; ++p) memcpy(&amax[p], &mx[p], 8);
    int st = nfs::tci_set_tables_dev(P->tci, d_tt, d_rr, amax.data(), amax.data() + nt, P->stream);
    if (st == 2) {
      // the exact int8 phase cannot represent this basis (some |t'_p r_p| > 2^12 turns)
      nfs::tci_destroy(P->tci);
      P->tci = nullptr;
      NFS_TRY(f16x3_fallback(P, "this basis (phase range)"));
    } else if (st) {
      return fail(NFS_ERR_INVALID, "tci tables: " + std::string(nfs::tci_last_error()));
    }
  }
  return NFS_OK;
}

// scratch device buffers freed on scope exit (after a stream sync)
struct DevScratch {
  cudaStream_t st;
  std::vector<void*> bufs;
  ~DevScratch() {
    cudaStreamSynchronize(st);
    for (void* b : bufs) nfs::dev_free(b);
  }
  template <typename T>
  cudaError_t get(T** p, size_t bytes) {
    cudaError_t e = nfs::dev_alloc((void**)p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) bufs.push_back(*p);
    return e;
  }
};

// spatial_lp: the spatial table is voxel-major [L][P1] (nfs_set_tables_t) instead of [P1][L]
static int set_tables_impl(nfs_plan* P, const double* temporal, const double* spatial, bool spatial_lp) {
  if (!P || (!temporal && P->K > 0) || !spatial) return fail(NFS_ERR_INVALID, "null table");
  NFS_CUDA(cudaSetDevice(P->device));
  const int nt = P->NT, p1 = P->P1;
  const int64_t K = P->K, L = P->L;
  // raw tables up, scaling / transposition / padding on the device
  DevScratch sc{P->stream, {}};
  double *d_temp = nullptr, *d_spat = nullptr, *d_tt = nullptr, *d_rr = nullptr;
  NFS_CUDA(sc.get(&d_temp, (size_t)K * p1 * 8));
  NFS_CUDA(sc.get(&d_spat, (size_t)p1 * L * 8));
  NFS_CUDA(sc.get(&d_tt, (size_t)K * nt * 8));
  NFS_CUDA(sc.get(&d_rr, (size_t)L * nt * 8));
  if (K > 0) NFS_CUDA(nfs::h2d(d_temp, temporal, (size_t)K * p1 * 8, P->stream));
  NFS_CUDA(nfs::h2d(d_spat, spatial, (size_t)p1 * L * 8, P->stream));
  NFS_CUDA(nfs::launch_prep_tables(d_temp, d_spat, K, L, p1, nt, d_tt, d_rr, P->stream, spatial_lp,
                                   P->prec == NFS_PREC_FP64));
  return finish_tables(P, d_tt, d_rr);
}

extern "C" int nfs_set_tables(nfs_plan* P, const double* temporal, const double* spatial) {
  return set_tables_impl(P, temporal, spatial, false);
}

extern "C" int nfs_set_tables_t(nfs_plan* P, const double* temporal, const double* spatial_t) {
  return set_tables_impl(P, temporal, spatial_t, true);
}

// Spatial table evaluated on the device from the masked voxel indices: same
// tables as nfs_set_tables(temporal, build_bases(...)[0]) bit for bit.
extern "C" int nfs_set_tables_grid(nfs_plan* P, const double* temporal, const int64_t* vox_index,
                                   const double* b0_masked, const int32_t* dims, const double* fov, int32_t order) {
  if (!P || (!temporal && P->K > 0) || !vox_index || !b0_masked || !dims || !fov)
    return fail(NFS_ERR_INVALID, "null argument");
  if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || !(fov[0] > 0) || !(fov[1] > 0) || !(fov[2] > 0))
    return fail(NFS_ERR_INVALID, "grid extents and FOV must be positive");
  const int ndim = dims[2] == 1 ? 2 : 3;
  const int nh = nfs::harmonic_terms(order, ndim);
  if (nh < 0) return fail(NFS_ERR_INVALID, "unsupported harmonic order " + std::to_string(order));
  if (1 + nh != P->P1)
    return fail(NFS_ERR_INVALID, "order " + std::to_string(order) + " gives " + std::to_string(1 + nh) +
                                     " basis rows but the plan has " + std::to_string(P->P1));
  const int64_t nvox = (int64_t)dims[0] * dims[1] * dims[2];
  for (int64_t l = 0; l < P->L; ++l)
    if (vox_index[l] < 0 || vox_index[l] >= nvox) return fail(NFS_ERR_INVALID, "voxel index outside the grid");
  NFS_CUDA(cudaSetDevice(P->device));
  const int nt = P->NT, p1 = P->P1;
  const int64_t K = P->K, L = P->L;
  DevScratch sc{P->stream, {}};
  int64_t* d_vox = nullptr;
  double *d_b0 = nullptr, *d_temp = nullptr, *d_tt = nullptr, *d_rr = nullptr;
  NFS_CUDA(sc.get(&d_vox, (size_t)L * 8));
  NFS_CUDA(sc.get(&d_b0, (size_t)L * 8));
  NFS_CUDA(sc.get(&d_temp, (size_t)K * p1 * 8));
  NFS_CUDA(sc.get(&d_tt, (size_t)K * nt * 8));
  NFS_CUDA(sc.get(&d_rr, (size_t)L * nt * 8));
  NFS_CUDA(cudaMemcpyAsync(d_vox, vox_index, L * 8, cudaMemcpyHostToDevice, P->stream));
  NFS_CUDA(cudaMemcpyAsync(d_b0, b0_masked, L * 8, cudaMemcpyHostToDevice, P->stream));
  if (K > 0) NFS_CUDA(nfs::h2d(d_temp, temporal, (size_t)K * p1 * 8, P->stream));
  NFS_CUDA(nfs::launch_prep_tables(d_temp, nullptr, K, 0, p1, nt, d_tt, nullptr, P->stream, false,
                                   P->prec == NFS_PREC_FP64));
  NFS_CUDA(nfs::launch_spatial_from_grid(d_vox, d_b0, L, nt, dims, fov, order, d_rr, P->stream));
  return finish_tables(P, d_tt, d_rr);
}

extern "C" int nfs_set_sens(nfs_plan* P, const double* sens, const double* intensity) {
  if (!P || !sens) return fail(NFS_ERR_INVALID, "null sensitivities");
  NFS_CUDA(cudaSetDevice(P->device));
  const int64_t L = P->L;
  DevScratch sc{P->stream, {}};
  double2* d_sens = nullptr;
  double* d_j = nullptr;
  NFS_CUDA(sc.get(&d_sens, (size_t)L * P->G * sizeof(double2)));
  NFS_CUDA(nfs::h2d(d_sens, sens, (size_t)L * P->G * sizeof(double2), P->stream));
  if (intensity) {
    NFS_CUDA(sc.get(&d_j, (size_t)L * 8));
    NFS_CUDA(cudaMemcpyAsync(d_j, intensity, (size_t)L * 8, cudaMemcpyHostToDevice, P->stream));
  }
  NFS_CUDA(nfs::launch_prep_sens(d_sens, d_j, L, P->G, P->ldc, P->esz == 8, P->d_S, P->stream));   // S' = S o j
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  P->have_sens = true;
  if (P->tc) {
    int s = nfs::tc_set_sens(P->tc, P->d_S, P->ldc, P->stream);
    if (s) return fail(NFS_ERR_CUDA, "tc sens: " + std::string(nfs::tc_last_error()));
  }
  if (P->tci) {
    int s = nfs::tci_set_sens(P->tci, P->d_S, P->ldc, P->stream);
    if (s) return fail(NFS_ERR_CUDA, "tci sens: " + std::string(nfs::tci_last_error()));
  }
  return NFS_OK;
}

// S' from the FULL-grid maps (f3: the mask restriction and, with intensity == NULL, the intensity
// correction run on the device): S'[l] = S_full[vox_index[l]] o j[l].
extern "C" int nfs_set_sens_grid(nfs_plan* P, const double* sens_full, int64_t n_full, const int64_t* vox_index,
                                 const double* intensity, double* j_out) {
  if (!P || !sens_full || !vox_index || n_full < P->L) return fail(NFS_ERR_INVALID, "bad full-grid sensitivities");
  NFS_CUDA(cudaSetDevice(P->device));
  const int64_t L = P->L;
  for (int64_t l = 0; l < L; ++l)
    if (vox_index[l] < 0 || vox_index[l] >= n_full) return fail(NFS_ERR_INVALID, "voxel index outside the grid");
  DevScratch sc{P->stream, {}};
  double2* d_full = nullptr;
  int64_t* d_idx = nullptr;
  double* d_j = nullptr;
  NFS_CUDA(sc.get(&d_full, (size_t)n_full * P->G * sizeof(double2)));
  NFS_CUDA(sc.get(&d_idx, (size_t)L * sizeof(int64_t)));
  NFS_CUDA(sc.get(&d_j, (size_t)L * 8));
  NFS_CUDA(nfs::h2d(d_full, sens_full, (size_t)n_full * P->G * sizeof(double2), P->stream));
  NFS_CUDA(cudaMemcpyAsync(d_idx, vox_index, (size_t)L * sizeof(int64_t), cudaMemcpyHostToDevice, P->stream));
  if (intensity) NFS_CUDA(cudaMemcpyAsync(d_j, intensity, (size_t)L * 8, cudaMemcpyHostToDevice, P->stream));
  else NFS_CUDA(nfs::launch_intensity(d_full, d_idx, L, P->G, d_j, P->stream));
  NFS_CUDA(nfs::launch_prep_sens_gather(d_full, d_idx, d_j, L, P->G, P->ldc, P->esz == 8, P->d_S, P->stream));
  if (j_out) NFS_CUDA(cudaMemcpyAsync(j_out, d_j, (size_t)L * 8, cudaMemcpyDeviceToHost, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  P->have_sens = true;
  if (P->tc) {
    int s = nfs::tc_set_sens(P->tc, P->d_S, P->ldc, P->stream);
    if (s) return fail(NFS_ERR_CUDA, "tc sens: " + std::string(nfs::tc_last_error()));
  }
  if (P->tci) {
    int s = nfs::tci_set_sens(P->tci, P->d_S, P->ldc, P->stream);
    if (s) return fail(NFS_ERR_CUDA, "tci sens: " + std::string(nfs::tci_last_error()));
  }
  return NFS_OK;
}

// Stateless device intensity correction (nfs/sensmaps.py:145-152) of the reconstructed voxels.
extern "C" int nfs_intensity_correction(int32_t device, const double* sens_full, int64_t n_full, int32_t n_coils,
                                        const int64_t* vox_index, int64_t n_r, double* j_out) {
  if (!sens_full || !vox_index || !j_out || n_full < 0 || n_r < 0 || n_coils < 1)
    return fail(NFS_ERR_INVALID, "bad arguments");
  for (int64_t l = 0; l < n_r; ++l)
    if (vox_index[l] < 0 || vox_index[l] >= n_full) return fail(NFS_ERR_INVALID, "voxel index outside the grid");
  NFS_CUDA(cudaSetDevice(device));
  cudaStream_t st = nfs::alloc_stream();
  DevScratch sc{st, {}};
  double2* d_full = nullptr;
  int64_t* d_idx = nullptr;
  double* d_j = nullptr;
  NFS_CUDA(sc.get(&d_full, (size_t)n_full * n_coils * sizeof(double2)));
  NFS_CUDA(sc.get(&d_idx, (size_t)n_r * sizeof(int64_t)));
  NFS_CUDA(sc.get(&d_j, (size_t)n_r * 8));
  NFS_CUDA(nfs::h2d(d_full, sens_full, (size_t)n_full * n_coils * sizeof(double2), st));
  NFS_CUDA(cudaMemcpyAsync(d_idx, vox_index, (size_t)n_r * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  NFS_CUDA(nfs::launch_intensity(d_full, d_idx, n_r, n_coils, d_j, st));
  NFS_CUDA(cudaMemcpyAsync(j_out, d_j, (size_t)n_r * 8, cudaMemcpyDeviceToHost, st));
  NFS_CUDA(cudaStreamSynchronize(st));
  return NFS_OK;
}

static int upload_samples(nfs_plan* P, const double* sigma, void* dst) {
  const size_t n = (size_t)P->K * P->G;
  NFS_TRY(ensure_io(P, std::max<size_t>(n, (size_t)P->L)));
  NFS_CUDA(nfs::h2d(P->d_io, sigma, n * sizeof(double2), P->stream));
  NFS_CUDA(nfs::launch_pack(P->prec == NFS_PREC_FP64 ? 1 : 0, P->d_io, dst, P->K, P->G, P->ldc, P->stream));
  return NFS_OK;
}

static int finish_samples(nfs_plan* P);

extern "C" int nfs_set_samples(nfs_plan* P, const double* sigma) {
  if (!P || (!sigma && P->K > 0)) return fail(NFS_ERR_INVALID, "null samples");
  NFS_CUDA(cudaSetDevice(P->device));
  const size_t n = (size_t)P->K * P->G;
  NFS_TRY(ensure_io(P, std::max<size_t>(n, (size_t)P->L)));
  NFS_CUDA(nfs::h2d(P->d_io, sigma, n * sizeof(double2), P->stream));
  return finish_samples(P);
}

// Samples straight from a dataset file: rows [row0, row0 + K) of a raw little-endian complex128
// (K_total, n_coils) array (the reference's `sigma.c128`, nfs/core.py:292-328) -- a sharded rank
// reads only its own rows from disk.
extern "C" int nfs_set_samples_file(nfs_plan* P, const char* path, int64_t row0) {
  if (!P || !path || row0 < 0) return fail(NFS_ERR_INVALID, "bad sample file arguments");
  NFS_CUDA(cudaSetDevice(P->device));
  const size_t n = (size_t)P->K * P->G;
  NFS_TRY(ensure_io(P, std::max<size_t>(n, (size_t)P->L)));
  const cudaError_t e = nfs::h2d_file(P->d_io, path, row0 * (int64_t)P->G * 16, n * sizeof(double2), P->stream);
  if (e == cudaErrorInvalidValue) return fail(NFS_ERR_INVALID, std::string("cannot read the sample rows from ") + path);
  NFS_CUDA(e);
  return finish_samples(P);
}

static int finish_samples(nfs_plan* P) {
  const size_t n = (size_t)P->K * P->G;
  unsigned int bad = 0;
  unsigned int* d_bad = reinterpret_cast<unsigned int*>(P->d_partials);   // reduction scratch
  NFS_CUDA(nfs::launch_count_nonfinite(reinterpret_cast<const double*>(P->d_io), (int64_t)n * 2, d_bad, P->stream));
  NFS_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  if (bad) return fail(NFS_ERR_NONFINITE, "raw data contains non-finite values");
  NFS_CUDA(nfs::launch_pack(P->prec == NFS_PREC_FP64 ? 1 : 0, P->d_io, P->d_sig, P->K, P->G, P->ldc, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  P->have_samples = true;
  return NFS_OK;
}

// ------------------------------------------------------------------ operator sequences
static nfs::ContractLaunch base_launch(const nfs_plan* P, bool fwd) {
  nfs::ContractLaunch L{};
  L.prec = (P->prec == NFS_PREC_FP64) ? NFS_PREC_FP64 : NFS_PREC_FP32;
  L.forward = fwd;
  L.nc = P->NC;
  L.nt = P->NT;
  L.n_groups = P->NG;
  L.ldc = P->ldc;
  L.sens = P->d_S;
  if (fwd) {
    L.n_own = P->K; L.n_str = P->L; L.own_tab = P->d_T; L.str_tab = P->d_R; L.n_split = P->split_f;
  } else {
    L.n_own = P->L; L.n_str = P->K; L.own_tab = P->d_R; L.str_tab = P->d_T; L.n_split = P->split_a;
  }
  return L;
}

// y = E p  (device p -> device y [K][ldc] in operator precision)
static int run_forward(nfs_plan* P, const double2* p, const int* stop) {
  if (P->tc) {
    int s = nfs::tc_forward(P->tc, p, P->d_y, stop, P->stream);
    if (s) return fail(NFS_ERR_CUDA, std::string("tc forward: ") + nfs::tc_last_error());
    return NFS_OK;
  }
  if (P->tci) {
    int s = nfs::tci_forward_parts(P->tci, p, P->d_y, stop, P->stream, 0);
    if (!s) s = nfs::tci_forward_parts(P->tci, p, P->d_y, stop, P->stream, 1);
    if (s) return fail(NFS_ERR_CUDA, std::string("tci forward: ") + nfs::tci_last_error());
    return NFS_OK;
  }
  if (P->K == 0) return NFS_OK;
  nfs::ContractLaunch L = base_launch(P, true);
  NFS_CUDA(nfs::launch_make_w(L.prec, P->d_S, p, P->d_w, P->L, P->ldc, stop, P->stream));
  L.x = P->d_w;
  L.stop = stop;
  L.out = (P->split_f > 1) ? P->d_party : P->d_y;
  NFS_CUDA(nfs::launch_contract(L, P->stream));
  if (P->split_f > 1)
    NFS_CUDA(nfs::launch_reduce_parts(L.prec == NFS_PREC_FP64 ? 1 : 0, P->d_party, P->d_y,
                                      P->K * P->ldc, P->split_f, stop, P->stream));
  return NFS_OK;
}

// q = E^H y (device y [K][ldc] -> device q, all-reduced over ranks)
static int run_adjoint(nfs_plan* P, const void* y, double2* q, const int* stop) {
  if (P->tc) {
    int s = nfs::tc_adjoint(P->tc, y, q, stop, P->stream);
    if (s) return fail(NFS_ERR_CUDA, std::string("tc adjoint: ") + nfs::tc_last_error());
  } else if (P->tci) {
    int s = nfs::tci_adjoint_parts(P->tci, y, q, stop, P->stream, 0);
    if (!s) s = nfs::tci_adjoint_parts(P->tci, y, q, stop, P->stream, 1);
    if (s) return fail(NFS_ERR_CUDA, std::string("tci adjoint: ") + nfs::tci_last_error());
  } else if (P->K == 0) {
    NFS_CUDA(cudaMemsetAsync(q, 0, P->L * sizeof(double2), P->stream));
  } else {
    nfs::ContractLaunch L = base_launch(P, false);
    L.x = y;
    L.stop = stop;
    L.out = P->d_partq;
    NFS_CUDA(nfs::launch_contract(L, P->stream));
    NFS_CUDA(nfs::launch_reduce_image(1, P->d_partq, q, P->L,
                                      P->split_a * P->NG, stop, P->stream));
  }
  if (P->comm) {   // sample-sharded: sum the adjoint images of all ranks (in place)
    int r = nccl_api().allreduce(q, q, (size_t)P->L * 2, kNcclDouble, kNcclSum, P->comm, P->stream);
    if (r != 0) return fail(NFS_ERR_NCCL, "ncclAllReduce failed");
  }
  return NFS_OK;
}

static int run_ehe(nfs_plan* P, const double2* p, double2* q, const int* stop) {
  NFS_TRY(run_forward(P, p, stop));
  NFS_TRY(run_adjoint(P, P->d_y, q, stop));
  return NFS_OK;
}

static int need_ready(nfs_plan* P) {
  if (!P) return fail(NFS_ERR_INVALID, "null plan");
  if (!P->have_tables || !P->have_sens) return fail(NFS_ERR_INVALID, "tables and sensitivities must be set first");
  NFS_CUDA(cudaSetDevice(P->device));
  return NFS_OK;
}

extern "C" int nfs_apply_E(nfs_plan* P, const double* p, double* y) {
  NFS_TRY(need_ready(P));
  NFS_TRY(ensure_io(P, std::max<size_t>((size_t)P->K * P->G, (size_t)P->L)));
  NFS_CUDA(cudaMemcpyAsync(P->d_p, p, P->L * sizeof(double2), cudaMemcpyHostToDevice, P->stream));
  NFS_TRY(run_forward(P, P->d_p, nullptr));
  NFS_CUDA(nfs::launch_unpack(P->prec == NFS_PREC_FP64 ? 1 : 0, P->d_y, P->d_io, P->K, P->G, P->ldc, P->stream));
  NFS_CUDA(cudaMemcpyAsync(y, P->d_io, (size_t)P->K * P->G * sizeof(double2), cudaMemcpyDeviceToHost, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  return NFS_OK;
}

extern "C" int nfs_apply_EH(nfs_plan* P, const double* sigma, double* q) {
  NFS_TRY(need_ready(P));
  NFS_TRY(upload_samples(P, sigma, P->d_y));
  NFS_TRY(run_adjoint(P, P->d_y, P->d_q, nullptr));
  NFS_CUDA(cudaMemcpyAsync(q, P->d_q, P->L * sizeof(double2), cudaMemcpyDeviceToHost, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  return NFS_OK;
}

extern "C" int nfs_apply_EHE(nfs_plan* P, const double* p, double* q) {
  NFS_TRY(need_ready(P));
  NFS_CUDA(cudaMemcpyAsync(P->d_p, p, P->L * sizeof(double2), cudaMemcpyHostToDevice, P->stream));
  NFS_TRY(run_ehe(P, P->d_p, P->d_q, nullptr));
  NFS_CUDA(cudaMemcpyAsync(q, P->d_q, P->L * sizeof(double2), cudaMemcpyDeviceToHost, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  return NFS_OK;
}

extern "C" int nfs_phase_rows(nfs_plan* P, int64_t lo, int64_t hi, double* out) {
  if (!P || !P->have_tables) return fail(NFS_ERR_INVALID, "tables must be set first");
  if (lo < 0 || hi > P->K || hi < lo) return fail(NFS_ERR_INVALID, "row range out of bounds");
  if (hi == lo) return NFS_OK;
  NFS_CUDA(cudaSetDevice(P->device));
  const size_t n = (size_t)(hi - lo) * P->L;
  double2* d = nullptr;
  NFS_CUDA(nfs::dev_alloc((void**)&d, n * sizeof(double2)));
  cudaError_t e = nfs::launch_phase_rows(P->prec == NFS_PREC_FP64 ? 1 : 0, P->NT, P->d_T, P->d_R,
                                         lo, hi - lo, P->L, d, P->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, n * sizeof(double2), cudaMemcpyDeviceToHost, P->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(P->stream);
  nfs::dev_free(d);
  if (e != cudaSuccess) return fail(NFS_ERR_CUDA, std::string("phase rows: ") + cudaGetErrorString(e));
  return NFS_OK;
}

// ------------------------------------------------------------------ CG
static int cg_iteration(nfs_plan* P) {
  const int* stop = &P->d_cg->stop;
  NFS_TRY(run_ehe(P, P->d_p, P->d_q, stop));
  NFS_CUDA(nfs::launch_cg_iter_tail(P->d_q, P->d_p, P->d_r, P->d_rho, P->L, P->d_cg,
                                    P->d_partials, P->d_res, P->d_sol, P->stream));
  if (P->rmse_on)
    NFS_CUDA(nfs::launch_cg_rmse(P->d_rho, P->d_rmse_ref, P->d_rmse_w, P->L, P->d_cg, P->d_partials,
                                 P->rmse_outside, P->rmse_ref_sq, P->d_rmse_log, P->stream));
  if (P->ssim_on)
    NFS_CUDA(nfs::launch_cg_ssim(P->d_rho, P->d_ssim_w, P->d_ssim_vox, P->L, P->d_ssim_img, P->d_ssim_ref,
                                 P->ssim_nx, P->ssim_ny, P->d_ssim_kern, P->ssim_win, P->ssim_c1, P->ssim_c2,
                                 P->d_ssim_sel, P->ssim_nsel, P->d_cg, P->d_partials, P->d_ssim_log, P->stream));
  return NFS_OK;
}

// Device-side per-iteration mean SSIM of |rho o j| on an nx x ny grid against
// ref_img (nx*ny, x fastest), window kernel kern (win x win), constants c1, c2 (from the
// reference's dynamic range), optional window selection sel ((nx-win+1) x (ny-win+1), x
// fastest).  vox_index: grid index of every reconstructed voxel; weight: j.  NULL ref_img off.
extern "C" int nfs_set_ssim_reference(nfs_plan* P, const int64_t* vox_index, const double* weight, int32_t nx,
                                      int32_t ny, const double* ref_img, const double* kern, int32_t win,
                                      double c1, double c2, const uint8_t* sel) {
  if (!P) return fail(NFS_ERR_INVALID, "null plan");
  if (!ref_img) {
    P->ssim_on = false;
    return NFS_OK;
  }
  if (!vox_index || !weight || !kern || nx < win || ny < win || win < 1)
    return fail(NFS_ERR_INVALID, "image smaller than the SSIM window");
  const int64_t npix = (int64_t)nx * ny, nwin = (int64_t)(nx - win + 1) * (ny - win + 1);
  for (int64_t l = 0; l < P->L; ++l)
    if (vox_index[l] < 0 || vox_index[l] >= npix) return fail(NFS_ERR_INVALID, "voxel index outside the image");
  double n_sel = (double)nwin;
  if (sel) {
    n_sel = 0;
    for (int64_t o = 0; o < nwin; ++o) n_sel += sel[o] ? 1.0 : 0.0;
    if (n_sel == 0) return fail(NFS_ERR_INVALID, "mask covers no valid windows");
  }
  NFS_CUDA(cudaSetDevice(P->device));
  cudaStreamSynchronize(P->stream);
  void* old[] = {P->d_ssim_vox, P->d_ssim_w, P->d_ssim_img, P->d_ssim_ref, P->d_ssim_kern, P->d_ssim_sel};
  for (void* b : old) nfs::dev_free(b);
  P->d_ssim_vox = nullptr; P->d_ssim_w = P->d_ssim_img = P->d_ssim_ref = P->d_ssim_kern = nullptr;
  P->d_ssim_sel = nullptr;
  NFS_CUDA(nfs::dev_alloc((void**)&P->d_ssim_vox, std::max<int64_t>(P->L, 1) * 8));
  NFS_CUDA(nfs::dev_alloc((void**)&P->d_ssim_w, std::max<int64_t>(P->L, 1) * 8));
  NFS_CUDA(nfs::dev_alloc((void**)&P->d_ssim_img, npix * 8));
  NFS_CUDA(nfs::dev_alloc((void**)&P->d_ssim_ref, npix * 8));
  NFS_CUDA(nfs::dev_alloc((void**)&P->d_ssim_kern, (size_t)win * win * 8));
  if (sel) NFS_CUDA(nfs::dev_alloc((void**)&P->d_ssim_sel, nwin));
  NFS_CUDA(cudaMemcpyAsync(P->d_ssim_vox, vox_index, P->L * 8, cudaMemcpyHostToDevice, P->stream));
  NFS_CUDA(cudaMemcpyAsync(P->d_ssim_w, weight, P->L * 8, cudaMemcpyHostToDevice, P->stream));
  NFS_CUDA(cudaMemcpyAsync(P->d_ssim_ref, ref_img, npix * 8, cudaMemcpyHostToDevice, P->stream));
  NFS_CUDA(cudaMemcpyAsync(P->d_ssim_kern, kern, (size_t)win * win * 8, cudaMemcpyHostToDevice, P->stream));
  if (sel) NFS_CUDA(cudaMemcpyAsync(P->d_ssim_sel, sel, nwin, cudaMemcpyHostToDevice, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  P->ssim_nx = nx; P->ssim_ny = ny; P->ssim_win = win; P->ssim_c1 = c1; P->ssim_c2 = c2; P->ssim_nsel = n_sel;
  P->ssim_on = true;
  return NFS_OK;
}

extern "C" int nfs_ssim_log(nfs_plan* P, double* out, int32_t n) {
  if (!P || !out || n < 0) return fail(NFS_ERR_INVALID, "bad arguments");
  if (!P->ssim_on || n > P->ssim_cap) return fail(NFS_ERR_INVALID, "no SSIM log of that length");
  if (n > 0) NFS_CUDA(cudaMemcpy(out, P->d_ssim_log, n * sizeof(double), cudaMemcpyDeviceToHost));
  return NFS_OK;
}

// Device-side per-iteration relative RMSE of rho o j vs a reference image: no
// host copy of the iterate per iteration.  ref_masked: reference on the reconstruction mask
// (L_R complex, zero off the RMSE support); weight: j on the support, 0 off it; outside_sq: the
// support's |ref|^2 outside the reconstruction mask; ref_sq: the support's total |ref|^2.
// ref_masked == NULL switches the diagnostic off.
extern "C" int nfs_set_rmse_reference(nfs_plan* P, const double* ref_masked, const double* weight,
                                      double outside_sq, double ref_sq) {
  if (!P) return fail(NFS_ERR_INVALID, "null plan");
  if (!ref_masked) {
    P->rmse_on = false;
    return NFS_OK;
  }
  if (!weight || !(ref_sq > 0.0) || !std::isfinite(ref_sq) || !(outside_sq >= 0.0))
    return fail(NFS_ERR_INVALID, "RMSE reference is zero on the support");
  NFS_CUDA(cudaSetDevice(P->device));
  if (!P->d_rmse_ref) {
    NFS_CUDA(nfs::dev_alloc((void**)&P->d_rmse_ref, std::max<int64_t>(P->L, 1) * sizeof(double2)));
    NFS_CUDA(nfs::dev_alloc((void**)&P->d_rmse_w, std::max<int64_t>(P->L, 1) * sizeof(double)));
  }
  NFS_CUDA(cudaMemcpyAsync(P->d_rmse_ref, ref_masked, P->L * sizeof(double2), cudaMemcpyHostToDevice, P->stream));
  NFS_CUDA(cudaMemcpyAsync(P->d_rmse_w, weight, P->L * sizeof(double), cudaMemcpyHostToDevice, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  P->rmse_outside = outside_sq;
  P->rmse_ref_sq = ref_sq;
  P->rmse_on = true;
  return NFS_OK;
}

// per-iteration RMSE values of the last nfs_cg_solve (n <= iterations done)
extern "C" int nfs_rmse_log(nfs_plan* P, double* out, int32_t n) {
  if (!P || !out || n < 0) return fail(NFS_ERR_INVALID, "bad arguments");
  if (!P->rmse_on || n > P->rmse_cap) return fail(NFS_ERR_INVALID, "no RMSE log of that length");
  if (n > 0) NFS_CUDA(cudaMemcpy(out, P->d_rmse_log, n * sizeof(double), cudaMemcpyDeviceToHost));
  return NFS_OK;
}

extern "C" int nfs_cg_solve(nfs_plan* P, int32_t n_iter, nfs_iter_callback cb, void* user,
                            double* rho, double* res_norms, double* sol_norms, int32_t* n_done,
                            double* timings) {
  NFS_TRY(need_ready(P));
  if (!P->have_samples) return fail(NFS_ERR_INVALID, "samples must be set first");
  if (n_iter < 0) return fail(NFS_ERR_INVALID, "negative iteration count");
  if (n_done) *n_done = 0;
  if (n_iter > P->log_cap) {
    cudaStreamSynchronize(P->stream);
    if (P->d_res) nfs::dev_free(P->d_res);
    if (P->d_sol) nfs::dev_free(P->d_sol);
    P->d_res = P->d_sol = nullptr;
    NFS_CUDA(nfs::dev_alloc((void**)&P->d_res, std::max(n_iter, 1) * sizeof(double)));
    NFS_CUDA(nfs::dev_alloc((void**)&P->d_sol, std::max(n_iter, 1) * sizeof(double)));
    P->log_cap = n_iter;
  }
  if (P->ssim_on && n_iter > P->ssim_cap) {
    cudaStreamSynchronize(P->stream);
    nfs::dev_free(P->d_ssim_log);
    P->d_ssim_log = nullptr;
    NFS_CUDA(nfs::dev_alloc((void**)&P->d_ssim_log, std::max(n_iter, 1) * sizeof(double)));
    P->ssim_cap = n_iter;
  }
  if (P->rmse_on && n_iter > P->rmse_cap) {
    cudaStreamSynchronize(P->stream);
    nfs::dev_free(P->d_rmse_log);
    P->d_rmse_log = nullptr;
    NFS_CUDA(nfs::dev_alloc((void**)&P->d_rmse_log, std::max(n_iter, 1) * sizeof(double)));
    P->rmse_cap = n_iter;
  }
  std::vector<cudaEvent_t> ev(n_iter + 2);
  for (auto& e : ev) NFS_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    std::vector<cudaEvent_t>& v;
    ~EvGuard() { for (auto e : v) cudaEventDestroy(e); }
  } guard{ev};

  NFS_CUDA(cudaMemsetAsync(P->d_cg, 0, sizeof(CGState), P->stream));
  NFS_CUDA(cudaEventRecord(ev[0], P->stream));
  NFS_TRY(run_adjoint(P, P->d_sig, P->d_q0, nullptr));                 // initial_adjoint
  NFS_CUDA(nfs::launch_cg_init(P->d_q0, P->d_r, P->d_p, P->d_rho, P->L, P->d_cg, P->d_partials, P->stream));
  NFS_CUDA(cudaEventRecord(ev[1], P->stream));

  // capture one iteration as a CUDA graph (falls back to direct launches)
  cudaGraphExec_t gexec = nullptr;
  if (n_iter > 1) {
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      int s = cg_iteration(P);
      cudaError_t ce = cudaStreamEndCapture(P->stream, &graph);
      if (s == NFS_OK && ce == cudaSuccess && graph &&
          cudaGraphInstantiate(&gexec, graph, 0) != cudaSuccess)
        gexec = nullptr;
      if (graph) cudaGraphDestroy(graph);
    }
    cudaGetLastError();
  }
  std::vector<double> host_rho;
  if (cb) host_rho.resize((size_t)P->L * 2);
  int done = 0, aborted = 0;
  CGState st{};
  for (int n = 1; n <= n_iter; ++n) {
    if (gexec) NFS_CUDA(cudaGraphLaunch(gexec, P->stream));
    else NFS_TRY(cg_iteration(P));
    NFS_CUDA(cudaEventRecord(ev[n + 1], P->stream));
    if (cb) {
      NFS_CUDA(cudaMemcpyAsync(&st, P->d_cg, sizeof st, cudaMemcpyDeviceToHost, P->stream));
      NFS_CUDA(cudaStreamSynchronize(P->stream));
      if (st.err || st.iter < n) break;
      NFS_CUDA(cudaMemcpy(host_rho.data(), P->d_rho, P->L * sizeof(double2), cudaMemcpyDeviceToHost));
      if (cb(n, host_rho.data(), user) != 0) {
        aborted = n;
        break;
      }
      if (st.stop) break;
    }
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  NFS_CUDA(cudaMemcpyAsync(&st, P->d_cg, sizeof st, cudaMemcpyDeviceToHost, P->stream));
  NFS_CUDA(cudaStreamSynchronize(P->stream));
  done = st.iter;
  if (n_done) *n_done = st.err ? st.err_iter : done;
  if (st.err == NFS_ERR_BREAKDOWN)
    return fail(NFS_ERR_BREAKDOWN, "CG breakdown at iteration " + std::to_string(st.err_iter));
  if (st.err == NFS_ERR_NONFINITE_ITERATE)
    return fail(NFS_ERR_NONFINITE_ITERATE, "non-finite iterate at iteration " + std::to_string(st.err_iter));
  if (aborted) {
    if (n_done) *n_done = aborted;
    return fail(NFS_ERR_ABORTED, "solve aborted by the iteration callback at iteration " + std::to_string(aborted));
  }
  if (rho) NFS_CUDA(cudaMemcpy(rho, P->d_rho, P->L * sizeof(double2), cudaMemcpyDeviceToHost));
  if (done > 0) {
    if (res_norms) NFS_CUDA(cudaMemcpy(res_norms, P->d_res, done * sizeof(double), cudaMemcpyDeviceToHost));
    if (sol_norms) NFS_CUDA(cudaMemcpy(sol_norms, P->d_sol, done * sizeof(double), cudaMemcpyDeviceToHost));
  }
  if (timings) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[0], ev[1]);
    timings[0] = ms * 1e-3;
    const int last = cb ? std::min(done, n_iter) : n_iter;
    cudaEventElapsedTime(&ms, ev[0], ev[std::max(last, 0) + 1]);
    timings[1] = ms * 1e-3;
    for (int n = 1; n <= n_iter; ++n) {
      timings[1 + n] = 0.0;
      if (n <= done && n <= last) {
        cudaEventElapsedTime(&ms, ev[n], ev[n + 1]);
        timings[1 + n] = ms * 1e-3;
      }
    }
  }
  return NFS_OK;
}

// ------------------------------------------------------------------ benchmarking hooks
extern "C" int nfs_apply_EHE_resident(nfs_plan* P, int32_t n) {
  NFS_TRY(need_ready(P));
  for (int i = 0; i < n; ++i) NFS_TRY(run_ehe(P, P->d_p, P->d_q, nullptr));
  return NFS_OK;
}

// Benchmark steps: n E^H E applies on the resident p, each preceded by a device write of
// flush_bytes (evicts L2; outside the timed events) and timed with CUDA events on the plan
// stream: step_ms[i] = the whole apply (both operators, reductions, the NCCL all-reduce when a
// communicator is attached); kern_ms[0] / [1] = summed durations of the forward / adjoint main
// contraction kernel over the n steps (events around each launch, same timed steps).
extern "C" int nfs_bench_applies(nfs_plan* P, int32_t n, int64_t flush_bytes, float* step_ms, float* kern_ms) {
  NFS_TRY(need_ready(P));
  if (n < 1 || !step_ms || !kern_ms || flush_bytes < 0) return fail(NFS_ERR_INVALID, "bad arguments");
  void* flush = nullptr;
  if (flush_bytes > 0) NFS_CUDA(nfs::dev_alloc(&flush, (size_t)flush_bytes));
  std::vector<cudaEvent_t> ev((size_t)n * 6);
  int status = NFS_OK;
  for (auto& e : ev) {
    if (cudaEventCreate(&e) != cudaSuccess) { status = fail(NFS_ERR_CUDA, "cudaEventCreate"); break; }
  }
  nfs::KernelEvents& kev = nfs::kernel_events();
  for (int i = 0; i < n && status == NFS_OK; ++i) {
    if (flush) cudaMemsetAsync(flush, i & 0xff, (size_t)flush_bytes, P->stream);
    cudaEvent_t* e = &ev[(size_t)i * 6];
    for (int k = 0; k < 4; ++k) kev.ev[k] = e[1 + k];
    kev.on = 1;
    cudaEventRecord(e[0], P->stream);
    status = run_ehe(P, P->d_p, P->d_q, nullptr);
    cudaEventRecord(e[5], P->stream);
    kev.on = 0;
  }
  kev.on = 0;
  if (status == NFS_OK && cudaStreamSynchronize(P->stream) != cudaSuccess) status = fail(NFS_ERR_CUDA, "bench sync");
  kern_ms[0] = kern_ms[1] = 0.f;
  for (int i = 0; i < n && status == NFS_OK; ++i) {
    cudaEvent_t* e = &ev[(size_t)i * 6];
    float a = 0.f, f = 0.f, d = 0.f;
    cudaEventElapsedTime(&a, e[0], e[5]);
    cudaEventElapsedTime(&f, e[1], e[2]);
    cudaEventElapsedTime(&d, e[3], e[4]);
    step_ms[i] = a;
    kern_ms[0] += f;
    kern_ms[1] += d;
  }
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  if (flush) {
    cudaStreamSynchronize(P->stream);
    nfs::dev_free(flush);
  }
  return status;
}

extern "C" int nfs_kernel_times(nfs_plan* P, int32_t reps, float* ms_out) {
  NFS_TRY(need_ready(P));
  if (reps < 1 || !ms_out) return fail(NFS_ERR_INVALID, "bad arguments");
  cudaEvent_t e[5];
  for (auto& x : e) NFS_CUDA(cudaEventCreate(&x));
  double acc[4] = {0, 0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    if (P->tci) {
      NFS_CUDA(cudaEventRecord(e[0], P->stream));
      if (nfs::tci_forward_parts(P->tci, P->d_p, P->d_y, nullptr, P->stream, 0)) return fail(NFS_ERR_CUDA, nfs::tci_last_error());
      NFS_CUDA(cudaEventRecord(e[1], P->stream));
      if (nfs::tci_forward_parts(P->tci, P->d_p, P->d_y, nullptr, P->stream, 1)) return fail(NFS_ERR_CUDA, nfs::tci_last_error());
      NFS_CUDA(cudaEventRecord(e[2], P->stream));
      if (nfs::tci_adjoint_parts(P->tci, P->d_y, P->d_q, nullptr, P->stream, 0)) return fail(NFS_ERR_CUDA, nfs::tci_last_error());
      NFS_CUDA(cudaEventRecord(e[3], P->stream));
      if (nfs::tci_adjoint_parts(P->tci, P->d_y, P->d_q, nullptr, P->stream, 1)) return fail(NFS_ERR_CUDA, nfs::tci_last_error());
      NFS_CUDA(cudaEventRecord(e[4], P->stream));
    } else if (P->tc) {
      NFS_CUDA(cudaEventRecord(e[0], P->stream));
      if (nfs::tc_forward_parts(P->tc, P->d_p, P->d_y, nullptr, P->stream, 0))
        return fail(NFS_ERR_CUDA, nfs::tc_last_error());
      NFS_CUDA(cudaEventRecord(e[1], P->stream));
      if (nfs::tc_forward_parts(P->tc, P->d_p, P->d_y, nullptr, P->stream, 1))
        return fail(NFS_ERR_CUDA, nfs::tc_last_error());
      NFS_CUDA(cudaEventRecord(e[2], P->stream));
      if (nfs::tc_adjoint_parts(P->tc, P->d_y, P->d_q, nullptr, P->stream, 0))
        return fail(NFS_ERR_CUDA, nfs::tc_last_error());
      NFS_CUDA(cudaEventRecord(e[3], P->stream));
      if (nfs::tc_adjoint_parts(P->tc, P->d_y, P->d_q, nullptr, P->stream, 1))
        return fail(NFS_ERR_CUDA, nfs::tc_last_error());
      NFS_CUDA(cudaEventRecord(e[4], P->stream));
    } else {
      const int cp = (P->prec == NFS_PREC_FP64) ? 1 : 0;
      nfs::ContractLaunch F = base_launch(P, true);
      F.x = P->d_w;
      F.out = (P->split_f > 1) ? P->d_party : P->d_y;
      nfs::ContractLaunch A = base_launch(P, false);
      A.x = P->d_y;
      A.out = P->d_partq;
      NFS_CUDA(nfs::launch_make_w(F.prec, P->d_S, P->d_p, P->d_w, P->L, P->ldc, nullptr, P->stream));
      NFS_CUDA(cudaEventRecord(e[0], P->stream));
      NFS_CUDA(nfs::launch_contract(F, P->stream));
      NFS_CUDA(cudaEventRecord(e[1], P->stream));
      if (P->split_f > 1)
        NFS_CUDA(nfs::launch_reduce_parts(cp, P->d_party, P->d_y, P->K * P->ldc, P->split_f, nullptr, P->stream));
      NFS_CUDA(cudaEventRecord(e[2], P->stream));
      NFS_CUDA(nfs::launch_contract(A, P->stream));
      NFS_CUDA(cudaEventRecord(e[3], P->stream));
      NFS_CUDA(nfs::launch_reduce_image(1, P->d_partq, P->d_q, P->L, P->split_a * P->NG, nullptr, P->stream));
      NFS_CUDA(cudaEventRecord(e[4], P->stream));
    }
    NFS_CUDA(cudaEventSynchronize(e[4]));
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e[i], e[i + 1]);
      acc[i] += ms;
    }
  }
  for (auto& x : e) cudaEventDestroy(x);
  for (int i = 0; i < 4; ++i) ms_out[i] = (float)(acc[i] / reps);
  return NFS_OK;
}

extern "C" int nfs_launches_per_apply(nfs_plan* P) {
  if (!P) return 0;
  if (P->tc) return nfs::tc_launches_per_apply(P->tc);
  if (P->tci) return nfs::tci_launches_per_apply(P->tci);
  return 2 + (P->split_f > 1 ? 1 : 0) + 2;
}

extern "C" const char* nfs_plan_describe(nfs_plan* P) { return P ? P->desc.c_str() : ""; }
