// nfs_tci.cuh -- tensor-core operator with the phase computed EXACTLY on the INT8 tensor cores
// (NFS_PREC_F16X3).  Operates on the FP32 layouts of nfs_common.cuh for S' and the samples.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace nfs {

struct TciPlan;
TciPlan* tci_create(int64_t K, int64_t L, int G, int nt, int sms, std::string* why);
void tci_destroy(TciPlan* t);
const char* tci_describe(TciPlan* t);
const char* tci_last_error();
// tables from FP64 device tables (temporal in turns [K][nt], spatial [L][nt], zero padded) and
// their per-term max |value| (host arrays); returns 2 when the exact fixed-point phase range is
// exceeded (the caller then uses the FP32 CUDA-core contraction)
int tci_set_tables_dev(TciPlan* t, const double* d_tt, const double* d_rr, const double* amax_t,
                       const double* amax_r, cudaStream_t st);
int tci_set_sens(TciPlan* t, const void* d_S, int ldc, cudaStream_t st);
// part 0 = prep + main kernel, part 1 = split reduction
int tci_forward_parts(TciPlan* t, const double2* p, void* y, const int* stop, cudaStream_t st, int part);
int tci_adjoint_parts(TciPlan* t, const void* y, double2* q, const int* stop, cudaStream_t st, int part);
int tci_launches_per_apply(TciPlan* t);
int tci_coil_width(int G);

}  // namespace nfs
