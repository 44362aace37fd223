// nfs_tc.cuh -- tensor-core (tcgen05) split-precision operator path, NFS_PREC_TF32X3 / F16X3.
// Operates on the FP32 layouts of nfs_common.cuh: T_tab/R_tab (float, NT terms),
// S' float2 [L][ldc], samples float2 [K][ldc].
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace nfs {

struct TcPlan;
// coil group width of the tensor-core path (8, 16 or 32); the plan pads its coil stride to it
int tc_coil_width(int G);
TcPlan* tc_create(int64_t K, int64_t L, int G, int nt, int sms, bool f16, std::string* why);
void tc_destroy(TcPlan* t);
const char* tc_describe(TcPlan* t);
const char* tc_last_error();
int tc_set_tables(TcPlan* t, const void* d_T, const void* d_R, cudaStream_t st);
int tc_set_sens(TcPlan* t, const void* d_S, int ldc, cudaStream_t st);
// y (float2 [K][ldc]) = E p
int tc_forward(TcPlan* t, const double2* p, void* y, const int* stop, cudaStream_t st);
// q (complex128, L) = E^H y
int tc_adjoint(TcPlan* t, const void* y, double2* q, const int* stop, cudaStream_t st);
// the two launch groups of each operator (part 0 = main kernel, 1 = epilogue/reduce)
int tc_forward_parts(TcPlan* t, const double2* p, void* y, const int* stop, cudaStream_t st, int part);
int tc_adjoint_parts(TcPlan* t, const void* y, double2* q, const int* stop, cudaStream_t st, int part);
int tc_launches_per_apply(TcPlan* t);

}  // namespace nfs
