// nfs_vec.cuh -- device CG state and host launchers of nfs_vec.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nfs {

struct CGState {
  double2 alpha;     // vdot(r, r) (real)
  double2 step;      // alpha / beta
  double ratio;      // alpha_new / alpha_old
  double r0;         // ||r_0||
  int iter;          // completed iterations
  int stop;          // 0 running, 1 error/zero rhs, 2 early stop
  int err;           // 0, NFS_ERR_BREAKDOWN, NFS_ERR_NONFINITE_ITERATE
  int err_iter;
  unsigned int ticket;
};

cudaError_t launch_pack(int prec, const double2* src, void* dst, int64_t rows, int g, int ldc,
                        cudaStream_t st);
cudaError_t launch_unpack(int prec, const void* src, double2* dst, int64_t rows, int g, int ldc,
                          cudaStream_t st);
cudaError_t launch_reduce_parts(int prec, const void* part, void* out, int64_t n, int n_part,
                                const int* stop, cudaStream_t st);
cudaError_t launch_reduce_image(int prec, const void* part, double2* q, int64_t n, int n_part,
                                const int* stop, cudaStream_t st);
int cg_grid(int64_t n);
cudaError_t launch_cg_ssim(const double2* rho, const double* w, const int64_t* vox, int64_t n, double* img,
                           const double* ref, int nx, int ny, const double* kern, int win, double c1, double c2,
                           const unsigned char* sel, double n_sel, CGState* s, double* partials, double* log,
                           cudaStream_t st);
cudaError_t launch_cg_rmse(const double2* rho, const double2* ref, const double* w, int64_t n, CGState* s,
                           double* partials, double outside, double ref_sq, double* log, cudaStream_t st);
cudaError_t launch_cg_init(const double2* q0, double2* r, double2* p, double2* rho, int64_t n,
                           CGState* s, double* partials, cudaStream_t st);
cudaError_t launch_cg_iter_tail(const double2* q, double2* p, double2* r, double2* rho, int64_t n,
                                CGState* s, double* partials, double* res_log, double* sol_log,
                                cudaStream_t st);
cudaError_t launch_phase_rows(int prec, int nt, const void* ttab, const void* rtab,
                              int64_t row_lo, int64_t rows, int64_t n_vox, double2* out,
                              cudaStream_t st);

}  // namespace nfs
