// nfs_bases.cuh -- device-side input preparation (tables, device bases, S', checks), see nfs_bases.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nfs {
int harmonic_terms(int order, int ndim);   // -1 for an unsupported order
cudaError_t launch_spatial_from_grid(const int64_t* d_vox, const double* d_b0, int64_t L, int nt, const int* dims,
                                     const double* fov, int order, double* d_rr, cudaStream_t st);
cudaError_t launch_col_absmax(const double* d_tab, int64_t n, int nt, unsigned long long* d_out, cudaStream_t st);
cudaError_t launch_to_float(const double* d_in, float* d_out, int64_t n, cudaStream_t st);
cudaError_t launch_prep_tables(const double* d_temporal, const double* d_spatial, int64_t K, int64_t L, int p1,
                               int nt, double* d_tt, double* d_rr, cudaStream_t st,
                               bool spatial_lp = false, bool radians = false);
cudaError_t launch_prep_sens(const double2* d_sens, const double* d_j, int64_t L, int g, int ldc, bool fp64,
                             void* d_out, cudaStream_t st);
cudaError_t launch_intensity(const double2* d_full, const int64_t* d_idx, int64_t n_r, int g, double* d_j,
                             cudaStream_t st);
cudaError_t launch_prep_sens_gather(const double2* d_full, const int64_t* d_idx, const double* d_j, int64_t n_r, int g,
                                    int ldc, bool fp64, void* d_out, cudaStream_t st);
cudaError_t launch_count_nonfinite(const double* d_x, int64_t n, unsigned int* d_out, cudaStream_t st);
}  // namespace nfs
