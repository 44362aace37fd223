// nfs_bases.cuh -- device-side spatial basis, see nfs_bases.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nfs {
int harmonic_terms(int order, int ndim);   // -1 for an unsupported order
cudaError_t launch_spatial_from_grid(const int64_t* d_vox, const double* d_b0, int64_t L, int nt, const int* dims,
                                     const double* fov, int order, double* d_rr, cudaStream_t st);
cudaError_t launch_col_absmax(const double* d_tab, int64_t n, int nt, unsigned long long* d_out, cudaStream_t st);
cudaError_t launch_to_float(const double* d_in, float* d_out, int64_t n, cudaStream_t st);
}  // namespace nfs
