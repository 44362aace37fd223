// nfs_bases.cu -- device-side input preparation: basis tables (incl. the spatial basis evaluated
// from voxel indices), S' = S o j, and the raw-data finiteness check.
//
// R[l, 0] = B0 (rad/s) of masked voxel l, R[l, 1..] = the zero-Laplacian solid harmonics of its
// grid coordinates (order 1 / 2 / 3: 2-or-3 / 8 / 15 terms), in the plan's [L_R][NT] FP64 table
// layout.  Restates engine.build_bases (nfs/engine.py:252-280), solid_harmonics
// (nfs/simulate.py:26-59) and grid_coordinates (nfs/core.py:102-113) with explicitly rounded
// IEEE operations in numpy's evaluation order, so the table is bit-identical to the host build.
// Only the voxel index (8 B) and B0 (8 B) cross PCIe per voxel instead of P+1 doubles.
#include <cuda_runtime.h>
#include <stdint.h>

#include "nfs_bases.cuh"

namespace nfs {

__device__ __forceinline__ double axis_coord(int64_t m, int n, double fov) {
  const double pitch = __ddiv_rn(fov, (double)n);                   // fov / n
  const double off = __dsub_rn((double)m, __ddiv_rn((double)(n - 1), 2.0));   // m - (n-1)/2
  return __dmul_rn(pitch, off);
}

__global__ void spatial_from_grid_kernel(const int64_t* __restrict__ vox, const double* __restrict__ b0,
                                         int64_t L, int nt, int nx, int ny, int nz, double fx, double fy,
                                         double fz, int ndim, int order, double* __restrict__ rr) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = vox[l];
    const int64_t ix = idx % nx, iy = (idx / nx) % ny, iz = idx / ((int64_t)nx * ny);
    const double x = axis_coord(ix, nx, fx), y = axis_coord(iy, ny, fy), z = axis_coord(iz, nz, fz);
    double* r = rr + l * nt;
    int p = 0;
    r[p++] = b0[l];
    r[p++] = x;
    r[p++] = y;
    if (!(ndim == 2 && order == 1)) r[p++] = z;
    const double x2 = __dmul_rn(x, x), y2 = __dmul_rn(y, y), z2 = __dmul_rn(z, z);
    if (order >= 2) {
      r[p++] = __dmul_rn(x, y);
      r[p++] = __dmul_rn(z, y);
      r[p++] = __dsub_rn(__dsub_rn(__dmul_rn(2.0, z2), x2), y2);           // 2 z^2 - x^2 - y^2
      r[p++] = __dmul_rn(z, x);
      r[p++] = __dsub_rn(x2, y2);
    }
    if (order >= 3) {
      r[p++] = __dmul_rn(y, __dsub_rn(__dmul_rn(3.0, x2), y2));                           // y (3x^2 - y^2)
      r[p++] = __dmul_rn(__dmul_rn(x, y), z);                                              // x y z
      r[p++] = __dmul_rn(y, __dsub_rn(__dsub_rn(__dmul_rn(4.0, z2), x2), y2));           // y (4z^2 - x^2 - y^2)
      r[p++] = __dmul_rn(z, __dsub_rn(__dsub_rn(__dmul_rn(2.0, z2), __dmul_rn(3.0, x2)), __dmul_rn(3.0, y2)));
      r[p++] = __dmul_rn(x, __dsub_rn(__dsub_rn(__dmul_rn(4.0, z2), x2), y2));           // x (4z^2 - x^2 - y^2)
      r[p++] = __dmul_rn(z, __dsub_rn(x2, y2));                                            // z (x^2 - y^2)
      r[p++] = __dmul_rn(x, __dsub_rn(x2, __dmul_rn(3.0, y2)));                           // x (x^2 - 3y^2)
    }
    for (; p < nt; ++p) r[p] = 0.0;
  }
}

// per-column max |v| of a [n][nt] FP64 table (for the fixed-point scales of the int8 phase)
__global__ void col_absmax_kernel(const double* __restrict__ tab, int64_t n, int nt, unsigned long long* out) {
  for (int p = 0; p < nt; ++p) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      m = fmax(m, fabs(tab[i * nt + p]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&out[p], (unsigned long long)__double_as_longlong(m));   // m >= 0
  }
}

__global__ void to_float_kernel(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

// temporal [K][P1] (rad) -> tt [K][nt] (turns, zero padded); spatial [P1][L] -> rr [L][nt]
__global__ void prep_tables_kernel(const double* __restrict__ temporal, const double* __restrict__ spatial,
                                   int64_t K, int64_t L, int p1, int nt, bool spatial_lp, double tscale,
                                   double* __restrict__ tt, double* __restrict__ rr) {
  const int64_t nk = K * nt, total = nk + L * nt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nk) {
      const int64_t k = i / nt;
      const int p = (int)(i - k * nt);
      tt[i] = p < p1 ? temporal[k * p1 + p] * tscale : 0.0;
    } else {
      const int64_t j = i - nk, l = j / nt;
      const int p = (int)(j - l * nt);
      rr[j] = p < p1 ? spatial[spatial_lp ? l * p1 + p : (int64_t)p * L + l] : 0.0;
    }
  }
}

// S' = S o j with the coil stride padded to ldc (FP32 or FP64 layout)
template <typename T2>
__global__ void prep_sens_kernel(const double2* __restrict__ sens, const double* __restrict__ j, int64_t L, int g,
                                 int ldc, T2* __restrict__ out) {
  const int64_t n = L * ldc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / ldc;
    const int c = (int)(i - l * ldc);
    T2 v;
    v.x = 0; v.y = 0;
    if (c < g) {
      const double w = j ? j[l] : 1.0;
      const double2 s = sens[l * g + c];
      v.x = s.x * w;
      v.y = s.y * w;
    }
    out[i] = v;
  }
}

// Intensity correction on the device (nfs/sensmaps.py:145-152): for every reconstructed voxel
// (grid index idx[l]) j = 1/sqrt(sum_c |S_c|^2) if that sum is > 0, else 0.  |S|^2 is formed as
// abs(S)^2 with abs = hypot, like numpy's np.abs(maps) ** 2; the coil sum runs in numpy's
// pairwise order for rows of <= 128 coils (8 interleaved partial sums, combined as
// ((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7)), then the remainder sequentially), so j matches the
// reference to the last bit up to the hypot rounding (CUDA hypot: <= 1 ulp).
__global__ void intensity_kernel(const double2* __restrict__ full, const int64_t* __restrict__ idx, int64_t n_r,
                                 int g, double* __restrict__ j) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n_r; l += (int64_t)gridDim.x * blockDim.x) {
    const double2* row = full + idx[l] * g;
    auto sq = [&](int c) {
      const double a = hypot(row[c].x, row[c].y);
      return a * a;
    };
    double ssq;
    if (g < 8) {
      ssq = 0.0;
      for (int c = 0; c < g; ++c) ssq += sq(c);
    } else {
      double r[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = sq(k);
      int c = 8;
      for (; c + 8 <= g; c += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] += sq(c + k);
      ssq = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; c < g; ++c) ssq += sq(c);
    }
    j[l] = ssq > 0.0 ? 1.0 / sqrt(ssq) : 0.0;
  }
}

// S' = S[idx] o j: the mask restriction as a gather of the full-grid maps (coils padded to ldc)
template <typename T2>
__global__ void prep_sens_gather_kernel(const double2* __restrict__ full, const int64_t* __restrict__ idx,
                                        const double* __restrict__ j, int64_t n_r, int g, int ldc, T2* __restrict__ out) {
  const int64_t n = n_r * ldc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / ldc;
    const int c = (int)(i - l * ldc);
    T2 v;
    v.x = 0; v.y = 0;
    if (c < g) {
      const double w = j[l];
      const double2 s = full[idx[l] * g + c];
      v.x = s.x * w;
      v.y = s.y * w;
    }
    out[i] = v;
  }
}

// count of non-finite doubles (raw data check of nfs_set_samples)
__global__ void count_nonfinite_kernel(const double* __restrict__ x, int64_t n, unsigned int* out) {
  unsigned int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad += isfinite(x[i]) ? 0u : 1u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(out, bad);
}

int harmonic_terms(int order, int ndim) {
  if (order == 1) return ndim == 2 ? 2 : 3;
  if (order == 2) return 8;
  if (order == 3) return 15;
  return -1;
}

static int grid_for(int64_t n) { return (int)(n / 256 + 1 < 148 * 8 ? n / 256 + 1 : 148 * 8); }

cudaError_t launch_spatial_from_grid(const int64_t* d_vox, const double* d_b0, int64_t L, int nt, const int* dims,
                                     const double* fov, int order, double* d_rr, cudaStream_t st) {
  const int ndim = dims[2] == 1 ? 2 : 3;
  spatial_from_grid_kernel<<<grid_for(L), 256, 0, st>>>(d_vox, d_b0, L, nt, dims[0], dims[1], dims[2], fov[0], fov[1],
                                                        fov[2], ndim, order, d_rr);
  return cudaGetLastError();
}

cudaError_t launch_col_absmax(const double* d_tab, int64_t n, int nt, unsigned long long* d_out, cudaStream_t st) {
  cudaMemsetAsync(d_out, 0, nt * sizeof(unsigned long long), st);
  col_absmax_kernel<<<grid_for(n), 256, 0, st>>>(d_tab, n, nt, d_out);
  return cudaGetLastError();
}

cudaError_t launch_to_float(const double* d_in, float* d_out, int64_t n, cudaStream_t st) {
  to_float_kernel<<<grid_for(n), 256, 0, st>>>(d_in, d_out, n);
  return cudaGetLastError();
}

// temporal table in turns (temporal / 2pi: the FP32 and tensor-core paths) or, radians = true, as
// given (the FP64 parity path computes phi = temporal . spatial exactly like the reference's dgemm
// and takes sin/cos of phi itself)
cudaError_t launch_prep_tables(const double* d_temporal, const double* d_spatial, int64_t K, int64_t L, int p1,
                               int nt, double* d_tt, double* d_rr, cudaStream_t st, bool spatial_lp, bool radians) {
  const double tscale = radians ? 1.0 : 1.0 / 6.283185307179586476925286766559;
  prep_tables_kernel<<<grid_for((K + L) * nt), 256, 0, st>>>(d_temporal, d_spatial, K, L, p1, nt, spatial_lp, tscale,
                                                             d_tt, d_rr);
  return cudaGetLastError();
}

cudaError_t launch_prep_sens(const double2* d_sens, const double* d_j, int64_t L, int g, int ldc, bool fp64,
                             void* d_out, cudaStream_t st) {
  if (fp64) prep_sens_kernel<double2><<<grid_for(L * ldc), 256, 0, st>>>(d_sens, d_j, L, g, ldc, (double2*)d_out);
  else prep_sens_kernel<float2><<<grid_for(L * ldc), 256, 0, st>>>(d_sens, d_j, L, g, ldc, (float2*)d_out);
  return cudaGetLastError();
}

cudaError_t launch_intensity(const double2* d_full, const int64_t* d_idx, int64_t n_r, int g, double* d_j,
                             cudaStream_t st) {
  if (n_r > 0) intensity_kernel<<<grid_for(n_r), 256, 0, st>>>(d_full, d_idx, n_r, g, d_j);
  return cudaGetLastError();
}

cudaError_t launch_prep_sens_gather(const double2* d_full, const int64_t* d_idx, const double* d_j, int64_t n_r, int g,
                                    int ldc, bool fp64, void* d_out, cudaStream_t st) {
  if (n_r <= 0) return cudaSuccess;
  if (fp64) prep_sens_gather_kernel<double2><<<grid_for(n_r * ldc), 256, 0, st>>>(d_full, d_idx, d_j, n_r, g, ldc, (double2*)d_out);
  else prep_sens_gather_kernel<float2><<<grid_for(n_r * ldc), 256, 0, st>>>(d_full, d_idx, d_j, n_r, g, ldc, (float2*)d_out);
  return cudaGetLastError();
}

cudaError_t launch_count_nonfinite(const double* d_x, int64_t n, unsigned int* d_out, cudaStream_t st) {
  cudaMemsetAsync(d_out, 0, sizeof(unsigned int), st);
  count_nonfinite_kernel<<<grid_for(n), 256, 0, st>>>(d_x, n, d_out);
  return cudaGetLastError();
}

}  // namespace nfs
