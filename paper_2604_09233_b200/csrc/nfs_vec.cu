// nfs_vec.cu -- split reductions, sample packing and the device-side CG recurrence.
//
// CG follows nfs/engine.py:154-178 exactly (same update order, complex step alpha/beta with
// beta = vdot(p, q), early stop ||r|| <= 1e-15 ||r0|| checked before each iteration,
// breakdown on beta == 0 / non-finite, non-finite iterate).  All reductions are
// deterministic: fixed per-thread strides, fixed warp-shuffle trees, and the last CTA to
// finish (ticket counter) sums the per-CTA partials in index order -- no float atomics.
#include <cuda_runtime.h>
#include <stdint.h>

#include "nfs_common.cuh"
#include "nfs_vec.cuh"
#include "nfs_phase.cuh"

namespace nfs {

// ------------------------------------------------------------------ packing
template <typename T2>
__global__ void pack_samples_kernel(const double2* __restrict__ src, T2* __restrict__ dst,
                                    int64_t rows, int g, int ldc) {
  const int64_t n = rows * ldc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / ldc;
    const int c = (int)(i - k * ldc);
    T2 v;
    if (c < g) { const double2 s = src[k * g + c]; v.x = s.x; v.y = s.y; }
    else { v.x = 0; v.y = 0; }
    dst[i] = v;
  }
}

template <typename T2>
__global__ void unpack_samples_kernel(const T2* __restrict__ src, double2* __restrict__ dst,
                                      int64_t rows, int g, int ldc) {
  const int64_t n = rows * g;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / g;
    const int c = (int)(i - k * g);
    const T2 s = src[k * ldc + c];
    dst[i] = make_double2(s.x, s.y);
  }
}

// sum of n_part partial arrays of length n (T2), fixed order, into T2 out
template <typename T2>
__global__ void reduce_parts_kernel(const T2* __restrict__ part, T2* __restrict__ out,
                                    int64_t n, int n_part, const int* stop) {
  if (stop && *stop) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    T2 a = part[i];
    for (int s = 1; s < n_part; ++s) { const T2 b = part[(int64_t)s * n + i]; a.x += b.x; a.y += b.y; }
    out[i] = a;
  }
}

// adjoint partials -> double2 image (accumulate in double, fixed order)
template <typename T2>
__global__ void reduce_image_kernel(const T2* __restrict__ part, double2* __restrict__ q,
                                    int64_t n, int n_part, const int* stop) {
  if (stop && *stop) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double ax = 0.0, ay = 0.0;
    for (int s = 0; s < n_part; ++s) { const T2 b = part[(int64_t)s * n + i]; ax += b.x; ay += b.y; }
    q[i] = make_double2(ax, ay);
  }
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum of NV values; result valid in thread 0.  Fixed tree -> deterministic.
template <int NV>
__device__ void block_sum(double (&v)[NV]) {
  __shared__ double sm[NV][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) sm[j][w] = v[j];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) { v[j] = (lane < nw) ? sm[j][lane] : 0.0; v[j] = warp_sum(v[j]); }
  }
  __syncthreads();
}

// Write this CTA's NV partials; returns true in the LAST CTA, which then holds the totals
// (summed in CTA index order) in tot[].
template <int NV>
__device__ bool grid_sum(double (&v)[NV], double* partials, unsigned int* ticket,
                         double (&tot)[NV]) {
  __shared__ bool last;
  block_sum<NV>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) partials[(int64_t)j * gridDim.x + blockIdx.x] = v[j];
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double w[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    w[j] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
      w[j] += ((volatile double*)partials)[(int64_t)j * gridDim.x + b];
  }
  block_sum<NV>(w);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) tot[j] = w[j];
    *ticket = 0u;   // re-arm for the next launch (stream order guarantees no overlap)
  }
  return true;
}

// ------------------------------------------------------------------ CG kernels
__device__ __forceinline__ bool finite2(double2 a) { return isfinite(a.x) && isfinite(a.y); }

// r = p = q0, rho = 0, alpha = vdot(r, r), r0 = ||r||
__global__ void cg_init_kernel(const double2* __restrict__ q0, double2* __restrict__ r,
                               double2* __restrict__ p, double2* __restrict__ rho, int64_t n,
                               CGState* st, double* partials) {
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = q0[i];
    r[i] = a; p[i] = a; rho[i] = make_double2(0.0, 0.0);
    v[0] = fma(a.x, a.x, fma(a.y, a.y, v[0]));
  }
  double tot[1];
  if (grid_sum<1>(v, partials, &st->ticket, tot) && threadIdx.x == 0) {
    st->alpha = make_double2(tot[0], 0.0);
    st->r0 = sqrt(tot[0]);
    st->iter = 0;
    st->err = 0;
    st->err_iter = 0;
    // iteration-1 check of nfs/engine.py:158: ||r|| <= 1e-15 * r0 (true only for r0 == 0)
    st->stop = (st->r0 <= 1e-15 * st->r0) ? 1 : 0;
  }
}

// beta = vdot(p, q); breakdown check; step = alpha / beta
__global__ void cg_dot_kernel(const double2* __restrict__ p, const double2* __restrict__ q,
                              int64_t n, CGState* st, double* partials) {
  if (st->stop) return;
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = p[i], b = q[i];   // conj(a) * b
    v[0] = fma(a.x, b.x, fma(a.y, b.y, v[0]));
    v[1] = fma(a.x, b.y, fma(-a.y, b.x, v[1]));
  }
  double tot[2];
  if (grid_sum<2>(v, partials, &st->ticket, tot) && threadIdx.x == 0) {
    const double2 beta = make_double2(tot[0], tot[1]);
    if ((beta.x == 0.0 && beta.y == 0.0) || !finite2(beta)) {
      st->err = 3;   // NFS_ERR_BREAKDOWN
      st->err_iter = st->iter + 1;
      st->stop = 1;
      return;
    }
    // complex division alpha / beta, Smith's algorithm as numpy's complex128 scalar math
    const double2 al = st->alpha;
    if (fabs(beta.x) >= fabs(beta.y)) {
      const double rat = __ddiv_rn(beta.y, beta.x);
      const double scl = __ddiv_rn(1.0, __dadd_rn(beta.x, __dmul_rn(beta.y, rat)));
      st->step = make_double2(__dmul_rn(__dadd_rn(al.x, __dmul_rn(al.y, rat)), scl),
                              __dmul_rn(__dsub_rn(al.y, __dmul_rn(al.x, rat)), scl));
    } else {
      const double rat = __ddiv_rn(beta.x, beta.y);
      const double scl = __ddiv_rn(1.0, __dadd_rn(beta.y, __dmul_rn(beta.x, rat)));
      st->step = make_double2(__dmul_rn(__dadd_rn(__dmul_rn(al.x, rat), al.y), scl),
                              __dmul_rn(__dsub_rn(__dmul_rn(al.y, rat), al.x), scl));
    }
  }
}

// rho += step p; r -= step q; alpha_new = vdot(r, r); log; finiteness; early stop
__global__ void cg_update_kernel(const double2* __restrict__ p, const double2* __restrict__ q,
                                 double2* __restrict__ r, double2* __restrict__ rho, int64_t n,
                                 CGState* st, double* partials, double* res_log,
                                 double* sol_log) {
  if (st->stop) return;
  const double2 s = st->step;
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 pv = p[i], qv = q[i];
    double2 x = rho[i], y = r[i];
    x.x += s.x * pv.x - s.y * pv.y;
    x.y += s.x * pv.y + s.y * pv.x;
    y.x -= s.x * qv.x - s.y * qv.y;
    y.y -= s.x * qv.y + s.y * qv.x;
    rho[i] = x; r[i] = y;
    v[0] = fma(y.x, y.x, fma(y.y, y.y, v[0]));
    v[1] = fma(x.x, x.x, fma(x.y, x.y, v[1]));
    if (!finite2(x)) v[2] += 1.0;
  }
  double tot[3];
  if (grid_sum<3>(v, partials, &st->ticket, tot) && threadIdx.x == 0) {
    const double alpha_old = st->alpha.x;
    st->alpha = make_double2(tot[0], 0.0);
    st->ratio = tot[0] / alpha_old;     // (alpha / beta) with beta := old alpha, both real
    const int it = st->iter + 1;
    st->iter = it;
    if (tot[2] != 0.0 || !isfinite(tot[1])) {
      st->err = 7;   // NFS_ERR_NONFINITE_ITERATE
      st->err_iter = it;
      st->stop = 1;
      return;
    }
    res_log[it - 1] = sqrt(tot[0]);
    sol_log[it - 1] = sqrt(tot[1]);
    // next iteration's top-of-loop check (nfs/engine.py:158)
    if (sqrt(tot[0]) <= 1e-15 * st->r0) st->stop = 2;
  }
}

// p = r + ratio p
__global__ void cg_dir_kernel(const double2* __restrict__ r, double2* __restrict__ p, int64_t n,
                              const CGState* st) {
  if (st->stop) return;
  const double a = st->ratio;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 rv = r[i], pv = p[i];
    p[i] = make_double2(rv.x + a * pv.x, rv.y + a * pv.y);
  }
}

// per-iteration relative RMSE of the image rho o j against a reference, on the device (SURVEY 8f
// f4; the reference's metrics.rmse, nfs/metrics.py:73-88, evaluated in a convergence study's
// callback): err^2 = (sum_l w_l^2-weighted |rho_l w_l - ref_l|^2 + outside) / ref_sq, where
// w_l = j_l on the RMSE support and 0 off it (then ref_l = 0 too), and `outside` is the
// support's energy outside the reconstruction mask (the image is zero there).
__global__ void cg_rmse_kernel(const double2* __restrict__ rho, const double2* __restrict__ ref,
                               const double* __restrict__ w, int64_t n, CGState* st, double* partials,
                               double outside, double ref_sq, double* log) {
  if (st->err || st->iter < 1) return;
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = rho[i], r = ref[i];
    const double dx = x.x * w[i] - r.x, dy = x.y * w[i] - r.y;
    v[0] = fma(dx, dx, fma(dy, dy, v[0]));
  }
  double tot[1];
  if (grid_sum<1>(v, partials, &st->ticket, tot) && threadIdx.x == 0)
    log[st->iter - 1] = sqrt((tot[0] + outside) / ref_sq);
}

cudaError_t launch_cg_rmse(const double2* rho, const double2* ref, const double* w, int64_t n, CGState* s,
                           double* partials, double outside, double ref_sq, double* log, cudaStream_t st);

// per-iteration mean SSIM of |rho o j| scattered to the 2D grid against a reference image (SURVEY
// 8f f4; the reference's metrics.ssim, nfs/metrics.py:20-70: Gaussian-weighted local statistics
// over all windows that fit, dynamic range from the reference, optional window selection).
__global__ void ssim_scatter_kernel(const double2* __restrict__ rho, const double* __restrict__ w,
                                    const int64_t* __restrict__ vox, int64_t n, const CGState* st,
                                    double* __restrict__ img) {
  if (st->err || st->iter < 1) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = rho[i];
    img[vox[i]] = hypot(x.x * w[i], x.y * w[i]);   // |rho_l j_l|
  }
}

__global__ void ssim_eval_kernel(const double* __restrict__ img, const double* __restrict__ ref, int nx, int ny,
                                 const double* __restrict__ kern, int win, double c1, double c2,
                                 const unsigned char* __restrict__ sel, double n_sel, CGState* st,
                                 double* partials, double* log) {
  if (st->err || st->iter < 1) return;
  const int ox_n = nx - win + 1, oy_n = ny - win + 1;
  const int64_t n = (int64_t)ox_n * oy_n;
  double v[1] = {0.0};
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    const int ox = (int)(o % ox_n), oy = (int)(o / ox_n);
    if (sel && !sel[o]) continue;
    double m1 = 0, m2 = 0, e11 = 0, e22 = 0, e12 = 0;
    for (int b = 0; b < win; ++b)
      for (int a = 0; a < win; ++a) {
        const double k = kern[a * win + b];
        const int64_t idx = (int64_t)(ox + a) + (int64_t)nx * (oy + b);
        const double t = img[idx], r = ref[idx];
        m1 = fma(k, t, m1);
        m2 = fma(k, r, m2);
        e11 = fma(k, t * t, e11);
        e22 = fma(k, r * r, e22);
        e12 = fma(k, t * r, e12);
      }
    const double v1 = e11 - m1 * m1, v2 = e22 - m2 * m2, cov = e12 - m1 * m2;
    v[0] += ((2 * m1 * m2 + c1) * (2 * cov + c2)) / ((m1 * m1 + m2 * m2 + c1) * (v1 + v2 + c2));
  }
  double tot[1];
  if (grid_sum<1>(v, partials, &st->ticket, tot) && threadIdx.x == 0) log[st->iter - 1] = tot[0] / n_sel;
}

cudaError_t launch_cg_ssim(const double2* rho, const double* w, const int64_t* vox, int64_t n, double* img,
                           const double* ref, int nx, int ny, const double* kern, int win, double c1, double c2,
                           const unsigned char* sel, double n_sel, CGState* s, double* partials, double* log,
                           cudaStream_t st);

// ------------------------------------------------------------------ phase materialisation
template <typename T, int NT>
__global__ void phase_rows_kernel(const T* __restrict__ ttab, const T* __restrict__ rtab,
                                  int64_t row_lo, int64_t rows, int64_t n_vox,
                                  double2* __restrict__ out) {
  const int64_t n = rows * n_vox;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = row_lo + i / n_vox, l = i % n_vox;
    T a[NT];
#pragma unroll
    for (int p = 0; p < NT; ++p) a[p] = ttab[k * NT + p];
    const T t = phase_turns_generic<T, NT>(a, rtab + l * NT);
    T s, c;
    turns_sincos_generic(t, s, c);
    out[i] = make_double2((double)c, (double)s);
  }
}

// ------------------------------------------------------------------ host wrappers
static inline int grid_for(int64_t n, int cap) {
  int64_t b = (n + 255) / 256;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_pack(int prec, const double2* src, void* dst, int64_t rows, int g, int ldc,
                        cudaStream_t st) {
  const int gb = grid_for(rows * ldc, 148 * 8);
  if (prec == 1) pack_samples_kernel<double2><<<gb, 256, 0, st>>>(src, (double2*)dst, rows, g, ldc);
  else pack_samples_kernel<float2><<<gb, 256, 0, st>>>(src, (float2*)dst, rows, g, ldc);
  return cudaGetLastError();
}

cudaError_t launch_unpack(int prec, const void* src, double2* dst, int64_t rows, int g, int ldc,
                          cudaStream_t st) {
  const int gb = grid_for(rows * g, 148 * 8);
  if (prec == 1) unpack_samples_kernel<double2><<<gb, 256, 0, st>>>((const double2*)src, dst, rows, g, ldc);
  else unpack_samples_kernel<float2><<<gb, 256, 0, st>>>((const float2*)src, dst, rows, g, ldc);
  return cudaGetLastError();
}

cudaError_t launch_reduce_parts(int prec, const void* part, void* out, int64_t n, int n_part,
                                const int* stop, cudaStream_t st) {
  const int gb = grid_for(n, 148 * 8);
  if (prec == 1) reduce_parts_kernel<double2><<<gb, 256, 0, st>>>((const double2*)part, (double2*)out, n, n_part, stop);
  else reduce_parts_kernel<float2><<<gb, 256, 0, st>>>((const float2*)part, (float2*)out, n, n_part, stop);
  return cudaGetLastError();
}

cudaError_t launch_reduce_image(int prec, const void* part, double2* q, int64_t n, int n_part,
                                const int* stop, cudaStream_t st) {
  const int gb = grid_for(n, 148 * 8);
  if (prec == 1) reduce_image_kernel<double2><<<gb, 256, 0, st>>>((const double2*)part, q, n, n_part, stop);
  else reduce_image_kernel<float2><<<gb, 256, 0, st>>>((const float2*)part, q, n, n_part, stop);
  return cudaGetLastError();
}

int cg_grid(int64_t n) { return grid_for(n, 2 * 148); }

cudaError_t launch_cg_init(const double2* q0, double2* r, double2* p, double2* rho, int64_t n,
                           CGState* s, double* partials, cudaStream_t st) {
  cg_init_kernel<<<cg_grid(n), 256, 0, st>>>(q0, r, p, rho, n, s, partials);
  return cudaGetLastError();
}

cudaError_t launch_cg_iter_tail(const double2* q, double2* p, double2* r, double2* rho, int64_t n,
                                CGState* s, double* partials, double* res_log, double* sol_log,
                                cudaStream_t st) {
  const int gb = cg_grid(n);
  cg_dot_kernel<<<gb, 256, 0, st>>>(p, q, n, s, partials);
  cg_update_kernel<<<gb, 256, 0, st>>>(p, q, r, rho, n, s, partials, res_log, sol_log);
  cg_dir_kernel<<<gb, 256, 0, st>>>(r, p, n, s);
  return cudaGetLastError();
}

cudaError_t launch_cg_rmse(const double2* rho, const double2* ref, const double* w, int64_t n, CGState* s,
                           double* partials, double outside, double ref_sq, double* log, cudaStream_t st) {
  cg_rmse_kernel<<<cg_grid(n), 256, 0, st>>>(rho, ref, w, n, s, partials, outside, ref_sq, log);
  return cudaGetLastError();
}

cudaError_t launch_cg_ssim(const double2* rho, const double* w, const int64_t* vox, int64_t n, double* img,
                           const double* ref, int nx, int ny, const double* kern, int win, double c1, double c2,
                           const unsigned char* sel, double n_sel, CGState* s, double* partials, double* log,
                           cudaStream_t st) {
  cudaMemsetAsync(img, 0, (size_t)nx * ny * sizeof(double), st);
  ssim_scatter_kernel<<<cg_grid(n), 256, 0, st>>>(rho, w, vox, n, s, img);
  const int64_t nw = (int64_t)(nx - win + 1) * (ny - win + 1);
  ssim_eval_kernel<<<cg_grid(nw), 256, 0, st>>>(img, ref, nx, ny, kern, win, c1, c2, sel, n_sel, s, partials, log);
  return cudaGetLastError();
}

cudaError_t launch_phase_rows(int prec, int nt, const void* ttab, const void* rtab,
                              int64_t row_lo, int64_t rows, int64_t n_vox, double2* out,
                              cudaStream_t st) {
  const int gb = grid_for(rows * n_vox, 148 * 8);
#define NFS_PR(T, N)                                                                       \
  phase_rows_kernel<T, N><<<gb, 256, 0, st>>>((const T*)ttab, (const T*)rtab, row_lo, rows, \
                                               n_vox, out)
#define NFS_PR_T(T)                        \
  switch (nt) {                            \
    case 4: NFS_PR(T, 4); break;           \
    case 8: NFS_PR(T, 8); break;           \
    case 16: NFS_PR(T, 16); break;         \
    case 20: NFS_PR(T, 20); break;         \
    case 32: NFS_PR(T, 32); break;         \
    default: return cudaErrorInvalidValue; \
  }
  if (prec == 1) { NFS_PR_T(double) } else { NFS_PR_T(float) }
#undef NFS_PR_T
#undef NFS_PR
  return cudaGetLastError();
}

}  // namespace nfs
