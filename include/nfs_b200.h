/*
 * nfs_b200.h -- C ABI of the B200-native non-Fourier SENSE hot path.
 *
 * The reference (arXiv 2604.09233, /root/reference/pkg/src/nfsense) is pure Python; it has
 * no FFI.  Its boundary for this path is the Python engine API (nfs/__init__.py:18-27,
 * pkg/README.md:86-99).  The entry points below are what a Python binding of that API
 * needs (plain pointers and sizes, no torch types); paper_2604_09233_b200/_native.py is
 * the ctypes binding and INTEGRATION.md shows the stub a reference maintainer would add.
 *
 * Array conventions (all host arrays are caller-owned, never aliased or mutated):
 *   complex arrays are interleaved (re, im) float64 pairs (numpy complex128);
 *   temporal  (K, P+1)   row-major: column 0 = sample time [s], then field terms
 *   spatial   (P+1, L_R) row-major: row 0 = B0 [rad/s], then basis terms
 *   sens      (L_R, G)   row-major complex, sigma (K, G) row-major complex (coil fastest)
 *   p, q, rho (L_R,)     complex
 * phase[k,l] = exp(+i * sum_p temporal[k,p] * spatial[p,l])          (nfs/engine.py:93-95)
 *
 * Status codes map onto the reference's exception classes:
 *   NFS_ERR_INVALID / NFS_ERR_NONFINITE / NFS_ERR_BREAKDOWN / NFS_ERR_NONFINITE_ITERATE
 *     -> EngineError        (nfs/engine.py:22, raised at :49-69, :139-140, :164-165, :173-174)
 *   NFS_ERR_ABORTED (the iteration callback returned non-zero) -> the callback's own exception
 *   NFS_ERR_BUDGET -> MemoryBudgetError (nfs/engine.py:26, :132-137)
 * nfs_last_error() returns the thread-local message of the last failing call.
 */
#ifndef NFS_B200_H
#define NFS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NFS_OK 0
#define NFS_ERR_INVALID 1
#define NFS_ERR_NONFINITE 2
#define NFS_ERR_BREAKDOWN 3
#define NFS_ERR_BUDGET 4
#define NFS_ERR_CUDA 5
#define NFS_ERR_NCCL 6
#define NFS_ERR_NONFINITE_ITERATE 7
#define NFS_ERR_ABORTED 8

/* operator arithmetic */
#define NFS_PREC_FP32 0   /* FP32 phase + MUFU sincos + FP32 FMA contraction (fast mode)  */
#define NFS_PREC_FP64 1   /* FP64 phase, FP64 sincospi, FP64 FMA (parity mode)            */
#define NFS_PREC_TF32X3 2 /* tcgen05 3xTF32 split contraction, FP32 phase (tensor mode)   */
#define NFS_PREC_F16X3 3  /* tcgen05 3xFP16 split contraction (scaled B), exact int8 tcgen05 phase */

typedef struct nfs_plan nfs_plan;

/* Called once per CG iteration when registered: n (1-based) and the restricted iterate
 * (host copy, complex128, L_R entries).  Mirrors `callback(n, rho)` of nfs/engine.py:177.
 * A non-zero return aborts the solve right there (the reference's CG stops at a callback that
 * raises): nfs_cg_solve returns NFS_ERR_ABORTED with *n_done = n. */
typedef int32_t (*nfs_iter_callback)(int32_t n, const double* rho, void* user);

/* Plan for one device.  n_samples = rows held by THIS rank (sample sharding).
 * Replaces the implicit state of recon_full/recon_split (nfs/engine.py:125,182). */
int nfs_plan_create(nfs_plan** plan, int64_t n_samples, int64_t n_voxels, int32_t n_coils,
                    int32_t n_terms, int32_t precision, int32_t device);
void nfs_plan_destroy(nfs_plan* plan);
/* Launch on a caller stream (cudaStream_t as void*); NULL = the plan's own stream. */
int nfs_plan_set_stream(nfs_plan* plan, void* stream);
/* Sample-sharded multi-GPU: join an NCCL communicator (128-byte ncclUniqueId). The adjoint
 * image is all-reduced (sum) once per CG iteration.  world == 1 needs no call (a 1-rank
 * communicator is accepted and exercises the same all-reduce path). */
int nfs_plan_attach_comm(nfs_plan* plan, const void* nccl_unique_id, int32_t rank, int32_t world);
/* A communicator shared by all plans of a process (created once per rank, borrowed by every
 * plan with nfs_plan_use_comm and destroyed by nfs_comm_destroy after the last plan), so
 * repeated reconstructions do not pay ncclCommInitRank each time. */
int nfs_comm_create(const void* nccl_unique_id, int32_t rank, int32_t world, int32_t device, void** comm);
void nfs_comm_destroy(void* comm);
int nfs_plan_use_comm(nfs_plan* plan, void* comm, int32_t rank, int32_t world);

/* Basis tables: temporal rows of this rank (K x P1) and spatial (P1 x L_R). */
int nfs_set_tables(nfs_plan* plan, const double* temporal, const double* spatial);
/* Same, with the spatial table voxel-major (L_R x P1): the memory of the Fortran-ordered
 * (P1, L_R) array that np.vstack([b0, harm.T]) in build_bases (nfs/engine.py:252-280)
 * returns, so the caller uploads it as is instead of transposing on the host. */
int nfs_set_tables_t(nfs_plan* plan, const double* temporal, const double* spatial_t);
/* Same, with the spatial table evaluated ON THE DEVICE from the masked voxels' linear grid
 * indices (ix + nx (iy + ny iz)), their B0 (rad/s), the grid extents dims[3], FOV fov[3] (m)
 * and the harmonic order 1..3 -- replaces engine.build_bases (nfs/engine.py:252-280) +
 * solid_harmonics (nfs/simulate.py:26-59) + grid_coordinates (nfs/core.py:102-113); the table
 * is bit-identical to the host build.  P1 must equal 1 + the order's harmonic count. */
int nfs_set_tables_grid(nfs_plan* plan, const double* temporal, const int64_t* vox_index,
                        const double* b0_masked, const int32_t* dims, const double* fov, int32_t order);
/* Sensitivities (L_R x G complex) and optional intensity correction j (L_R) -> S' = S o j
 * (nfs/engine.py:143).  intensity == NULL means j = 1 (apply_E / apply_EH semantics). */
int nfs_set_sens(nfs_plan* plan, const double* sens, const double* intensity);
/* Same from the FULL-grid maps sens_full [n_full][n_coils] (complex): the mask restriction
 * (vox_index[L_R] = grid index of each reconstructed voxel, nfs/pipeline.py:202) and, when
 * intensity is NULL, the intensity correction j = 1/sqrt(sum_c |S|^2) (nfs/sensmaps.py:145-152)
 * run on the device; j_out (L_R, optional) receives the j used. */
int nfs_set_sens_grid(nfs_plan* plan, const double* sens_full, int64_t n_full, const int64_t* vox_index,
                      const double* intensity, double* j_out);
/* Stateless device intensity correction of the n_r voxels vox_index of the full-grid maps. */
int nfs_intensity_correction(int32_t device, const double* sens_full, int64_t n_full, int32_t n_coils,
                             const int64_t* vox_index, int64_t n_r, double* j_out);
/* Raw samples of this rank (K x G complex); non-finite -> NFS_ERR_NONFINITE. */
int nfs_set_samples(nfs_plan* plan, const double* sigma);
/* Samples read straight from a dataset file: rows [row0, row0 + n_samples) of a
 * raw little-endian complex128 (K_total, n_coils) array -- the reference's `sigma.c128`
 * (nfs/core.py:292-328) -- through the pinned staging ring; a sharded rank reads only its rows.
 * Same finiteness check as nfs_set_samples; NFS_ERR_INVALID on a short read. */
int nfs_set_samples_file(nfs_plan* plan, const char* path, int64_t row0);

/* Per-iteration diagnostic on the device: relative RMSE of the image rho o j vs
 * a reference (nfs/metrics.py:73-88 as called from a convergence-study callback) is logged by
 * nfs_cg_solve without copying the iterate to the host.  ref_masked: reference on the
 * reconstruction mask (L_R complex, zero off the RMSE support); weight: j on the support, 0 off;
 * outside_sq: the support's |ref|^2 outside the mask; ref_sq: the support's |ref|^2.
 * ref_masked == NULL turns it off.  nfs_rmse_log copies the first n logged values. */
int nfs_set_rmse_reference(nfs_plan* plan, const double* ref_masked, const double* weight,
                           double outside_sq, double ref_sq);
int nfs_rmse_log(nfs_plan* plan, double* out, int32_t n);
/* Same for the mean SSIM (nfs/metrics.py:20-70) of |rho o j| scattered to an nx x ny image
 * (x fastest) against ref_img: vox_index = grid index of each reconstructed voxel, weight = j,
 * kern = the win x win Gaussian window, c1 / c2 from the reference's dynamic range, sel = optional
 * selection of the (nx-win+1) x (ny-win+1) valid windows.  ref_img == NULL turns it off. */
int nfs_set_ssim_reference(nfs_plan* plan, const int64_t* vox_index, const double* weight, int32_t nx,
                           int32_t ny, const double* ref_img, const double* kern, int32_t win, double c1,
                           double c2, const uint8_t* sel);
int nfs_ssim_log(nfs_plan* plan, double* out, int32_t n);

/* Operators with host buffers (copies inside).  nfs/engine.py:98-108. */
int nfs_apply_E(nfs_plan* plan, const double* p, double* y);
int nfs_apply_EH(nfs_plan* plan, const double* sigma, double* q);
int nfs_apply_EHE(nfs_plan* plan, const double* p, double* q);
/* phase rows [row_lo, row_hi) of this rank as complex128 (row_hi-row_lo) x L_R, computed on
 * the device with the operators' own phase generator.  nfs/engine.py:93-95. */
int nfs_phase_rows(nfs_plan* plan, int64_t row_lo, int64_t row_hi, double* out);

/* CG on E^H E rho = E^H sigma with the reference's update order and early stop
 * (nfs/engine.py:151-178).  Outputs (host): rho (L_R complex), res_norms/sol_norms
 * (n_iter entries, first *n_done valid), timings_s (2 + n_iter entries: initial_adjoint,
 * solve_total, cg_iteration_1..n).  cb may be NULL.  On breakdown / non-finite iterate the
 * call returns the matching code with *n_done = the failing iteration. */
int nfs_cg_solve(nfs_plan* plan, int32_t n_iter, nfs_iter_callback cb, void* user,
                 double* rho, double* res_norms, double* sol_norms, int32_t* n_done,
                 double* timings_s);

/* Benchmark hooks: n applies of E^H E on the device-resident p (no host copies), timed by
 * the caller on the plan stream; and per-kernel average durations (ms) measured with CUDA
 * events on the plan stream over `reps` applies: [fwd, fwd_reduce, adj, adj_reduce]. */
int nfs_apply_EHE_resident(nfs_plan* plan, int32_t n_applies);
int nfs_kernel_times(nfs_plan* plan, int32_t reps, float* ms_out);
/* Timed benchmark steps (bench.py): n applies of E^H E on the device-resident p, each after a
 * flush_bytes device write (L2 eviction, outside the timing); step_ms[n] = each apply's duration,
 * kern_ms[2] = summed durations of the forward / adjoint main contraction kernel over the same
 * steps (CUDA events around each launch on the plan stream). */
int nfs_bench_applies(nfs_plan* plan, int32_t n, int64_t flush_bytes, float* step_ms, float* kern_ms);
/* Number of kernel launches one E^H E apply issues (for the bench's launch count). */
int nfs_launches_per_apply(nfs_plan* plan);
/* Human-readable kernel configuration (tile sizes, splits), for logs. */
const char* nfs_plan_describe(nfs_plan* plan);

const char* nfs_last_error(void);
const char* nfs_version(void);

#ifdef __cplusplus
}
#endif

#endif /* NFS_B200_H */
