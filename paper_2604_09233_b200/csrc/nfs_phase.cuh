// nfs_phase.cuh -- the single phase generator shared by every kernel of the path.
//
// phase[k,l] = exp(+i * phi[k,l]),  phi = sum_p T[k,p] R[l,p]  (nfs/engine.py:93-95,
// exp(1j * temporal @ spatial)).  FP32 / tensor paths: T' = temporal / 2pi, so the sum is in
// turns and its fraction feeds MUFU sin/cos.  FP64 parity path: T = temporal (radians), the sum
// in the SAME order as OpenBLAS's dgemm for these shapes (p = 0 product, then fma for
// p = 1..P; bit-identical to numpy's `temporal @ spatial` for >= 99.8% of the entries of
// configs A/B) and sin/cos of phi itself, so the parity path perturbs the reference's phasors
// by ulps, not by the 1e-14-rad rounding of a turns conversion.  Forward, adjoint and phase
// materialisation all call these two functions, so E and E^H use bit-identical phasors.
#pragma once
#include <cuda_runtime.h>

namespace nfs {

template <typename T, int NT>
__device__ __forceinline__ T phase_turns_generic(const T (&a)[NT], const T* __restrict__ b) {
  // fixed order p = 0..NT-1; fma(a,b,c) == fma(b,a,c), so owner/streamed roles commute.
  T t;
  if constexpr (sizeof(T) == 4) t = __fmul_rn(a[0], b[0]); else t = __dmul_rn(a[0], b[0]);
#pragma unroll
  for (int p = 1; p < NT; ++p) t = fma(a[p], b[p], t);
  return t;
}

__device__ __forceinline__ void turns_sincos_generic(float t, float& s, float& c) {
  const float f = t - rintf(t);                    // exact, |f| <= 1/2 turn
  __sincosf(f * 6.28318530717958647692f, &s, &c);  // MUFU.SIN / MUFU.COS (fast mode)
}
__device__ __forceinline__ void turns_sincos_generic(double phi, double& s, double& c) {
  sincos(phi, &s, &c);                             // FP64 parity mode: phi in radians
}

}  // namespace nfs
