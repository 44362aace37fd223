// Microbenchmark: FP32 FFMA vs packed FFMA2 issue/throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float x = a, y = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fmaf(x, acc[i], y);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_ffma2(float* out, int iters, float a, float b) {
  float2 acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  float2 x = make_float2(a, a), y = make_float2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = __ffma2_rn(x, acc[i], y);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// complex MAC pattern: x from smem broadcast, 2 owners, 32 coils, scalar FFMA
template <bool PACKED>
__global__ void k_cmac(float* out, int iters) {
  __shared__ float2 sx[64 * 32];
  __shared__ float2 sxs[64 * 32];
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) {
    sx[i] = make_float2(i * 1e-3f, -i * 1e-3f);
    sxs[i] = make_float2(i * 1e-3f, i * 2e-3f);
  }
  __syncthreads();
  float2 acc[2][32];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[r][c] = make_float2(0.f, 0.f);
  float cs0 = threadIdx.x * 1e-4f, sn0 = 1.f - cs0, cs1 = cs0 * 0.5f, sn1 = sn0 * 0.25f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int si = 0; si < 64; ++si) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float2 x = sx[si * 32 + c];
        if (PACKED) {
          const float2 xs = sxs[si * 32 + c];
          acc[0][c] = __ffma2_rn(make_float2(cs0, cs0), x, acc[0][c]);
          acc[0][c] = __ffma2_rn(make_float2(sn0, sn0), xs, acc[0][c]);
          acc[1][c] = __ffma2_rn(make_float2(cs1, cs1), x, acc[1][c]);
          acc[1][c] = __ffma2_rn(make_float2(sn1, sn1), xs, acc[1][c]);
        } else {
          acc[0][c].x = fmaf(cs0, x.x, acc[0][c].x); acc[0][c].x = fmaf(-sn0, x.y, acc[0][c].x);
          acc[0][c].y = fmaf(cs0, x.y, acc[0][c].y); acc[0][c].y = fmaf(sn0, x.x, acc[0][c].y);
          acc[1][c].x = fmaf(cs1, x.x, acc[1][c].x); acc[1][c].x = fmaf(-sn1, x.y, acc[1][c].x);
          acc[1][c].y = fmaf(cs1, x.y, acc[1][c].y); acc[1][c].y = fmaf(sn1, x.x, acc[1][c].y);
        }
      }
      cs0 += 1e-7f; sn0 -= 1e-7f; cs1 += 2e-7f; sn1 -= 3e-7f;
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 32; ++c) s += acc[r][c].x + acc[r][c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// owner-pair packing: acc_re[c] = (owner0.re, owner1.re), coefficients as pairs, x as scalars
template <int NC>
__global__ void k_cmac_pair(float* out, int iters) {
  __shared__ float4 sx[64 * NC / 2];
  for (int i = threadIdx.x; i < 64 * NC / 2; i += blockDim.x)
    sx[i] = make_float4(i * 1e-3f, -i * 1e-3f, i * 2e-3f, i * 3e-3f);
  __syncthreads();
  float2 are[NC], aim[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) { are[c] = make_float2(0.f, 0.f); aim[c] = make_float2(0.f, 0.f); }
  float2 cs = make_float2(threadIdx.x * 1e-4f, threadIdx.x * 2e-4f);
  float2 sn = make_float2(1.f - cs.x, 1.f - cs.y);
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int si = 0; si < 64; ++si) {
      const float2 nsn = make_float2(-sn.x, -sn.y);
#pragma unroll
      for (int c2 = 0; c2 < NC / 2; ++c2) {
        const float4 x = sx[si * (NC / 2) + c2];
        are[2 * c2] = __ffma2_rn(cs, make_float2(x.x, x.x), are[2 * c2]);
        are[2 * c2] = __ffma2_rn(nsn, make_float2(x.y, x.y), are[2 * c2]);
        aim[2 * c2] = __ffma2_rn(cs, make_float2(x.y, x.y), aim[2 * c2]);
        aim[2 * c2] = __ffma2_rn(sn, make_float2(x.x, x.x), aim[2 * c2]);
        are[2 * c2 + 1] = __ffma2_rn(cs, make_float2(x.z, x.z), are[2 * c2 + 1]);
        are[2 * c2 + 1] = __ffma2_rn(nsn, make_float2(x.w, x.w), are[2 * c2 + 1]);
        aim[2 * c2 + 1] = __ffma2_rn(cs, make_float2(x.w, x.w), aim[2 * c2 + 1]);
        aim[2 * c2 + 1] = __ffma2_rn(sn, make_float2(x.z, x.z), aim[2 * c2 + 1]);
      }
      cs.x += 1e-7f; cs.y += 2e-7f; sn.x -= 1e-7f; sn.y -= 3e-7f;
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += are[c].x + are[c].y + aim[c].x + aim[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double run(F launch, double flops, const char* name) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double tf = flops / (ms * 1e-3) / 1e12;
  printf("%-28s %8.3f ms  %7.2f TFLOP/s  err=%s\n", name, ms, tf, cudaGetErrorString(cudaGetLastError()));
  return tf;
}

int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int bpsm : {2, 4, 8}) {
    dim3 g(sms * bpsm), t(256);
    double th = (double)g.x * t.x;
    char nm[64];
    snprintf(nm, 64, "ffma  acc16 blk/sm=%d", bpsm);
    run([&] { k_ffma<16><<<g, t>>>(out, iters, 1.0001f, 0.5f); }, th * iters * 16 * 2, nm);
    snprintf(nm, 64, "ffma2 acc16 blk/sm=%d", bpsm);
    run([&] { k_ffma2<16><<<g, t>>>(out, iters, 1.0001f, 0.5f); }, th * iters * 16 * 4, nm);
  }
  for (int bpsm : {1, 2}) {
    dim3 g(sms * bpsm * 2), t(128);
    double th = (double)g.x * t.x;
    const int it2 = 200;
    char nm[64];
    snprintf(nm, 64, "cmac scalar 128thr x%d", bpsm * 2);
    run([&] { k_cmac<false><<<g, t>>>(out, it2); }, th * it2 * 64 * 32 * 2 * 8, nm);
    snprintf(nm, 64, "cmac packed 128thr x%d", bpsm * 2);
    run([&] { k_cmac<true><<<g, t>>>(out, it2); }, th * it2 * 64 * 32 * 2 * 8, nm);
  }
  for (int bpsm : {1, 2}) {
    dim3 g(sms * bpsm * 2), t(128);
    double th = (double)g.x * t.x;
    const int it2 = 200;
    char nm[64];
    snprintf(nm, 64, "cmac pair32 128thr x%d", bpsm * 2);
    run([&] { k_cmac_pair<32><<<g, t>>>(out, it2); }, th * it2 * 64 * 32 * 2 * 8, nm);
    snprintf(nm, 64, "cmac pair16 128thr x%d", bpsm * 2);
    run([&] { k_cmac_pair<16><<<g, t>>>(out, it2); }, th * it2 * 64 * 16 * 2 * 8, nm);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d clock(attr)=%d kHz nominal fp32=%.1f TF\n", sms, clk, sms * 128 * 2 * clk * 1e3 / 1e12);
  return 0;
}
