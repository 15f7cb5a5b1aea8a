// Measurement diagnostics (not part of the reference interface): the FP64 roofline denominators.
// bench.py reports max(cuBLAS DGEMM 8192^3, the DMMA peak below) as the FP64 tensor peak, and the
// mixed kernel tells whether DMMA and DFMA issue to one FP64 pipe (their times add) or to two.
#include "common.cuh"
#include "ptx.cuh"

namespace mi {

__global__ void diag_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// MIX = 0: DMMA only; 1: DMMA + the same issue count of DFMA per warp as diag_dfma does per thread / 8
template <int MIX>
__global__ void diag_dmma(double* out, int iters, double fa, double fb) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2], x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0, x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dmma(c[k][0], c[k][1], a, b);
      if (MIX) {
#pragma unroll
        for (int r = 0; r < 2; ++r) x[k] = fma(x[k], fa, fb);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + (MIX ? x[k] : 0.0);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace mi

extern "C" {

int mi_diag_fp64_peak(int device, int kind, double* tflops, double* ms_out) {
  MI_REQUIRE(tflops != nullptr, MI_ERR_ARG, "tflops is NULL");
  MI_REQUIRE(kind >= 0 && kind <= 2, MI_ERR_ARG, "kind: 0 DMMA, 1 DFMA, 2 DMMA+DFMA mixed");
  mi::DeviceGuard guard(device);
  const int sms = mi::num_sms();
  const int tpb = 256, blocks = sms * 8, iters = 4000;
  double* out = nullptr;
  MI_CUDA(cudaMalloc(&out, sizeof(double) * blocks * tpb));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](int it) {
    if (kind == 0) mi::diag_dmma<0><<<blocks, tpb>>>(out, it, 1.0000001, 1e-9);
    if (kind == 1) mi::diag_dfma<<<blocks, tpb>>>(out, it, 1.0000001, 1e-9);
    if (kind == 2) mi::diag_dmma<1><<<blocks, tpb>>>(out, it, 1.0000001, 1e-9);
  };
  run(20);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    run(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return mi::fail("mi_diag_fp64_peak", err);
  const double warps = (double)blocks * tpb / 32, thr = (double)blocks * tpb;
  double flops = 0;
  if (kind == 0) flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * warps;
  if (kind == 1) flops = 2.0 * 128 * (double)iters * thr;
  if (kind == 2) flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * warps + 2.0 * 16 * (double)iters * thr;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms_out) *ms_out = best;
  return MI_OK;
}

}  // extern "C"
