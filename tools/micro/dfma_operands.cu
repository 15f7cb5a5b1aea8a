// DFMA throughput with the operand patterns of the reaction time stage (how many distinct 64-bit
// register operands a DFMA reads decides whether the FP64 pipe can issue every 2 cycles).
//   A: x = fma(x, a, b), a / b uniform              (the roofline microbenchmark's pattern)
//   B: acc[k] = fma(c[j], x[k][j], acc[k])          (time interpolation: 3 register operands, c shared)
//   C: y[j][k] = fma(w[j], v[k], y[j][k])           (time projection)
//   D: B + C interleaved like one Gauss-point step
// nvcc -arch=sm_100a -O3 -o dfma_operands dfma_operands.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(256, 1) kern(double* out, int iters, double a, double b) {
  double x[12][4], acc[12], c[4], y[4][4], v[4];
  for (int k = 0; k < 12; ++k) {
    acc[k] = threadIdx.x * 1e-3 + k;
    for (int j = 0; j < 4; ++j) x[k][j] = 1.0 + 1e-9 * (threadIdx.x + 4 * k + j);
  }
  for (int j = 0; j < 4; ++j) {
    c[j] = 1e-3 * (j + 1) + 1e-12 * threadIdx.x;
    v[j] = 1e-3 * (j + 2) + 1e-12 * threadIdx.x;
    for (int k = 0; k < 4; ++k) y[j][k] = threadIdx.x + j + k;
  }
  for (int i = 0; i < iters; ++i) {
    if (KIND == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 12; ++k) acc[k] = fma(acc[k], a, b);
    } else if (KIND == 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 12; ++k) acc[k] = fma(c[j], x[k][j], acc[k]);
    } else if (KIND == 2) {
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) y[j][k] = fma(c[j], v[k], y[j][k]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = fma(c[j], x[k][j], acc[k]);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) y[j][k] = fma(c[j], acc[k], y[j][k]);
    }
  }
  double s = 0;
  for (int k = 0; k < 12; ++k) s += acc[k];
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 4; ++k) s += y[j][k] + x[j][k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
void run(const char* name, int tpb, int bps) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * bps, iters = 20000;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * tpb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<KIND><<<blocks, tpb>>>(out, 100, 1.0000001, 1e-9);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    kern<KIND><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double per_iter = 48;
  const double flops = 2.0 * per_iter * iters * (double)blocks * tpb;
  printf("%-28s %4d threads x %d blocks/SM: %7.2f TF/s\n", name, tpb, bps, flops / (best * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  for (int tpb : {256, 512}) {
    run<0>("A x=fma(x,a,b) uniform", tpb, 1);
    run<1>("B interp 3 reg operands", tpb, 1);
    run<2>("C proj 3 reg operands", tpb, 1);
    run<3>("D interp+proj", tpb, 1);
  }
  return 0;
}
