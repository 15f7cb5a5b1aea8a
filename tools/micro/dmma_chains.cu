// DMMA throughput vs independent accumulator chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[C][2];
#pragma unroll
  for (int j = 0; j < C; ++j) c[j][0] = c[j][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < C; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < C; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C>
void run(double* out, int warps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  k<C><<<148, 32 * warps>>>(out, 10);
  cudaEventRecord(e0);
  k<C><<<148, 32 * warps>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * C * (double)iters * warps * 148;
  printf("chains=%d warps/SM=%2d: %6.2f TFLOP/s  (cycles per dmma per warp-chain ~ %.1f)\n", C, warps, flops / ms / 1e9,
         ms * 1e-3 * 1.965e9 / iters);
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  for (int w : {4, 8, 16, 32}) { run<1>(out, w); run<2>(out, w); run<3>(out, w); run<4>(out, w); run<8>(out, w); }
  return 0;
}
