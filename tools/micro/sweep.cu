// Isolated DMMA sweep: 16 warps/SM, B fragments in registers (KH per warp),
// A fragments from smem with compile-time offsets (the stencil_dmma inner loop).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
constexpr int TSTR = 20;
__host__ __device__ constexpr int koff(int ks) { return ((ks / 2) / 7 * 8 + (ks / 2) % 7) * 8 + 4 * (ks % 2); }
template <int KH, int MT>
__global__ void __launch_bounds__(512, 1) sweep(double* out, const double* bsrc, int reps) {
  extern __shared__ double X[];
  for (int i = threadIdx.x; i < 512 * TSTR * 2; i += 512) X[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = warp & 1;
  double breg[KH];
#pragma unroll
  for (int j = 0; j < KH; ++j) breg[j] = bsrc[(j * 32 + lane) % 4096];
  const int kl = lane & 3, mrow = lane >> 2;
  const double* Xb = X + (kl + (warp >> 1)) * TSTR + mrow;
  double acc[MT][2] = {};
  for (int r = 0; r < reps; ++r) {
    const double* Xr = Xb + (r & 1) * 512 * TSTR / 2;
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      const double* xa = Xr + koff(half * KH + j) * TSTR;
#pragma unroll
      for (int m = 0; m < MT; ++m) dmma(acc[m][0], acc[m][1], xa[m * 8], breg[j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int m = 0; m < MT; ++m) s += acc[m][0] + acc[m][1];
  out[blockIdx.x * 512 + threadIdx.x] = s;
}
template <int KH, int MT>
void run(double* out, double* b) {
  cudaFuncSetAttribute(sweep<KH, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int reps = 200;
  sweep<KH, MT><<<148, 512, 512 * TSTR * 2 * 8>>>(out, b, 2);
  cudaEventRecord(e0);
  sweep<KH, MT><<<148 * 4, 512, 512 * TSTR * 2 * 8>>>(out, b, reps);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * KH * MT * (double)reps * 16 * 148 * 4;
  printf("KH=%d MT=%d: %.2f TFLOP/s\n", KH, MT, fl / ms / 1e9);
}
int main() {
  double *out, *b; cudaMalloc(&out, 1 << 24); cudaMalloc(&b, 1 << 20); cudaMemset(b, 0, 1 << 20);
  run<49, 2>(out, b); run<49, 3>(out, b); run<32, 2>(out, b); run<24, 2>(out, b); run<24, 4>(out, b); run<16, 4>(out, b);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
