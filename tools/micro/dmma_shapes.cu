// Microbenchmark: FP64 mma.sync shape throughput on sm_100a.
// m8n8k4 (the sm_80 DMMA shape) vs the sm_90+ shapes m16n8k4 / m16n8k8 / m16n8k16.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_shapes dmma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void mma_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (threadIdx.x + k) * 1e-3;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 1.0 - (threadIdx.x + k) * 1e-4;
  double c[8][4];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if constexpr (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a[0]), "d"(b[0]));
      } else if constexpr (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if constexpr (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                     "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
void run(double* out, int sms, const char* name, double flop_per_mma) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int tpb : {128, 256, 512}) {
    const int blocks = sms * (1024 / tpb);
    const int iters = SHAPE == 3 ? 500 : 2000;
    mma_kernel<SHAPE><<<blocks, tpb>>>(out, 10);
    cudaEventRecord(e0);
    mma_kernel<SHAPE><<<blocks, tpb>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * tpb / 32;
    const double flops = flop_per_mma * 8 * (double)iters * warps;
    printf("%-8s tpb=%4d warps/SM=%2d: %6.2f TFLOP/s (%.3f ms)\n", name, tpb, 1024 / 32, flops / ms / 1e9, ms);
  }
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  printf("device %s SMs %d\n", prop.name, prop.multiProcessorCount);
  double* out;
  cudaMalloc(&out, 1 << 26);
  const int sms = prop.multiProcessorCount;
  run<0>(out, sms, "m8n8k4", 2.0 * 8 * 8 * 4);
  run<1>(out, sms, "m16n8k4", 2.0 * 16 * 8 * 4);
  run<2>(out, sms, "m16n8k8", 2.0 * 16 * 8 * 8);
  run<3>(out, sms, "m16n8k16", 2.0 * 16 * 8 * 16);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
