// Microbenchmark: FP64 DMMA (m8n8k4) throughput vs warps per SM and independent
// accumulator chains per warp, one block per SM.  Answers how many warps x chains
// the FP64 tensor pipe needs on sm_100a, and whether a single warp's back-to-back
// DMMAs (the compiler pads them with NOPs) limit it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_issue dmma_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, bool SHARE_A>
__global__ void chains(double* out, int iters) {
  double a[CH], b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int k = 0; k < CH; ++k) a[k] = (threadIdx.x + k) * 1e-3;
  double c[CH][2];
#pragma unroll
  for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(SHARE_A ? a[0] : a[k]), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// A operand from shared memory (one conflict-free LDS.64 per DMMA, like the resident-factor mode
// products), K loop of KS steps over CH independent accumulators
template <int CH, int KS>
__global__ void lds_fed(double* out, int iters) {
  __shared__ double sA[KS * CH * 32];
  for (int i = threadIdx.x; i < KS * CH * 32; i += blockDim.x) sA[i] = i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const double b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll 2
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int k = 0; k < CH; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1])
                     : "d"(sA[(ks * CH + k) * 32 + lane]), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH, int KS>
void run_lds(double* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {8, 12, 16, 24}) {
    const int tpb = 32 * warps, iters = 2000 / (CH * KS / 8 > 0 ? CH * KS / 8 : 1);
    lds_fed<CH, KS><<<sms, tpb>>>(out, 10);
    cudaEventRecord(e0);
    lds_fed<CH, KS><<<sms, tpb>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 512.0 * CH * KS * (double)iters * warps * sms;
    printf("lds-fed chains=%2d ks=%2d warps/SM=%2d: %6.2f TFLOP/s\n", CH, KS, warps, flops / ms / 1e9);
  }
}

template <int CH, bool SHARE_A>
void run(double* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 12, 16, 24, 32}) {
    const int tpb = 32 * warps, iters = 20000 / CH;
    chains<CH, SHARE_A><<<sms, tpb>>>(out, 10);
    cudaEventRecord(e0);
    chains<CH, SHARE_A><<<sms, tpb>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 512.0 * CH * (double)iters * warps * sms;
    printf("chains=%2d shareA=%d warps/SM=%2d: %6.2f TFLOP/s\n", CH, (int)SHARE_A, warps, flops / ms / 1e9);
  }
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  double* out;
  cudaMalloc(&out, 1 << 26);
  const int sms = prop.multiProcessorCount;
  run_lds<1, 26>(out, sms);
  run_lds<2, 26>(out, sms);
  run_lds<4, 26>(out, sms);
  run_lds<8, 12>(out, sms);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
