// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) batched GEMM used for the
// dense eigenvector mode products of the fast-diagonalisation
// preconditioner (reference: mode_apply inside FastDiagPreconditioner.apply,
// linalg.py:329-346 / tensorops.py:13-26).
//
// C[b] = A[b] * B[b]  (row-major, arbitrary leading dimensions and batch
// strides; a zero stride broadcasts one matrix over the batch).
// Tile 64x64x32, 8 warps (each 2x4 DMMA tiles), cp.async double buffering.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "ptx.cuh"

namespace mi {

struct GemmArgs {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  long long lda, ldb, ldc;
  long long sA, sB, sC;  // batch strides (elements)
};

constexpr int GT_M = 64, GT_N = 64, GT_K = 32;
constexpr int GA_LD = GT_K + 4;   // 36: conflict-free A fragment reads
constexpr int GB_LD = GT_N + 4;   // 68: conflict-free B fragment reads
constexpr int GEMM_SMEM = 2 * (GT_M * GA_LD + GT_K * GB_LD) * 8;

static __global__ void __launch_bounds__(256) dgemm_dmma(GemmArgs g) {
  extern __shared__ double smem[];
  double* As = smem;                              // [2][64][36]
  double* Bs = smem + 2 * GT_M * GA_LD;           // [2][32][68]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.y * GT_M, n0 = blockIdx.x * GT_N;
  const long long b = blockIdx.z;
  const double* A = g.A + b * g.sA;
  const double* B = g.B + b * g.sB;
  double* C = g.C + b * g.sC;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;
  const int gq = lane >> 2, t4 = lane & 3;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load = [&](int stage, int k0) {
    double* as = As + stage * GT_M * GA_LD;
    double* bs = Bs + stage * GT_K * GB_LD;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + 256 * e;
      int r = idx >> 5, k = idx & 31;
      bool v = (m0 + r < g.M) && (k0 + k < g.K);
      const double* src = v ? A + (long long)(m0 + r) * g.lda + k0 + k : A;
      cp_async8(as + r * GA_LD + k, src, v);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + 256 * e;
      int k = idx >> 6, n = idx & 63;
      bool v = (k0 + k < g.K) && (n0 + n < g.N);
      const double* src = v ? B + (long long)(k0 + k) * g.ldb + n0 + n : B;
      cp_async8(bs + k * GB_LD + n, src, v);
    }
    cp_async_commit();
  };

  const int nk = (g.K + GT_K - 1) / GT_K;
  load(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      load((kc + 1) & 1, (kc + 1) * GT_K);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + (kc & 1) * GT_M * GA_LD;
    const double* bs = Bs + (kc & 1) * GT_K * GB_LD;
#pragma unroll
    for (int ks = 0; ks < GT_K / 4; ++ks) {
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = as[(wm + 8 * i + gq) * GA_LD + ks * 4 + t4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(ks * 4 + t4) * GB_LD + wn + 8 * j + gq];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    int r = m0 + wm + 8 * i + gq;
    if (r >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int cidx = n0 + wn + 8 * j + 2 * t4;
      double* dst = C + (long long)r * g.ldc + cidx;
      if (cidx < g.N) dst[0] = acc[i][j][0];
      if (cidx + 1 < g.N) dst[1] = acc[i][j][1];
    }
  }
}

// Launch helper: returns cudaError_t of the launch.
static inline cudaError_t launch_dgemm(const GemmArgs& g, int batch, cudaStream_t st) {
  MI_DEV_FLAG(attr);
  if (!attr) {
    cudaFuncSetAttribute(dgemm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
    attr = true;
  }
  dim3 grid((g.N + GT_N - 1) / GT_N, (g.M + GT_M - 1) / GT_M, batch);
  dgemm_dmma<<<grid, 256, GEMM_SMEM, st>>>(g);
  return cudaGetLastError();
}

}  // namespace mi

namespace mi {

// Panel DMMA GEMM for the small-n mode products: one block covers ALL n rows
// (ALONG_N: C = A(n x n) B(n x cols), warps along the columns) or ALL n
// columns (!ALONG_N: C = X(rows x n) U(n x n), warps along the rows), so the
// only padding is n -> 8*ceil(n/8).  K chunks of 20 (5 k-steps), cp.async
// double buffering; smem strides chosen for conflict-free fragment loads.
template <int TILES, bool ALONG_N>
__global__ void __launch_bounds__(256) dgemm_panel(GemmArgs g) {
  constexpr int KC = 20;
  constexpr int BM = ALONG_N ? 8 * TILES : 64;     // block rows
  constexpr int BN = ALONG_N ? 64 : 8 * TILES;     // block cols
  constexpr int ALD = KC + 8;                      // 28 doubles: rows shift by 24 banks
  constexpr int BLD = BN + ((BN % 16 == 0) ? 4 : (BN % 16 == 8 ? 12 : 4));
  extern __shared__ double smem[];
  double* As = smem;                               // [2][BM][ALD]
  double* Bs = smem + 2 * BM * ALD;                // [2][KC][BLD]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const long long bz = blockIdx.z;
  const double* A = g.A + bz * g.sA;
  const double* B = g.B + bz * g.sB;
  double* C = g.C + bz * g.sC;
  const int gq = lane >> 2, t4 = lane & 3;
  // warp sub-tile: ALONG_N -> all TILES m-tiles x 1 n-tile (column 8*warp);
  //               !ALONG_N -> 1 m-tile (row 8*warp) x all TILES n-tiles
  double acc[TILES][2];
#pragma unroll
  for (int i = 0; i < TILES; ++i) acc[i][0] = acc[i][1] = 0.0;
  auto load = [&](int stage, int k0) {
    double* as = As + stage * BM * ALD;
    double* bs = Bs + stage * KC * BLD;
    for (int e = tid; e < BM * KC; e += 256) {
      const int r = e / KC, k = e % KC;
      const bool v = (m0 + r < g.M) && (k0 + k < g.K);
      cp_async8(as + r * ALD + k, v ? A + (long long)(m0 + r) * g.lda + k0 + k : A, v);
    }
    for (int e = tid; e < KC * BN; e += 256) {
      const int k = e / BN, n = e % BN;
      const bool v = (k0 + k < g.K) && (n0 + n < g.N);
      cp_async8(bs + k * BLD + n, v ? B + (long long)(k0 + k) * g.ldb + n0 + n : B, v);
    }
    cp_async_commit();
  };
  const int nk = (g.K + KC - 1) / KC;
  load(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      load((kc + 1) & 1, (kc + 1) * KC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + (kc & 1) * BM * ALD;
    const double* bs = Bs + (kc & 1) * KC * BLD;
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      if (ALONG_N) {
        const double bf = bs[(ks * 4 + t4) * BLD + 8 * warp + gq];
#pragma unroll
        for (int i = 0; i < TILES; ++i) dmma(acc[i][0], acc[i][1], as[(8 * i + gq) * ALD + ks * 4 + t4], bf);
      } else {
        const double af = as[(8 * warp + gq) * ALD + ks * 4 + t4];
#pragma unroll
        for (int j = 0; j < TILES; ++j) dmma(acc[j][0], acc[j][1], af, bs[(ks * 4 + t4) * BLD + 8 * j + gq]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TILES; ++i) {
    const int r = ALONG_N ? m0 + 8 * i + gq : m0 + 8 * warp + gq;
    const int cidx = ALONG_N ? n0 + 8 * warp + 2 * t4 : n0 + 8 * i + 2 * t4;
    if (r >= g.M) continue;
    double* dst = C + (long long)r * g.ldc + cidx;
    if (cidx < g.N) dst[0] = acc[i][0];
    if (cidx + 1 < g.N) dst[1] = acc[i][1];
  }
}

template <int TILES, bool ALONG_N>
inline cudaError_t launch_panel(const GemmArgs& g, int batch, cudaStream_t st) {
  constexpr int KC = 20;
  constexpr int BM = ALONG_N ? 8 * TILES : 64;
  constexpr int BN = ALONG_N ? 64 : 8 * TILES;
  constexpr int BLD = BN + ((BN % 16 == 0) ? 4 : (BN % 16 == 8 ? 12 : 4));
  constexpr int SM = 2 * (BM * (KC + 8) + KC * BLD) * 8;
  MI_DEV_FLAG(attr);
  if (!attr) {
    cudaFuncSetAttribute(dgemm_panel<TILES, ALONG_N>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    attr = true;
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, batch);
  dgemm_panel<TILES, ALONG_N><<<grid, 256, SM, st>>>(g);
  return cudaGetLastError();
}

// Dispatch on the small dimension n (rows for ALONG_N, cols otherwise).
template <bool ALONG_N>
inline cudaError_t launch_panel_n(const GemmArgs& g, int n, int batch, cudaStream_t st) {
  const int t = (n + 7) / 8;
  if (t <= 1) return launch_panel<1, ALONG_N>(g, batch, st);
  if (t <= 2) return launch_panel<2, ALONG_N>(g, batch, st);
  if (t <= 4) return launch_panel<4, ALONG_N>(g, batch, st);
  if (t <= 8) return launch_panel<8, ALONG_N>(g, batch, st);
  if (t <= 9) return launch_panel<9, ALONG_N>(g, batch, st);
  if (t <= 13) return launch_panel<13, ALONG_N>(g, batch, st);
  if (t <= 17) return launch_panel<17, ALONG_N>(g, batch, st);
  if (t <= 26) return launch_panel<13, ALONG_N>(g, batch, st);   // two row (column) blocks of 104
  return launch_dgemm(g, batch, st);
}

}  // namespace mi
