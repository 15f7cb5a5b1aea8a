// Persistent mode products for the small (n <= 8*TN) spatial eigenvector
// factors of the fast-diagonalisation preconditioner (reference mode_apply,
// tensorops.py:13-26, inside FastDiagPreconditioner.apply, linalg.py:329-346).
//
// One 256-thread block per SM keeps the whole n x n factor resident in shared
// memory as DMMA fragments (laid out fragment-major at block start, so every
// fragment read is one conflict-free 8-byte load) and streams full-K panels of
// the data through double-buffered cp.async, so the factor is read once per
// block instead of once per tile and K chunk, and tile i+1's loads overlap
// tile i's tensor-core work.
//
//   COLS (strided modes): out[o][i][c] = sum_j A[i][j] in[o][j][c].  Columns
//        are flattened over o (column g = o * inner + c), 64 per tile, so short
//        rows (the y transform, inner = n_1) need no per-batch padding.
//   ROWS (contiguous mode): out[r][i] = sum_j in[r][j] A[j][i], 64 rows per tile.
#pragma once
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace mi {

template <int TN>
struct ModeRes {
  static constexpr int KS = 2 * TN;                 // k-steps: K padded to 8 * TN
  static constexpr int KP = 4 * KS;                 // padded K
  static constexpr int FR = TN * KS * 32;           // resident fragments (doubles)
  static constexpr int BLD = 68;                    // COLS panel row stride (conflict-free B reads)
  // ROWS panel row stride: >= KP and = 4 or 12 (mod 16) doubles -> conflict-free A reads
  static constexpr int ALD = (KP % 16 == 4 || KP % 16 == 12) ? KP : KP + ((4 - KP % 16) + 16) % 16;
  static constexpr size_t SMEM_COLS = (size_t)(FR + 2 * KP * BLD) * 8;
  static constexpr size_t SMEM_ROWS = (size_t)(FR + 2 * 64 * ALD) * 8;
};

template <int TN, bool ROWS>
__global__ void __launch_bounds__(256, 1) mode_resident(const double* __restrict__ A, const double* __restrict__ in,
                                                         double* __restrict__ out, int n, long long inner,
                                                         long long outer) {
  using G = ModeRes<TN>;
  constexpr int KS = G::KS, KP = G::KP;
  extern __shared__ double smem[];
  double* frag = smem;                               // [TN][KS][32]
  double* pan = smem + G::FR;                        // [2][panel]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  // resident fragments.  COLS: A operand, lane holds A[8 i + gq][4 ks + t4].
  //                       ROWS: B operand, lane holds A[4 ks + t4][8 j + gq].
  for (int e = tid; e < G::FR; e += 256) {
    const int l = e & 31, ks = (e >> 5) % KS, i = (e >> 5) / KS;
    const int q = l >> 2, t = l & 3;
    const int r = ROWS ? 4 * ks + t : 8 * i + q;
    const int c = ROWS ? 8 * i + q : 4 * ks + t;
    frag[e] = (r < n && c < n) ? __ldg(A + (long long)r * n + c) : 0.0;
  }
  const long long total = ROWS ? outer : outer * inner;   // rows (ROWS) or flattened columns (COLS)
  const long long ntiles = (total + 63) / 64;
  if constexpr (!ROWS) {
    // ---- COLS: panel [KP][BLD], thread loads column tid & 63, rows (tid >> 6) + 4 m
    const int lc = tid & 63, lk = tid >> 6;
    auto load = [&](long long tile, int buf) {
      const long long g = tile * 64 + lc;
      const bool okc = g < total;
      long long base = 0;
      if (okc) {
        const long long o = g / inner;
        base = o * n * inner + (g - o * inner);
      }
      double* dst = pan + buf * KP * G::BLD + lc;
#pragma unroll 4
      for (int m = 0; m < KS; ++m) {
        const int k = lk + 4 * m;
        const bool v = okc && k < n;
        cp_async8(dst + k * G::BLD, v ? in + base + (long long)k * inner : in, v);
      }
      cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) load(tile, 0);
    __syncthreads();                                  // fragments visible
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
      const int buf = it & 1;
      const long long next = tile + gridDim.x;
      if (next < ntiles) {
        load(next, buf ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* bs = pan + buf * KP * G::BLD;
      double acc[TN][2];
#pragma unroll
      for (int i = 0; i < TN; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll 2
      for (int ks = 0; ks < KS; ++ks) {
        const double bf = bs[(4 * ks + t4) * G::BLD + 8 * warp + gq];
#pragma unroll
        for (int i = 0; i < TN; ++i) dmma(acc[i][0], acc[i][1], frag[(i * KS + ks) * 32 + lane], bf);
      }
      // store: rows 8 i + gq, flattened columns tile*64 + 8 warp + 2 t4 + e
      long long ob[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long long g = tile * 64 + 8 * warp + 2 * t4 + e;
        ob[e] = -1;
        if (g < total) {
          const long long o = g / inner;
          ob[e] = o * n * inner + (g - o * inner);
        }
      }
#pragma unroll
      for (int i = 0; i < TN; ++i) {
        const int r = 8 * i + gq;
        if (r < n) {
          if (ob[0] >= 0) out[ob[0] + (long long)r * inner] = acc[i][0];
          if (ob[1] >= 0) out[ob[1] + (long long)r * inner] = acc[i][1];
        }
      }
      __syncthreads();                                // panel buf is refilled two tiles later
    }
  } else {
    // ---- ROWS: panel [64][ALD], rows r0..r0+63, K along the row (8-byte cp.async, rows of n doubles)
    auto load = [&](long long tile, int buf) {
      double* dst = pan + buf * 64 * G::ALD;
      for (int e = tid; e < 64 * KP; e += 256) {
        const int r = e / KP, k = e - r * KP;
        const long long row = tile * 64 + r;
        const bool v = row < total && k < n;
        cp_async8(dst + r * G::ALD + k, v ? in + row * n + k : in, v);
      }
      cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) load(tile, 0);
    __syncthreads();
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
      const int buf = it & 1;
      const long long next = tile + gridDim.x;
      if (next < ntiles) {
        load(next, buf ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* as = pan + buf * 64 * G::ALD;
      double acc[TN][2];
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 2
      for (int ks = 0; ks < KS; ++ks) {
        const double af = as[(8 * warp + gq) * G::ALD + 4 * ks + t4];
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma(acc[j][0], acc[j][1], af, frag[(j * KS + ks) * 32 + lane]);
      }
      const long long row = tile * 64 + 8 * warp + gq;
      if (row < total) {
        double* dst = out + row * n;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const int c = 8 * j + 2 * t4;
          if (c < n) dst[c] = acc[j][0];
          if (c + 1 < n) dst[c + 1] = acc[j][1];
        }
      }
      __syncthreads();
    }
  }
}

// Launch for n <= 8 * TN; returns false (nothing launched) when n is outside the resident range.
template <bool ROWS>
inline bool launch_mode_resident(const double* A, const double* in, double* out, int n, long long inner,
                                 long long outer, int nsm, cudaStream_t st, cudaError_t* err) {
#define MI_MR(TNV)                                                                                       \
  if (n <= 8 * TNV) {                                                                                    \
    constexpr size_t sm = ROWS ? ModeRes<TNV>::SMEM_ROWS : ModeRes<TNV>::SMEM_COLS;                      \
    MI_DEV_FLAG(attr);                                                                            \
    if (!attr) {                                                                                         \
      cudaFuncSetAttribute(mode_resident<TNV, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
      attr = true;                                                                                       \
    }                                                                                                    \
    const long long total = ROWS ? outer : outer * inner;                                                \
    const long long ntiles = (total + 63) / 64;                                                          \
    const int grid = (int)(ntiles < nsm ? ntiles : nsm);                                                 \
    mode_resident<TNV, ROWS><<<grid > 0 ? grid : 1, 256, sm, st>>>(A, in, out, n, inner, outer);         \
    *err = cudaGetLastError();                                                                           \
    return true;                                                                                         \
  }
  MI_MR(2) MI_MR(4) MI_MR(8) MI_MR(9) MI_MR(13)
#undef MI_MR
  return false;
}

}  // namespace mi
