// Even/odd (folded) mode products for CENTROSYMMETRIC spatial eigenbases of
// the fast-diagonalisation preconditioner (reference mode_apply,
// tensorops.py:13-26, inside FastDiagPreconditioner.apply, linalg.py:329-346).
//
// On a uniform open knot vector the univariate pencil (K_l, M_l) commutes
// with the index reversal J, so its eigenvectors split into hs = n - n/2
// symmetric (J v = v) and h = n/2 skew (J v = -v) ones
// (factors._centro_eigh builds them that way, exactly mirrored, symmetric
// modes first).  With c_m[k] = v_m[k] (k < hs):
//
//   forward  (U^T x)_m      = sum_{k<hs} c_m[k] f_s[k]   (m symmetric),
//                             sum_{k<h}  c_m[k] f_a[k]   (m skew),
//            f_s[k] = x[k] + x[n-1-k] (k < h), f_s[h] = x[h] (n odd), f_a[k] = x[k] - x[n-1-k];
//   inverse  g_s[k] = sum_{m sym} c_m[k] y_m,  g_a[k] = sum_{m skew} c_m[k] y_m,
//            x[k] = g_s[k] + g_a[k], x[n-1-k] = g_s[k] - g_a[k] (k < h), x[h] = g_s[h] (n odd).
//
// Two half-size dense products instead of one n x n: half the DMMAs.  The
// fold is applied to the operand fragments as they are read from shared
// memory (one add per fragment, reused by every tile of its block); the
// unfold happens in registers at the store (the lane holding g_s[k] also
// holds g_a[k]).  Structure otherwise as mode_resident.cuh: one 256-thread
// block per SM, both half factors resident in shared memory as DMMA
// fragments, full-K data panels double-buffered by cp.async.
#pragma once
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace mi {

template <int TH>
struct ModeFold {
  static constexpr int KS = 2 * TH;                 // k-steps per half block: K padded to 8 * TH >= hs
  static constexpr int KP = 16 * TH;                // panel depth: both halves (>= n)
  static constexpr int FH = TH * KS * 32;           // fragments of one half factor (doubles)
  static constexpr int BLD = 68;                    // COLS panel row stride (conflict-free B reads)
  static constexpr int ALD = (KP % 16 == 4 || KP % 16 == 12) ? KP : KP + ((4 - KP % 16) + 16) % 16;
  static constexpr size_t SMEM_COLS = (size_t)(2 * FH + 2 * KP * BLD) * 8;
  static constexpr size_t SMEM_ROWS = (size_t)(2 * FH + 2 * 64 * ALD) * 8;
  static_assert(SMEM_COLS <= 227 * 1024 && SMEM_ROWS <= 227 * 1024, "folded mode product exceeds shared memory");
};

// U: n x n row-major eigenvector matrix (columns = modes, symmetric first).  INV = false applies
// U^T (into mode space), INV = true applies U.  ROWS: the mode is the contiguous index
// (out[r][.] from in[r][.], `outer` rows); COLS: out[o][.][c] from in[o][.][c] (stride `inner`).
template <int TH, bool ROWS, bool INV>
__global__ void __launch_bounds__(256, 1) mode_fold(const double* __restrict__ U, const double* __restrict__ in,
                                                     double* __restrict__ out, int n, long long inner,
                                                     long long outer) {
  using G = ModeFold<TH>;
  constexpr int KS = G::KS, KP = G::KP;
  extern __shared__ double smem[];
  double* frag = smem;                               // [half][TH][KS][32]
  double* pan = smem + 2 * G::FH;                    // [2][panel]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  const int h = n >> 1, hs = n - h;
  const bool odd = (n & 1) != 0;
  // Half factor b (0 = symmetric, 1 = skew): C_b[m][k] = U[k][b * hs + m], m < size_b, k < size_b
  // (size_0 = hs, size_1 = h).  Tile index i / k-step ks select
  //   COLS fwd : A[m = 8 i + q][k = 4 ks + t]      COLS inv : A[k = 8 i + q][m = 4 ks + t]
  //   ROWS fwd : B[k = 4 ks + t][m = 8 i + q]      ROWS inv : B[m = 4 ks + t][k = 8 i + q]
  for (int e = tid; e < 2 * G::FH; e += 256) {
    const int l = e & 31, ks = (e >> 5) % KS, i = ((e >> 5) / KS) % TH, b = (e >> 5) / (KS * TH);
    const int q = l >> 2, t = l & 3;
    const int r8 = 8 * i + q, c4 = 4 * ks + t;
    const int m = INV ? c4 : r8, k = INV ? r8 : c4;  // the forward tiles run over modes, the inverse over k
    const int sz = b == 0 ? hs : h;
    frag[e] = (m < sz && k < sz) ? __ldg(U + (long long)k * n + b * hs + m) : 0.0;
  }
  const double* fs = frag;
  const double* fa = frag + G::FH;
  const long long total = ROWS ? outer : outer * inner;
  const long long ntiles = (total + 63) / 64;
  if constexpr (!ROWS) {
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
      for (int m = 0; m < KP / 4; ++m) {
        const int k = lk + 4 * m;
        const bool v = okc && k < n;
        cp_async8(dst + k * G::BLD, v ? in + base + (long long)k * inner : in, v);
      }
      cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) load(tile, 0);
    __syncthreads();
    const int col = 8 * warp + gq;
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
      double as_[TH][2], aa_[TH][2];
#pragma unroll
      for (int i = 0; i < TH; ++i) as_[i][0] = as_[i][1] = aa_[i][0] = aa_[i][1] = 0.0;
#pragma unroll 2
      for (int ks = 0; ks < KS; ++ks) {
        const int k = 4 * ks + t4;
        double bsym, bskw;
        if constexpr (!INV) {
          const double xk = bs[k * G::BLD + col];
          const double xr = bs[(k < h ? n - 1 - k : k) * G::BLD + col];
          bsym = k < h ? xk + xr : ((odd && k == h) ? xk : 0.0);
          bskw = k < h ? xk - xr : 0.0;
        } else {
          bsym = k < hs ? bs[k * G::BLD + col] : 0.0;
          bskw = k < h ? bs[(hs + k) * G::BLD + col] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < TH; ++i) {
          dmma(as_[i][0], as_[i][1], fs[(i * KS + ks) * 32 + lane], bsym);
          dmma(aa_[i][0], aa_[i][1], fa[(i * KS + ks) * 32 + lane], bskw);
        }
      }
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
      for (int i = 0; i < TH; ++i) {
        const int r = 8 * i + gq;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (ob[e] < 0) continue;
          double* o = out + ob[e];
          if constexpr (!INV) {
            if (r < hs) o[(long long)r * inner] = as_[i][e];
            if (r < h) o[(long long)(hs + r) * inner] = aa_[i][e];
          } else {
            if (r < h) {
              o[(long long)r * inner] = as_[i][e] + aa_[i][e];
              o[(long long)(n - 1 - r) * inner] = as_[i][e] - aa_[i][e];
            } else if (odd && r == h) {
              o[(long long)r * inner] = as_[i][e];
            }
          }
        }
      }
      __syncthreads();
    }
  } else {
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
      const double* arow = pan + buf * 64 * G::ALD + (8 * warp + gq) * G::ALD;
      double as_[TH][2], aa_[TH][2];
#pragma unroll
      for (int j = 0; j < TH; ++j) as_[j][0] = as_[j][1] = aa_[j][0] = aa_[j][1] = 0.0;
#pragma unroll 2
      for (int ks = 0; ks < KS; ++ks) {
        const int k = 4 * ks + t4;
        double asym, askw;
        if constexpr (!INV) {
          const double xk = arow[k];
          const double xr = arow[k < h ? n - 1 - k : k];
          asym = k < h ? xk + xr : ((odd && k == h) ? xk : 0.0);
          askw = k < h ? xk - xr : 0.0;
        } else {
          asym = k < hs ? arow[k] : 0.0;
          askw = k < h ? arow[hs + k] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < TH; ++j) {
          dmma(as_[j][0], as_[j][1], asym, fs[(j * KS + ks) * 32 + lane]);
          dmma(aa_[j][0], aa_[j][1], askw, fa[(j * KS + ks) * 32 + lane]);
        }
      }
      const long long row = tile * 64 + 8 * warp + gq;
      if (row < total) {
        double* dst = out + row * n;
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * j + 2 * t4 + e;
            if constexpr (!INV) {
              if (c < hs) dst[c] = as_[j][e];
              if (c < h) dst[hs + c] = aa_[j][e];
            } else {
              if (c < h) {
                dst[c] = as_[j][e] + aa_[j][e];
                dst[n - 1 - c] = as_[j][e] - aa_[j][e];
              } else if (odd && c == h) {
                dst[c] = as_[j][e];
              }
            }
          }
      }
      __syncthreads();
    }
  }
}

// Launch for hs = n - n/2 <= 8 * TH; returns false (nothing launched) outside the instantiated range.
template <bool ROWS>
inline bool launch_mode_fold(const double* U, const double* in, double* out, int n, bool inverse, long long inner,
                             long long outer, int nsm, cudaStream_t st, cudaError_t* err) {
  const int hs = n - n / 2;
#define MI_MF(THV)                                                                                       \
  if (hs <= 8 * THV) {                                                                                   \
    constexpr size_t sm = ROWS ? ModeFold<THV>::SMEM_ROWS : ModeFold<THV>::SMEM_COLS;                    \
    static bool attr = false;                                                                            \
    if (!attr) {                                                                                         \
      cudaFuncSetAttribute(mode_fold<THV, ROWS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
      cudaFuncSetAttribute(mode_fold<THV, ROWS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);  \
      attr = true;                                                                                       \
    }                                                                                                    \
    const long long total = ROWS ? outer : outer * inner;                                                \
    const long long ntiles = (total + 63) / 64;                                                          \
    const int grid = (int)(ntiles < nsm ? ntiles : nsm);                                                 \
    if (inverse)                                                                                         \
      mode_fold<THV, ROWS, true><<<grid > 0 ? grid : 1, 256, sm, st>>>(U, in, out, n, inner, outer);     \
    else                                                                                                 \
      mode_fold<THV, ROWS, false><<<grid > 0 ? grid : 1, 256, sm, st>>>(U, in, out, n, inner, outer);    \
    *err = cudaGetLastError();                                                                           \
    return true;                                                                                         \
  }
  MI_MF(1) MI_MF(2) MI_MF(3) MI_MF(5) MI_MF(7)
#undef MI_MF
  return false;
}

}  // namespace mi
