// Fused channel-stencil + banded-time-filter operator kernel on the FP64
// tensor cores (DMMA m8n8k4).  Reference: KroneckerOperator.matvec
// (assembly.py:430-444) over the Galerkin + Spline Upwind term list
// (solver.py:213-236, stabilization.py:439-445).
//
//   y[t, i] (+)= sum_c sum_k T_c[t, t-pt+k] W_c[t-pt+k, i],
//   W_c[t, i]   = sum_s S_c[s, i] x[t, i + off(s)]          (8 channels / launch)
//
// Tensor-core mapping, per output point i:  M = 8 time slices, N = 8
// channels, K = stencil points (4 per DMMA).  A[m][k] = x[t0+m, i+off(k)]
// comes from a shared-memory halo tile, B[k][n] = S_n[k, i] is loaded ONCE
// per point into registers (fragment-major storage, coalesced 256 B per
// k-step) and reused for all N_t time slices.  A block owns 8 points
// (2x2x2 for d=3) and sweeps time in chunks of TT=16 with a cp.async
// double-buffered halo tile; two warps per point split K.  The time filter
// consumes a ring of W rows in shared memory, so W never touches HBM.
#pragma once
#include "common.cuh"
#include "ptx.cuh"
#include <cuda.h>

namespace mi {

template <int D, int P>
struct DmmaSten {
  static constexpr int W = 2 * P + 1;
  static constexpr int S = D == 3 ? W * W * W : (D == 2 ? W * W : W);
  // K order: x-offset a1 padded to W1P (multiple of 4) so every k-step covers
  // 4 consecutive x-offsets of one (a2, a3) row (zero coefficients in the pad)
  static constexpr int W1P = (W + 3) / 4 * 4;
  static constexpr int QR = W1P / 4;                // k-steps per stencil row
  static constexpr int NROW = D == 3 ? W * W : (D == 2 ? W : 1);
  static constexpr int KS = QR * NROW;              // k-steps per point
  static constexpr int KH = (KS + 1) / 2;           // k-steps per warp (2 warps / point)
  static constexpr int B1 = D == 3 ? 2 : (D == 2 ? 4 : 8);
  static constexpr int B2 = D == 3 ? 2 : (D == 2 ? 2 : 1);
  static constexpr int B3 = D == 3 ? 2 : 1;
  static constexpr int H1 = B1 + 2 * P;
  static constexpr int H2 = D >= 2 ? B2 + 2 * P : 1;
  static constexpr int H3 = D >= 3 ? B3 + 2 * P : 1;
  static constexpr int HS = H1 * H2 * H3;
  static constexpr int MT = 2;                      // M-tiles (8 time rows each) per chunk
  static constexpr int TT = 8 * MT;                 // time rows per chunk
  static constexpr int TSTR = TT + 4;               // smem stride per halo point (= 4 mod 16)
  static constexpr int PTMAX = 4;
  static constexpr int BW = 2 * PTMAX + 1;
  static constexpr int WL = 2 * TT + 2 * PTMAX;     // circular W buffer length (rows)
  static constexpr int PSTR = 8 * WL + 4;           // point stride in the W buffer (= 4 mod 16)
  static constexpr int THREADS = 512;
  static constexpr int FK = 8 * 16;                 // filter K: 8 channels x 16 time taps
  static constexpr size_t SMEM = (size_t)2 * HS * TSTR * 8       // X halo [buf][h][t]
                                 + (size_t)2 * 8 * PSTR * 8       // W partials [half][pt][ch*WL + row]
                                 + (size_t)2 * 2 * 4 * 64 * 8     // filter partials [buf][mtile][cpair][64]
                                 + 16;                            // TMA mbarriers
  // halo offset of lane-k 0 of k-step ks (lane kl adds kl)
  static constexpr __host__ __device__ int koff(int ks) {
    return ((D >= 3 ? (ks / QR) / W : 0) * H2 + (D >= 2 ? (ks / QR) % W : 0)) * H1 + 4 * (ks % QR);
  }
};

struct DmmaArgs {
  const double* xt;     // time-innermost copy of x: xt[i * ntp + t]
  const double* afr;    // time-filter A fragments [tau][32 ks][32 lanes] of this group
  int ntau;
  const double* frag;   // fragment-major coefficients of this channel group
  const double* band;   // time bands (nchan_total, nt, 2pt+1)
  double* y;
  int c0, nc;           // channel group [c0, c0+nc)
  int pt, accumulate;
  int n1, n2, n3, nt, ntp;
  int C1, C2, C3;       // cube grid
  long long ns;
};

// x (nt, ns) -> xt (ns, ntp), zero padded in time; 32x32 smem tiles.
__global__ void transpose_time_inner(const double* __restrict__ x, double* __restrict__ xt, int nt, int ntp,
                                     long long ns) {
  __shared__ double tile[32][33];
  const long long s0 = (long long)blockIdx.x * 32;
  const int t0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int t = t0 + r;
    const long long s = s0 + threadIdx.x;
    tile[r][threadIdx.x] = (t < nt && s < ns) ? x[(long long)t * ns + s] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const long long s = s0 + r;
    const int t = t0 + threadIdx.x;
    if (s < ns && t < ntp) xt[s * ntp + t] = tile[threadIdx.x][r];
  }
}

// One warp's K-half of the DMMA sweep over a time chunk: per k-step two
// immediate-offset LDS.64 (lane kl reads x-offset 4q+kl: conflict-free) and
// two DMMAs; no per-step address arithmetic, no branches.
template <class G, int HALF>
__device__ __forceinline__ void dmma_sweep(const double* X, const double (&breg)[G::KH],
                                           double (&acc)[G::MT][2]) {
#pragma unroll
  for (int j = 0; j < G::KH; ++j) {
    const int ks = HALF * G::KH + j;
    if (ks < G::KS) {
      const double* xa = X + G::koff(ks) * G::TSTR;
#pragma unroll
      for (int m = 0; m < G::MT; ++m) dmma(acc[m][0], acc[m][1], xa[m * 8], breg[j]);
    }
  }
}

template <int D, int P>
__global__ void __launch_bounds__(512, 1) stencil_dmma(DmmaArgs a, const __grid_constant__ CUtensorMap tmap) {
  using G = DmmaSten<D, P>;
  extern __shared__ __align__(128) double sm[];
  double* Xs = sm;                                   // [2][HS][TSTR]
  double* Wp = Xs + 2 * G::HS * G::TSTR;             // [2 half][8 pt][PSTR]
  double* ys = Wp + 2 * 8 * G::PSTR;                 // [2 buf][2 mtile][4 cpair][64]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ys + 2 * 2 * 4 * 64);   // 2 mbarriers

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pt = warp >> 1, half = warp & 1;
  const int cube = blockIdx.x;
  const int c1 = cube % a.C1, c2 = (cube / a.C1) % a.C2, c3 = cube / (a.C1 * a.C2);
  const int o1 = c1 * G::B1, o2 = c2 * G::B2, o3 = c3 * G::B3;

  for (int e = tid; e < 2 * 8 * G::PSTR; e += G::THREADS) Wp[e] = 0.0;

  double breg[G::KH];
  {
    const double* f = a.frag + ((long long)cube * 8 + pt) * G::KS * 32 + lane;
#pragma unroll
    for (int j = 0; j < G::KH; ++j) {
      const int ks = half * G::KH + j;
      breg[j] = ks < G::KS ? __ldg(f + ks * 32) : 0.0;
    }
  }

  const int W2pt = 2 * a.pt + 1;
  // ---- async loads of chunk t0: halo tile (16 B copies) + band rows of the
  // halo tile of chunk t0 by ONE TMA bulk-tensor copy: box (TSTR time rows, H1, H2, H3) of the
  // time-innermost copy; out-of-range halo coordinates (incl. negative) are zero-filled by TMA
  constexpr unsigned TILE_BYTES = (unsigned)(G::TSTR * G::HS * 8);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto load_chunk = [&](int buf, int t0) {
    if (tid == 0 && t0 < a.nt) {
      mbar_expect_tx(&bars[buf], TILE_BYTES);
      tma_load_4d(Xs + buf * G::HS * G::TSTR, &tmap, &bars[buf], t0, o1 - P, D >= 2 ? o2 - P : 0,
                  D >= 3 ? o3 - P : 0);
    }
  };

  // time filter on the tensor cores: warps 0..7 -> (mtile fm, channel pair fcq)
  const int fm = warp & 1, fcq = (warp >> 1) & 3;
  // output write of the previous filter: warps 8..11 (tid 256..383) -> (mtile, row m, point n);
  // warps 0..7 run the tensor-core filter, so the extra work is spread over 12 warps
  auto write_y = [&](int ch_buf, int tbase) {
    const int wt_ = tid - 256;
    const int om = (wt_ >> 6) & 1, orow = (wt_ >> 3) & 7, opt = wt_ & 7;
    const int q1 = o1 + opt % G::B1, q2 = o2 + (opt / G::B1) % G::B2, q3 = o3 + opt / (G::B1 * G::B2);
    const int t = tbase + 8 * om + orow;
    if (t >= 0 && t < a.nt && q1 < a.n1 && q2 < a.n2 && q3 < a.n3) {
      const double* yp = ys + (ch_buf * 2 + om) * 4 * 64 + orow * 8 + opt;
      const double v = (yp[0] + yp[64]) + (yp[128] + yp[192]);
      double* dst = a.y + (long long)t * a.ns + ((long long)q3 * a.n2 + q2) * a.n1 + q1;
      if (a.accumulate) *dst += v; else *dst = v;
    }
  };

  const int base = ((pt / (G::B1 * G::B2)) * G::H2 + (pt / G::B1) % G::B2) * G::H1 + pt % G::B1;
  const int kl = lane & 3, mrow = lane >> 2;
  double* wmine = Wp + (half * 8 + pt) * G::PSTR + 2 * kl * G::WL;   // channels 2kl, 2kl+1

  const int nchunks = (a.nt + a.pt + G::TT - 1) / G::TT + 1;   // +1: filter of the last chunk
  (void)W2pt;
  load_chunk(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int t0 = ch * G::TT;
    if (t0 < a.nt) mbar_wait(&bars[ch & 1], (ch >> 1) & 1);   // X(ch) landed (k-th use of buffer -> parity k&1)
    __syncthreads();                  // other buffer free; W rows of chunk ch-1 complete
    if (ch + 1 < nchunks) load_chunk((ch + 1) & 1, t0 + G::TT);
    // ---- write y of the filter of chunk ch-2 (partials summed over channel pairs)
#ifndef MI_EXP_NOFILTER
    if (ch >= 2 && tid >= 256 && tid < 384) write_y(ch & 1, t0 - 2 * G::TT - a.pt);
#endif
    // ---- time filter of chunk ch-1 on the tensor cores (warps 0..7)
#ifdef MI_EXP_NOFILTER
    if (false) {
#else
    if (ch >= 1 && warp < 8) {
#endif
      const int tau = 2 * (ch - 1) + fm;                   // M-tile rows tb = 8 tau - pt
      const int tb = 8 * tau - a.pt;
      const double* af = a.afr + ((long long)tau * 32 + 8 * fcq) * 32 + lane;
      const int n = lane >> 2;                             // point (B column)
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
      const int r0 = (tb - a.pt + 2 * G::PTMAX) % G::WL;  // row of time tb - pt
#pragma unroll
      for (int kq = 0; kq < 8; ++kq) {
        const int k = 4 * (8 * fcq + kq) + kl;             // K index: channel k/16, tap j = k%16
        const int c = k >> 4, j = k & 15;
        int r = r0 + j;
        r = r >= G::WL ? r - G::WL : r;
        const double* wp = Wp + n * G::PSTR + c * G::WL + r;
        const double bv = wp[0] + wp[8 * G::PSTR];
        const double av = __ldg(af + kq * 32);
        if (kq & 1) dmma(d0, d1, av, bv); else dmma(c0, c1, av, bv);
      }
      double* yp = ys + (((ch + 1) & 1) * 2 + fm) * 4 * 64 + fcq * 64;
      yp[mrow * 8 + 2 * kl] = c0 + d0;
      yp[mrow * 8 + 2 * kl + 1] = c1 + d1;
    }
    // ---- DMMA sweep of chunk ch into this half's W partial rows
    if (t0 < a.nt + a.pt) {
      double acc[G::MT][2];
#pragma unroll
      for (int m = 0; m < G::MT; ++m) acc[m][0] = acc[m][1] = 0.0;
      if (t0 < a.nt) {
        const double* X = Xs + (ch & 1) * G::HS * G::TSTR + (base + kl) * G::TSTR + mrow;
        if (half == 0)
          dmma_sweep<G, 0>(X, breg, acc);
        else
          dmma_sweep<G, 1>(X, breg, acc);
      }
#pragma unroll
      for (int m = 0; m < G::MT; ++m) {
        const int r = (t0 + m * 8 + mrow + 2 * G::PTMAX) % G::WL;
        wmine[r] = acc[m][0];
        wmine[G::WL + r] = acc[m][1];
      }
    }
  }
  // flush the last filter's partials (chunk nchunks-2)
  __syncthreads();
  if (tid >= 256 && tid < 384) write_y(nchunks & 1, nchunks * G::TT - 2 * G::TT - a.pt);
}

// Time-filter A fragments: afr[tau][ks][lane] = T_{c0+c}[t, t'] with
// t = 8 tau - pt + lane/4, k = 4 ks + lane%4 = 16 c + j, t' = t - (lane/4) - pt + j
// (zero outside the band, the channel group or [0, nt)).
__global__ void build_filter_frag(double* __restrict__ afr, const double* __restrict__ band, int c0, int nc,
                                  int nt, int pt, int ntau) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ntau * 32 * 32) return;
  const int lane = e & 31, ks = (e >> 5) & 31, tau = e >> 10;
  const int m = lane >> 2, k = 4 * ks + (lane & 3);
  const int c = k >> 4, j = k & 15;
  const int t = 8 * tau - pt + m;
  const int tap = j - m;                                  // t' - t + pt
  double v = 0.0;
  if (c < nc && t >= 0 && t < nt && tap >= 0 && tap <= 2 * pt)
    v = band[((long long)(c0 + c) * nt + t) * (2 * pt + 1) + tap];
  afr[e] = v;
}

// Repack channel stencils [c][s][i] into the fragment-major layout
// frag[(cube*8 + pt)][ks][lane] = S_{c0 + lane/4}[4 ks + lane%4][i(cube, pt)].
template <int D, int P>
__global__ void repack_frag(const double* __restrict__ sten, double* __restrict__ frag, int c0, int nc,
                            int n1, int n2, int n3, int C1, int C2, long long ns, long long total) {
  using G = DmmaSten<D, P>;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int lane = (int)(e & 31);
  const long long r = e >> 5;
  const int ks = (int)(r % G::KS);
  const long long pid = r / G::KS;
  const int pt = (int)(pid & 7);
  const long long cube = pid >> 3;
  const int cc1 = (int)(cube % C1), cc2 = (int)((cube / C1) % C2), cc3 = (int)(cube / ((long long)C1 * C2));
  const int i1 = cc1 * G::B1 + pt % G::B1, i2 = cc2 * G::B2 + (pt / G::B1) % G::B2,
            i3 = cc3 * G::B3 + pt / (G::B1 * G::B2);
  const int ch = lane >> 2;
  const int a1 = 4 * (ks % G::QR) + (lane & 3), row = ks / G::QR;
  const int s = row * G::W + a1;                   // unpadded stencil index
  double v = 0.0;
  if (ch < nc && a1 < G::W && i1 < n1 && i2 < n2 && i3 < n3) {
    const long long i = ((long long)i3 * n2 + i2) * n1 + i1;
    v = sten[((long long)(c0 + ch) * G::S + s) * ns + i];
  }
  frag[e] = v;
}

}  // namespace mi
