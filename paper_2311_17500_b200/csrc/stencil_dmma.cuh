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
  static constexpr int THREADS = 512;
  static constexpr size_t SMEM = (size_t)2 * HS * TSTR * 8       // X halo [buf][h][t]
                                 + (size_t)2 * 8 * 8 * WL * 8;    // W partials [half][pt][ch][row mod WL]
  // halo offset of lane-k 0 of k-step ks (lane kl adds kl)
  static constexpr __host__ __device__ int koff(int ks) {
    return ((D >= 3 ? (ks / QR) / W : 0) * H2 + (D >= 2 ? (ks / QR) % W : 0)) * H1 + 4 * (ks % QR);
  }
};

struct DmmaArgs {
  const double* xt;     // time-innermost copy of x: xt[i * ntp + t]
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
__global__ void __launch_bounds__(512, 1) stencil_dmma(DmmaArgs a) {
  using G = DmmaSten<D, P>;
  extern __shared__ double sm[];
  double* Xs = sm;                                   // [2][HS][TSTR]
  double* Wp = Xs + 2 * G::HS * G::TSTR;             // [2 half][8 pt][8 ch][WL]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pt = warp >> 1, half = warp & 1;
  const int cube = blockIdx.x;
  const int c1 = cube % a.C1, c2 = (cube / a.C1) % a.C2, c3 = cube / (a.C1 * a.C2);
  const int o1 = c1 * G::B1, o2 = c2 * G::B2, o3 = c3 * G::B3;

  for (int e = tid; e < 2 * 8 * 8 * G::WL; e += G::THREADS) Wp[e] = 0.0;

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
  constexpr int PAIRS = G::TT / 2;
  auto load_chunk = [&](int buf, int t0) {
    if (t0 >= a.nt) return;
    double* dst = Xs + buf * G::HS * G::TSTR;
    for (int e = tid; e < G::HS * PAIRS; e += G::THREADS) {
      const int h = e / PAIRS, pr = e - h * PAIRS;
      const int h1 = h % G::H1, h2 = (h / G::H1) % G::H2, h3 = h / (G::H1 * G::H2);
      const int g1 = o1 - P + h1;
      const int g2 = D >= 2 ? o2 - P + h2 : 0;
      const int g3 = D >= 3 ? o3 - P + h3 : 0;
      const bool v = g1 >= 0 && g1 < a.n1 && g2 >= 0 && g2 < a.n2 && g3 >= 0 && g3 < a.n3;
      const double* src = v ? a.xt + (((long long)g3 * a.n2 + g2) * a.n1 + g1) * a.ntp + t0 + 2 * pr : a.xt;
      cp_async16(dst + h * G::TSTR + 2 * pr, src, v);
    }
  };

  // filter item of this thread: (point fq, channel fc, rows fr + 8*hh)
  const int fc = tid & 7, fr = (tid >> 3) & 7, fq = tid >> 6;
  const int f1 = o1 + fq % G::B1, f2 = o2 + (fq / G::B1) % G::B2, f3 = o3 + fq / (G::B1 * G::B2);
  const bool fvalid = f1 < a.n1 && f2 < a.n2 && f3 < a.n3;
  const long long fidx = ((long long)f3 * a.n2 + f2) * a.n1 + f1;
  const double* w0 = Wp + (fq * 8 + fc) * G::WL;
  const double* w1 = Wp + ((8 + fq) * 8 + fc) * G::WL;

  const int base = ((pt / (G::B1 * G::B2)) * G::H2 + (pt / G::B1) % G::B2) * G::H1 + pt % G::B1;
  const int kl = lane & 3, mrow = lane >> 2;
  double* wmine = Wp + ((half * 8 + pt) * 8 + 2 * kl) * G::WL;   // channels 2kl, 2kl+1

  const int nchunks = (a.nt + a.pt + G::TT - 1) / G::TT + 1;   // +1: filter of the last chunk
  load_chunk(0, 0);
  cp_async_commit();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int t0 = ch * G::TT;
    cp_async_wait<0>();
    __syncthreads();                  // X(ch), bands(ch) visible; W rows of chunk ch-1 complete
    if (ch + 1 < nchunks) load_chunk((ch + 1) & 1, t0 + G::TT);
    cp_async_commit();
    // ---- time filter of chunk ch-1: y[t], t in [t0 - TT - pt, t0 - pt)
    if (ch > 0) {
      const int tp0 = t0 - G::TT;
#pragma unroll
      for (int hh = 0; hh < G::TT / 8; ++hh) {
        const int tl = fr + 8 * hh;
        const int t = tp0 - a.pt + tl;
        double v = 0.0;
        if (fc < a.nc && t >= 0 && t < a.nt) {
          const double* bd = a.band + ((long long)(a.c0 + fc) * a.nt + t) * W2pt;
          for (int k = 0; k < W2pt; ++k) {
            int r = t - a.pt + k + 2 * G::PTMAX;           // row of time t-pt+k (shifted >= 0)
            r = r % G::WL;
            v = fma(__ldg(bd + k), w0[r] + w1[r], v);
          }
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        if (fc == 0 && t >= 0 && t < a.nt && fvalid) {
          double* dst = a.y + (long long)t * a.ns + fidx;
          if (a.accumulate) *dst += v; else *dst = v;
        }
      }
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
