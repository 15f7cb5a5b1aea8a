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
  static constexpr int KS = (S + 3) / 4;            // k-steps per point
  static constexpr int KH = (KS + 1) / 2;           // k-steps per warp (2 warps / point)
  static constexpr int B1 = D == 3 ? 2 : (D == 2 ? 4 : 8);
  static constexpr int B2 = D == 3 ? 2 : (D == 2 ? 2 : 1);
  static constexpr int B3 = D == 3 ? 2 : 1;
  static constexpr int H1 = B1 + 2 * P;
  static constexpr int H2 = D >= 2 ? B2 + 2 * P : 1;
  static constexpr int H3 = D >= 3 ? B3 + 2 * P : 1;
  static constexpr int HS = H1 * H2 * H3;
  static constexpr int TS = HS + ((4 - HS % 16) + 16) % 16;   // row stride = 4 mod 16 doubles
  static constexpr int MT = 3;                      // M-tiles (8 time rows each) per chunk
  static constexpr int TT = 8 * MT;                 // time rows per chunk
  static constexpr int PTMAX = 4;
  static constexpr int RING = TT + 2 * PTMAX;
  static constexpr int THREADS = 512;
  static constexpr size_t SMEM = (size_t)2 * TT * TS * 8      // X halo, double buffered
                                 + (size_t)8 * 8 * RING * 8    // W ring [pt][ch][row]
                                 + (size_t)KS * 4 * 4;         // stencil offsets
};

struct DmmaArgs {
  const double* x;
  const double* frag;   // fragment-major coefficients of this channel group
  const double* band;   // time bands (nchan_total, nt, 2pt+1)
  double* y;
  int c0, nc;           // channel group [c0, c0+nc)
  int pt, accumulate;
  int n1, n2, n3, nt;
  int C1, C2, C3;       // cube grid
  long long ns;
};

__device__ __forceinline__ void pair_sync(int id) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory");
}

template <int D, int P>
__global__ void __launch_bounds__(512, 1) stencil_dmma(DmmaArgs a) {
  using G = DmmaSten<D, P>;
  extern __shared__ double sm[];
  double* Xs = sm;                                   // [2][TT][TS]
  double* ring = Xs + 2 * G::TT * G::TS;             // [8 pt][8 ch][RING]
  int* offs = reinterpret_cast<int*>(ring + 8 * 8 * G::RING);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pt = warp >> 1, half = warp & 1;
  const int cube = blockIdx.x;
  const int c1 = cube % a.C1, c2 = (cube / a.C1) % a.C2, c3 = cube / (a.C1 * a.C2);
  const int o1 = c1 * G::B1, o2 = c2 * G::B2, o3 = c3 * G::B3;

  for (int s = tid; s < G::KS * 4; s += G::THREADS) {
    int v = 0;
    if (s < G::S) {
      const int a1 = s % G::W, a2 = D >= 2 ? (s / G::W) % G::W : 0, a3 = D >= 3 ? s / (G::W * G::W) : 0;
      v = (a3 * G::H2 + a2) * G::H1 + a1;
    }
    offs[s] = v;
  }
  double* myring = ring + pt * 8 * G::RING;          // this point's W ring [ch][row]
  for (int e = (tid & 63); e < 8 * G::RING; e += 64) myring[e] = 0.0;

  // this warp's point
  const int l1 = pt % G::B1, l2 = (pt / G::B1) % G::B2, l3 = pt / (G::B1 * G::B2);
  const int p1 = o1 + l1, p2 = o2 + l2, p3 = o3 + l3;
  const bool pvalid = p1 < a.n1 && p2 < a.n2 && p3 < a.n3;
  const long long pidx = ((long long)p3 * a.n2 + p2) * a.n1 + p1;
  const int base = (l3 * G::H2 + l2) * G::H1 + l1;

  // coefficient fragments for this warp's half of K (registers, whole sweep)
  double breg[G::KH];
  {
    const double* f = a.frag + ((long long)cube * 8 + pt) * G::KS * 32 + lane;
#pragma unroll
    for (int j = 0; j < G::KH; ++j) {
      const int ks = half * G::KH + j;
      breg[j] = ks < G::KS ? __ldg(f + ks * 32) : 0.0;
    }
  }

  const int nchunks = (a.nt + a.pt + G::TT - 1) / G::TT;
  auto load_chunk = [&](int buf, int t0) {
    if (t0 >= a.nt) return;
    double* dst = Xs + buf * G::TT * G::TS;
    const int rows = min(G::TT, a.nt - t0);
    for (int e = tid; e < rows * G::HS; e += G::THREADS) {
      const int t = e / G::HS, h = e - t * G::HS;
      const int h1 = h % G::H1, h2 = (h / G::H1) % G::H2, h3 = h / (G::H1 * G::H2);
      const int g1 = o1 - P + h1;
      const int g2 = D >= 2 ? o2 - P + h2 : 0;
      const int g3 = D >= 3 ? o3 - P + h3 : 0;
      const bool v = g1 >= 0 && g1 < a.n1 && g2 >= 0 && g2 < a.n2 && g3 >= 0 && g3 < a.n3;
      const double* src = v ? a.x + (long long)(t0 + t) * a.ns + ((long long)g3 * a.n2 + g2) * a.n1 + g1 : a.x;
      cp_async8(dst + t * G::TS + h, src, v);
    }
  };

  load_chunk(0, 0);
  cp_async_commit();
  const int W2pt = 2 * a.pt + 1;
  const int bar_id = 1 + pt;
  // filter work split: 64 threads of the pair = TT rows x (64/TT) channel slices
  const int ptid = tid & 63;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int t0 = ch * G::TT;
    cp_async_wait<0>();
    __syncthreads();                                  // chunk ch visible; buffer (ch+1)&1 free
    if (ch + 1 < nchunks) load_chunk((ch + 1) & 1, t0 + G::TT);
    cp_async_commit();
    const double* X = Xs + (ch & 1) * G::TT * G::TS;
    double acc[G::MT][2];
#pragma unroll
    for (int m = 0; m < G::MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    const int mt_live = t0 < a.nt ? min(G::MT, (a.nt - t0 + 7) / 8) : 0;
    if (mt_live > 0) {
      const double* xa = X + (lane >> 2) * G::TS + base;
#pragma unroll
      for (int j = 0; j < G::KH; ++j) {
        const int ks = half * G::KH + j;
        if (ks < G::KS) {
          const int o = offs[ks * 4 + (lane & 3)];
#pragma unroll
          for (int m = 0; m < G::MT; ++m)
            if (m < mt_live) dmma(acc[m][0], acc[m][1], xa[m * 8 * G::TS + o], breg[j]);
        }
      }
    }
    // K-split reduction in place in the ring rows of this chunk
    const int mr = lane >> 2, n0 = 2 * (lane & 3);
    if (half == 1) {
#pragma unroll
      for (int m = 0; m < G::MT; ++m) {
        const int row = 2 * G::PTMAX + m * 8 + mr;
        myring[n0 * G::RING + row] = acc[m][0];
        myring[(n0 + 1) * G::RING + row] = acc[m][1];
      }
    }
    pair_sync(bar_id);
    if (half == 0) {
#pragma unroll
      for (int m = 0; m < G::MT; ++m) {
        const int row = 2 * G::PTMAX + m * 8 + mr;
        myring[n0 * G::RING + row] += acc[m][0];
        myring[(n0 + 1) * G::RING + row] += acc[m][1];
      }
    }
    pair_sync(bar_id);
    // time filter: y[t] for t in [t0 - pt, t0 + TT - pt), by the warp pair
    for (int e = ptid; e < G::TT; e += 64) {
      const int tl = e;
      const int t = t0 - a.pt + tl;
      if (t >= 0 && t < a.nt && pvalid) {
        double v = 0.0;
        for (int c = 0; c < a.nc; ++c) {
          const double* bd = a.band + ((long long)(a.c0 + c) * a.nt + t) * W2pt;
          const double* rw = myring + c * G::RING + 2 * (G::PTMAX - a.pt) + tl;
          for (int k = 0; k < W2pt; ++k) v = fma(__ldg(bd + k), rw[k], v);
        }
        double* dst = a.y + (long long)t * a.ns + pidx;
        if (a.accumulate) *dst += v; else *dst = v;
      }
    }
    pair_sync(bar_id);
    // shift the ring: keep the last 2*PTMAX rows, clear the rest
    for (int e = ptid; e < 8 * 2 * G::PTMAX; e += 64) {
      const int r = e % (2 * G::PTMAX), c = e / (2 * G::PTMAX);
      myring[c * G::RING + r] = myring[c * G::RING + G::TT + r];
    }
    pair_sync(bar_id);
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
  const int ch = lane >> 2, s = ks * 4 + (lane & 3);
  double v = 0.0;
  if (ch < nc && s < G::S && i1 < n1 && i2 < n2 && i3 < n3) {
    const long long i = ((long long)i3 * n2 + i2) * n1 + i1;
    v = sten[((long long)(c0 + ch) * G::S + s) * ns + i];
  }
  frag[e] = v;
}

}  // namespace mi
