// Spline Upwind residual indicator on the device (reference compute_theta,
// stabilization.py:235-339; strong residual stabilization.py:148-174):
//
//   res = C_m u_t / T - sum_l D_l d2u/dx_l^2 + c1 u (u - a)(u - 1) + c2 u w - f
//
// (D scalar in the reference; one value per direction here)
// at the q = p+1 Gauss points of every space-time element, reduced to
// per-element maxima of |res|, plus the global maxima max|u|, max|u_t| of
// the denominator.  The per-function window maxima (separable along t, x, y,
// z) and the clamped ratio are separate HBM-bound kernels.
//
// The element kernel is the reaction kernel's time-streamed tile sweep
// (reaction.cu) with different stage channels: a block owns 2^d spatial
// elements and streams the time functions.  Each entering slice of (u, w) is
// interpolated to the tile's spatial Gauss grid as five channels -- u, the
// three second parametric derivatives of u and w -- with the last direction's
// DMMA accumulators kept in registers.  The Laplacian is linear, so it is
// summed (1/L_l^2 weighted) at entry.  The window therefore holds three
// values (u, lap u, w) per point per slice, and the time stage forms u,
// u_t, lap u, w and |res| on the thread's own points.  Element maxima use
// atomicMax on the bit patterns of non-negative doubles, which is exact and
// order independent.
#include "common.cuh"
#include "ptx.cuh"

namespace mi {

struct ThArgs {
  const double* u;
  const double* w;
  const double* src;              // NULL or f at the Gauss points of elements [et0, et1)
  double* emax;                   // [nel_t][nel_3][nel_2][nel_1]
  unsigned long long* maxes;      // [2] max|u|, max|u_t| (bit patterns of non-negative doubles)
  const double* B0[4];            // element tables [e][g][a]: values
  const double* B1[4];            // space: second parametric derivative; time: first
  int nel[4];
  int n[3];
  int ntc, rowoff;
  long long ns, gs;               // spatial DoFs; spatial Gauss points (src row length)
  int G[3];                       // spatial Gauss points per direction
  int et0, et1;
  double il2[3];                  // D_l / L_l^2
  double cmT, c1, a, c2;          // C_m / T, Rogers-McCulloch constants
  const double* u0;               // u0 lifting: u coefficients of the dropped first time function (null: zero)
};

template <int D, int P>
struct ThTile {
  static constexpr int E = 2, QE = P + 1, L = E + P, Q = E * QE;
  static constexpr int L1 = L, L2 = D >= 2 ? L : 1, L3 = D >= 3 ? L : 1;
  static constexpr int Q1 = Q, Q2 = D >= 2 ? Q : 1;
  static constexpr int LS = L1 * L2 * L3, KI = (L + 3) / 4;
  static constexpr int QL = D == 3 ? Q1 * Q2 : (D == 2 ? Q1 : 1);   // lines of the last stage
  static constexpr int NT = (QL + 7) / 8, MT = (NT + 7) / 8;
  static constexpr int NLX = L3 * L2, TX = (NLX + 7) / 8;           // x stage: lines / tiles per channel
  static constexpr int NLY = L3 * Q1, TY = (NLY + 7) / 8;           // y stage
  static constexpr int CA = L3 * L2 * Q1, CB = L3 * Q2 * Q1;        // channel strides of the stage buffers
  static constexpr int ev(int n) { return (n + 1) & ~1; }
  static constexpr int SIN = ev(2 * LS);
  static constexpr int SA = D >= 2 ? ev(3 * CA) : 2;
  static constexpr int SB = D >= 3 ? ev(4 * CB) : 2;
  static constexpr int NPRE = (2 * LS + 255) / 256;
  static constexpr int NEL = D == 3 ? 8 : (D == 2 ? 4 : 2);          // elements per tile
  static constexpr size_t SMEM = (size_t)(SIN + SA + SB + 64 + 256) * 8 + 2 * 8 * sizeof(unsigned long long);
};

__device__ __forceinline__ unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }

template <int D, int P, int PT>
__global__ void __launch_bounds__(256, 2) theta_elements(ThArgs r) {
  using G = ThTile<D, P>;
  constexpr int E = G::E, QE = G::QE, L = G::L, Q = G::Q;
  constexpr int L1 = G::L1, L2 = G::L2, Q1 = G::Q1, Q2 = G::Q2;
  constexpr int LS = G::LS, KI = G::KI, QL = G::QL, NT = G::NT, MT = G::MT;
  constexpr int PW = PT + 1, QT = PT + 1, NBT = 2 * QT * PW;
  static_assert(NBT <= 32, "time tables too large");
  static_assert(Q1 % 2 == 0, "paired stores need an even Gauss count");
  extern __shared__ double sm[];
  double* sIn = sm;                                 // [u, w][j3][j2][j1]
  double* sA = sIn + G::SIN;                        // x stage [3][j3][j2][q1]
  double* sB = sA + G::SA;                          // y stage [4][j3][q2][q1]
  double* sBt = sB + G::SB;                         // [2][32] time tables (values, derivatives)
  unsigned long long* emx = reinterpret_cast<unsigned long long*>(sm + G::SIN + G::SA + G::SB + 64 + 256);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  for (int i = tid; i < G::SIN + G::SA + G::SB + 64 + 256; i += 256) sm[i] = 0.0;
  if (tid < 16) emx[tid] = 0ull;
  int b = blockIdx.x, k[3], ne[3];
  for (int l = 0; l < 3; ++l) {
    const int ntile = l < D ? (r.nel[l] + E - 1) / E : 1;
    const int m = b % ntile;
    b /= ntile;
    k[l] = l < D ? m * E : 0;
    ne[l] = l < D ? min(E, r.nel[l] - k[l]) : 1;
  }
  auto table = [&](const double* const* T, int l, int j, int q) -> double {
    if (l >= D || q >= Q || j >= L) return 0.0;
    const int le = q / QE, gq = q % QE, aa = j - le;
    if (le >= ne[l] || aa < 0 || aa > P) return 0.0;
    return __ldg(T[l] + ((long long)(k[l] + le) * QE + gq) * (P + 1) + aa);
  };
  double b0[D][KI], b2[D][KI];                      // B fragments: values / second derivatives (K = j, N = q)
#pragma unroll
  for (int l = 0; l < D; ++l)
#pragma unroll
    for (int ks = 0; ks < KI; ++ks) {
      b0[l][ks] = table(r.B0, l, 4 * ks + fk, fr);
      b2[l][ks] = table(r.B1, l, 4 * ks + fk, fr);
    }
  // the thread's Gauss points (line = 8 t + fr, q_last = 2 fk + e): validity, tile element, source index
  int pel[MT][2];                                   // tile-local element, -1 if outside the domain
  long long psrc[MT][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int line = 8 * (warp + 8 * mi) + fr, ql = 2 * fk + e;
      int q[3] = {0, 0, 0};
      if (D == 3) { q[0] = line % Q1; q[1] = line / Q1; q[2] = ql; }
      if (D == 2) { q[0] = line; q[1] = ql; }
      if (D == 1) { q[0] = ql; }
      bool ok = line < QL && ql < Q;
      int lidx = 0, mul = 1;
      long long gi = 0;
      for (int l = D - 1; l >= 0; --l) {
        const int le = q[l] / QE;
        ok = ok && le < ne[l];
        gi = gi * r.G[l] + (long long)k[l] * QE + q[l];
      }
      for (int l = 0; l < D; ++l) {
        lidx += (q[l] / QE) * mul;
        mul *= E;
      }
      pel[mi][e] = ok ? lidx : -1;
      psrc[mi][e] = gi;
    }
  const long long ns = r.ns;
  long long gsp[G::NPRE];
#pragma unroll
  for (int m = 0; m < G::NPRE; ++m) {
    const int i = tid + 256 * m;
    const int s = i % LS;
    const int j1 = s % L1, j2 = (s / L1) % L2, j3 = s / (L1 * L2);
    const int g1 = k[0] + j1, g2 = k[1] + j2, g3 = k[2] + j3;
    const bool ok = i < 2 * LS && g1 < r.n[0] && g2 < r.n[1] && g3 < r.n[2];
    gsp[m] = ok ? ((long long)g3 * r.n[1] + g2) * r.n[0] + g1 : -1;
  }
  double pre[G::NPRE];
  auto prefetch = [&](int ft) {
    const int ct = ft + r.rowoff;
    const bool vt = ct >= 0 && ct < r.ntc;
#pragma unroll
    for (int m = 0; m < G::NPRE; ++m) {
      const bool isu = (tid + 256 * m) < LS;
      const double* src = isu ? r.u : r.w;
      double v = 0.0;
      if (gsp[m] >= 0) {
        if (vt) v = __ldg(src + (long long)ct * ns + gsp[m]);
        else if (ct == -1 && isu && r.u0 != nullptr) v = __ldg(r.u0 + gsp[m]);
      }
      pre[m] = v;
    }
  };
  double btp = 0.0;
  auto prefetch_bt = [&](int et) {
    if (tid < NBT && et >= r.et0 && et < r.et1) {
      const int ga = tid % (QT * PW);
      btp = __ldg((tid < QT * PW ? r.B0[3] : r.B1[3]) + (long long)et * QT * PW + ga);
    }
  };
  auto flush = [&](int et) {                       // element maxima of time element et -> global
    if (tid < G::NEL) {
      const int le1 = tid % E, le2 = (tid / E) % E, le3 = tid / (E * E);
      const bool ok = le1 < ne[0] && (D < 2 || le2 < ne[1]) && (D < 3 || le3 < ne[2]);
      if (ok) {
        const long long el = ((long long)(k[2] + (D >= 3 ? le3 : 0)) * r.nel[1] + (k[1] + (D >= 2 ? le2 : 0))) *
                                  r.nel[0] + (k[0] + le1);
        const long long nes = (long long)r.nel[0] * r.nel[1] * r.nel[2];
        r.emax[(long long)et * nes + el] = __longlong_as_double((long long)emx[(et & 1) * 8 + tid]);
      }
      emx[(et & 1) * 8 + tid] = 0ull;
    }
  };
  double X[MT][PW][3][2];                          // window: (u, lap u, w) of slices et..et+PT
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int a = 0; a < PW; ++a)
#pragma unroll
      for (int f = 0; f < 3; ++f) X[mi][a][f][0] = X[mi][a][f][1] = 0.0;
  double umax = 0.0, utmax = 0.0;
  const double cmT = r.cmT, rc1 = r.c1, ra = r.a, rc2 = r.c2;

  const int nsl = r.et1 - r.et0 + PT;              // slices: full time functions et0 .. et1 + PT - 1
  prefetch(r.et0);
  for (int j = 0; j < nsl; ++j) {
    const int ft = r.et0 + j;
    if constexpr (D == 1) __syncthreads();         // sIn is read by the last stage directly
#pragma unroll
    for (int m = 0; m < G::NPRE; ++m)
      if (tid + 256 * m < 2 * LS) sIn[tid + 256 * m] = pre[m];
    if (tid < NBT) sBt[(j & 1) * 32 + tid] = btp;
    __syncthreads();                               // B1
    if (ft - PT - 1 >= r.et0) flush(ft - PT - 1);
    if (j + 1 < nsl) prefetch(ft + 1);
    prefetch_bt(ft + 1 - PT);
    const double* fin = sIn;
    int cstr = LS;                                 // channel stride of the last stage's input
    if constexpr (D >= 2) {
      // x stage: channels (u B, u B'', w B): lines (j3, j2), K = j1, N = q1 -> sA [c][j3][j2][q1]
      for (int tt = warp; tt < 3 * G::TX; tt += 8) {
        const int cx = tt / G::TX, line = (tt % G::TX) * 8 + fr;
        const double* src = sIn + (cx == 2 ? LS : 0);
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KI; ++ks) dmma(c0, c1, src[line * L1 + 4 * ks + fk], cx == 1 ? b2[0][ks] : b0[0][ks]);
        const int n0 = 2 * fk;
        if (line < G::NLX && n0 < Q1)
          *reinterpret_cast<double2*>(sA + cx * G::CA + line * Q1 + n0) = make_double2(c0, c1);
      }
      __syncthreads();                             // B2
      fin = sA;
      cstr = G::CA;
    }
    if constexpr (D == 3) {
      // y stage: channels (x0 B, x0 B'', x1 B, x2 B): lines (j3, q1), K = j2, N = q2 -> sB [c][j3][q2][q1]
      for (int tt = warp; tt < 4 * G::TY; tt += 8) {
        const int cy = tt / G::TY, line = (tt % G::TY) * 8 + fr;
        const int sx = cy == 0 ? 0 : cy - 1;
        const int q1 = line % Q1, j3 = line / Q1;
        const double* src = sA + sx * G::CA;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KI; ++ks)
          dmma(c0, c1, src[(j3 * L2 + 4 * ks + fk) * Q1 + q1], cy == 1 ? b2[1][ks] : b0[1][ks]);
        const int n0 = 2 * fk;
        if (line < G::NLY) {
          if (n0 < Q2) sB[cy * G::CB + (j3 * Q2 + n0) * Q1 + q1] = c0;
          if (n0 + 1 < Q2) sB[cy * G::CB + (j3 * Q2 + n0 + 1) * Q1 + q1] = c1;
        }
      }
      __syncthreads();                             // B3
      fin = sB;
      cstr = G::CB;
    }
    // last direction: channels (c0 B, c0 B'', c1 B, .., c_last B) -> (u, lap u, w) into the window
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
#pragma unroll
      for (int a = 0; a < PW - 1; ++a)
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          X[mi][a][f][0] = X[mi][a + 1][f][0];
          X[mi][a][f][1] = X[mi][a + 1][f][1];
        }
      const int t = warp + 8 * mi;
      double ch[D + 2][2];
#pragma unroll
      for (int c = 0; c < D + 2; ++c) ch[c][0] = ch[c][1] = 0.0;
      if (t < NT) {
        const int line = 8 * t + fr;
#pragma unroll
        for (int c = 0; c < D + 2; ++c) {
          const int sc = c == 0 ? 0 : c - 1;
          const double* src = fin + sc * cstr;
#pragma unroll
          for (int ks = 0; ks < KI; ++ks)
            dmma(ch[c][0], ch[c][1], src[(4 * ks + fk) * QL + line], c == 1 ? b2[D - 1][ks] : b0[D - 1][ks]);
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        // channel 1 = d2/dx_last^2; channels 2..D = the earlier directions (last-but-one first)
        double lap = ch[1][e] * r.il2[D - 1];
        if constexpr (D == 3) lap += ch[2][e] * r.il2[1] + ch[3][e] * r.il2[0];
        if constexpr (D == 2) lap += ch[2][e] * r.il2[0];
        X[mi][PW - 1][0][e] = ch[0][e];
        X[mi][PW - 1][1][e] = lap;
        X[mi][PW - 1][2][e] = ch[D + 1][e];
      }
    }
    const int et = ft - PT;
    if (et < r.et0) continue;
    // time element et: u, u_t, lap u, w and |res| at the thread's points, element maxima
    const double* bt = sBt + (j & 1) * 32;
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (pel[mi][e] < 0) continue;
        double amax = 0.0;
#pragma unroll
        for (int g = 0; g < QT; ++g) {
          double uu = 0.0, ut = 0.0, lp = 0.0, ww = 0.0;
#pragma unroll
          for (int a = 0; a < PW; ++a) {
            const double b0t = bt[g * PW + a], b1t = bt[QT * PW + g * PW + a];
            uu = fma(b0t, X[mi][a][0][e], uu);
            ut = fma(b1t, X[mi][a][0][e], ut);
            lp = fma(b0t, X[mi][a][1][e], lp);
            ww = fma(b0t, X[mi][a][2][e], ww);
          }
          double res = cmT * ut - lp + rc1 * uu * (uu - ra) * (uu - 1.0) + rc2 * uu * ww;
          if (r.src) res -= __ldg(r.src + ((long long)(et - r.et0) * QT + g) * r.gs + psrc[mi][e]);
          amax = fmax(amax, fabs(res));
          umax = fmax(umax, fabs(uu));
          utmax = fmax(utmax, fabs(ut));
        }
        atomicMax(&emx[(et & 1) * 8 + pel[mi][e]], dbits(amax));
      }
  }
  __syncthreads();
  if (r.et1 > r.et0) flush(r.et1 - 1);
  // denominator maxima: warp max, then one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    utmax = fmax(utmax, __shfl_xor_sync(0xffffffffu, utmax, o));
  }
  if (lane == 0) {
    atomicMax(&r.maxes[0], dbits(umax));
    atomicMax(&r.maxes[1], dbits(utmax));
  }
}

// out[o][i][r] = max_{e in [w0[i], w1[i])} in[o][e][r]   (values >= 0)
__global__ void window_max_kernel(const double* __restrict__ in, double* __restrict__ out, long long outer, int n_in,
                                  int n_out, long long inner, const int* __restrict__ w0, const int* __restrict__ w1) {
  const long long total = outer * n_out * inner;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long rr = idx % inner;
    const int i = (int)((idx / inner) % n_out);
    const long long o = idx / (inner * n_out);
    double m = 0.0;
    for (int e = w0[i]; e < w1[i]; ++e) m = fmax(m, in[(o * n_in + e) * inner + rr]);
    out[idx] = m;
  }
}

__global__ void theta_ratio_kernel(const double* __restrict__ numer, double* __restrict__ theta, long long n,
                                   double denom) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    theta[i] = fmin(numer[i] / denom, 1.0);
}

// Mapped geometries (stabilization.py:273-295): the strong residual at the Gauss points of time
// elements [et0, et1) from precomputed Gauss-point fields (rows = time Gauss points of the chunk,
// G_s spatial Gauss points per row):
//   fields[f][row][s], f = u, u_tau, w, d_i u (i < d), d_ab u (aa first, then a < b)
//   coef[c][s],        c = cg_i (i < d), cm_ab (same order as the second derivatives)
// with  lap = sum_i cg_i d_i u + sum_ab cm_ab d_ab u  (cm_ab = (J^-1 J^-T)_ab, doubled for a != b;
// cg_i = -sum_ab (J^-1 J^-T)_ab sum_c H_abc (J^-1)_ic), so
//   res = C_m u_tau / T - D lap + c1 u (u - a)(u - 1) + c2 u w - f.
// |res| goes to its element's maximum (bit-pattern atomicMax of non-negative doubles: exact and order
// independent, as theta_elements), max|u| and max|u_tau| to the denominator maxima.
__global__ void mapped_residual_kernel(const double* __restrict__ fields, const double* __restrict__ coef,
                                       const double* __restrict__ src, double* __restrict__ emax,
                                       unsigned long long* __restrict__ maxes, int d, int rows, long long gs,
                                       int G1, int G2, int q, int qt, int et0, int E1, int E2, int E3,
                                       double D, double cmT, double c1, double a, double c2) {
  const int nd2 = d * (d + 1) / 2;
  const long long total = (long long)rows * gs;
  double umax = 0.0, utmax = 0.0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long sp = idx % gs;
    const int row = (int)(idx / gs);
    const double u = fields[idx], ut = fields[total + idx], w = fields[2 * total + idx];
    double lap = 0.0;
    for (int i = 0; i < d; ++i) lap = fma(coef[i * gs + sp], fields[(3 + i) * total + idx], lap);
    for (int k = 0; k < nd2; ++k) lap = fma(coef[(d + k) * gs + sp], fields[(3 + d + k) * total + idx], lap);
    double res = cmT * ut - D * lap + c1 * u * (u - a) * (u - 1.0) + c2 * u * w;
    if (src) res -= src[idx];
    const int g1 = (int)(sp % G1), g2 = (int)((sp / G1) % G2), g3 = (int)(sp / ((long long)G1 * G2));
    const long long el = (((long long)(et0 + row / qt) * E3 + g3 / q) * E2 + g2 / q) * E1 + g1 / q;
    atomicMax(reinterpret_cast<unsigned long long*>(emax) + el, dbits(fabs(res)));
    umax = fmax(umax, fabs(u));
    utmax = fmax(utmax, fabs(ut));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    utmax = fmax(utmax, __shfl_xor_sync(0xffffffffu, utmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&maxes[0], dbits(umax));
    atomicMax(&maxes[1], dbits(utmax));
  }
}

#define MI_TH_CASE(dv, pv, ptv, ...)                                 \
  case ((dv) * 8 + (pv)) * 8 + (ptv): {                              \
    constexpr int D_ = (dv), P_ = (pv), PT_ = (ptv);                 \
    __VA_ARGS__;                                                     \
  } break;
#define MI_TH_DISPATCH(d, p, pt, ...)                                                           \
  switch (((d) * 8 + (p)) * 8 + (pt)) {                                                         \
    MI_TH_CASE(1, 1, 1, __VA_ARGS__) MI_TH_CASE(1, 2, 2, __VA_ARGS__)                           \
    MI_TH_CASE(1, 3, 3, __VA_ARGS__) MI_TH_CASE(2, 1, 1, __VA_ARGS__)                           \
    MI_TH_CASE(2, 2, 2, __VA_ARGS__) MI_TH_CASE(2, 3, 3, __VA_ARGS__)                           \
    MI_TH_CASE(3, 1, 1, __VA_ARGS__) MI_TH_CASE(3, 2, 2, __VA_ARGS__)                           \
    MI_TH_CASE(3, 3, 3, __VA_ARGS__)                                                            \
    default:                                                                                    \
      ::mi::set_error("residual indicator: unsupported (d, p, p_t) (need p = p_t <= 3)");       \
      return MI_ERR_ARG;                                                                        \
  }

}  // namespace mi

using namespace mi;

extern "C" {

int mi_theta_setup(mi_ctx* c, const int* nel, const double* B0, const double* B1, const double* lengths,
                   const double* diffusion, double final_time, double C_m, double c1, double a, double c2) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr && nel && B0 && B1 && lengths && diffusion, MI_ERR_ARG, "NULL argument to mi_theta_setup");
  MI_REQUIRE(final_time > 0.0, MI_ERR_ARG, "final time must be positive");
  MI_REQUIRE(c->p == c->pt && c->p <= 3, MI_ERR_ARG, "residual indicator: need p = p_t <= 3");
  size_t tot = 0;
  for (int l = 0; l < 4; ++l) {
    const bool present = l == 3 || l < c->d;
    const int src = l == 3 ? c->d : l;
    c->th_nel[l] = present ? nel[src] : 1;
    c->th_off[l] = tot;
    tot += (size_t)c->th_nel[l] * ((l == 3 ? c->pt : c->p) + 1) * ((l == 3 ? c->pt : c->p) + 1);
  }
  std::vector<double> h0(tot, 0.0), h1(tot, 0.0);
  size_t s = 0;
  for (int l = 0; l < 4; ++l) {
    const bool present = l == 3 || l < c->d;
    const int pl = l == 3 ? c->pt : c->p;
    const size_t cnt = (size_t)c->th_nel[l] * (pl + 1) * (pl + 1);
    if (!present) continue;
    for (size_t i = 0; i < cnt; ++i) {
      h0[c->th_off[l] + i] = B0[s + i];
      h1[c->th_off[l] + i] = B1[s + i];
    }
    s += cnt;
  }
  int rc;
  if ((rc = dalloc(c->th_B0, tot)) || (rc = dalloc(c->th_B1, tot))) return rc;
  MI_CUDA(cudaMemcpy(c->th_B0.p, h0.data(), sizeof(double) * tot, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->th_B1.p, h1.data(), sizeof(double) * tot, cudaMemcpyHostToDevice));
  for (int l = 0; l < 3; ++l) c->th_il2[l] = l < c->d ? diffusion[l] / (lengths[l] * lengths[l]) : 0.0;
  c->th_cmT = C_m / final_time;
  c->th_c1 = c1;
  c->th_a = a;
  c->th_c2 = c2;
  c->th_ready = true;
  return MI_OK;
}

int mi_theta_elements(mi_ctx* c, const double* u, const double* w, const double* src, int et0, int et1,
                      double* emax, double* maxes) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->th_ready, MI_ERR_STATE, "mi_theta_setup must be called first");
  MI_REQUIRE(u && w && emax && maxes, MI_ERR_ARG, "NULL argument to mi_theta_elements");
  MI_REQUIRE(0 <= et0 && et0 <= et1 && et1 <= c->th_nel[3], MI_ERR_ARG, "time element range out of bounds");
  if (et0 == et1) return MI_OK;
  ThArgs r{};
  r.u = u;
  r.w = w;
  r.src = src;
  r.emax = emax;
  r.maxes = reinterpret_cast<unsigned long long*>(maxes);
  for (int l = 0; l < 4; ++l) {
    r.B0[l] = c->th_B0.p + c->th_off[l];
    r.B1[l] = c->th_B1.p + c->th_off[l];
    r.nel[l] = c->th_nel[l];
  }
  r.gs = 1;
  for (int l = 0; l < 3; ++l) {
    r.n[l] = c->n[l];
    r.G[l] = l < c->d ? c->th_nel[l] * (c->p + 1) : 1;
    r.gs *= r.G[l];
    r.il2[l] = c->th_il2[l];
  }
  r.ntc = c->nt;
  r.rowoff = -1;
  r.ns = c->ns;
  r.et0 = et0;
  r.et1 = et1;
  r.cmT = c->th_cmT;
  r.c1 = c->th_c1;
  r.a = c->th_a;
  r.c2 = c->th_c2;
  r.u0 = c->th_u0.n ? c->th_u0.p : nullptr;
  long long nb = 1;
  for (int l = 0; l < c->d; ++l) nb *= (c->th_nel[l] + 1) / 2;
  MI_TH_DISPATCH(c->d, c->p, c->pt, {
    using G = ThTile<D_, P_>;
    MI_DEV_FLAG(attr);
    if (!attr) {
      MI_CUDA(cudaFuncSetAttribute(theta_elements<D_, P_, PT_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)G::SMEM));
      attr = true;
    }
    theta_elements<D_, P_, PT_><<<(unsigned)nb, 256, G::SMEM, c->stream>>>(r);
    MI_CHECK_LAUNCH("theta_elements");
  });
  return MI_OK;
}

int mi_theta_set_lift(mi_ctx* c, const double* u0) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->th_ready, MI_ERR_STATE, "mi_theta_setup must be called first");
  if (u0 == nullptr) {
    mi::dfree(c->th_u0);
    return MI_OK;
  }
  int rc;
  if ((rc = mi::dalloc(c->th_u0, (size_t)c->ns))) return rc;
  MI_CUDA(cudaMemcpyAsync(c->th_u0.p, u0, sizeof(double) * c->ns, cudaMemcpyDeviceToDevice, c->stream));
  return MI_OK;
}

int mi_theta_mapped_elements(mi_ctx* c, const double* fields, const double* coef, const double* src, int et0,
                             int et1, const int* G, int q, int qt, const int* nel, double D, double cmT, double c1,
                             double a, double c2, double* emax, double* maxes) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && fields && coef && G && nel && emax && maxes, MI_ERR_ARG, "NULL argument to mi_theta_mapped_elements");
  MI_REQUIRE(0 <= et0 && et0 <= et1 && q >= 1 && qt >= 1, MI_ERR_ARG, "bad element range or rule");
  if (et0 == et1) return MI_OK;
  const int d = c->d;
  long long gs = 1;
  int Gl[3] = {1, 1, 1}, El[3] = {1, 1, 1};
  for (int l = 0; l < d; ++l) {
    Gl[l] = G[l];
    El[l] = nel[l];
    MI_REQUIRE(G[l] == nel[l] * q, MI_ERR_ARG, "Gauss grid does not match the element count");
    gs *= G[l];
  }
  const int rows = (et1 - et0) * qt;
  const long long total = (long long)rows * gs;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  mapped_residual_kernel<<<grid, 256, 0, c->stream>>>(fields, coef, src, emax,
                                                     reinterpret_cast<unsigned long long*>(maxes), d, rows, gs,
                                                     Gl[0], Gl[1], q, qt, et0, El[0], El[1], El[2], D, cmT, c1, a, c2);
  MI_CHECK_LAUNCH("mapped_residual_kernel");
  return MI_OK;
}

int mi_window_max(mi_ctx* c, const double* in, double* out, long long outer, int n_in, int n_out, long long inner,
                  const int* w0, const int* w1) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && in && out && w0 && w1 && in != out, MI_ERR_ARG, "bad arguments to mi_window_max");
  MI_REQUIRE(outer >= 0 && n_in > 0 && n_out >= 0 && inner >= 0, MI_ERR_ARG, "bad shape in mi_window_max");
  for (int i = 0; i < n_out; ++i)
    MI_REQUIRE(0 <= w0[i] && w0[i] < w1[i] && w1[i] <= n_in, MI_ERR_ARG, "window out of range");
  if (c->th_nwin < 2 * n_out) {
    if (c->th_win) cudaFree(c->th_win);
    c->th_win = nullptr;
    MI_CUDA(cudaMalloc(&c->th_win, sizeof(int) * 2 * n_out));
    c->th_nwin = 2 * n_out;
  }
  MI_CUDA(cudaMemcpyAsync(c->th_win, w0, sizeof(int) * n_out, cudaMemcpyHostToDevice, c->stream));
  MI_CUDA(cudaMemcpyAsync(c->th_win + n_out, w1, sizeof(int) * n_out, cudaMemcpyHostToDevice, c->stream));
  const long long total = outer * n_out * inner;
  if (total == 0) return MI_OK;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  window_max_kernel<<<grid, 256, 0, c->stream>>>(in, out, outer, n_in, n_out, inner, c->th_win, c->th_win + n_out);
  MI_CHECK_LAUNCH("window_max_kernel");
  // the window tables are consumed by this launch before the next call can overwrite them
  MI_CUDA(cudaStreamSynchronize(c->stream));
  return MI_OK;
}

int mi_theta_ratio(mi_ctx* c, const double* numer, double* theta, long long n, double denom) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && numer && theta && n >= 0, MI_ERR_ARG, "bad arguments to mi_theta_ratio");
  MI_REQUIRE(denom > 0.0, MI_ERR_ARG, "denominator must be positive");
  if (n == 0) return MI_OK;
  const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 32);
  theta_ratio_kernel<<<grid, 256, 0, c->stream>>>(numer, theta, n, denom);
  MI_CHECK_LAUNCH("theta_ratio_kernel");
  return MI_OK;
}

}  // extern "C"
