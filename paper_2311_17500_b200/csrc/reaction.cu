// Reaction correction y += M_R x with the Rogers-McCulloch linearisation
// (reference reaction_mass, assembly.py:287-347):
//
//   M_R[i, j] = int int C_r B_i B_j,   C_r = c1 (u - a)(u - 1) + c2 w,
//
// u, w = the frozen iterate, evaluated at q = p+1 Gauss points per element
// in every direction (space and time; assembly.py:313-318 -- the rule is
// parity-critical).  Matrix-free: a block owns a tile
// of p elements per direction (incl. time), loads the local coefficients of
// u, w, x, interpolates them to the tile's Gauss grid one time point at a
// time (sum factorisation: t, then x, y, z), evaluates the ionic
// linearisation pointwise, and projects back (z, y, x, t).  Tiles are
// processed in 2^(d+1) colour classes so concurrently running blocks never
// touch the same output DoF: no atomics, bitwise deterministic.
#include "common.cuh"
#include "dispatch.cuh"
#include "ptx.cuh"

#include <type_traits>

#ifndef RX_UNROLL
#define RX_UNROLL 0   // unroll the slice loop by p_t+1 (no window rotation; more registers / code)
#endif

namespace mi {

struct RxArgs {
  const double* u;
  const double* w;
  const double* x;
  double* y;
  // per direction l = 0 (x), 1 (y), 2 (z), 3 (t): basis values at Gauss points
  // B_l[(e * q + g) * (p_l + 1) + a] of function e + a, weights W_l[e * q + g]
  const double* B[4];
  const double* Wq[4];
  int nel[4];          // elements per direction (1 for absent dims)
  int n[3];            // spatial functions per direction
  int color[3];        // colour class of this launch (element index mod (p+1))
  int ncol[3];         // elements of this colour per direction
  int ntc;             // constrained time functions (rows of this context)
  int rowoff;          // row of full time function ft is ft + rowoff (-1 unsharded)
  long long ns;
  double c1, a, c2;
#ifdef RX_ABL_CBT
  double btc[32];
#endif
};

// One warp per spatial element (colour class: elements p+1 apart never
// share a basis function), sweeping all time elements with a sliding
// window of p_t+1 coefficient slices and p_t+1 output slices in shared
// memory.  Sum factorisation per time Gauss point as LINE operations: a lane
// takes one line of LD coefficients along a direction and produces its Q
// Gauss values with the element's 1D basis matrix held in registers
// (LD loads -> LD*Q FMAs -> Q stores), then C_r(u, w) x W pointwise and the
// transposed line operations back.  q = p+1 is the reference rule.
template <int D, int P, int PT>
__global__ void __launch_bounds__(128, 8) reaction_warp(RxArgs r) {
  constexpr int LD = P + 1, Q = P + 1;
  constexpr int L1 = LD, L2 = D >= 2 ? LD : 1, L3 = D >= 3 ? LD : 1;
  constexpr int LS = L1 * L2 * L3;                   // local spatial functions (= quad points)
  constexpr int PW = PT + 1;                         // time window
  constexpr int QT = PT + 1;                         // time Gauss points
  constexpr int NL = LS / LD;                        // lines per field along a direction
  constexpr int WARP_SM = 3 * PW * LS + PW * LS + 2 * 3 * LS + 3 * Q * LD;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* base = sm + wib * WARP_SM;
  double* win = base;                                // [3][PW][LS]
  double* outw = win + 3 * PW * LS;                  // [PW][LS]
  double* ta = outw + PW * LS;                       // [3][LS]
  double* tb = ta + 3 * LS;                          // [3][LS]
  double* bsm = tb + 3 * LS;                         // [3 dirs][Q][LD] basis of this element

  long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long long nw = (long long)r.ncol[0] * r.ncol[1] * r.ncol[2];
  if (wid >= nw) return;
  int e[3];
  {
    long long t = wid;
    for (int l = 0; l < 3; ++l) {
      const int m = (int)(t % r.ncol[l]);
      t /= r.ncol[l];
      e[l] = (l < D) ? m * LD + r.color[l] : 0;
    }
  }
  // the element's 1D basis matrices B_l[g][j] (shared by the warp's lanes: broadcast loads)
  for (int i = lane; i < 3 * Q * LD; i += 32) {
    const int l = i / (Q * LD), gj = i % (Q * LD);
    bsm[i] = l < D ? __ldg(r.B[l] + (long long)e[l] * Q * LD + gj) : 0.0;
  }
  __syncwarp();
  const double* bx = bsm;
  const double* by = bsm + Q * LD;
  const double* bz = bsm + 2 * Q * LD;
  double wsp[(LS + 31) / 32];
#pragma unroll
  for (int k = 0; k < (LS + 31) / 32; ++k) {
    const int s = lane + 32 * k;
    double wv = 0.0;
    if (s < LS) {
      const int g1 = s % L1, g2 = (s / L1) % L2, g3 = s / (L1 * L2);
      wv = r.Wq[0][e[0] * Q + g1];
      if (D >= 2) wv *= r.Wq[1][e[1] * Q + g2];
      if (D >= 3) wv *= r.Wq[2][e[2] * Q + g3];
    }
    wsp[k] = wv;
  }
  auto gidx = [&](int s) -> long long {
    const int j1 = s % L1, j2 = (s / L1) % L2, j3 = s / (L1 * L2);
    return ((long long)(e[2] + j3) * r.n[1] + (e[1] + j2)) * r.n[0] + (e[0] + j1);
  };
  auto load_slice = [&](int ft) {                     // full-basis time function ft
    const int ct = ft + r.rowoff, slot = ft % PW;
    const bool v = ct >= 0 && ct < r.ntc;
    for (int s = lane; s < LS; s += 32) {
      const long long gi = (long long)ct * r.ns + gidx(s);
      win[(0 * PW + slot) * LS + s] = v ? r.u[gi] : 0.0;
      win[(1 * PW + slot) * LS + s] = v ? r.w[gi] : 0.0;
      win[(2 * PW + slot) * LS + s] = v ? r.x[gi] : 0.0;
      outw[slot * LS + s] = 0.0;
    }
  };
  auto flush_slice = [&](int ft) {
    const int ct = ft + r.rowoff, slot = ft % PW;
    if (ct >= 0 && ct < r.ntc)
      for (int s = lane; s < LS; s += 32) r.y[(long long)ct * r.ns + gidx(s)] += outw[slot * LS + s];
  };
  // line op along a direction with stride `st` (1, L1, L1*L2): in[line base + j*st] -> out[.. + g*st]
  auto line_fwd = [&](const double* in, double* out, const double* bm, int lb, int st) {
    double v[LD];
#pragma unroll
    for (int j = 0; j < LD; ++j) v[j] = in[lb + j * st];
#pragma unroll
    for (int g = 0; g < Q; ++g) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < LD; ++j) acc = fma(bm[g * LD + j], v[j], acc);
      out[lb + g * st] = acc;
    }
  };
  auto line_bwd = [&](const double* in, double* out, const double* bm, int lb, int st) {
    double v[Q];
#pragma unroll
    for (int g = 0; g < Q; ++g) v[g] = in[lb + g * st];
#pragma unroll
    for (int j = 0; j < LD; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int g = 0; g < Q; ++g) acc = fma(bm[g * LD + j], v[g], acc);
      out[lb + j * st] = acc;
    }
  };
  // line base index of line `li` (0..NL) along direction dir
  auto line_base = [&](int dir, int li) -> int {
    if (dir == 0) return li * L1;                                // (j2, j3) -> rows of L1
    if (dir == 1) return (li / L1) * (L1 * L2) + (li % L1);      // (g1, j3)
    return li;                                                   // (g1, g2)
  };

  for (int ft = 0; ft < PT; ++ft) load_slice(ft);
  for (int et = 0; et < r.nel[3]; ++et) {
    load_slice(et + PT);
    __syncwarp();
    for (int g = 0; g < QT; ++g) {
      const double* bt = r.B[3] + ((long long)et * QT + g) * (PT + 1);
      const double wt = r.Wq[3][et * QT + g];
      double btv[PT + 1];
#pragma unroll
      for (int aa = 0; aa <= PT; ++aa) btv[aa] = __ldg(bt + aa);
      // time interpolation -> ta[3][LS]
      for (int i = lane; i < 3 * LS; i += 32) {
        const int fld = i / LS, s = i % LS;
        double v = 0.0;
#pragma unroll
        for (int aa = 0; aa <= PT; ++aa) v = fma(btv[aa], win[(fld * PW + (et + aa) % PW) * LS + s], v);
        ta[i] = v;
      }
      __syncwarp();
      // x, y, z interpolation as line ops: ta -> tb -> ta -> tb
      for (int i = lane; i < 3 * NL; i += 32) line_fwd(ta + (i / NL) * LS, tb + (i / NL) * LS, bx, line_base(0, i % NL), 1);
      __syncwarp();
      if (D >= 2) {
        for (int i = lane; i < 3 * NL; i += 32) line_fwd(tb + (i / NL) * LS, ta + (i / NL) * LS, by, line_base(1, i % NL), L1);
      } else {
        for (int i = lane; i < 3 * LS; i += 32) ta[i] = tb[i];
      }
      __syncwarp();
      if (D >= 3) {
        for (int i = lane; i < 3 * NL; i += 32) line_fwd(ta + (i / NL) * LS, tb + (i / NL) * LS, bz, line_base(2, i % NL), L1 * L2);
      } else {
        for (int i = lane; i < 3 * LS; i += 32) tb[i] = ta[i];
      }
      __syncwarp();
      // pointwise: C_r(u, w) * x * weights -> ta[0..LS)
#pragma unroll
      for (int k = 0; k < (LS + 31) / 32; ++k) {
        const int s = lane + 32 * k;
        if (s < LS) {
          const double uu = tb[s], ww = tb[LS + s], xx = tb[2 * LS + s];
          const double cr = r.c1 * (uu - r.a) * (uu - 1.0) + r.c2 * ww;
          ta[s] = cr * xx * (wt * wsp[k]);
        }
      }
      __syncwarp();
      // projections z, y, x: ta -> tb -> ta -> tb
      if (D >= 3) {
        for (int i = lane; i < NL; i += 32) line_bwd(ta, tb, bz, line_base(2, i), L1 * L2);
      } else {
        for (int i = lane; i < LS; i += 32) tb[i] = ta[i];
      }
      __syncwarp();
      if (D >= 2) {
        for (int i = lane; i < NL; i += 32) line_bwd(tb, ta, by, line_base(1, i), L1);
      } else {
        for (int i = lane; i < LS; i += 32) ta[i] = tb[i];
      }
      __syncwarp();
      for (int i = lane; i < NL; i += 32) line_bwd(ta, tb, bx, line_base(0, i), 1);
      __syncwarp();
      // time projection into the output window
      for (int s = lane; s < LS; s += 32) {
        const double v = tb[s];
#pragma unroll
        for (int aa = 0; aa <= PT; ++aa) outw[((et + aa) % PW) * LS + s] += btv[aa] * v;
      }
      __syncwarp();
    }
    flush_slice(et);
    __syncwarp();
  }
  for (int ft = r.nel[3]; ft < r.nel[3] + PT; ++ft) flush_slice(ft);
}

// R3: one block per tile of E x E x E spatial elements (E = 2), sweeping all
// time elements with sliding windows.  Stages per time Gauss point run over
// the whole tile (x, y, z interpolation of u, w, x; pointwise C_r * x * W;
// z, y, x projection; time projection), so neighbouring elements share the
// interpolation work.  Tiles are coloured by (tile index mod RC) per
// direction, RC = ceil((E + p) / E): same-colour tiles never share a basis
// function.  Deterministic, no atomics.
template <int D, int P, int PT>
struct RxTile {
  static constexpr int E = 2;
  static constexpr int LD = P + 1, Q = P + 1;
  static constexpr int E1 = E, E2 = D >= 2 ? E : 1, E3 = D >= 3 ? E : 1;
  static constexpr int L1 = E1 + P, L2 = D >= 2 ? E2 + P : 1, L3 = D >= 3 ? E3 + P : 1;   // local functions
  static constexpr int Q1 = E1 * Q, Q2 = D >= 2 ? E2 * Q : 1, Q3 = D >= 3 ? E3 * Q : 1;   // Gauss points
  static constexpr int LS = L1 * L2 * L3, QS = Q1 * Q2 * Q3;
  static constexpr int PW = PT + 1, QT = PT + 1;
  static constexpr int RC = (E + P + E - 1) / E;          // colours per direction
  static constexpr int S1 = Q1 * L2 * L3, S2 = Q1 * Q2 * L3;   // intermediate sizes
  static constexpr int BIG = QS > S2 ? (QS > S1 ? QS : S1) : (S2 > S1 ? S2 : S1);
  static constexpr int THREADS = 256;
  // smem: coefficient window [3][PW][LS], output window [PW][LS], f0 [3][LS],
  // two work buffers [3][BIG], basis tables [3 dirs][E][Q][LD], weights [3][E*Q]
  static constexpr size_t SMEM = (size_t)(3 * PW * LS + PW * LS + 3 * LS + 6 * BIG + 3 * E * Q * LD + 3 * E * Q) * 8;
};

template <int D, int P, int PT>
__global__ void __launch_bounds__(256) reaction_tile3(RxArgs r) {
  using G = RxTile<D, P, PT>;
  constexpr int E = G::E, LD = G::LD, Q = G::Q, PW = G::PW, QT = G::QT;
  constexpr int L1 = G::L1, L2 = G::L2, L3 = G::L3, Q1 = G::Q1, Q2 = G::Q2, Q3 = G::Q3;
  constexpr int LS = G::LS, QS = G::QS, BIG = G::BIG;
  extern __shared__ double sm[];
  double* win = sm;                               // [3][PW][LS]
  double* outw = win + 3 * PW * LS;               // [PW][LS]
  double* f0 = outw + PW * LS;                    // [3][LS]
  double* s1 = f0 + 3 * LS;                       // [3][BIG]
  double* s2 = s1 + 3 * BIG;                      // [3][BIG]
  double* bt = s2 + 3 * BIG;                      // [3][E][Q][LD]
  double* wq = bt + 3 * E * Q * LD;               // [3][E*Q]
  const int tid = threadIdx.x;
  // tile of this block (colour class)
  int b = blockIdx.x, k[3], ne[3];
  for (int l = 0; l < 3; ++l) {
    const int m = b % r.ncol[l];
    b /= r.ncol[l];
    k[l] = l < D ? (m * G::RC + r.color[l]) * E : 0;     // first element of the tile
    ne[l] = l < D ? min(E, r.nel[l] - k[l]) : 1;
  }
  // basis tables / weights of the tile's elements (zero for elements beyond the mesh)
  for (int i = tid; i < 3 * E * Q * LD; i += G::THREADS) {
    const int l = i / (E * Q * LD), rem = i % (E * Q * LD), le = rem / (Q * LD);
    const bool ok = l < D && le < ne[l];
    bt[i] = ok ? __ldg(r.B[l] + (long long)(k[l] + le) * Q * LD + rem % (Q * LD)) : (l >= D && le == 0 && rem % (Q * LD) == 0 ? 1.0 : 0.0);
  }
  for (int i = tid; i < 3 * E * Q; i += G::THREADS) {
    const int l = i / (E * Q), rem = i % (E * Q), le = rem / Q;
    wq[i] = (l < D && le < ne[l]) ? __ldg(r.Wq[l] + (long long)(k[l] + le) * Q + rem % Q) : (l >= D ? 1.0 : 0.0);
  }
  auto gfun = [&](int s, int& g1, int& g2, int& g3) {
    const int j1 = s % L1, j2 = (s / L1) % L2, j3 = s / (L1 * L2);
    g1 = k[0] + j1;
    g2 = k[1] + j2;
    g3 = k[2] + j3;
  };
  auto load_slice = [&](int ft) {
    const int ct = ft + r.rowoff, slot = ft % PW;
    const bool vt = ct >= 0 && ct < r.ntc;
    for (int s = tid; s < LS; s += G::THREADS) {
      int g1, g2, g3;
      gfun(s, g1, g2, g3);
      const bool v = vt && g1 < r.n[0] && g2 < r.n[1] && g3 < r.n[2];
      const long long gi = (long long)ct * r.ns + ((long long)g3 * r.n[1] + g2) * r.n[0] + g1;
      win[(0 * PW + slot) * LS + s] = v ? r.u[gi] : 0.0;
      win[(1 * PW + slot) * LS + s] = v ? r.w[gi] : 0.0;
      win[(2 * PW + slot) * LS + s] = v ? r.x[gi] : 0.0;
      outw[slot * LS + s] = 0.0;
    }
  };
  auto flush_slice = [&](int ft) {
    const int ct = ft + r.rowoff, slot = ft % PW;
    if (ct < 0 || ct >= r.ntc) return;
    for (int s = tid; s < LS; s += G::THREADS) {
      int g1, g2, g3;
      gfun(s, g1, g2, g3);
      if (g1 < r.n[0] && g2 < r.n[1] && g3 < r.n[2])
        r.y[(long long)ct * r.ns + ((long long)g3 * r.n[1] + g2) * r.n[0] + g1] += outw[slot * LS + s];
    }
  };
  const double* bx = bt;
  const double* by = bt + E * Q * LD;
  const double* bz = bt + 2 * E * Q * LD;
  for (int ft = 0; ft < PT; ++ft) load_slice(ft);
  for (int et = 0; et < r.nel[3]; ++et) {
    load_slice(et + PT);
    __syncthreads();
    for (int g = 0; g < QT; ++g) {
      const double* btt = r.B[3] + ((long long)et * QT + g) * (PT + 1);
      const double wt = __ldg(r.Wq[3] + et * QT + g);
      double btv[PT + 1];
#pragma unroll
      for (int aa = 0; aa <= PT; ++aa) btv[aa] = __ldg(btt + aa);
      // time interpolation -> f0[3][LS]
      for (int i = tid; i < 3 * LS; i += G::THREADS) {
        const int fld = i / LS, s = i % LS;
        double v = 0.0;
#pragma unroll
        for (int aa = 0; aa <= PT; ++aa) v = fma(btv[aa], win[(fld * PW + (et + aa) % PW) * LS + s], v);
        f0[i] = v;
      }
      __syncthreads();
      // x: f0 [3][L3][L2][L1] -> s1 [3][L3][L2][Q1]
      for (int i = tid; i < 3 * L3 * L2 * Q1; i += G::THREADS) {
        const int q1 = i % Q1, rest = i / Q1;       // rest = (fld, j3, j2)
        const int le = q1 / Q, gq = q1 % Q;
        const double* src = f0 + rest * L1 + le;
        const double* bb = bx + (le * Q + gq) * LD;
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < LD; ++j) v = fma(bb[j], src[j], v);
        s1[(rest / (L3 * L2)) * BIG + (rest % (L3 * L2)) * Q1 + q1] = v;
      }
      __syncthreads();
      // y: s1 [3][L3][L2][Q1] -> s2 [3][L3][Q2][Q1]
      if (D >= 2) {
        for (int i = tid; i < 3 * L3 * Q2 * Q1; i += G::THREADS) {
          const int q1 = i % Q1, q2 = (i / Q1) % Q2, j3 = (i / (Q1 * Q2)) % L3, fld = i / (Q1 * Q2 * L3);
          const int le = q2 / Q, gq = q2 % Q;
          const double* src = s1 + fld * BIG + (j3 * L2 + le) * Q1 + q1;
          const double* bb = by + (le * Q + gq) * LD;
          double v = 0.0;
#pragma unroll
          for (int j = 0; j < LD; ++j) v = fma(bb[j], src[j * Q1], v);
          s2[fld * BIG + (j3 * Q2 + q2) * Q1 + q1] = v;
        }
      } else {
        for (int i = tid; i < 3 * BIG; i += G::THREADS) s2[i] = s1[i];
      }
      __syncthreads();
      // z: s2 [3][L3][Q2][Q1] -> s1 [3][Q3][Q2][Q1]
      if (D >= 3) {
        for (int i = tid; i < 3 * QS; i += G::THREADS) {
          const int q12 = i % (Q1 * Q2), q3 = (i / (Q1 * Q2)) % Q3, fld = i / QS;
          const int le = q3 / Q, gq = q3 % Q;
          const double* src = s2 + fld * BIG + le * Q2 * Q1 + q12;
          const double* bb = bz + (le * Q + gq) * LD;
          double v = 0.0;
#pragma unroll
          for (int j = 0; j < LD; ++j) v = fma(bb[j], src[j * Q1 * Q2], v);
          s1[fld * BIG + q3 * Q1 * Q2 + q12] = v;
        }
      } else {
        for (int i = tid; i < 3 * BIG; i += G::THREADS) s1[i] = s2[i];
      }
      __syncthreads();
      // pointwise: C_r(u, w) * x * weights -> s2[0..QS)
      for (int i = tid; i < QS; i += G::THREADS) {
        const int q1 = i % Q1, q2 = (i / Q1) % Q2, q3 = i / (Q1 * Q2);
        const double uu = s1[i], ww = s1[BIG + i], xx = s1[2 * BIG + i];
        const double cr = r.c1 * (uu - r.a) * (uu - 1.0) + r.c2 * ww;
        s2[i] = cr * xx * (wt * wq[q1] * wq[E * Q + q2] * wq[2 * E * Q + q3]);
      }
      __syncthreads();
      // z projection: s2 [Q3][Q2][Q1] -> s1 [L3][Q2][Q1]
      if (D >= 3) {
        for (int i = tid; i < L3 * Q2 * Q1; i += G::THREADS) {
          const int q12 = i % (Q1 * Q2), j3 = i / (Q1 * Q2);
          double v = 0.0;
          for (int le = 0; le < E; ++le) {
            const int aa = j3 - le;
            if (aa < 0 || aa > P) continue;
#pragma unroll
            for (int gq = 0; gq < Q; ++gq) v = fma(bz[(le * Q + gq) * LD + aa], s2[(le * Q + gq) * Q1 * Q2 + q12], v);
          }
          s1[i] = v;
        }
      } else {
        for (int i = tid; i < QS; i += G::THREADS) s1[i] = s2[i];
      }
      __syncthreads();
      // y projection: s1 [L3][Q2][Q1] -> s2 [L3][L2][Q1]
      if (D >= 2) {
        for (int i = tid; i < L3 * L2 * Q1; i += G::THREADS) {
          const int q1 = i % Q1, j2 = (i / Q1) % L2, j3 = i / (Q1 * L2);
          double v = 0.0;
          for (int le = 0; le < E; ++le) {
            const int aa = j2 - le;
            if (aa < 0 || aa > P) continue;
#pragma unroll
            for (int gq = 0; gq < Q; ++gq) v = fma(by[(le * Q + gq) * LD + aa], s1[(j3 * Q2 + le * Q + gq) * Q1 + q1], v);
          }
          s2[i] = v;
        }
      } else {
        for (int i = tid; i < L3 * L2 * Q1; i += G::THREADS) s2[i] = s1[i];
      }
      __syncthreads();
      // x projection + time projection into the output window
      for (int i = tid; i < LS; i += G::THREADS) {
        const int j1 = i % L1, rest = i / L1;
        double v = 0.0;
        for (int le = 0; le < E; ++le) {
          const int aa = j1 - le;
          if (aa < 0 || aa > P) continue;
#pragma unroll
          for (int gq = 0; gq < Q; ++gq) v = fma(bx[(le * Q + gq) * LD + aa], s2[rest * Q1 + le * Q + gq], v);
        }
#pragma unroll
        for (int aa = 0; aa <= PT; ++aa) outw[((et + aa) % PW) * LS + i] += btv[aa] * v;
      }
      __syncthreads();
    }
    flush_slice(et);
    __syncthreads();
  }
  for (int ft = r.nel[3]; ft < r.nel[3] + PT; ++ft) flush_slice(ft);
}

// R4: the R3 tile sweep with every sum-factorisation stage on the FP64
// tensor cores.  Per direction the tile's 2 elements give a dense
// (L = 2 + p functions) x (Q = 2 (p+1) Gauss points) basis block; a stage is
// C[lines, Q] = A[lines, L] B_l[L, Q] (interpolation) or C[lines, L] =
// A[lines, Q] B_l^T (projection), with M = 8 lines, N = Q or L <= 8, K = L or
// Q (<= 8, 1-2 k-steps).  The B fragments of all six stage matrices live in
// registers for the whole sweep; each DMMA needs one shared load.
#ifndef RX4_GB
#define RX4_GB 1   // time Gauss points per pass (2 halves the barriers but costs occupancy: 653 vs 615 ms at cfg4)
#endif
template <int D, int P>
struct RxT4 {
  static constexpr int E = 2, LD = P + 1, QE = P + 1;
  static constexpr int L = E + P, Q = E * QE;                    // per present direction
  static constexpr int L1 = L, L2 = D >= 2 ? L : 1, L3 = D >= 3 ? L : 1;
  static constexpr int Q1 = Q, Q2 = D >= 2 ? Q : 1, Q3 = D >= 3 ? Q : 1;
  static constexpr int LS = L1 * L2 * L3, QS = Q1 * Q2 * Q3;
  static constexpr int KI = (L + 3) / 4, KP = (Q + 3) / 4;      // k-steps interp / proj
  static constexpr int RC = (E + P + E - 1) / E;
};

template <int D, int P, int PT>
__global__ void __launch_bounds__(256) reaction_tile4(RxArgs r) {
  using G = RxT4<D, P>;
  constexpr int E = G::E, LD = G::LD, QE = G::QE, L = G::L, Q = G::Q;
  constexpr int L1 = G::L1, L2 = G::L2, L3 = G::L3, Q1 = G::Q1, Q2 = G::Q2, Q3 = G::Q3;
  constexpr int LS = G::LS, QS = G::QS, KI = G::KI, KP = G::KP;
  constexpr int PW = PT + 1, QT = PT + 1;
  constexpr int GB = RX4_GB;                        // time Gauss points per pass
  constexpr int F = 3 * GB;                       // (g, field) pairs per pass
  // stage buffer sizes
  constexpr int SX = F * L3 * L2 * Q1, SY = F * L3 * Q2 * Q1, SZ = F * QS;
  constexpr int BUF = (SX > SY ? (SX > SZ ? SX : SZ) : (SY > SZ ? SY : SZ));
  extern __shared__ double sm[];
  double* win = sm;                               // [3][PW][LS]
  double* outw = win + 3 * PW * LS;               // [PW][LS]
  double* f0 = outw + PW * LS;                    // [GB][3][LS]
  double* sa = f0 + F * LS;                       // [BUF]
  double* sb = sa + BUF;                          // [BUF]
  double* wq = sb + BUF;                          // [3][Q]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;        // fragment row / col
  int b = blockIdx.x, k[3], ne[3];
  for (int l = 0; l < 3; ++l) {
    const int m = b % r.ncol[l];
    b /= r.ncol[l];
    k[l] = l < D ? (m * G::RC + r.color[l]) * E : 0;
    ne[l] = l < D ? min(E, r.nel[l] - k[l]) : 1;
  }
  // basis value of local function j at tile Gauss point q (direction l)
  auto basis = [&](int l, int j, int q) -> double {
    if (q >= Q || j >= L) return 0.0;
    const int le = q / QE, gq = q % QE, aa = j - le;
    if (le >= ne[l] || aa < 0 || aa > P) return 0.0;
    return __ldg(r.B[l] + ((long long)(k[l] + le) * QE + gq) * LD + aa);
  };
  // B fragments: interpolation (K = j, N = q) and projection (K = q, N = j), per direction
  double bI[3][2], bP[3][2];
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const bool pres = l < D;
      bI[l][ks] = pres ? basis(l, 4 * ks + fk, fr) : 0.0;
      bP[l][ks] = pres ? basis(l, fr, 4 * ks + fk) : 0.0;
    }
  for (int i = tid; i < 3 * Q; i += 256) {
    const int l = i / Q, q = i % Q, le = q / QE;
    wq[i] = (l < D) ? ((le < ne[l]) ? __ldg(r.Wq[l] + (long long)(k[l] + le) * QE + q % QE) : 0.0) : (q == 0 ? 1.0 : 0.0);
  }
  auto gidx = [&](int s, bool& ok) -> long long {
    const int j1 = s % L1, j2 = (s / L1) % L2, j3 = s / (L1 * L2);
    const int g1 = k[0] + j1, g2 = k[1] + j2, g3 = k[2] + j3;
    ok = g1 < r.n[0] && g2 < r.n[1] && g3 < r.n[2];
    return ((long long)g3 * r.n[1] + g2) * r.n[0] + g1;
  };
  auto load_slice = [&](int ft) {
    const int ct = ft + r.rowoff, slot = ft % PW;
    const bool vt = ct >= 0 && ct < r.ntc;
    for (int s = tid; s < LS; s += 256) {
      bool ok;
      const long long gs = gidx(s, ok);
      const bool v = vt && ok;
      const long long gi = (long long)ct * r.ns + gs;
      win[(0 * PW + slot) * LS + s] = v ? r.u[gi] : 0.0;
      win[(1 * PW + slot) * LS + s] = v ? r.w[gi] : 0.0;
      win[(2 * PW + slot) * LS + s] = v ? r.x[gi] : 0.0;
      outw[slot * LS + s] = 0.0;
    }
  };
  auto flush_slice = [&](int ft) {
    const int ct = ft + r.rowoff, slot = ft % PW;
    if (ct < 0 || ct >= r.ntc) return;
    for (int s = tid; s < LS; s += 256) {
      bool ok;
      const long long gs = gidx(s, ok);
      if (ok) r.y[(long long)ct * r.ns + gs] += outw[slot * LS + s];
    }
  };
  const int nL13 = L3 * L2, lines_x = F * nL13, lines_y = F * L3 * Q1, lines_z = F * Q2 * Q1;
  for (int ft = 0; ft < PT; ++ft) load_slice(ft);
  for (int et = 0; et < r.nel[3]; ++et) {
    load_slice(et + PT);
    __syncthreads();
    static_assert(QT % GB == 0, "GB must divide the time Gauss count");
    for (int g0 = 0; g0 < QT; g0 += GB) {
      // time interpolation of GB Gauss points -> f0[(gb, fld)][LS] (layout [gb][fld][j3][j2][j1])
      for (int i = tid; i < F * LS; i += 256) {
        const int gf = i / LS, s = i % LS, gb = gf / 3, fld = gf % 3;
        const double* btt = r.B[3] + ((long long)et * QT + g0 + gb) * (PT + 1);
        double v = 0.0;
#pragma unroll
        for (int aa = 0; aa <= PT; ++aa) v = fma(__ldg(btt + aa), win[(fld * PW + (et + aa) % PW) * LS + s], v);
        f0[i] = v;
      }
      __syncthreads();
      // x interpolation: lines (fld, j3, j2), K = j1, N = q1 -> sa [fld][j3][j2][q1]
      for (int mt = warp; mt < (lines_x + 7) / 8; mt += 8) {
        const int line = mt * 8 + fr;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KI; ++ks) {
          const int j = 4 * ks + fk;
          const double av = (line < lines_x && j < L1) ? f0[line * L1 + j] : 0.0;
          dmma(c0, c1, av, bI[0][ks]);
        }
        const int lo = mt * 8 + fr, n0 = 2 * fk;
        if (lo < lines_x) {
          if (n0 < Q1) sa[lo * Q1 + n0] = c0;
          if (n0 + 1 < Q1) sa[lo * Q1 + n0 + 1] = c1;
        }
      }
      __syncthreads();
      // y interpolation: lines (fld, j3, q1), K = j2, N = q2 -> sb [fld][j3][q2][q1]
      if (D >= 2) {
        for (int mt = warp; mt < (lines_y + 7) / 8; mt += 8) {
          const int line = mt * 8 + fr;
          const int q1 = line % Q1, fj3 = line / Q1;
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KI; ++ks) {
            const int j = 4 * ks + fk;
            const double av = (line < lines_y && j < L2) ? sa[(fj3 * L2 + j) * Q1 + q1] : 0.0;
            dmma(c0, c1, av, bI[1][ks]);
          }
          const int n0 = 2 * fk;
          if (line < lines_y) {
            if (n0 < Q2) sb[(fj3 * Q2 + n0) * Q1 + q1] = c0;
            if (n0 + 1 < Q2) sb[(fj3 * Q2 + n0 + 1) * Q1 + q1] = c1;
          }
        }
        // note: stores are per (line, n) with line = this lane's row
      } else {
        for (int i = tid; i < SX; i += 256) sb[i] = sa[i];
      }
      __syncthreads();
      // z interpolation: lines (fld, q2, q1), K = j3, N = q3 -> sa [fld][q3][q2][q1]
      if (D >= 3) {
        for (int mt = warp; mt < (lines_z + 7) / 8; mt += 8) {
          const int line = mt * 8 + fr;
          const int q12 = line % (Q1 * Q2), fld = line / (Q1 * Q2);
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KI; ++ks) {
            const int j = 4 * ks + fk;
            const double av = (line < lines_z && j < L3) ? sb[(fld * L3 + j) * Q1 * Q2 + q12] : 0.0;
            dmma(c0, c1, av, bI[2][ks]);
          }
          const int n0 = 2 * fk;
          if (line < lines_z) {
            if (n0 < Q3) sa[(fld * Q3 + n0) * Q1 * Q2 + q12] = c0;
            if (n0 + 1 < Q3) sa[(fld * Q3 + n0 + 1) * Q1 * Q2 + q12] = c1;
          }
        }
      } else {
        for (int i = tid; i < SY; i += 256) sa[i] = sb[i];
      }
      __syncthreads();
      // pointwise: C_r(u, w) * x * weights -> sb[gb][QS]
      for (int i = tid; i < GB * QS; i += 256) {
        const int gb = i / QS, qi = i % QS;
        const int q1 = qi % Q1, q2 = (qi / Q1) % Q2, q3 = qi / (Q1 * Q2);
        const double wt = __ldg(r.Wq[3] + et * QT + g0 + gb);
        const double* src = sa + gb * 3 * QS + qi;
        const double uu = src[0], ww = src[QS], xx = src[2 * QS];
        const double cr = r.c1 * (uu - r.a) * (uu - 1.0) + r.c2 * ww;
        sb[i] = cr * xx * (wt * wq[q1] * wq[Q + q2] * wq[2 * Q + q3]);
      }
      __syncthreads();
      // z projection: lines (gb, q2, q1), K = q3, N = j3 -> sa [gb][j3][q2][q1]
      if (D >= 3) {
        constexpr int NL = GB * Q1 * Q2;
        for (int mt = warp; mt < (NL + 7) / 8; mt += 8) {
          const int line = mt * 8 + fr;
          const int gb = line / (Q1 * Q2), q12 = line % (Q1 * Q2);
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KP; ++ks) {
            const int q = 4 * ks + fk;
            const double av = (line < NL && q < Q3) ? sb[gb * QS + q * Q1 * Q2 + q12] : 0.0;
            dmma(c0, c1, av, bP[2][ks]);
          }
          const int n0 = 2 * fk;
          if (line < NL) {
            if (n0 < L3) sa[(gb * L3 + n0) * Q1 * Q2 + q12] = c0;
            if (n0 + 1 < L3) sa[(gb * L3 + n0 + 1) * Q1 * Q2 + q12] = c1;
          }
        }
      } else {
        for (int i = tid; i < GB * QS; i += 256) sa[i] = sb[i];
      }
      __syncthreads();
      // y projection: lines (gb, j3, q1), K = q2, N = j2 -> sb [gb][j3][j2][q1]
      if (D >= 2) {
        constexpr int NL = GB * L3 * Q1;
        for (int mt = warp; mt < (NL + 7) / 8; mt += 8) {
          const int line = mt * 8 + fr;
          const int q1 = line % Q1, gj3 = line / Q1;    // gj3 = gb * L3 + j3
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KP; ++ks) {
            const int q = 4 * ks + fk;
            const double av = (line < NL && q < Q2) ? sa[(gj3 * Q2 + q) * Q1 + q1] : 0.0;
            dmma(c0, c1, av, bP[1][ks]);
          }
          const int n0 = 2 * fk;
          if (line < NL) {
            if (n0 < L2) sb[(gj3 * L2 + n0) * Q1 + q1] = c0;
            if (n0 + 1 < L2) sb[(gj3 * L2 + n0 + 1) * Q1 + q1] = c1;
          }
        }
      } else {
        for (int i = tid; i < GB * L3 * Q1; i += 256) sb[i] = sa[i];
      }
      __syncthreads();
      // x projection: lines (gb, j3, j2), K = q1, N = j1 -> f0 [gb][j3][j2][j1]  (then time projection)
      {
        constexpr int NL = GB * L3 * L2;
        for (int mt = warp; mt < (NL + 7) / 8; mt += 8) {
          const int line = mt * 8 + fr;
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KP; ++ks) {
            const int q = 4 * ks + fk;
            const double av = (line < NL && q < Q1) ? sb[line * Q1 + q] : 0.0;
            dmma(c0, c1, av, bP[0][ks]);
          }
          const int n0 = 2 * fk;
          if (line < NL) {
            if (n0 < L1) f0[line * L1 + n0] = c0;
            if (n0 + 1 < L1) f0[line * L1 + n0 + 1] = c1;
          }
        }
      }
      __syncthreads();
      for (int i = tid; i < LS; i += 256) {
#pragma unroll
        for (int gb = 0; gb < GB; ++gb) {
          const double v = f0[gb * LS + i];
          const double* btt = r.B[3] + ((long long)et * QT + g0 + gb) * (PT + 1);
#pragma unroll
          for (int aa = 0; aa <= PT; ++aa) outw[((et + aa) % PW) * LS + i] += __ldg(btt + aa) * v;
        }
      }
      __syncthreads();
    }
    flush_slice(et);
    __syncthreads();
  }
  for (int ft = r.nel[3]; ft < r.nel[3] + PT; ++ft) flush_slice(ft);
}

// R5: time-streamed sum factorisation.  The block still owns a 2^d tile of
// spatial elements and sweeps all time elements, but the spatial stages now
// run once per TIME FUNCTION instead of once per time Gauss point:
//   * each time slice entering the window is interpolated to the tile's
//     spatial Gauss grid (x, y on the tensor cores through shared memory;
//     the last direction's DMMA accumulators stay in registers, which fixes
//     the Gauss points every thread owns);
//   * per time element the thread does the time interpolation, the
//     Rogers-McCulloch linearisation and the time projection on its own
//     points in registers (a rotating window of p_t+1 slices, no barriers);
//   * the slice leaving the window is projected back (last direction from
//     registers via quad shuffles into the A fragments, then y, x) and added
//     straight into y.
// 5 block barriers per time element (R4: 9 per time Gauss point).
template <int D, int P>
struct RxT5 : RxT4<D, P> {
  using B4 = RxT4<D, P>;
  static constexpr int QL = D == 3 ? B4::Q1 * B4::Q2 : (D == 2 ? B4::Q1 : 1);  // lines of the last stage
  static constexpr int NT = (QL + 7) / 8;                                          // its M tiles
  static constexpr int MT = (NT + 7) / 8;                                          // tiles per warp
  static constexpr int ev(int n) { return (n + 1) & ~1; }                        // 16-byte aligned buffers
  static constexpr int SIN = ev(3 * B4::LS);
  static constexpr int SA = D >= 2 ? ev(3 * B4::L3 * B4::L2 * B4::Q1) : 2;
  static constexpr int SB = D >= 3 ? ev(3 * B4::L3 * B4::Q2 * B4::Q1) : 2;
  static constexpr int SC = D >= 2 ? ev(B4::L * QL) : 2;
  static constexpr int SD = D >= 3 ? ev(B4::L3 * B4::L2 * B4::Q1) : 2;
  static constexpr int NIN = 3 * B4::LS;                                          // input items per slice
  static constexpr int NPRE = (NIN + 255) / 256;
  static constexpr size_t SMEM = (size_t)(SIN + SA + SB + SC + SD + 64 + 256) * 8;   // + time tables + read pad
};

template <int D, int P, int PT>
__global__ void __launch_bounds__(256, 2) reaction_tile5(RxArgs r) {
  using G = RxT5<D, P>;
  constexpr int E = G::E, QE = G::QE, L = G::L, Q = G::Q;
  constexpr int L1 = G::L1, L2 = G::L2, L3 = G::L3, Q1 = G::Q1, Q2 = G::Q2;
  constexpr int LS = G::LS, KI = G::KI, KP = G::KP, QL = G::QL, NT = G::NT, MT = G::MT;
  constexpr int PW = PT + 1, QT = PT + 1;
  constexpr int NBT = 2 * QT * PW;                  // time basis (interpolation) + weighted (projection)
  constexpr int NLX = L3 * L2;                      // x-projection lines (j3, j2)
  static_assert(NBT <= 32 && (NLX + 7) / 8 <= 8, "reaction tile too large");
  static_assert(Q1 % 2 == 0, "paired stores need an even Gauss count");
  extern __shared__ double sm[];
  double* sIn = sm;                // [fld][j3][j2][j1]
  double* sA = sIn + G::SIN;       // x-interp out [fld][j3][j2][q1]
  double* sB = sA + G::SA;         // y-interp out [fld][j3][q2][q1]
  double* sC = sB + G::SB;         // last-direction projection out [j_last][QL]
  double* sD = sC + G::SC;         // y-projection out [j3][j2][q1]
  double* sBt = sD + G::SD;        // [2][32] time tables (double-buffered by iteration parity)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  // A-fragment loads run unpredicated over padded rows / k columns: whatever they read is finite
  // (the buffers start zeroed) and meets a zero B entry or lands in a discarded output row
  for (int i = tid; i < (int)(G::SMEM / 8); i += 256) sm[i] = 0.0;
  int b = blockIdx.x, k[3], ne[3];
  for (int l = 0; l < 3; ++l) {
    const int m = b % r.ncol[l];
    b /= r.ncol[l];
    k[l] = l < D ? (m * G::RC + r.color[l]) * E : 0;
    ne[l] = l < D ? min(E, r.nel[l] - k[l]) : 1;
  }
  auto basis = [&](int l, int j, int q) -> double {
    if (l >= D || q >= Q || j >= L) return 0.0;
    const int le = q / QE, gq = q % QE, aa = j - le;
    if (le >= ne[l] || aa < 0 || aa > P) return 0.0;
    return __ldg(r.B[l] + ((long long)(k[l] + le) * QE + gq) * (P + 1) + aa);
  };
  auto wgt = [&](int l, int q) -> double {
    const int le = q / QE;
    return (q < Q && le < ne[l]) ? __ldg(r.Wq[l] + (long long)(k[l] + le) * QE + q % QE) : 0.0;
  };
  double bI[D][KI], bP[D][KP];
#pragma unroll
  for (int l = 0; l < D; ++l) {
#pragma unroll
    for (int ks = 0; ks < KI; ++ks) bI[l][ks] = basis(l, 4 * ks + fk, fr);
#pragma unroll
    for (int ks = 0; ks < KP; ++ks) bP[l][ks] = basis(l, fr, 4 * ks + fk);
  }
  // the thread's Gauss points: (line = 8 t + fr, q_last = 2 fk + e), t = warp + 8 mi.  The spatial
  // weight is folded into the x field and c2 into the w field as the slice enters the window.
  double wsp[MT][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int line = 8 * (warp + 8 * mi) + fr, ql = 2 * fk + e;
      double v = 0.0;
      if (line < QL && ql < Q) {
        v = wgt(D - 1, ql);
        if (D == 3) v *= wgt(0, line % Q1) * wgt(1, line / Q1);
        if (D == 2) v *= wgt(0, line);
      }
      wsp[mi][e] = v;
    }
  const long long ns = r.ns;
  auto spatial = [&](int j3, int j2, int j1, bool& ok) -> long long {
    const int g1 = k[0] + j1, g2 = k[1] + j2, g3 = k[2] + j3;
    ok = j1 < L1 && g1 < r.n[0] && g2 < r.n[1] && g3 < r.n[2];
    return ((long long)g3 * r.n[1] + g2) * r.n[0] + g1;
  };
  // input slice items of this thread: (fld, s) -> global spatial index (-1: padding)
  long long gsp[G::NPRE];
#pragma unroll
  for (int m = 0; m < G::NPRE; ++m) {
    const int i = tid + 256 * m;
    const int s = i % LS;
    bool ok;
    const long long gs = spatial(s / (L1 * L2), (s / L1) % L2, s % L1, ok);
    gsp[m] = (i < G::NIN && ok) ? gs : -1;
  }
  double pre[G::NPRE];
  auto prefetch = [&](int ft) {
    const int ct = ft + r.rowoff;
    const bool vt = ct >= 0 && ct < r.ntc;
#pragma unroll
    for (int m = 0; m < G::NPRE; ++m) {
      const int f = (tid + 256 * m) / LS;
      const double* src = f == 0 ? r.u : (f == 1 ? r.w : r.x);
      pre[m] = (vt && gsp[m] >= 0) ? __ldg(src + (long long)ct * ns + gsp[m]) : 0.0;
    }
  };
  double btp = 0.0;
  auto prefetch_bt = [&](int et) {
    if (tid < NBT && et >= 0 && et < r.nel[3]) {
      const int ga = tid % (QT * PW);
      const double bv = __ldg(r.B[3] + (long long)et * QT * PW + ga);
      btp = tid < QT * PW ? bv : bv * __ldg(r.Wq[3] + (long long)et * QT + ga / PW);
    }
  };
  // x-projection outputs of this thread: line 8 warp + fr, j1 = 2 fk + e (old y prefetched a phase early)
  const int xline = 8 * warp + fr;
  long long yidx[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    bool ok = false;
    long long gs = 0;
    if (xline < NLX) gs = spatial(D >= 2 ? xline / L2 : 0, D >= 2 ? xline % L2 : 0, 2 * fk + e, ok);
    yidx[e] = ok ? gs : -1;
  }
  double yold[2] = {0.0, 0.0};
  auto yrow = [&](int ft) -> long long {           // row offset of time function ft, -1 if constrained / foreign
    const int ct = ft + r.rowoff;
    return (ct >= 0 && ct < r.ntc) ? (long long)ct * ns : -1;
  };
  const double rc1 = r.c1, rk1 = -r.c1 * (1.0 + r.a), rk0 = r.c1 * r.a, rc2 = r.c2;

  // window slot of time function f is f % PW (compile-time below: the slice loop is unrolled by PW)
  double X[MT][PW][3][2], Y[MT][PW][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int a = 0; a < PW; ++a) {
#pragma unroll
      for (int f = 0; f < 3; ++f) X[mi][a][f][0] = X[mi][a][f][1] = 0.0;
      Y[mi][a][0] = Y[mi][a][1] = 0.0;
    }

  // x projection of function ft: lines (j3, j2), K = q1, N = j1 -> y (from sC for D = 2, sD for D = 3)
  auto xproj = [&](int ft, const double* xb) {
    if (warp < (NLX + 7) / 8) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KP; ++ks) dmma(c0, c1, xb[xline * Q1 + 4 * ks + fk], bP[0][ks]);
      const long long row = yrow(ft);
      if (row >= 0) {
        if (yidx[0] >= 0) r.y[row + yidx[0]] = yold[0] + c0;
        if (yidx[1] >= 0) r.y[row + yidx[1]] = yold[1] + c1;
      }
    }
  };

  const int nfull = r.nel[3] + PT;                   // full-basis time functions
  const int jmax = nfull + PT;
  auto step = [&](auto phc, int j) {
    constexpr int PH = decltype(phc)::value;         // j % PW: slot of the entering slice
    const int et = j - PT;                           // time element (0 <= et < nel_t); z-projection of function et
    const int fp = j - PT - 1;                       // function whose y / x projections run in this iteration
    const bool has_in = j < nfull, has_fp = fp >= 0 && fp < nfull;
    if constexpr (D == 1) __syncthreads();           // sIn is read by the last stage directly
    if (has_in) {
#pragma unroll
      for (int m = 0; m < G::NPRE; ++m)
        if (tid + 256 * m < G::NIN) sIn[tid + 256 * m] = pre[m];
    }
    if (tid < NBT) sBt[(j & 1) * 32 + tid] = btp;
    if constexpr (D >= 2) {
      if (has_fp) {
        const long long row = yrow(fp);
#pragma unroll
        for (int e = 0; e < 2; ++e) yold[e] = (row >= 0 && yidx[e] >= 0) ? r.y[row + yidx[e]] : 0.0;
      }
    }
    __syncthreads();                                 // B1
    if (j + 1 < nfull) prefetch(j + 1);
    prefetch_bt(et + 1);
    const double* fin = sIn;
    if constexpr (D >= 2) {
      // phase 2: x interpolation of slice j: lines (fld, j3, j2), K = j1, N = q1 -> sA [fld][j3][j2][q1]
#ifdef RX_ABL_NOXY
      if (false) {
#else
      if (has_in) {
#endif
        constexpr int NL = 3 * L3 * L2;
        for (int mt = warp; mt < (NL + 7) / 8; mt += 8) {
          const int line = mt * 8 + fr;
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KI; ++ks) dmma(c0, c1, sIn[line * L1 + 4 * ks + fk], bI[0][ks]);
          const int n0 = 2 * fk;
          if (line < NL && n0 < Q1) *reinterpret_cast<double2*>(sA + line * Q1 + n0) = make_double2(c0, c1);
        }
      }
      // ... and the y projection of function fp: lines (j3, q1), K = q2, N = j2 -> sD [j3][j2][q1]
      if (has_fp) {
        if constexpr (D == 3) {
          constexpr int NL = L3 * Q1;
          for (int mt = warp; mt < (NL + 7) / 8; mt += 8) {
            const int line = mt * 8 + fr;
            const int q1 = line % Q1, j3 = line / Q1;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < KP; ++ks) dmma(c0, c1, sC[(j3 * Q2 + 4 * ks + fk) * Q1 + q1], bP[1][ks]);
            const int n0 = 2 * fk;
            if (line < NL) {
              if (n0 < L2) sD[(j3 * L2 + n0) * Q1 + q1] = c0;
              if (n0 + 1 < L2) sD[(j3 * L2 + n0 + 1) * Q1 + q1] = c1;
            }
          }
        } else {
          xproj(fp, sC);
        }
      }
      __syncthreads();                               // B2
      fin = sA;
    }
    if constexpr (D == 3) {
      // phase 3: y interpolation of slice j: lines (fld, j3, q1), K = j2, N = q2 -> sB [fld][j3][q2][q1]
#ifdef RX_ABL_NOXY
      if (false) {
#else
      if (has_in) {
#endif
        constexpr int NL = 3 * L3 * Q1;
        for (int mt = warp; mt < (NL + 7) / 8; mt += 8) {
          const int line = mt * 8 + fr;
          const int q1 = line % Q1, fj3 = line / Q1;
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KI; ++ks) dmma(c0, c1, sA[(fj3 * L2 + 4 * ks + fk) * Q1 + q1], bI[1][ks]);
          const int n0 = 2 * fk;
          if (line < NL) {
            if (n0 < Q2) sB[(fj3 * Q2 + n0) * Q1 + q1] = c0;
            if (n0 + 1 < Q2) sB[(fj3 * Q2 + n0 + 1) * Q1 + q1] = c1;
          }
        }
      }
      // ... and the x projection of function fp (from sD) -> y
      if (has_fp) xproj(fp, sD);
      __syncthreads();                               // B3
      fin = sB;
    }
    // phase 4: last-direction interpolation of slice j -> window slot PH ...
    if (has_in) {
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) {
        const int t = warp + 8 * mi;
        if (t < NT) {
          const int line = 8 * t + fr;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < KI; ++ks) dmma(c0, c1, fin[(f * L + 4 * ks + fk) * QL + line], bI[D - 1][ks]);
            const double sc0 = f == 0 ? 1.0 : (f == 1 ? rc2 : wsp[mi][0]);
            const double sc1 = f == 0 ? 1.0 : (f == 1 ? rc2 : wsp[mi][1]);
            X[mi][PH][f][0] = f == 0 ? c0 : c0 * sc0;
            X[mi][PH][f][1] = f == 0 ? c1 : c1 * sc1;
          }
        }
      }
    }
    if (et < 0 || et >= nfull) return;
    constexpr int S0 = (PH + 1) % PW;                // slot of function et
    // ... time element et (slots S0 + a = functions et + a): interpolate in time, linearise, project
    // in time, all on the thread's own points ...
#ifndef RX_ABL_NOTIME
    if (et < r.nel[3]) {
#else
    if (et < 0) {
#endif
#ifdef RX_ABL_CBT
      const double* bt = r.btc;          // timing experiment: one table for every element (wrong results)
#else
      const double* bt = sBt + (j & 1) * 32;
#endif
#pragma unroll
      for (int g = 0; g < QT; ++g) {
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double uu = 0.0, ww = 0.0, xx = 0.0;
#pragma unroll
            for (int a = 0; a < PW; ++a) {
              const double ba = bt[g * PW + a];
              uu = fma(ba, X[mi][(S0 + a) % PW][0][e], uu);
              ww = fma(ba, X[mi][(S0 + a) % PW][1][e], ww);
              xx = fma(ba, X[mi][(S0 + a) % PW][2][e], xx);
            }
            // C_r = c1 (u - a)(u - 1) + c2 w = u (c1 u - c1 (1 + a)) + c1 a + c2 w
            const double cr = fma(uu, fma(rc1, uu, rk1), ww + rk0);
            const double v = cr * xx;
#pragma unroll
            for (int a = 0; a < PW; ++a)
              Y[mi][(S0 + a) % PW][e] = fma(bt[QT * PW + g * PW + a], v, Y[mi][(S0 + a) % PW][e]);
          }
      }
    }
    // ... and the last-direction projection of the completed function et (quad shuffles -> A fragments)
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      const int t = warp + 8 * mi;
      if (t < NT) {                                  // warp-uniform
        const int line = 8 * t + fr;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KP; ++ks) {
          const int c = 4 * ks + fk, src = (lane & ~3) | (c >> 1);
          const double v0 = __shfl_sync(0xffffffffu, Y[mi][S0][0], src);
          const double v1 = __shfl_sync(0xffffffffu, Y[mi][S0][1], src);
          dmma(c0, c1, (c & 1) ? v1 : v0, bP[D - 1][ks]);
        }
        const int n0 = 2 * fk;
        if (line < QL) {
          if constexpr (D == 1) {
            const long long row = yrow(et);
            if (row >= 0) {
              if (yidx[0] >= 0) r.y[row + yidx[0]] += c0;
              if (yidx[1] >= 0) r.y[row + yidx[1]] += c1;
            }
          } else {
            if (n0 < L) sC[n0 * QL + line] = c0;
            if (n0 + 1 < L) sC[(n0 + 1) * QL + line] = c1;
          }
        }
      }
      Y[mi][S0][0] = Y[mi][S0][1] = 0.0;
    }
  };
  prefetch(0);
#if RX_UNROLL
  for (int j0 = 0; j0 <= jmax; j0 += PW) {
    step(std::integral_constant<int, 0>{}, j0);
    if (j0 + 1 <= jmax) step(std::integral_constant<int, 1 % PW>{}, j0 + 1);
    if constexpr (PW > 2) if (j0 + 2 <= jmax) step(std::integral_constant<int, 2 % PW>{}, j0 + 2);
    if constexpr (PW > 3) if (j0 + 3 <= jmax) step(std::integral_constant<int, 3 % PW>{}, j0 + 3);
  }
#else
  // one copy of the step with fixed slots (entering slice -> slot PT, function et -> slot 0) and a
  // cyclic rotation of both windows after it (fewer registers and instruction bytes than unrolling)
  for (int j = 0; j <= jmax; ++j) {
    step(std::integral_constant<int, PT>{}, j);
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      double xs[3][2], ys[2];
#pragma unroll
      for (int f = 0; f < 3; ++f) xs[f][0] = X[mi][0][f][0], xs[f][1] = X[mi][0][f][1];
      ys[0] = Y[mi][0][0], ys[1] = Y[mi][0][1];
#pragma unroll
      for (int a = 0; a < PW - 1; ++a) {
#pragma unroll
        for (int f = 0; f < 3; ++f) X[mi][a][f][0] = X[mi][a + 1][f][0], X[mi][a][f][1] = X[mi][a + 1][f][1];
        Y[mi][a][0] = Y[mi][a + 1][0], Y[mi][a][1] = Y[mi][a + 1][1];
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) X[mi][PW - 1][f][0] = xs[f][0], X[mi][PW - 1][f][1] = xs[f][1];
      Y[mi][PW - 1][0] = ys[0], Y[mi][PW - 1][1] = ys[1];
    }
  }
#endif
}

template <int D, int P, int PT>
static constexpr size_t rx4_smem() {
  using G = RxT4<D, P>;
  constexpr int GB = RX4_GB, F = 3 * GB;
  constexpr int SX = F * G::L3 * G::L2 * G::Q1, SY = F * G::L3 * G::Q2 * G::Q1, SZ = F * G::QS;
  constexpr int BUF = (SX > SY ? (SX > SZ ? SX : SZ) : (SY > SZ ? SY : SZ));
  return (size_t)(3 * (PT + 1) * G::LS + (PT + 1) * G::LS + F * G::LS + 2 * BUF + 3 * G::Q) * 8;
}

template <int D, int P, int PT>
static constexpr size_t rx_warp_smem() {
  constexpr int LD = P + 1;
  constexpr int LS = LD * (D >= 2 ? LD : 1) * (D >= 3 ? LD : 1);
  constexpr int PW = PT + 1;
  return (size_t)(3 * PW * LS + PW * LS + 2 * 3 * LS + 3 * (P + 1) * LD) * 8;
}

#define MI_RX_CASE(dv, pv, ptv, ...)                                 \
  case ((dv) * 8 + (pv)) * 8 + (ptv): {                              \
    constexpr int D_ = (dv), P_ = (pv), PT_ = (ptv);                 \
    __VA_ARGS__;                                                     \
  } break;
#define MI_RX_DISPATCH(d, p, pt, ...)                                            \
  switch (((d) * 8 + (p)) * 8 + (pt)) {                                          \
    MI_RX_CASE(1, 1, 1, __VA_ARGS__) MI_RX_CASE(1, 2, 2, __VA_ARGS__)            \
    MI_RX_CASE(1, 3, 3, __VA_ARGS__) MI_RX_CASE(2, 1, 1, __VA_ARGS__)            \
    MI_RX_CASE(2, 2, 2, __VA_ARGS__) MI_RX_CASE(2, 3, 3, __VA_ARGS__)            \
    MI_RX_CASE(3, 1, 1, __VA_ARGS__) MI_RX_CASE(3, 2, 2, __VA_ARGS__)            \
    MI_RX_CASE(3, 3, 3, __VA_ARGS__)                                             \
    default:                                                                     \
      ::mi::set_error("reaction: unsupported (d, p, p_t) (need p = p_t <= 3)");  \
      return MI_ERR_ARG;                                                         \
  }

int reaction_apply(mi_ctx* c, const double* x, double* y) {
  RxArgs r{};
  r.u = c->u_it.p;
  r.w = c->w_it.p;
  r.x = x;
  r.y = y;
  for (int l = 0; l < 4; ++l) {
    r.B[l] = c->rx_B.p + c->rx_Boff[l];
    r.Wq[l] = c->rx_W.p + c->rx_Woff[l];
    r.nel[l] = c->rx_nel[l];
  }
  r.n[0] = c->n[0];
  r.n[1] = c->n[1];
  r.n[2] = c->n[2];
  r.ntc = c->nt;
  r.rowoff = c->rx_rowoff;
  r.ns = c->ns;
  r.c1 = c->c1;
  r.a = c->a;
  r.c2 = c->c2;
  MI_RX_DISPATCH(c->d, c->p, c->pt, {
    using G = RxT5<D_, P_>;
    constexpr size_t smem = G::SMEM;
    static bool attr = false;
    if (!attr) {
      MI_CUDA(cudaFuncSetAttribute(reaction_tile5<D_, P_, PT_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      attr = true;
    }
    const int RC = G::RC;
    const int ncolors = RC * (c->d >= 2 ? RC : 1) * (c->d >= 3 ? RC : 1);
    for (int col = 0; col < ncolors; ++col) {
      int cc = col;
      long long nb = 1;
      for (int l = 0; l < 3; ++l) {
        if (l < c->d) {
          r.color[l] = cc % RC;
          cc /= RC;
          const int ntile = (c->rx_nel[l] + G::E - 1) / G::E;
          r.ncol[l] = (ntile - r.color[l] + RC - 1) / RC;
        } else {
          r.color[l] = 0;
          r.ncol[l] = 1;
        }
        nb *= r.ncol[l] > 0 ? r.ncol[l] : 0;
      }
      if (nb == 0) continue;
      reaction_tile5<D_, P_, PT_><<<(unsigned)nb, 256, smem, c->stream>>>(r);
      MI_CHECK_LAUNCH("reaction_tile5");
    }
  });
  return MI_OK;
}

}  // namespace mi

using namespace mi;

extern "C" {

int mi_op_set_reaction(mi_ctx* c, const double* u, const double* w, double c1, double a, double c2,
                       const int* q, const int* nel, const double* B, const double* Wq) {
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(u && w && q && nel && B && Wq, MI_ERR_ARG, "NULL argument to mi_op_set_reaction");
  int rc;
  if ((rc = dalloc(c->u_it, c->N)) || (rc = dalloc(c->w_it, c->N))) return rc;
  MI_CUDA(cudaMemcpyAsync(c->u_it.p, u, sizeof(double) * c->N, cudaMemcpyDeviceToDevice, c->stream));
  MI_CUDA(cudaMemcpyAsync(c->w_it.p, w, sizeof(double) * c->N, cudaMemcpyDeviceToDevice, c->stream));
  // per direction tables, direction order x, y, z, t; absent spatial dims get q=1, p=0
  size_t nb = 0, nw = 0;
  for (int l = 0; l < 4; ++l) {
    const bool present = l == 3 || l < c->d;
    const int src = l == 3 ? c->d : l;           // host arrays: x, y, ..., t
    c->rx_q[l] = present ? q[src] : 1;
    c->rx_p[l] = present ? (l == 3 ? c->pt : c->p) : 0;
    c->rx_nel[l] = present ? nel[src] : 1;
    c->rx_E[l] = present ? std::max(1, c->rx_p[l]) : 1;
    c->rx_Boff[l] = nb;
    c->rx_Woff[l] = nw;
    nb += (size_t)c->rx_nel[l] * c->rx_q[l] * (c->rx_p[l] + 1);
    nw += (size_t)c->rx_nel[l] * c->rx_q[l];
  }
  std::vector<double> hb(nb), hw(nw);
  size_t sb = 0, sw = 0;
  for (int l = 0; l < 4; ++l) {
    const bool present = l == 3 || l < c->d;
    const size_t cb = (size_t)c->rx_nel[l] * c->rx_q[l] * (c->rx_p[l] + 1);
    const size_t cw = (size_t)c->rx_nel[l] * c->rx_q[l];
    for (size_t i = 0; i < cb; ++i) hb[c->rx_Boff[l] + i] = present ? B[sb + i] : 1.0;
    for (size_t i = 0; i < cw; ++i) hw[c->rx_Woff[l] + i] = present ? Wq[sw + i] : 1.0;
    if (present) {
      sb += cb;
      sw += cw;
    }
  }
  if ((rc = dalloc(c->rx_B, nb)) || (rc = dalloc(c->rx_W, nw))) return rc;
  MI_CUDA(cudaMemcpy(c->rx_B.p, hb.data(), sizeof(double) * nb, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->rx_W.p, hw.data(), sizeof(double) * nw, cudaMemcpyHostToDevice));
  c->c1 = c1;
  c->a = a;
  c->c2 = c2;
  MI_REQUIRE(c->p == c->pt && c->p <= 3, MI_ERR_ARG, "reaction: need p = p_t <= 3");
  for (int l = 0; l < 4; ++l)
    MI_REQUIRE(c->rx_q[l] == ((l == 3 || l < c->d) ? c->p + 1 : 1), MI_ERR_ARG, "reaction: need q = p + 1");
  c->reaction_on = true;
  return MI_OK;
}

int mi_op_set_reaction_rows(mi_ctx* c, int row_offset) {
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  c->rx_rowoff = row_offset;
  return MI_OK;
}

int mi_op_clear_reaction(mi_ctx* c) {
  if (c) c->reaction_on = false;
  return MI_OK;
}

}  // extern "C"
