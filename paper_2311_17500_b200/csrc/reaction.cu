// Reaction correction y += M_R x with the Rogers-McCulloch linearisation
// (reference reaction_mass, assembly.py:287-347):
//
//   M_R[i, j] = int int C_r B_i B_j,   C_r = c1 (u - a)(u - 1) + c2 w,
//
// u, w = the frozen iterate, evaluated at q = p+1 Gauss points per element
// in every direction (space and time; assembly.py:313-318 -- the rule is
// parity-critical).  Matrix-free, sum factorised: a
// block owns a tile of 2^d spatial elements and streams through all time
// elements (see reaction_tile below).  Tiles run in RC^d colour classes so
// concurrently running blocks never touch the same output DoF: every y entry
// has one writer per colour launch (its atomicAdd never races) and the
// launches are stream-ordered, so the result is bitwise deterministic.
//
// History (cfg 4, 96^3 x 192, p = 3): warp per element 1259 ms, line ops
// 1123, block tile sweep 813, DMMA stages 615, time-streamed 281, pipelined
// projections 229 (profiles/r01_optimisation_log.md), reaction_tile 202; the
// fused mode at d = 3, p = 3 now runs the warp-specialised reaction_ws
// (reaction_ws.cuh, 112.8 ms; profiles/r02_optimisation_log.md R15-R22).
#include "common.cuh"
#include "dispatch.cuh"
#include "ptx.cuh"

#include <cstdlib>
#include <type_traits>

#ifndef MI_RX_BAL
#define MI_RX_BAL 1    // projection tiles on the warps with the fewest interpolation tiles (phase balance)
#endif
#ifndef MI_RX_NOCW
#define MI_RX_NOCW 0   // timing ablation only (wrong results): the stored mode skips its coefficient reads
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
  const double* jw;    // mapped geometry: |det J| at the spatial Gauss points, C order (Q_3, Q_2, Q_1); null: box
  double* cw;          // stored weighted coefficient C_r w_x (RX_PRE writes it, RX_STORED reads it)
  // u0 lifting: coefficients of the dropped first time function (constrained row -1) for the u field
  // (the lifted iterate) and for the x field (mi_op_apply_lift); null = zero slab (the reference)
  const double* lift_u;
  const double* lift_x;
};

// Kernel modes.  RX_FUSED interpolates u, w and x and evaluates C_r on the fly every apply.  The
// iterate is frozen for a whole GMRES solve, so when the Gauss-point coefficients fit in memory
// RX_PRE evaluates c_w = C_r x (spatial weight) once per operator build and RX_STORED applies M_R
// with it: one interpolated field instead of three, and the time stage reads c_w (coalesced: the
// store is laid out in the order each thread consumes its own points) instead of forming C_r.
enum RxMode { RX_FUSED = 0, RX_PRE = 1, RX_STORED = 2 };

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
struct RxTile {
  static constexpr int E = 2, LD = P + 1, QE = P + 1;
  static constexpr int L = E + P, Q = E * QE;                    // per present direction
  static constexpr int L1 = L, L2 = D >= 2 ? L : 1, L3 = D >= 3 ? L : 1;
  static constexpr int Q1 = Q, Q2 = D >= 2 ? Q : 1, Q3 = D >= 3 ? Q : 1;
  static constexpr int LS = L1 * L2 * L3, QS = Q1 * Q2 * Q3;
  static constexpr int KI = (L + 3) / 4, KP = (Q + 3) / 4;      // k-steps interp / proj
  static constexpr int RC = (E + P + E - 1) / E;
  using B4 = RxTile;
  static constexpr int QL = D == 3 ? B4::Q1 * B4::Q2 : (D == 2 ? B4::Q1 : 1);  // lines of the last stage
  static constexpr int NT = (QL + 7) / 8;                                          // its M tiles
  static constexpr int NW = NT < 8 ? NT : 8;                                       // warps: one last-stage tile each
  static constexpr int NTH = 32 * NW;
  static constexpr int MT = (NT + NW - 1) / NW;                                    // last-stage tiles per warp
  static constexpr int ev(int n) { return (n + 1) & ~1; }                        // 16-byte aligned buffers
  static constexpr int SIN = ev(3 * B4::LS);
  static constexpr int SA = D >= 2 ? ev(3 * B4::L3 * B4::L2 * B4::Q1) : 2;
  // bank-conflict padding (d = 3, 8 Gauss points per direction, i.e. p = 3): the y-interpolation
  // output rows (q2 stride BS1 = 4 mod 8) and planes (j3 stride BJ = 8 mod 16), and the last-direction
  // projection output (j stride CS = 4 mod 8), so that the DMMA accumulator stores (lanes 2 fk, fr) and
  // the A-fragment reads (lanes fk, fr) each touch every bank pair exactly twice.  ncu before: 47% of
  // the kernel's shared wavefronts were conflict replays.
  static constexpr bool PADB = D == 3 && Q1 % 8 == 0;
  static constexpr int BS1 = PADB ? Q1 + 4 : Q1;
  static constexpr int BJ = PADB ? Q2 * BS1 + ((8 - (Q2 * BS1) % 16) + 16) % 16 : Q2 * Q1;
  static constexpr int CS = PADB ? QL + 4 : QL;
  static constexpr int SB = D >= 3 ? ev(3 * B4::L3 * BJ) : 2;
  static constexpr int SC = D >= 2 ? ev(B4::L * CS) : 2;
  static constexpr int SD = D >= 3 ? ev(B4::L3 * B4::L2 * B4::Q1) : 2;
  static constexpr int NIN = 3 * B4::LS;                                          // input items per slice
  static constexpr int NPRE = (NIN + NTH - 1) / NTH;
  static constexpr size_t SMEM = (size_t)(SIN + SA + SB + SC + SD + 64 + 256) * 8;   // + time tables + read pad
  // resident blocks per SM the register budget is sized for: the kernel is latency-bound, and at
  // d = 3, p = 2 a fourth 160-thread block (96 registers, a 100-byte spill) beats three (126
  // registers): 24.1 -> 20.6 ms at cfg 3; five or six blocks spill more and lose
  static constexpr int MINB = (D == 3 && P == 2) ? 640 / NTH : 512 / NTH;
};

template <int D, int P, int PT, int MODE>
__global__ void __launch_bounds__(RxTile<D, P>::NTH, RxTile<D, P>::MINB) reaction_tile(RxArgs r) {
  using G = RxTile<D, P>;
  constexpr int NF = MODE == RX_FUSED ? 3 : (MODE == RX_PRE ? 2 : 1);   // interpolated fields
  constexpr int NIN = NF * G::LS, NPRE = (NIN + G::NTH - 1) / G::NTH;
  constexpr int E = G::E, QE = G::QE, L = G::L, Q = G::Q;
  constexpr int L1 = G::L1, L2 = G::L2, L3 = G::L3, Q1 = G::Q1, Q2 = G::Q2;
  constexpr int LS = G::LS, KI = G::KI, KP = G::KP, QL = G::QL, NT = G::NT, MT = G::MT;
  constexpr int NW = G::NW, NTH = G::NTH;
  constexpr int BS1 = G::BS1, BJ = G::BJ, CS = G::CS;
  constexpr int PW = PT + 1, QT = PT + 1;
  constexpr int NBT = 2 * QT * PW;                  // time basis (interpolation) + weighted (projection)
  constexpr int NLX = L3 * L2;                      // x-projection lines (j3, j2)
  static_assert(NBT <= 32 && (NLX + 7) / 8 <= NW, "reaction tile too large");
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
  for (int i = tid; i < (int)(G::SMEM / 8); i += NTH) sm[i] = 0.0;
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
      const int line = 8 * (warp + NW * mi) + fr, ql = 2 * fk + e;
      double v = 0.0;
      if (line < QL && ql < Q) {
        v = wgt(D - 1, ql);
        if (D == 3) v *= wgt(0, line % Q1) * wgt(1, line / Q1);
        if (D == 2) v *= wgt(0, line);
        if (r.jw != nullptr && v != 0.0) {
          // global Gauss index of this point: element k[l] + local element, QE points per element
          int gq[3] = {0, 0, 0};
          if (D == 3) { gq[0] = k[0] * QE + line % Q1; gq[1] = k[1] * QE + line / Q1; gq[2] = k[2] * QE + ql; }
          if (D == 2) { gq[0] = k[0] * QE + line; gq[1] = k[1] * QE + ql; }
          if (D == 1) { gq[0] = k[0] * QE + ql; }
          const long long G1 = (long long)r.nel[0] * QE, G2 = D >= 2 ? (long long)r.nel[1] * QE : 1;
          v *= __ldg(r.jw + ((long long)gq[2] * G2 + gq[1]) * G1 + gq[0]);
        }
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
  long long gsp[NPRE];
#pragma unroll
  for (int m = 0; m < NPRE; ++m) {
    const int i = tid + NTH * m;
    const int s = i % LS;
    bool ok;
    const long long gs = spatial(s / (L1 * L2), (s / L1) % L2, s % L1, ok);
    gsp[m] = (i < NIN && ok) ? gs : -1;
  }
  double pre[NPRE];
  auto prefetch = [&](int ft) {
    const int ct = ft + r.rowoff;
    const bool vt = ct >= 0 && ct < r.ntc;
#pragma unroll
    for (int m = 0; m < NPRE; ++m) {
      const int f = (tid + NTH * m) / LS;
      const double* src = MODE == RX_STORED ? r.x : (f == 0 ? r.u : (f == 1 ? r.w : r.x));
      const double* lift = MODE == RX_STORED ? r.lift_x : (f == 0 ? r.lift_u : (f == 1 ? nullptr : r.lift_x));
      double v = 0.0;
      if (gsp[m] >= 0) {
        if (vt) v = __ldg(src + (long long)ct * ns + gsp[m]);
        else if (ct == -1 && lift != nullptr) v = __ldg(lift + gsp[m]);
      }
      pre[m] = v;
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
  // projection tiles run on the warps in reverse order (pwarp): the interpolation tiles of the same
  // phase fill the low warps first, so the phase's slowest warp does one tile fewer (d = 3, p = 3:
  // x-interpolation 10 tiles + y-projection 5 tiles over 8 warps -> at most 2 per warp, was 3)
  const int pwarp = MI_RX_BAL ? NW - 1 - warp : warp;
  // x-projection outputs of this thread: line 8 pwarp + fr, j1 = 2 fk + e
  const int xline = 8 * pwarp + fr;
  long long yidx[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    bool ok = false;
    long long gs = 0;
    if (xline < NLX) gs = spatial(D >= 2 ? xline / L2 : 0, D >= 2 ? xline % L2 : 0, 2 * fk + e, ok);
    yidx[e] = ok ? gs : -1;
  }
  auto yrow = [&](int ft) -> long long {           // row offset of time function ft, -1 if constrained / foreign
    const int ct = ft + r.rowoff;
    return (ct >= 0 && ct < r.ntc) ? (long long)ct * ns : -1;
  };
  const double rc1 = r.c1, rk1 = -r.c1 * (1.0 + r.a), rk0 = r.c1 * r.a, rc2 = r.c2;

  // window slot of time function f is f % PW (compile-time below: the slice loop is unrolled by PW)
  double X[MT][PW][NF][2], Y[MT][PW][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int a = 0; a < PW; ++a) {
#pragma unroll
      for (int f = 0; f < NF; ++f) X[mi][a][f][0] = X[mi][a][f][1] = 0.0;
      Y[mi][a][0] = Y[mi][a][1] = 0.0;
    }

  // x projection of function ft: lines (j3, j2), K = q1, N = j1 -> y (from sC for D = 2, sD for D = 3)
  auto xproj = [&](int ft, const double* xb) {
    if (pwarp < (NLX + 7) / 8) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KP; ++ks) dmma(c0, c1, xb[xline * Q1 + 4 * ks + fk], bP[0][ks]);
      const long long row = yrow(ft);
      if (row >= 0) {
        // fire-and-forget reduction (no old-y round trip): within one colour launch every y entry has
        // exactly one writer, and the launches are stream-ordered, so the sums stay deterministic
        if (yidx[0] >= 0) atomicAdd(r.y + row + yidx[0], c0);
        if (yidx[1] >= 0) atomicAdd(r.y + row + yidx[1], c1);
      }
    }
  };

  // c_w store layout: [tile][time element][g][line][q_last], valid Gauss points only (QL x Q per slice)
  const long long tile_id = ((long long)(k[2] / E) * ((r.nel[1] + E - 1) / E) + k[1] / E) * ((r.nel[0] + E - 1) / E) +
                            k[0] / E;
  auto cw_valid = [&](int mi, int e) -> bool { return 8 * (warp + NW * mi) + fr < QL && 2 * fk + e < Q; };
  auto cw_index = [&](int et, int g, int mi, int e) -> long long {
    return ((tile_id * r.nel[3] + et) * QT + g) * (long long)(QL * Q) + (8 * (warp + NW * mi) + fr) * Q + 2 * fk + e;
  };
  [[maybe_unused]] double cwp[QT][MT][2];
  const int nfull = r.nel[3] + PT;                   // full-basis time functions
  const int jmax = nfull + PT;
  auto step = [&](auto phc, int j) {
    constexpr int PH = decltype(phc)::value;         // j % PW: slot of the entering slice
    const int et = j - PT;                           // time element (0 <= et < nel_t); z-projection of function et
    const int fp = j - PT - 1;                       // function whose y / x projections run in this iteration
    const bool has_in = j < nfull;
    [[maybe_unused]] const bool has_fp = MODE != RX_PRE && fp >= 0 && fp < nfull;
    if constexpr (D == 1) __syncthreads();           // sIn is read by the last stage directly
    if (has_in) {
#pragma unroll
      for (int m = 0; m < NPRE; ++m)
        if (tid + NTH * m < NIN) sIn[tid + NTH * m] = pre[m];
    }
    if (tid < NBT) sBt[(j & 1) * 32 + tid] = btp;
    __syncthreads();                                 // B1
    if (j + 1 < nfull) prefetch(j + 1);
    prefetch_bt(et + 1);
    if constexpr (MODE == RX_STORED) {               // this step's c_w, consumed by its time stage
      if (et >= 0 && et < r.nel[3]) {
#pragma unroll
        for (int g = 0; g < QT; ++g)
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              cwp[g][mi][e] = MI_RX_NOCW ? 1.0 : (cw_valid(mi, e) ? __ldcs(r.cw + cw_index(et, g, mi, e)) : 0.0);
      }
    }
    const double* fin = sIn;
    if constexpr (D >= 2) {
      // phase 2: x interpolation of slice j: lines (fld, j3, j2), K = j1, N = q1 -> sA [fld][j3][j2][q1]
      if (has_in) {
        constexpr int NL = NF * L3 * L2;
        for (int mt = warp; mt < (NL + 7) / 8; mt += NW) {
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
          for (int mt = pwarp; mt < (NL + 7) / 8; mt += NW) {
            const int line = mt * 8 + fr;
            const int q1 = line % Q1, j3 = line / Q1;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < KP; ++ks) dmma(c0, c1, sC[j3 * CS + (4 * ks + fk) * Q1 + q1], bP[1][ks]);
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
      if (has_in) {
        constexpr int NL = NF * L3 * Q1;
        for (int mt = warp; mt < (NL + 7) / 8; mt += NW) {
          const int line = mt * 8 + fr;
          const int q1 = line % Q1, fj3 = line / Q1;
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KI; ++ks) dmma(c0, c1, sA[(fj3 * L2 + 4 * ks + fk) * Q1 + q1], bI[1][ks]);
          const int n0 = 2 * fk;
          if (line < NL) {
            if (n0 < Q2) sB[fj3 * BJ + n0 * BS1 + q1] = c0;
            if (n0 + 1 < Q2) sB[fj3 * BJ + (n0 + 1) * BS1 + q1] = c1;
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
        const int t = warp + NW * mi;
        if (t < NT) {
          const int line = 8 * t + fr;
          // sB (d = 3) holds (q2, q1) rows at stride BS1 and j3 planes at stride BJ
          const int loff = D == 3 ? (line / Q1) * BS1 + line % Q1 : line;
          constexpr int FS = D == 3 ? BJ : QL;
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < KI; ++ks) dmma(c0, c1, fin[(f * L + 4 * ks + fk) * FS + loff], bI[D - 1][ks]);
            // fused: (u, c2 w, w_x x); pre: (u, c2 w); stored: (x) -- the weight is in c_w
            const double sc0 = MODE == RX_STORED ? 1.0 : (f == 0 ? 1.0 : (f == 1 ? rc2 : wsp[mi][0]));
            const double sc1 = MODE == RX_STORED ? 1.0 : (f == 0 ? 1.0 : (f == 1 ? rc2 : wsp[mi][1]));
            X[mi][PH][f][0] = c0 * sc0;
            X[mi][PH][f][1] = c1 * sc1;
          }
        }
      }
    }
    if (et < 0 || et >= nfull) return;
    constexpr int S0 = (PH + 1) % PW;                // slot of function et
    // ... time element et (slots S0 + a = functions et + a): interpolate in time, linearise, project
    // in time, all on the thread's own points ...
    if (et < r.nel[3]) {
      const double* bt = sBt + (j & 1) * 32;
#pragma unroll
      for (int g = 0; g < QT; ++g) {
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if constexpr (MODE == RX_STORED) {
              double xx = 0.0;
#pragma unroll
              for (int a = 0; a < PW; ++a) xx = fma(bt[g * PW + a], X[mi][(S0 + a) % PW][0][e], xx);
              const double v = cwp[g][mi][e] * xx;
#pragma unroll
              for (int a = 0; a < PW; ++a)
                Y[mi][(S0 + a) % PW][e] = fma(bt[QT * PW + g * PW + a], v, Y[mi][(S0 + a) % PW][e]);
            } else {
              double uu = 0.0, ww = 0.0;
              [[maybe_unused]] double xx = 0.0;
#pragma unroll
              for (int a = 0; a < PW; ++a) {
                const double ba = bt[g * PW + a];
                uu = fma(ba, X[mi][(S0 + a) % PW][0][e], uu);
                ww = fma(ba, X[mi][(S0 + a) % PW][1][e], ww);
                if constexpr (MODE == RX_FUSED) xx = fma(ba, X[mi][(S0 + a) % PW][NF - 1][e], xx);
              }
              // C_r = c1 (u - a)(u - 1) + c2 w = u (c1 u - c1 (1 + a)) + c1 a + c2 w
              const double cr = fma(uu, fma(rc1, uu, rk1), ww + rk0);
              if constexpr (MODE == RX_PRE) {
                if (cw_valid(mi, e)) r.cw[cw_index(et, g, mi, e)] = cr * wsp[mi][e];
              } else {
                const double v = cr * xx;
#pragma unroll
                for (int a = 0; a < PW; ++a)
                  Y[mi][(S0 + a) % PW][e] = fma(bt[QT * PW + g * PW + a], v, Y[mi][(S0 + a) % PW][e]);
              }
            }
          }
      }
    }
    // ... and the last-direction projection of the completed function et (quad shuffles -> A fragments);
    // RX_PRE projects nothing back
#pragma unroll
    for (int mi = 0; mi < (MODE == RX_PRE ? 0 : MT); ++mi) {
      const int t = warp + NW * mi;
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
        [[maybe_unused]] const int n0 = 2 * fk;
        if (line < QL) {
          if constexpr (D == 1) {
            const long long row = yrow(et);
            if (row >= 0) {
              if (yidx[0] >= 0) atomicAdd(r.y + row + yidx[0], c0);
              if (yidx[1] >= 0) atomicAdd(r.y + row + yidx[1], c1);
            }
          } else {
            if (n0 < L) sC[n0 * CS + line] = c0;
            if (n0 + 1 < L) sC[(n0 + 1) * CS + line] = c1;
          }
        }
      }
      Y[mi][S0][0] = Y[mi][S0][1] = 0.0;
    }
  };
  prefetch(0);
  // one copy of the step with fixed slots (entering slice -> slot PT, function et -> slot 0) and a
  // cyclic rotation of both windows after it (fewer registers and instruction bytes than unrolling)
  for (int j = 0; j <= jmax; ++j) {
    step(std::integral_constant<int, PT>{}, j);
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      double xs[NF][2], ys[2];
#pragma unroll
      for (int f = 0; f < NF; ++f) xs[f][0] = X[mi][0][f][0], xs[f][1] = X[mi][0][f][1];
      ys[0] = Y[mi][0][0], ys[1] = Y[mi][0][1];
#pragma unroll
      for (int a = 0; a < PW - 1; ++a) {
#pragma unroll
        for (int f = 0; f < NF; ++f) X[mi][a][f][0] = X[mi][a + 1][f][0], X[mi][a][f][1] = X[mi][a + 1][f][1];
        Y[mi][a][0] = Y[mi][a + 1][0], Y[mi][a][1] = Y[mi][a + 1][1];
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) X[mi][PW - 1][f][0] = xs[f][0], X[mi][PW - 1][f][1] = xs[f][1];
      Y[mi][PW - 1][0] = ys[0], Y[mi][PW - 1][1] = ys[1];
    }
  }
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

}  // namespace mi

#include "reaction_ws.cuh"

namespace mi {

// the warp-specialised kernel serves the fused mode at d = 3, p = p_t in {2, 3} (MI_RX_WS=0: reaction_tile)
static bool use_reaction_ws(const mi_ctx* c) {
  static const bool on = [] {
    const char* e = std::getenv("MI_RX_WS");
    return e == nullptr || e[0] != '0';
  }();
  const bool can = c->d == 3 && (c->p == 3 || c->p == 2) && c->pt == c->p && c->ns_in < (1LL << 31) && c->c1 >= 0.0;
  return can && (c->rx_kernel == 1 || (c->rx_kernel < 0 && on));
}

template <int MODE>
static int reaction_ws_mode(mi_ctx* c, RxArgs r) {
  return c->p == 3 ? reaction_ws_launch<3, MODE>(c, r) : reaction_ws_launch<2, MODE>(c, r);
}

// y[t, owned planes] += y_in[t, same planes of the input slab] (z-slab contexts)
__global__ void add_owned_planes(double* __restrict__ y, const double* __restrict__ yin, long long ns,
                                 long long ns_in, long long off, int nt) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (i < ns && t < nt) y[(long long)t * ns + i] += yin[(long long)t * ns_in + off + i];
}

static void fill_args(mi_ctx* c, RxArgs& r) {
  r.u = c->u_it.p;
  r.w = c->w_it.p;
  for (int l = 0; l < 4; ++l) {
    r.B[l] = c->rx_B.p + c->rx_Boff[l];
    r.Wq[l] = c->rx_W.p + c->rx_Woff[l];
    r.nel[l] = c->rx_nel[l];
  }
  r.n[0] = c->n[0];
  r.n[1] = c->n[1];
  r.n[2] = c->n[2] + c->hz_lo + c->hz_hi;
  r.ntc = c->nt;
  r.rowoff = c->rx_rowoff;
  r.ns = c->ns_in;
  r.c1 = c->c1;
  r.a = c->a;
  r.c2 = c->c2;
  r.jw = c->rx_mapped ? c->rx_jw.p : nullptr;
  r.cw = c->rx_cw_ok ? c->rx_cw.p : nullptr;
  r.lift_u = c->lift_on ? c->lift_u0.p : nullptr;
  r.lift_x = nullptr;
}

// all colour classes of one kernel mode
template <int MODE>
static int reaction_launch(mi_ctx* c, RxArgs r) {
  MI_RX_DISPATCH(c->d, c->p, c->pt, {
    using G = RxTile<D_, P_>;
    constexpr size_t smem = G::SMEM;
    MI_DEV_FLAG(attr);
    if (!attr) {
      MI_CUDA(cudaFuncSetAttribute(reaction_tile<D_, P_, PT_, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
      reaction_tile<D_, P_, PT_, MODE><<<(unsigned)nb, G::NTH, smem, c->stream>>>(r);
      MI_CHECK_LAUNCH("reaction_tile");
    }
  });
  return MI_OK;
}

// bytes of the stored weighted coefficient c_w for this context (0: dims unsupported)
static size_t reaction_store_bytes(const mi_ctx* c) {
  size_t out = 0;
  if (use_reaction_ws(c)) {
    // reaction_ws: [tile (2 x 4 x 2 elements)][time element][g][8 E1 QE... valid Gauss points]
    const size_t qe = (size_t)c->p + 1, e2 = MI_RXWS_E2(c->p);
    size_t tiles = ((c->rx_nel[0] + 1) / 2) * (size_t)((c->rx_nel[1] + e2 - 1) / e2) * ((c->rx_nel[2] + 1) / 2);
    return tiles * c->rx_nel[3] * qe * (2 * qe) * (e2 * qe) * (2 * qe) * sizeof(double);
  }
  auto one = [&](auto dv, auto pv) {
    constexpr int D_ = decltype(dv)::value, P_ = decltype(pv)::value;
    using G = RxTile<D_, P_>;
    size_t tiles = 1;
    for (int l = 0; l < D_; ++l) tiles *= (size_t)((c->rx_nel[l] + G::E - 1) / G::E);
    out = tiles * c->rx_nel[3] * (P_ + 1) * (size_t)(G::QL * G::Q) * sizeof(double);
  };
  if (c->p == c->pt) {
    if (c->d == 3 && c->p == 3) one(std::integral_constant<int, 3>{}, std::integral_constant<int, 3>{});
    if (c->d == 3 && c->p == 2) one(std::integral_constant<int, 3>{}, std::integral_constant<int, 2>{});
    if (c->d == 3 && c->p == 1) one(std::integral_constant<int, 3>{}, std::integral_constant<int, 1>{});
    if (c->d == 2 && c->p == 3) one(std::integral_constant<int, 2>{}, std::integral_constant<int, 3>{});
    if (c->d == 2 && c->p == 2) one(std::integral_constant<int, 2>{}, std::integral_constant<int, 2>{});
    if (c->d == 2 && c->p == 1) one(std::integral_constant<int, 2>{}, std::integral_constant<int, 1>{});
    if (c->d == 1 && c->p == 3) one(std::integral_constant<int, 1>{}, std::integral_constant<int, 3>{});
    if (c->d == 1 && c->p == 2) one(std::integral_constant<int, 1>{}, std::integral_constant<int, 2>{});
    if (c->d == 1 && c->p == 1) one(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
  }
  return out;
}

// evaluate c_w once for the current iterate when it fits (store mode: -1 auto = at most 40% of the
// free device memory, 0 never, 1 always)
static int reaction_prepare_store(mi_ctx* c) {
  c->rx_cw_ok = false;
  if (c->rx_store_mode == 0) return MI_OK;
  const size_t bytes = reaction_store_bytes(c);
  if (bytes == 0) return MI_OK;
  if (c->rx_store_mode < 0 && c->rx_cw.n * sizeof(double) < bytes) {
    size_t free_b = 0, total_b = 0;
    MI_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (bytes > free_b / 10 * 4) return MI_OK;
  }
  int rc;
  if ((rc = dalloc(c->rx_cw, bytes / sizeof(double)))) return rc;
  RxArgs r{};
  fill_args(c, r);
  r.cw = c->rx_cw.p;
  c->rx_cw_ws = use_reaction_ws(c);
  if ((rc = c->rx_cw_ws ? reaction_ws_mode<RX_PRE>(c, r) : reaction_launch<RX_PRE>(c, r))) return rc;
  c->rx_cw_ok = true;
  return MI_OK;
}

// y += M_R x; x0 (nullable) = the x coefficients of the lifted slab (mi_op_apply_lift)
int reaction_apply(mi_ctx* c, const double* x, double* y, const double* x0) {
  if (c->rx_cw_dirty) {
    int rc = reaction_prepare_store(c);
    if (rc) return rc;
    c->rx_cw_dirty = false;
  }
  // the reaction runs on the input frame (owned + halo planes): element contributions to the owned
  // planes need the iterate and x on every function of the elements touching them
  const bool slab = c->ns_in != c->ns;
  if (slab) {
    int rc;
    if ((rc = dalloc(c->y_in, (size_t)c->N_in))) return rc;
    MI_CUDA(cudaMemsetAsync(c->y_in.p, 0, sizeof(double) * c->N_in, c->stream));
  }
  RxArgs r{};
  fill_args(c, r);
  r.x = x;
  r.lift_x = x0;
  r.y = slab ? c->y_in.p : y;
  int rc = c->rx_cw_ok ? (c->rx_cw_ws ? reaction_ws_mode<RX_STORED>(c, r) : reaction_launch<RX_STORED>(c, r))
                        : (use_reaction_ws(c) ? reaction_ws_mode<RX_FUSED>(c, r) : reaction_launch<RX_FUSED>(c, r));
  if (rc) return rc;
  if (slab) {
    dim3 g((unsigned)((c->ns + 255) / 256), c->nt);
    add_owned_planes<<<g, 256, 0, c->stream>>>(y, c->y_in.p, c->ns, c->ns_in,
                                               (long long)c->hz_lo * c->n[0] * c->n[1], c->nt);
    MI_CHECK_LAUNCH("add_owned_planes");
  }
  return MI_OK;
}

}  // namespace mi

using namespace mi;

extern "C" {

int mi_op_set_reaction(mi_ctx* c, const double* u, const double* w, double c1, double a, double c2,
                       const int* q, const int* nel, const double* B, const double* Wq) {
  MI_DEVICE_GUARD(c);
  if (c) c->rx_mapped = false;    // a mapped weight is re-attached by mi_op_set_reaction_weight
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(u && w && q && nel && B && Wq, MI_ERR_ARG, "NULL argument to mi_op_set_reaction");
  int rc;
  // u, w on the input slab (owned planes plus the z halo; = N unsharded)
  if ((rc = dalloc(c->u_it, c->N_in)) || (rc = dalloc(c->w_it, c->N_in))) return rc;
  MI_CUDA(cudaMemcpyAsync(c->u_it.p, u, sizeof(double) * c->N_in, cudaMemcpyDeviceToDevice, c->stream));
  MI_CUDA(cudaMemcpyAsync(c->w_it.p, w, sizeof(double) * c->N_in, cudaMemcpyDeviceToDevice, c->stream));
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
  c->rx_cw_dirty = true;
  return MI_OK;
}

int mi_op_set_reaction_weight(mi_ctx* c, const double* jw) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  if (jw == nullptr) {
    c->rx_mapped = false;
    return MI_OK;
  }
  MI_REQUIRE(c->ns_in == c->ns, MI_ERR_ARG, "mapped reaction weights are not supported on z-slab contexts");
  size_t nq = 1;
  for (int l = 0; l < c->d; ++l) nq *= (size_t)c->rx_nel[l] * c->rx_q[l];
  int rc;
  if ((rc = dalloc(c->rx_jw, nq))) return rc;
  MI_CUDA(cudaMemcpy(c->rx_jw.p, jw, sizeof(double) * nq, cudaMemcpyHostToDevice));
  c->rx_mapped = true;
  c->rx_cw_dirty = true;
  return MI_OK;
}

int mi_op_set_reaction_store(mi_ctx* c, int mode) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  MI_REQUIRE(mode >= -1 && mode <= 1, MI_ERR_ARG, "store mode must be -1, 0 or 1");
  c->rx_store_mode = mode;
  c->rx_cw_dirty = true;
  return MI_OK;
}

int mi_op_set_reaction_kernel(mi_ctx* c, int kernel) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  MI_REQUIRE(kernel >= -1 && kernel <= 1, MI_ERR_ARG, "kernel must be -1 (auto), 0 (reaction_tile) or 1 (reaction_ws)");
  MI_REQUIRE(kernel != 1 || (c->d == 3 && (c->p == 3 || c->p == 2) && c->pt == c->p), MI_ERR_ARG,
             "reaction_ws serves d = 3, p = p_t in {2, 3} only");
  c->rx_kernel = kernel;
  c->rx_cw_dirty = true;          // the stored coefficient's layout follows the kernel
  return MI_OK;
}

int mi_op_set_reaction_rows(mi_ctx* c, int row_offset) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  c->rx_rowoff = row_offset;
  c->rx_cw_dirty = true;
  return MI_OK;
}

int mi_op_clear_reaction(mi_ctx* c) {
  MI_DEVICE_GUARD(c);
  if (c) c->reaction_on = false;
  return MI_OK;
}

}  // extern "C"
