// Warp-specialised fused reaction kernel for d = 3, p = p_t in {2, 3} (BASELINE cfg 3 / 4 / 5 shapes):
// y += M_R x with C_r evaluated on the fly (reference reaction_mass, assembly.py:287-347; the
// algorithm is reaction_tile's, reaction.cu: time-streamed sum factorisation, q = p+1 Gauss rule).
//
// reaction_tile runs every stage on every warp with three block barriers per time slice; its ncu
// source page (gpurun rx12) puts 53% of the warp time into the x / y stages and their barriers,
// where almost no FP64 work issues, and the register window caps residency at 16 warps per SM.
// Here one 384-thread block per SM owns a 2 x 4 x 2 element tile (16 elements) and splits into
//   * CONSUMER warps (8 at p = 3, 4 Gauss points per thread; 9 at p = 2, 2 points per thread): z
//     interpolation of the entering slice (DMMA, accumulators = the window in registers), the
//     per-point time stage (DFMA) and the z projection of the finished function (DMMA, A fragments by
//     quad shuffles), software-pipelined in one basic block per slice;
//   * PRODUCER warps (4 / 3): the slice's u, w, x by cp.async into a double-buffered shared slice, x
//     and y interpolation of slice j + 1 and the y and x projections of a finished function (DMMA
//     through shared memory), the reductions into y.
// The two sides meet only on mbarriers (double-buffered y-interpolation output sB and z-projection
// output sC), so the consumers never stop at a block barrier; the producers synchronise among
// themselves on a named barrier.  Colour classes (3 x 2 x 3 = 18 launches) give every y entry one
// writer per launch, as in reaction_tile: deterministic sums.
#pragma once

#ifndef MI_RXWS_NPP
#define MI_RXWS_NPP 0      // > 0: projection warps (timing experiments)
#endif
#ifndef MI_RXWS_ST6
#define MI_RXWS_ST6 1
#endif
#ifndef MI_RXWS_E2
#define MI_RXWS_E2(p) ((p) == 2 ? 8 : 4)
#endif

namespace mi {

// MODE: RX_FUSED interpolates u, w, x and forms C_r every apply; RX_PRE (u, w) evaluates the weighted
// coefficient c_w = C_r w_x once per operator build into HBM; RX_STORED (x) applies M_R with it.
template <int P_, int MODE_>
struct RxWS {
  static constexpr int P = P_, QE = P + 1, PW = P + 1, QT = P + 1;
  static constexpr int MODE = MODE_, NF = MODE == RX_FUSED ? 3 : (MODE == RX_PRE ? 2 : 1);
  static constexpr int E1 = 2, E2 = MI_RXWS_E2(P), E3 = 2;          // p = 2: a longer tile, more work per slice step
  static constexpr int L1 = E1 + P, L2 = E2 + P, L3 = E3 + P;          // p = 3: 5, 7, 5 functions
  static constexpr int Q1 = E1 * QE, Q2 = E2 * QE, Q3 = E3 * QE;       // p = 3: 8, 16, 8 Gauss points
  static constexpr int RC1 = (L1 + E1 - 1) / E1, RC2 = (L2 + E2 - 1) / E2, RC3 = (L3 + E3 - 1) / E3;   // 3, 2, 3
  static constexpr int LS = L1 * L2 * L3;                               // functions per slice and field
  static constexpr int QL = Q1 * Q2;                                    // (q2, q1) lines of the z stage
  static constexpr int NT = (QL + 7) / 8;                               // their 8-line tiles: 16 (p = 3), 9 (p = 2)
  // consumer warps (the rest of the 12 produce).  The stored mode's consumers have little to do per
  // slice (one field, no C_r): p = 2 gives half of the warps to the producers there
  static constexpr int NCW = NT % 9 == 0 ? ((MODE == RX_STORED && NT == 18 && MI_RXWS_ST6) ? 6 : 9) : 8;
  static constexpr int MT = (NT + NCW - 1) / NCW;                       // line tiles per consumer warp
  static constexpr int NPW = 12 - NCW, NCT = 32 * NCW, NPT = 32 * NPW, NTH = NCT + NPT;
  static constexpr bool REGSPLIT = NCW % 4 == 0 && NPW % 4 == 0;       // setmaxnreg works on groups of 4 warps
  static_assert(MT * NCW == NT && NT * 8 == QL && Q3 <= 8 && Q1 <= 8 && L1 == L3 && Q1 == Q3, "tile shape");
  // the consumer's second line tile (mi = 1) sits a whole number of q2 rows above the first
  static_assert(MT == 1 || (8 * NCW) % Q1 == 0, "line tiles of a consumer warp");
  static constexpr int MIQ2 = 8 * NCW / Q1;                             // q2 rows between them
  // leading functions of a K = L interpolation taken as rank-1 updates on the CUDA cores, so that the
  // DMMA covers the last 4 functions in ONE k-step (p = 3: K = 5 = 1 + 4; p = 2: K = 4)
  static constexpr int R1 = L1 - 4;
  static_assert(R1 == 0 || R1 == 1, "x / z interpolation: one k-step plus at most one rank-1 update");
  static constexpr int KY = (L2 + 3) / 4, NY = (Q2 + 7) / 8;           // y interpolation k-steps / N tiles
  static constexpr int KZP = (Q3 + 3) / 4, KYP = (Q2 + 3) / 4, KXP = (Q1 + 3) / 4;   // projection k-steps
  static constexpr int NYP = (L2 + 7) / 8;                              // N tiles of the y projection
  // shared-memory strides (doubles), chosen so the DMMA operand loads / accumulator stores of the
  // p = 3 shapes touch each bank pair exactly twice (p = 2 keeps dense rows: a few 3-way conflicts)
  static constexpr int IS1 = P == 3 ? 6 : L1;                           // sIn rows
  static constexpr int BS1 = P == 3 ? Q1 + 4 : Q1;                      // sB q2 rows
  static constexpr int BJ = Q2 * BS1 + ((8 - (Q2 * BS1) % 16) + 16) % 16;   // sB planes = 8 mod 16
  static constexpr int CS = QL + ((4 - QL % 8) + 8) % 8;                // sC rows = 4 mod 8
  static constexpr int DS1 = P == 3 ? 12 : Q1;                          // sD rows
  static constexpr int SIN = NF * L3 * L2 * IS1;
  static constexpr int SA = NF * L3 * L2 * Q1 + (NF * L3 * L2 * Q1) % 2;
  static constexpr int SB = NF * L3 * BJ;                               // x2 buffers
  static constexpr int SC = L3 * CS;                                    // x2 buffers
  static constexpr int SD = L3 * L2 * DS1 + 96;                         // + over-read pad
  static constexpr int SBT = NCW * 64;                                  // per consumer warp [2][32] time tables
  // RX_STORED: the c_w block of one (tile, time element), [g][line][q3], streams through a ring of
  // NSW stages (one bulk copy per element, issued NSW - 1 elements ahead by a producer thread)
  static constexpr int NSW = 4, CWB = QT * QL * Q3;
  static constexpr int SW = MODE == RX_STORED ? NSW * CWB : 0;
  static constexpr int NDBL0 = 2 * SIN + SA + 2 * SB + 2 * SC + SD + SBT;
  static constexpr int NDBL = NDBL0 + NDBL0 % 2 + SW;                   // the ring starts 16-byte aligned
  static constexpr size_t SMEM = (size_t)NDBL * 8 + (8 + 2 * NSW) * 8;  // + mbarriers
  static_assert(CWB % 2 == 0 && SMEM <= 227 * 1024, "c_w ring");
  static_assert(BJ % 16 == 8 && CS % 8 == 4 && (2 * SIN) % 2 == 0 && SA % 2 == 0, "padding");
  // tiles of the producer stages
  static constexpr int XI_T = (NF * L3 * L2 + 7) / 8, YI_T = (NF * L3 * Q1 + 7) / 8;
  static constexpr int YP_T = (L3 * Q1 + 7) / 8, XP_T = (L3 * L2 + 7) / 8;
  // The producers split into an INTERPOLATION group (loads, x / y interpolation of the next slice) and a
  // PROJECTION group (y / x projection of a finished function, the reductions into y), each with its own
  // named barrier: their per-slice chains run side by side instead of one after the other (at p = 2 the
  // chain, not the FP64 pipe, bounds the kernel).  RX_PRE has nothing to project.
  static constexpr int NPP = MODE == RX_PRE ? 0 : (MI_RXWS_NPP > 0 ? MI_RXWS_NPP : (NPW >= 6 ? 2 : 1));
  static constexpr int NPI = NPW - NPP, NIT_T = 32 * NPI, NPR_T = 32 * (NPP > 0 ? NPP : NPW);
  static constexpr int NPJ = NPP > 0 ? NPP : NPW;                       // warps that project
  static constexpr int XI_U = (XI_T + NPI - 1) / NPI, YI_U = (YI_T + NPI - 1) / NPI;
  static constexpr int YP_U = (YP_T + NPJ - 1) / NPJ, XP_U = (XP_T + NPJ - 1) / NPJ;
  static constexpr int NIT = (LS + NIT_T - 1) / NIT_T;                  // input positions per interpolation thread
  // the unpredicated operand loads of padded rows / k columns stay inside the shared-memory carve-up
  static_assert(SIN + (XI_T * 8 - 1) * IS1 + R1 + 3 < 2 * SIN + SA, "x interpolation over-read");
  static_assert((((YI_T * 8 - 1) / Q1) * L2 + 4 * (KY - 1) + 3) * Q1 + Q1 - 1 < SA + SB, "y interpolation over-read");
  static_assert(((NF - 1) * L3 + R1 + 3) * BJ + MIQ2 * BS1 * (MT - 1) + (Q2 - 1) * BS1 + Q1 - 1 < SB + SC,
                "z interpolation over-read");
  static_assert(((YP_T * 8 - 1) / Q1) * CS + (4 * (KYP - 1) + 3) * Q1 + Q1 - 1 < SC + SD, "y projection over-read");
  static_assert((XP_T * 8 - 1) * DS1 + 4 * (KXP - 1) + 3 < SD, "x projection over-read");
};

#ifndef MI_RXWS_REGC
#define MI_RXWS_REGC 216   // consumer registers after the split (256 x REGC + 128 x REGP <= 384 x 168)
#endif
#ifndef MI_RXWS_REGP
#define MI_RXWS_REGP 72
#endif
#ifndef MI_RXWS_ABL
#define MI_RXWS_ABL 0      // timing ablations (wrong results): 1 no time stage, 2 no producer DMMAs, 4 no z stages
#endif
template <int N>
__device__ __forceinline__ void rxws_reg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void rxws_reg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N)); }

__device__ __forceinline__ void rxws_pdmma(double& c0, double& c1, double a, double b) {
  if (MI_RXWS_ABL & 2) { c0 += a; c1 += b; } else dmma(c0, c1, a, b);
}
__device__ __forceinline__ void rxws_cdmma(double& c0, double& c1, double a, double b) {
  if (MI_RXWS_ABL & 4) { c0 += a; c1 += b; } else dmma(c0, c1, a, b);
}
template <int ID, int NT>
__device__ __forceinline__ void rxws_bar_group() {
  asm volatile("bar.sync %0, %1;\n" ::"n"(ID), "n"(NT) : "memory");
}

template <int P_, int MODE>
__global__ void __launch_bounds__(RxWS<P_, MODE>::NTH, 1) reaction_ws(RxArgs r) {
  using G = RxWS<P_, MODE>;
  constexpr int P = G::P, QE = G::QE, PW = G::PW, QT = G::QT, NF = G::NF, PT = G::P;
  constexpr int L1 = G::L1, L2 = G::L2, L3 = G::L3, Q1 = G::Q1, Q2 = G::Q2;
  constexpr int BS1 = G::BS1, BJ = G::BJ, CS = G::CS, IS1 = G::IS1, DS1 = G::DS1, MT = G::MT, R1 = G::R1;
  extern __shared__ __align__(16) double sm[];
  double* sIn = sm;                 // [2][fld][j3][j2][IS1]
  double* sA = sIn + 2 * G::SIN;    // x-interpolation out [fld][j3][j2][q1]
  double* sB = sA + G::SA;          // [2] y-interpolation out [fld][j3] planes of (q2 rows BS1) + q1
  double* sC = sB + 2 * G::SB;      // [2] z-projection out [j3][CS: (q2, q1)]
  double* sD = sC + 2 * G::SC;      // y-projection out [j3][j2][DS1]
  double* sBt = sD + G::SD;         // [warp][2][32] time tables
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + G::NDBL);
  unsigned long long *fullB = bars, *emptyB = bars + 2, *fullC = bars + 4, *emptyC = bars + 6;
  [[maybe_unused]] unsigned long long *fullW = bars + 8, *emptyW = bars + 8 + G::NSW;
  [[maybe_unused]] double* sW = sm + (G::NDBL - G::SW);     // RX_STORED: c_w ring
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  // A-fragment loads run unpredicated over padded rows / k columns: whatever they read is finite (the
  // buffers start zeroed and only ever hold finite data) and meets a zero B entry or a discarded row
  for (int i = tid; i < G::NDBL; i += G::NTH) sm[i] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&fullB[b], G::NIT_T);
      mbar_init(&emptyB[b], G::NCT);
      mbar_init(&fullC[b], G::NCT);
      mbar_init(&emptyC[b], G::NPR_T);
    }
    if constexpr (MODE == RX_STORED) {
      for (int b = 0; b < G::NSW; ++b) {
        mbar_init(&fullW[b], 1);
        mbar_init(&emptyW[b], G::NCT);
      }
    }
    mbar_fence_init();
  }
  int k[3], ne[3];
  {
    const int EL[3] = {G::E1, G::E2, G::E3}, RCL[3] = {G::RC1, G::RC2, G::RC3};
    int b = blockIdx.x;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int m = b % r.ncol[l];
      b /= r.ncol[l];
      k[l] = (m * RCL[l] + r.color[l]) * EL[l];
      ne[l] = min(EL[l], r.nel[l] - k[l]);
    }
  }
  // local function j, local Gauss point q of direction l (0 outside the tile / the element's support)
  auto basis = [&](int l, int j, int q) -> double {
    const int Ll = l == 1 ? L2 : L1, Ql = l == 1 ? Q2 : Q1;       // L1 = L3, Q1 = Q3
    const int le = q / QE, gq = q % QE, aa = j - le;
    if (q >= Ql || j >= Ll || le >= ne[l] || aa < 0 || aa > P) return 0.0;
    return __ldg(r.B[l] + ((long long)(k[l] + le) * QE + gq) * (P + 1) + aa);
  };
  auto wgt = [&](int l, int q) -> double {
    const int Ql = l == 1 ? Q2 : Q1, le = q / QE;
    return (q < Ql && le < ne[l]) ? __ldg(r.Wq[l] + (long long)(k[l] + le) * QE + q % QE) : 0.0;
  };
  const int nelt = r.nel[3];
  const int nfull = nelt + PT;                       // full-basis time functions
  // c_w store: [tile][time element][g][line][q3], valid Gauss points only
  [[maybe_unused]] long long cw_tile = 0;
  if constexpr (MODE != RX_FUSED) {
    const long long nt1 = (r.nel[0] + G::E1 - 1) / G::E1, nt2 = (r.nel[1] + G::E2 - 1) / G::E2;
    cw_tile = (((long long)(k[2] / G::E3) * nt2 + k[1] / G::E2) * nt1 + k[0] / G::E1) * nelt;
  }
  __syncthreads();

  if (warp < G::NCW) {
    // =========================== consumers ===========================
    if constexpr (G::REGSPLIT) rxws_reg_inc<MI_RXWS_REGC>();   // the producers' released registers
    // z projection operand: B[k][n] = basis of function n at Gauss point q3 = 2 k + ks (the accumulator
    // layout of the z interpolation: lane k of a quad owns q3 = 2 k and 2 k + 1)
    static_assert(G::KZP <= 2, "z projection: two k-steps cover q3 = 2 k + ks < 8");
    double bP[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) bP[ks] = basis(2, fr, 2 * fk + ks);
    // z interpolation operands: the last 4 functions as the DMMA B fragment, a leading one (p = 3) at
    // this thread's two points
    const double bI1 = basis(2, R1 + fk, fr);
    const double bI0[2] = {R1 ? basis(2, 0, 2 * fk) : 0.0, R1 ? basis(2, 0, 2 * fk + 1) : 0.0};
    // the thread's Gauss points: line 8 (warp + NCW mi) + fr = (q2, q1), q3 = 2 fk + e.  The spatial
    // weight is folded into the x field as the slice enters the window.
    // (q2, q1) of line tile mi: q2 = q20 + MIQ2 mi, q1 = q10; offset in an sB plane loff0 + MIQ2 BS1 mi
    const int line0 = 8 * warp + fr, q20 = line0 / Q1, q10 = line0 % Q1, loff0 = q20 * BS1 + q10;
    double wsp[MT][2];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      const int q2 = q20 + G::MIQ2 * mi, q1 = q10;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int q3 = 2 * fk + e;
        double v = wgt(2, q3) * wgt(0, q1) * wgt(1, q2);
        if (r.jw != nullptr && v != 0.0) {
          const long long G1 = (long long)r.nel[0] * QE, G2 = (long long)r.nel[1] * QE;
          v *= __ldg(r.jw + ((long long)(k[2] * QE + q3) * G2 + k[1] * QE + q2) * G1 + k[0] * QE + q1);
        }
        wsp[mi][e] = v;
      }
    }
    double X[MT][PW][NF][2], Y[MT][PW][2];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int a = 0; a < PW; ++a) {
#pragma unroll
        for (int f = 0; f < NF; ++f) X[mi][a][f][0] = X[mi][a][f][1] = 0.0;
        Y[mi][a][0] = Y[mi][a][1] = 0.0;
      }
    // a thread's two points of a line tile are one aligned double2 of the c_w block
    constexpr int Q3 = G::Q3;
    [[maybe_unused]] const bool cw_lane = 2 * fk < Q3;
    [[maybe_unused]] auto cw_ptr = [&](int et, int g, int mi) -> double* {
      return r.cw + ((cw_tile + et) * QT + g) * (long long)(G::QL * Q3) + (8 * (warp + G::NCW * mi) + fr) * Q3 + 2 * fk;
    };
    double* myBt = sBt + warp * 64;
    const double* sBme = sB + loff0 + fk * BJ;       // this lane's DMMA operand column of buffer 0, function R1
    // time tables of element et: lanes 0-15 the basis values (interpolation), lanes 16-31 the same
    // times the Gauss weight (projection).  The loads are consumed one step later (no stall on them).
    double btb = 0.0, btw = 1.0;
    auto prefetch_bt = [&](int et) {
      btb = 0.0;                                     // no such element: all-zero tables (the step adds nothing)
      const int ga = lane & 15;
      if (et >= 0 && et < nelt && (QT * PW == 16 || ga < QT * PW)) {
        btb = __ldg(r.B[3] + (long long)et * QT * PW + ga);
        if (lane >= 16) btw = __ldg(r.Wq[3] + (long long)et * QT + ga / PW);
      }
    };
    // One software-pipelined slice step with compile-time window slots (PH = j % PW).  Three mutually
    // independent pieces share ONE basic block, so the DMMA / shuffle / shared-memory latencies of the
    // z stages hide behind the DFMA stream of the time stage of the same warp:
    //   * z interpolation of the entering slice j (its accumulators reach window slot PH only at the
    //     end of the step: the slot still holds function j - PW, the first one of this step's element);
    //   * the time stage of element et = j - PW (functions et + a in slot (PH + a) % PW);
    //   * the z projection of function fz = et - 1, completed by the previous step (its Y slot, copied
    //     out first, is the one this step starts to fill for function et + PT).
    // Steps without a valid element run the time stage on all-zero tables (no branch), steps without an
    // entering slice interpolate stale (finite) data into a slot nothing reads.
    auto step = [&](auto phc, int j) {
      constexpr int PH = decltype(phc)::value, SZ = (PH + PW - 1) % PW;
      const int et = j - PW, fz = et - 1;
      const bool has_in = j < nfull, has_fz = MODE != RX_PRE && fz >= 0;     // fz < nfull by the loop bound
      const int bb = j & 1, cb = fz & 1;
      myBt[bb * 32 + lane] = btb * btw;
      __syncwarp();
      prefetch_bt(et + 1);
      if (has_in) mbar_wait(&fullB[bb], (unsigned)((j >> 1) & 1));
      if (MODE != RX_PRE && fz >= 2) mbar_wait(&emptyC[cb], (unsigned)(((fz >> 1) - 1) & 1));
      // ---- RX_STORED: this element's c_w from the ring
      [[maybe_unused]] double2 cwl[QT][MT];
      if constexpr (MODE == RX_STORED) {
#pragma unroll
        for (int g = 0; g < QT; ++g)
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) cwl[g][mi] = make_double2(0.0, 0.0);
        if (et >= 0 && et < nelt) {
          const int sw = et % G::NSW;
          mbar_wait(&fullW[sw], (unsigned)((et / G::NSW) & 1));
          if (cw_lane) {
            const double* blk = sW + sw * G::CWB + (8 * warp + fr) * Q3 + 2 * fk;
#pragma unroll
            for (int g = 0; g < QT; ++g)
#pragma unroll
              for (int mi = 0; mi < MT; ++mi)
                cwl[g][mi] = *reinterpret_cast<const double2*>(blk + g * (G::QL * Q3) + 8 * G::NCW * mi * Q3);
          }
          mbar_arrive(&emptyW[sw]);
        }
      }
      // ---- z interpolation of slice j
      const double* fin = sBme + bb * G::SB;
      double zc[MT][NF][2], a0[MT][NF], za[MT][NF];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          a0[mi][f] = R1 ? fin[f * L3 * BJ + G::MIQ2 * BS1 * mi - fk * BJ] : 0.0;
          za[mi][f] = fin[(f * L3 + R1) * BJ + G::MIQ2 * BS1 * mi];
        }
      const double* bt = myBt + bb * 32;
      double btv[2][QT * PW];
#pragma unroll
      for (int i = 0; i < QT * PW; ++i) btv[0][i] = bt[i], btv[1][i] = bt[16 + i];
      if (has_in) mbar_arrive(&emptyB[bb]);
      // ---- z projection operands of function fz (slot SZ), and the slot's fresh start
      double yz[MT][2], zp[MT][2];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) {
        yz[mi][0] = Y[mi][SZ][0], yz[mi][1] = Y[mi][SZ][1];
        Y[mi][SZ][0] = Y[mi][SZ][1] = 0.0;
        zp[mi][0] = zp[mi][1] = 0.0;
      }
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          zc[mi][f][0] = zc[mi][f][1] = 0.0;
          rxws_cdmma(zc[mi][f][0], zc[mi][f][1], za[mi][f], bI1);
        }
      // (the K order of this product is q3 = 2 k + ks: k-step ks takes every lane's OWN point e = ks, so
      // the A fragments need no shuffles)
#pragma unroll
      for (int ks = 0; ks < (MODE == RX_PRE ? 0 : 2); ++ks)
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) rxws_cdmma(zp[mi][0], zp[mi][1], yz[mi][ks], bP[ks]);
      // ---- time element et on the thread's own points, all chains interleaved
      if (!(MI_RXWS_ABL & 1)) {
#pragma unroll
        for (int g = 0; g < QT; ++g) {
          double acc[MT][NF][2];                     // fused: (u', p, x'); pre: (u', p); stored: (x)
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int f = 0; f < NF; ++f) acc[mi][f][0] = acc[mi][f][1] = 0.0;
#pragma unroll
          for (int a = 0; a < PW; ++a) {
            const double ba = btv[0][g * PW + a];
#pragma unroll
            for (int mi = 0; mi < MT; ++mi)
#pragma unroll
              for (int f = 0; f < NF; ++f)
#pragma unroll
                for (int e = 0; e < 2; ++e) acc[mi][f][e] = fma(ba, X[mi][(PH + a) % PW][f][e], acc[mi][f][e]);
          }
          if constexpr (MODE == RX_PRE) {
            // c_w = C_r w_x = (u'^2 + p) w_x at the thread's points of this (element, g)
            if (et >= 0 && et < nelt && cw_lane) {
#pragma unroll
              for (int mi = 0; mi < MT; ++mi)
                *reinterpret_cast<double2*>(cw_ptr(et, g, mi)) =
                    make_double2(fma(acc[mi][0][0], acc[mi][0][0], acc[mi][1][0]) * wsp[mi][0],
                                 fma(acc[mi][0][1], acc[mi][0][1], acc[mi][1][1]) * wsp[mi][1]);
            }
          } else {
            double v[MT][2];                         // C_r w_x x
#pragma unroll
            for (int mi = 0; mi < MT; ++mi) {
              if constexpr (MODE == RX_FUSED) {
                v[mi][0] = fma(acc[mi][0][0], acc[mi][0][0], acc[mi][1][0]) * acc[mi][2][0];
                v[mi][1] = fma(acc[mi][0][1], acc[mi][0][1], acc[mi][1][1]) * acc[mi][2][1];
              } else {
                v[mi][0] = cwl[g][mi].x * acc[mi][0][0];
                v[mi][1] = cwl[g][mi].y * acc[mi][0][1];
              }
            }
#pragma unroll
            for (int a = 0; a < PW; ++a) {
              const double bw = btv[1][g * PW + a];
#pragma unroll
              for (int mi = 0; mi < MT; ++mi)
#pragma unroll
                for (int e = 0; e < 2; ++e) Y[mi][(PH + a) % PW][e] = fma(bw, v[mi][e], Y[mi][(PH + a) % PW][e]);
            }
          }
        }
      }
      // ---- the entering slice reaches its window slot: (sqrt(c1) u, p) arrive transformed by the
      // producers; x takes its spatial weight here (stored mode: the weight is in c_w)
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const double cf = R1 ? fma(a0[mi][f], bI0[e], zc[mi][f][e]) : zc[mi][f][e];
            X[mi][PH][f][e] = (MODE == RX_FUSED && f == 2) ? cf * wsp[mi][e] : cf;
          }
      // ---- projected function fz to the producers
      if (has_fz) {
        double* out = sC + cb * G::SC;
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) {
          const int line = 8 * (warp + G::NCW * mi) + fr, n0 = 2 * fk;
          if (n0 < L3) out[n0 * CS + line] = zp[mi][0];
          if (n0 + 1 < L3) out[(n0 + 1) * CS + line] = zp[mi][1];
        }
        mbar_arrive(&fullC[cb]);
      }
    };
    const int nsteps = nfull + PW + 1;               // the last step projects function nfull - 1
    for (int j0 = 0; j0 < nsteps; j0 += PW) {
      step(std::integral_constant<int, 0>{}, j0);
      if (j0 + 1 < nsteps) step(std::integral_constant<int, 1>{}, j0 + 1);
      if (j0 + 2 < nsteps) step(std::integral_constant<int, 2>{}, j0 + 2);
      if constexpr (PW > 3)
        if (j0 + 3 < nsteps) step(std::integral_constant<int, 3 % PW>{}, j0 + 3);
    }
  } else {
    // =========================== producers ===========================
    if constexpr (G::REGSPLIT) rxws_reg_dec<MI_RXWS_REGP>();
    const int pw = warp - G::NCW;
    const long long ns = r.ns;
    // spatial indices fit in 32 bits (the launcher checks N_s < 2^31)
    auto spatial = [&](int j3, int j2, int j1, bool& ok) -> int {
      const int g1 = k[0] + j1, g2 = k[1] + j2, g3 = k[2] + j3;
      ok = g1 < r.n[0] && g2 < r.n[1] && g3 < r.n[2];
      return (g3 * r.n[1] + g2) * r.n[0] + g1;
    };
    if (pw < G::NPI) {
      // ----------------- interpolation group: loads, x and y interpolation of slice i -----------------
      constexpr int NPI = G::NPI, NT_ = G::NIT_T;
      const int p = tid - G::NCT;
      double bIy[G::NY][G::KY];
      const double bIx1 = basis(0, R1 + fk, fr);
      const double bIx0[2] = {R1 ? basis(0, 0, 2 * fk) : 0.0, R1 ? basis(0, 0, 2 * fk + 1) : 0.0};
#pragma unroll
      for (int ks = 0; ks < G::KY; ++ks)
#pragma unroll
        for (int n2 = 0; n2 < G::NY; ++n2) bIy[n2][ks] = basis(1, 4 * ks + fk, 8 * n2 + fr);
      // Input slice items of this thread: spatial positions s = p + NT_ h (s < LS) of all the mode's fields.
      // The slice is copied asynchronously (cp.async, zeros for padding / constrained rows) straight into
      // the double-buffered sIn: no register staging, and no global-load scoreboard in front of the
      // x-interpolation DMMAs.
      int gsp[G::NIT];                               // global spatial index (-1: outside the domain, -2: no item)
      unsigned sdst[G::NIT];                         // shared address of the field-0 copy in buffer 0
      int sof[G::NIT];                               // ... and its offset in sIn (doubles)
#pragma unroll
      for (int h = 0; h < G::NIT; ++h) {
        const int sp = p + NT_ * h;
        const int j3 = sp / (L1 * L2), j2 = (sp / L1) % L2, j1 = sp % L1;
        bool ok;
        const int gs = spatial(j3, j2, j1, ok);
        gsp[h] = sp < G::LS ? (ok ? gs : -1) : -2;
        sof[h] = sp < G::LS ? (j3 * L2 + j2) * IS1 + j1 : 0;
        sdst[h] = (unsigned)__cvta_generic_to_shared(sIn + sof[h]);
      }
      // C_r = c1 (u - a)(u - 1) + c2 w = (sqrt(c1) u)^2 + p with p = c2 w - c1 (1 + a) u + c1 a LINEAR in
      // the coefficients: every thread turns its own landed (u, w) items into (sqrt(c1) u, p) in place, so
      // the consumers interpolate u' and p directly and form C_r with ONE fused multiply-add per Gauss
      // point.  (The constant c1 a rides on the coefficients because the basis sums to 1 at every Gauss
      // point in every direction; zero slabs and padding become p = c1 a, as C_r of u = w = 0 is.)
      [[maybe_unused]] const double rsq = sqrt(r.c1), rk1 = -r.c1 * (1.0 + r.a), rk0 = r.c1 * r.a, rc2 = r.c2;
      auto put = [&](unsigned dst, const double* src, bool valid) {   // one double: async copy, or a zero
        if (valid)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
        else
          asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(dst), "d"(0.0) : "memory");
      };
      auto issue = [&](int ft) {
        const int ct = ft + r.rowoff;
        const unsigned boff = (unsigned)((ft & 1) * G::SIN * 8);
        constexpr unsigned FO = L3 * L2 * IS1 * 8;   // field stride in sIn (bytes)
        // fields of this mode: fused (u, w, x), pre (u, w), stored (x)
        const double* fld[3] = {MODE == RX_STORED ? r.x : r.u, r.w, r.x};
        const double* lft[3] = {MODE == RX_STORED ? r.lift_x : r.lift_u, nullptr, r.lift_x};
        if (ct >= 0 && ct < r.ntc) {
          const long long off = (long long)ct * ns;
#pragma unroll
          for (int h = 0; h < G::NIT; ++h) {
            if (gsp[h] != -2) {
              const bool v = gsp[h] >= 0;
              const int g = v ? gsp[h] : 0;
              const unsigned d = sdst[h] + boff;
#pragma unroll
              for (int f = 0; f < NF; ++f) put(d + f * FO, fld[f] + off + g, v);
            }
          }
        } else {
          // the lifted slab (row -1: u and x from the lift, if set) or a row outside this context: zeros
#pragma unroll
          for (int h = 0; h < G::NIT; ++h) {
            if (gsp[h] != -2) {
              const bool v = gsp[h] >= 0;
              const int g = v ? gsp[h] : 0;
              const unsigned d = sdst[h] + boff;
#pragma unroll
              for (int f = 0; f < NF; ++f) {
                const double* l = ct == -1 ? lft[f] : nullptr;
                put(d + f * FO, l + g, v && l != nullptr);
              }
            }
          }
        }
        cp_async_commit();
      };
      issue(0);
      [[maybe_unused]] int e_next = 0;               // RX_STORED: next c_w block to request
      for (int i = 0; i < nfull; ++i) {
        if constexpr (MODE == RX_STORED) {
          // c_w blocks NSW - 1 elements ahead of the consumers (who are on element i - 1 - PW); a stage is
          // free once they have read element e - NSW, which they did steps ago
          if (p == 0) {
            for (; e_next < nelt && e_next <= i - PW + G::NSW - 2; ++e_next) {
              const int sw = e_next % G::NSW, kuse = e_next / G::NSW;
              if (kuse >= 1) mbar_wait(&emptyW[sw], (unsigned)((kuse - 1) & 1));
              mbar_expect_tx(&fullW[sw], (unsigned)(G::CWB * 8));
              bulk_g2s(sW + sw * G::CWB, r.cw + (cw_tile + e_next) * (long long)G::CWB, (unsigned)(G::CWB * 8),
                       &fullW[sw]);
            }
          }
        }
        cp_async_wait<0>();                          // this thread's copies of slice i have landed ...
        if constexpr (MODE != RX_STORED) {
          double* sI = sIn + (i & 1) * G::SIN;
#pragma unroll
          for (int h = 0; h < G::NIT; ++h) {
            if (gsp[h] != -2) {
              const double uv = sI[sof[h]], wv = sI[sof[h] + L3 * L2 * IS1];
              sI[sof[h]] = uv * rsq;
              sI[sof[h] + L3 * L2 * IS1] = fma(uv, rk1, fma(wv, rc2, rk0));
            }
          }
        }
        rxws_bar_group<1, NT_>();                    // ... and everyone's; the other sIn buffer is free
        if (i + 1 < nfull) issue(i + 1);
        {
          const double* sI = sIn + (i & 1) * G::SIN;
          // x interpolation of slice i: lines (fld, j3, j2), K = j1, N = q1 -> sA.  The last 4 functions in
          // ONE DMMA, a leading one (first element's Gauss points only) as a rank-1 update
          constexpr int NL = NF * L3 * L2;
          double c[G::XI_U][2], a0[G::XI_U];
#pragma unroll
          for (int u = 0; u < G::XI_U; ++u) {
            c[u][0] = c[u][1] = 0.0;
            a0[u] = 0.0;
            const int mt = pw + NPI * u;
            if (mt < G::XI_T) {
              const double* row = sI + (mt * 8 + fr) * IS1;
              if (R1) a0[u] = row[0];
              rxws_pdmma(c[u][0], c[u][1], row[R1 + fk], bIx1);
            }
          }
#pragma unroll
          for (int u = 0; u < G::XI_U; ++u) {
            const int line = (pw + NPI * u) * 8 + fr;
            if (line < NL && 2 * fk < Q1)
              *reinterpret_cast<double2*>(sA + line * Q1 + 2 * fk) =
                  make_double2(fma(a0[u], bIx0[0], c[u][0]), fma(a0[u], bIx0[1], c[u][1]));
          }
        }
        rxws_bar_group<1, NT_>();
        {
          // y interpolation of slice i: lines (fld j3, q1), K = j2, N = q2 -> sB[i & 1]
          const int bb = i & 1;
          constexpr int NL = NF * L3 * Q1;
          double* out = sB + bb * G::SB;
#pragma unroll
          for (int h = 0; h < (G::YI_U + 1) / 2; ++h) {   // two line tiles at a time (register budget)
            double c[2][G::NY][2];
            int fj3[2], q1[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
#pragma unroll
              for (int n2 = 0; n2 < G::NY; ++n2) c[u][n2][0] = c[u][n2][1] = 0.0;
              const int mt = pw + NPI * (2 * h + u), line = mt * 8 + fr;
              fj3[u] = Q1 == 8 ? mt : line / Q1, q1[u] = Q1 == 8 ? fr : line % Q1;
              if (2 * h + u < G::YI_U && mt < G::YI_T) {
#pragma unroll
                for (int ks = 0; ks < G::KY; ++ks) {
                  const double av = sA[(fj3[u] * L2 + 4 * ks + fk) * Q1 + q1[u]];
#pragma unroll
                  for (int n2 = 0; n2 < G::NY; ++n2) rxws_pdmma(c[u][n2][0], c[u][n2][1], av, bIy[n2][ks]);
                }
              }
            }
            if (h == 0 && i >= 2) mbar_wait(&emptyB[bb], (unsigned)(((i >> 1) - 1) & 1));
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int mt = pw + NPI * (2 * h + u), line = mt * 8 + fr;
              if (2 * h + u < G::YI_U && line < NL) {
#pragma unroll
                for (int n2 = 0; n2 < G::NY; ++n2) {
                  const int n0 = 8 * n2 + 2 * fk;
                  if (n0 < Q2) out[fj3[u] * BJ + n0 * BS1 + q1[u]] = c[u][n2][0];
                  if (n0 + 1 < Q2) out[fj3[u] * BJ + (n0 + 1) * BS1 + q1[u]] = c[u][n2][1];
                }
              }
            }
          }
          mbar_arrive(&fullB[bb]);
        }
      }
    } else if constexpr (G::NPP > 0) {
      // ----------------- projection group: y and x projection of function fq, reductions into y -----------------
      constexpr int NPP = G::NPP, NT_ = G::NPR_T;
      const int pp = pw - G::NPI;
      double bPy[G::NYP][G::KYP], bPx[G::KXP];
#pragma unroll
      for (int ks = 0; ks < G::KXP; ++ks) bPx[ks] = basis(0, fr, 4 * ks + fk);
#pragma unroll
      for (int ks = 0; ks < G::KYP; ++ks)
#pragma unroll
        for (int n2 = 0; n2 < G::NYP; ++n2) bPy[n2][ks] = basis(1, 8 * n2 + fr, 4 * ks + fk);
      // x-projection outputs of this thread: line tiles mt = pp + NPP u, xline = 8 mt + fr = (j3, j2), j1 = 2 fk + e
      int yidx[G::XP_U][2];
#pragma unroll
      for (int u = 0; u < G::XP_U; ++u)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int xline = 8 * (pp + NPP * u) + fr, j1 = 2 * fk + e;
          bool ok = false;
          int gs = 0;
          if (xline < L3 * L2 && j1 < L1) gs = spatial(xline / L2, xline % L2, j1, ok);
          yidx[u][e] = ok ? gs : -1;
        }
      for (int fq = 0; fq < nfull; ++fq) {
        {
          // y projection of function fq: lines (j3, q1), K = q2, N = j2: sC[fq & 1] -> sD
          const int cb = fq & 1;
          mbar_wait(&fullC[cb], (unsigned)((fq >> 1) & 1));
          const double* in = sC + cb * G::SC;
          constexpr int NL = L3 * Q1;
          double c[G::YP_U][G::NYP][2];
          int j3[G::YP_U], q1[G::YP_U];
#pragma unroll
          for (int u = 0; u < G::YP_U; ++u) {
#pragma unroll
            for (int n2 = 0; n2 < G::NYP; ++n2) c[u][n2][0] = c[u][n2][1] = 0.0;
            const int mt = pp + NPP * u, line = 8 * mt + fr;
            j3[u] = Q1 == 8 ? mt : line / Q1, q1[u] = Q1 == 8 ? fr : line % Q1;
            if (mt < G::YP_T) {
#pragma unroll
              for (int ks = 0; ks < G::KYP; ++ks) {
                const double av = in[j3[u] * CS + (4 * ks + fk) * Q1 + q1[u]];
#pragma unroll
                for (int n2 = 0; n2 < G::NYP; ++n2) rxws_pdmma(c[u][n2][0], c[u][n2][1], av, bPy[n2][ks]);
              }
            }
          }
          mbar_arrive(&emptyC[cb]);
#pragma unroll
          for (int u = 0; u < G::YP_U; ++u) {
            const int line = 8 * (pp + NPP * u) + fr;
            if (line < NL) {
#pragma unroll
              for (int n2 = 0; n2 < G::NYP; ++n2) {
                const int n0 = 8 * n2 + 2 * fk;
                if (n0 < L2) sD[(j3[u] * L2 + n0) * DS1 + q1[u]] = c[u][n2][0];
                if (n0 + 1 < L2) sD[(j3[u] * L2 + n0 + 1) * DS1 + q1[u]] = c[u][n2][1];
              }
            }
          }
        }
        rxws_bar_group<2, NT_>();
        {
          // x projection of function fq: lines (j3, j2), K = q1, N = j1 -> y (fire-and-forget reductions:
          // one writer per y entry per colour launch, stream-ordered launches: deterministic)
          const int ct = fq + r.rowoff;
          const long long row = (ct >= 0 && ct < r.ntc) ? (long long)ct * ns : -1;
#pragma unroll
          for (int u = 0; u < G::XP_U; ++u) {
            const int mt = pp + NPP * u;
            if (mt < G::XP_T) {
              const int xline = 8 * mt + fr;
              double c0 = 0.0, c1 = 0.0;
#pragma unroll
              for (int ks = 0; ks < G::KXP; ++ks) rxws_pdmma(c0, c1, sD[xline * DS1 + 4 * ks + fk], bPx[ks]);
              if (row >= 0) {
                if (yidx[u][0] >= 0) atomicAdd(r.y + row + yidx[u][0], c0);
                if (yidx[u][1] >= 0) atomicAdd(r.y + row + yidx[u][1], c1);
              }
            }
          }
        }
        rxws_bar_group<2, NT_>();                    // sD is free for the next function
      }
    }
  }
}

// all colour classes of the warp-specialised kernel (d = 3, p = p_t, fused mode)
template <int P_, int MODE>
static int reaction_ws_launch(mi_ctx* c, RxArgs r) {
  using G = RxWS<P_, MODE>;
  MI_DEV_FLAG(attr);
  if (!attr) {
    MI_CUDA(cudaFuncSetAttribute(reaction_ws<P_, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
    attr = true;
  }
  const int EL[3] = {G::E1, G::E2, G::E3}, RCL[3] = {G::RC1, G::RC2, G::RC3};
  for (int col = 0; col < G::RC1 * G::RC2 * G::RC3; ++col) {
    int cc = col;
    long long nb = 1;
    for (int l = 0; l < 3; ++l) {
      r.color[l] = cc % RCL[l];
      cc /= RCL[l];
      const int ntile = (c->rx_nel[l] + EL[l] - 1) / EL[l];
      r.ncol[l] = (ntile - r.color[l] + RCL[l] - 1) / RCL[l];
      nb *= r.ncol[l] > 0 ? r.ncol[l] : 0;
    }
    if (nb == 0) continue;
    reaction_ws<P_, MODE><<<(unsigned)nb, G::NTH, G::SMEM, c->stream>>>(r);
    MI_CHECK_LAUNCH("reaction_ws");
  }
  return MI_OK;
}

}  // namespace mi
