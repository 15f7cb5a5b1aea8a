// Warp-specialised fused reaction kernel for d = 3, p = p_t = 3 (BASELINE cfg 4 / cfg 5 shapes):
// y += M_R x with C_r evaluated on the fly (reference reaction_mass, assembly.py:287-347; the
// algorithm is reaction_tile's, reaction.cu: time-streamed sum factorisation, q = p+1 Gauss rule).
//
// reaction_tile runs every stage on every warp with three block barriers per time slice; its ncu
// source page (gpurun rx12) puts 53% of the warp time into the x / y stages and their barriers,
// where almost no FP64 work issues, and the register window caps residency at 16 warps per SM.
// Here one 384-thread block per SM owns a 2 x 4 x 2 element tile (16 elements, 8 x 16 x 8 spatial
// Gauss points) and splits into
//   * 8 CONSUMER warps: z interpolation of the entering slice (DMMA, accumulators = the window in
//     registers, 4 Gauss points per thread), the per-point time stage (DFMA) and the z projection
//     of the finished function (DMMA, A fragments by quad shuffles);
//   * 4 PRODUCER warps: global loads, x and y interpolation of slice j + 1 and the y and x
//     projections of function j - p_t - 1 (DMMA through shared memory), the reductions into y.
// The two sides meet only on mbarriers (double-buffered y-interpolation output sB and z-projection
// output sC), so the consumers never stop at a block barrier; the producers synchronise among
// themselves on a named barrier.  Colour classes (3 x 2 x 3 = 18 launches) give every y entry one
// writer per launch, as in reaction_tile: deterministic sums.
#pragma once

namespace mi {

struct RxWS {
  static constexpr int P = 3, QE = 4, PW = 4, QT = 4, NF = 3;
  static constexpr int E1 = 2, E2 = 4, E3 = 2;
  static constexpr int L1 = E1 + P, L2 = E2 + P, L3 = E3 + P;          // 5, 7, 5 functions
  static constexpr int Q1 = E1 * QE, Q2 = E2 * QE, Q3 = E3 * QE;       // 8, 16, 8 Gauss points
  static constexpr int RC1 = (L1 + E1 - 1) / E1, RC2 = (L2 + E2 - 1) / E2, RC3 = (L3 + E3 - 1) / E3;   // 3, 2, 3
  static constexpr int LS = L1 * L2 * L3, NIN = NF * LS;              // 175, 525
  static constexpr int NCW = 8, NPW = 4, NCT = 32 * NCW, NPT = 32 * NPW, NTH = NCT + NPT;
  static constexpr int QL = Q1 * Q2;                                    // 128 (q2, q1) lines of the z stage
  static constexpr int MT = QL / 8 / NCW;                               // 2 line tiles per consumer warp
  // shared-memory strides (doubles), chosen so every DMMA operand load / accumulator store touches each
  // bank pair exactly twice: sIn rows 6 (5 functions), sB q2 rows 12, sB planes = 8 mod 16, sC rows = 4
  // mod 8, sD rows 12
  static constexpr int IS1 = 6, BS1 = Q1 + 4, BJ = Q2 * BS1 + 8, CS = QL + 4, DS1 = 12;
  static constexpr int SIN = NF * L3 * L2 * IS1;                        // 630
  static constexpr int SA = NF * L3 * L2 * Q1;                          // 840
  static constexpr int SB = NF * L3 * BJ;                               // 3000 (x2 buffers)
  static constexpr int SC = L3 * CS;                                    // 660  (x2 buffers)
  static constexpr int SD = L3 * L2 * DS1 + 76;                         // 420 + over-read pad
  static constexpr int SBT = NCW * 64;                                  // per consumer warp [2][32] time tables
  static constexpr int NDBL = 2 * SIN + SA + 2 * SB + 2 * SC + SD + SBT;
  static constexpr size_t SMEM = (size_t)NDBL * 8 + 8 * 8;              // + 8 mbarriers
  static_assert(BJ % 16 == 8 && CS % 8 == 4 && NDBL % 2 == 0, "padding");
  static_assert(MT * NCW * 8 == QL, "consumer tiling");
};

#ifndef MI_RXWS_REGC
#define MI_RXWS_REGC 208   // consumer registers after the split (256 x REGC + 128 x REGP <= 384 x 168)
#endif
#ifndef MI_RXWS_REGP
#define MI_RXWS_REGP 88
#endif
#ifndef MI_RXWS_ABL
#define MI_RXWS_ABL 0      // timing ablations (wrong results): 1 no time stage, 2 no producer DMMAs, 4 no z stages
#endif
#ifndef MI_RXWS_SKEW
#define MI_RXWS_SKEW 0
#endif
#ifndef MI_RXWS_UNROLL
#define MI_RXWS_UNROLL 1   // consumer slice loop unrolled by p_t + 1 (compile-time window slots, no rotation copies)
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
__device__ __forceinline__ void rxws_bar_producers() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(RxWS::NPT) : "memory");
}

__global__ void __launch_bounds__(RxWS::NTH, 1) reaction_ws(RxArgs r) {
  using G = RxWS;
  constexpr int P = G::P, QE = G::QE, PW = G::PW, QT = G::QT, NF = G::NF, PT = G::P;
  constexpr int L1 = G::L1, L2 = G::L2, L3 = G::L3, Q1 = G::Q1, Q2 = G::Q2, Q3 = G::Q3;
  constexpr int BS1 = G::BS1, BJ = G::BJ, CS = G::CS, IS1 = G::IS1, DS1 = G::DS1, MT = G::MT;
  extern __shared__ __align__(16) double sm[];
  double* sIn = sm;                 // [2][fld][j3][j2][IS1]
  double* sA = sIn + 2 * G::SIN;    // x-interpolation out [fld][j3][j2][q1]
  double* sB = sA + G::SA;          // [2] y-interpolation out [fld][j3] planes of (q2 rows BS1) + q1
  double* sC = sB + 2 * G::SB;      // [2] z-projection out [j3][CS: (q2, q1)]
  double* sD = sC + 2 * G::SC;      // y-projection out [j3][j2][DS1]
  double* sBt = sD + G::SD;         // [warp][2][32] time tables
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sBt + G::SBT);
  unsigned long long *fullB = bars, *emptyB = bars + 2, *fullC = bars + 4, *emptyC = bars + 6;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  // A-fragment loads run unpredicated over padded rows / k columns: whatever they read is finite (the
  // buffers start zeroed and only ever hold finite data) and meets a zero B entry or a discarded row
  for (int i = tid; i < G::NDBL; i += G::NTH) sm[i] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&fullB[b], G::NPT);
      mbar_init(&emptyB[b], G::NCT);
      mbar_init(&fullC[b], G::NCT);
      mbar_init(&emptyC[b], G::NPT);
    }
    mbar_fence_init();
  }
  int k[3], ne[3];
  {
    constexpr int EL[3] = {G::E1, G::E2, G::E3}, RCL[3] = {G::RC1, G::RC2, G::RC3};
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
    const int le = q / QE;
    return le < ne[l] ? __ldg(r.Wq[l] + (long long)(k[l] + le) * QE + q % QE) : 0.0;
  };
  const int nelt = r.nel[3];
  const int nfull = nelt + PT;                       // full-basis time functions
  __syncthreads();

  if (warp < G::NCW) {
    // =========================== consumers ===========================
    rxws_reg_inc<MI_RXWS_REGC>();                    // the producers' released registers: window + ILP-4 time stage
    double bP[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) bP[ks] = basis(2, fr, 4 * ks + fk);
    // z interpolation operands: functions 1..4 as the DMMA B fragment, function 0 at this thread's two points
    const double bI1 = basis(2, 1 + fk, fr);
    const double bI0[2] = {basis(2, 0, 2 * fk), basis(2, 0, 2 * fk + 1)};
    // the thread's Gauss points: line tile t = warp + 8 mi (q2 = t, q1 = fr), q3 = 2 fk + e.  The spatial
    // weight is folded into the x field and c2 into the w field as the slice enters the window.
    double wsp[MT][2];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int q2 = warp + G::NCW * mi, q3 = 2 * fk + e;
        double v = wgt(2, q3) * wgt(0, fr) * wgt(1, q2);
        if (r.jw != nullptr && v != 0.0) {
          const long long G1 = (long long)r.nel[0] * QE, G2 = (long long)r.nel[1] * QE;
          v *= __ldg(r.jw + ((long long)(k[2] * QE + q3) * G2 + k[1] * QE + q2) * G1 + k[0] * QE + fr);
        }
        wsp[mi][e] = v;
      }
    const double rsq = sqrt(r.c1), rk1 = -r.c1 * (1.0 + r.a), rk0 = r.c1 * r.a, rc2 = r.c2;   // c1 >= 0 (launcher)
    double X[MT][PW][NF][2], Y[MT][PW][2];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int a = 0; a < PW; ++a) {
#pragma unroll
        for (int f = 0; f < NF; ++f) X[mi][a][f][0] = X[mi][a][f][1] = 0.0;
        Y[mi][a][0] = Y[mi][a][1] = 0.0;
      }
    double* myBt = sBt + warp * 64;
    // time tables of element et: lanes 0-15 the basis values (interpolation), lanes 16-31 the same
    // times the Gauss weight (projection).  The loads are consumed one step later (no stall on them).
    double btb = 0.0, btw = 1.0;
    auto prefetch_bt = [&](int et) {
      btb = 0.0;                                     // no such element: all-zero tables (the step adds nothing)
      if (et >= 0 && et < nelt) {
        const int ga = lane & 15;
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
      const bool has_in = j < nfull, has_fz = fz >= 0;     // fz < nfull by the loop bound
      const int bb = j & 1, cb = fz & 1;
      myBt[bb * 32 + lane] = btb * btw;
      __syncwarp();
      prefetch_bt(et + 1);
      if (has_in) mbar_wait(&fullB[bb], (unsigned)((j >> 1) & 1));
      if (fz >= 2) mbar_wait(&emptyC[cb], (unsigned)(((fz >> 1) - 1) & 1));
      // ---- z interpolation of slice j: functions 1..4 in ONE DMMA (k = fk), function 0 as a rank-1
      // update on the CUDA cores (it only reaches the first element's Gauss points: bI0 is zero elsewhere)
      const double* fin = sB + bb * G::SB + fr;
      double zc[MT][NF][2], a0[MT][NF], za[MT][NF];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const double* fp = fin + f * L3 * BJ + (warp + G::NCW * mi) * BS1;
          a0[mi][f] = fp[0];
          za[mi][f] = fp[(1 + fk) * BJ];
        }
      const double* bt = myBt + bb * 32;
      double btv[2 * QT * PW];
#pragma unroll
      for (int i = 0; i < 2 * QT * PW; ++i) btv[i] = bt[i];
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
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) {
          const int cc = 4 * ks + fk, src = (lane & ~3) | (cc >> 1);
          const double v0 = __shfl_sync(0xffffffffu, yz[mi][0], src);
          const double v1 = __shfl_sync(0xffffffffu, yz[mi][1], src);
          rxws_cdmma(zp[mi][0], zp[mi][1], (cc & 1) ? v1 : v0, bP[ks]);
        }
      // ---- time element et on the thread's own four points, all chains interleaved
      if (!(MI_RXWS_ABL & 1)) {
#pragma unroll
        for (int g = 0; g < QT; ++g) {
          double uu[MT][2], ww[MT][2], xx[MT][2];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int e = 0; e < 2; ++e) uu[mi][e] = ww[mi][e] = xx[mi][e] = 0.0;
#pragma unroll
          for (int a = 0; a < PW; ++a) {
            const double ba = btv[g * PW + a];
#pragma unroll
            for (int mi = 0; mi < MT; ++mi)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                uu[mi][e] = fma(ba, X[mi][(PH + a) % PW][0][e], uu[mi][e]);
                ww[mi][e] = fma(ba, X[mi][(PH + a) % PW][1][e], ww[mi][e]);
                xx[mi][e] = fma(ba, X[mi][(PH + a) % PW][2][e], xx[mi][e]);
              }
          }
          double v[MT][2];                           // C_r x w_x = (u'^2 + p) x'
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int e = 0; e < 2; ++e) v[mi][e] = fma(uu[mi][e], uu[mi][e], ww[mi][e]) * xx[mi][e];
#pragma unroll
          for (int a = 0; a < PW; ++a) {
            const double bw = btv[QT * PW + g * PW + a];
#pragma unroll
            for (int mi = 0; mi < MT; ++mi)
#pragma unroll
              for (int e = 0; e < 2; ++e) Y[mi][(PH + a) % PW][e] = fma(bw, v[mi][e], Y[mi][(PH + a) % PW][e]);
          }
        }
      }
      // ---- the entering slice reaches its window slot as (sqrt(c1) u, p, w_x x) with
      // p = c2 w - c1 (1 + a) u + c1 a, so that C_r = c1 (u - a)(u - 1) + c2 w = (sqrt(c1) u)^2 + p is ONE
      // fused multiply-add per Gauss point; p is linear in the coefficients, and its constant rides
      // along because the time basis sums to 1
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double cu = fma(a0[mi][0], bI0[e], zc[mi][0][e]), cw = fma(a0[mi][1], bI0[e], zc[mi][1][e]),
                       cx = fma(a0[mi][2], bI0[e], zc[mi][2][e]);
          X[mi][PH][0][e] = cu * rsq;
          X[mi][PH][1][e] = fma(cu, rk1, fma(cw, rc2, rk0));
          X[mi][PH][2][e] = cx * wsp[mi][e];
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
      if (j0 + 3 < nsteps) step(std::integral_constant<int, 3>{}, j0 + 3);
    }
  } else {
    // =========================== producers ===========================
    rxws_reg_dec<MI_RXWS_REGP>();
    const int p = tid - G::NCT, pw = warp - G::NCW;
    double bIy[2][2], bPy[4], bPx[2];
    const double bIx1 = basis(0, 1 + fk, fr);
    const double bIx0[2] = {basis(0, 0, 2 * fk), basis(0, 0, 2 * fk + 1)};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      bPx[ks] = basis(0, fr, 4 * ks + fk);
#pragma unroll
      for (int n2 = 0; n2 < 2; ++n2) bIy[n2][ks] = basis(1, 4 * ks + fk, 8 * n2 + fr);
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) bPy[ks] = basis(1, fr, 4 * ks + fk);
    const long long ns = r.ns;
    // spatial indices fit in 32 bits (the launcher checks N_s < 2^31)
    auto spatial = [&](int j3, int j2, int j1, bool& ok) -> int {
      const int g1 = k[0] + j1, g2 = k[1] + j2, g3 = k[2] + j3;
      ok = g1 < r.n[0] && g2 < r.n[1] && g3 < r.n[2];
      return (g3 * r.n[1] + g2) * r.n[0] + g1;
    };
    // Input slice items of this thread: spatial positions s = p + 128 h (h = 0, 1; s < LS) of all three
    // fields.  The slice is copied asynchronously (cp.async, zero fill for padding / constrained rows)
    // straight into the double-buffered sIn: no register staging, and no global-load scoreboard in
    // front of the x-interpolation DMMAs.
    int gsp[2];                                      // global spatial index (-1: outside the domain, -2: no item)
    unsigned sdst[2];                                // shared address of the field-0 copy in buffer 0
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sp = p + G::NPT * h;
      const int j3 = sp / (L1 * L2), j2 = (sp / L1) % L2, j1 = sp % L1;
      bool ok;
      const int gs = spatial(j3, j2, j1, ok);
      gsp[h] = sp < G::LS ? (ok ? gs : -1) : -2;
      sdst[h] = (unsigned)__cvta_generic_to_shared(sIn + (sp < G::LS ? (j3 * L2 + j2) * IS1 + j1 : 0));
    }
    auto put = [&](unsigned dst, const double* src, bool valid) {   // one double: async copy, or a zero
      if (valid)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
      else
        asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(dst), "d"(0.0) : "memory");
    };
    auto issue = [&](int ft) {
      const int ct = ft + r.rowoff;
      const unsigned boff = (unsigned)((ft & 1) * G::SIN * 8);
      constexpr unsigned FO = L3 * L2 * IS1 * 8;     // field stride in sIn (bytes)
      if (ct >= 0 && ct < r.ntc) {
        const long long off = (long long)ct * ns;
        const double *ru = r.u + off, *rw = r.w + off, *rx = r.x + off;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (gsp[h] != -2) {
            const bool v = gsp[h] >= 0;
            const int g = v ? gsp[h] : 0;
            const unsigned d = sdst[h] + boff;
            put(d, ru + g, v);
            put(d + FO, rw + g, v);
            put(d + 2 * FO, rx + g, v);
          }
        }
      } else {
        // the lifted slab (row -1: u and x from the lift, if set) or a row outside this context: zeros
        const double* lu = ct == -1 ? r.lift_u : nullptr;
        const double* lx = ct == -1 ? r.lift_x : nullptr;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (gsp[h] != -2) {
            const bool v = gsp[h] >= 0;
            const int g = v ? gsp[h] : 0;
            const unsigned d = sdst[h] + boff;
            put(d, lu + g, v && lu != nullptr);
            put(d + FO, nullptr, false);
            put(d + 2 * FO, lx + g, v && lx != nullptr);
          }
        }
      }
      cp_async_commit();
    };
    // x-projection outputs of this thread: line tiles mt = pw + 4 u, xline = 8 mt + fr = (j3, j2), j1 = 2 fk + e
    int yidx[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int xline = 8 * (pw + G::NPW * u) + fr, j1 = 2 * fk + e;
        bool ok = false;
        int gs = 0;
        if (xline < L3 * L2 && j1 < L1) gs = spatial(xline / L2, xline % L2, j1, ok);
        yidx[u][e] = ok ? gs : -1;
      }
    issue(0);
    for (int i = 0; i <= nfull + PW + 1; ++i) {
      const bool has_in = i < nfull;
      const int fq = i - PW - 2;                     // function whose y / x projections run now (its z
                                                     // projection ended with consumer step i - 1)
      const bool has_fq = fq >= 0 && fq < nfull;
      cp_async_wait<0>();                            // this thread's copies of slice i have landed ...
      rxws_bar_producers();                          // ... and everyone's; the other sIn buffer is free
      if (i + 1 < nfull) issue(i + 1);
      if (has_in) {
        const double* sI = sIn + (i & 1) * G::SIN;
        // x interpolation of slice i: lines (fld, j3, j2), K = j1, N = q1 -> sA
        constexpr int NL = NF * L3 * L2, NMT = (NL + 7) / 8;    // 105 lines, 14 tiles
        // functions 1..4 in ONE DMMA, function 0 (first element's Gauss points only) as a rank-1 update
        double c[4][2], a0[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          c[u][0] = c[u][1] = 0.0;
          a0[u] = 0.0;
          const int mt = pw + G::NPW * u;
          if (mt < NMT) {
            const double* row = sI + (mt * 8 + fr) * IS1;
            a0[u] = row[0];
            rxws_pdmma(c[u][0], c[u][1], row[1 + fk], bIx1);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int line = (pw + G::NPW * u) * 8 + fr;
          if (line < NL)
            *reinterpret_cast<double2*>(sA + line * Q1 + 2 * fk) =
                make_double2(fma(a0[u], bIx0[0], c[u][0]), fma(a0[u], bIx0[1], c[u][1]));
        }
      }
      rxws_bar_producers();
      if (has_in) {
        // y interpolation of slice i: lines (fld j3, q1), K = j2, N = q2 (two N tiles) -> sB[i & 1]
        const int bb = i & 1;
        constexpr int NMT = NF * L3;                 // 15 line tiles (one (fld, j3) plane each)
        double* out = sB + bb * G::SB;
#pragma unroll
        for (int h = 0; h < 2; ++h) {               // two line tiles at a time (register budget)
          double c[2][2][2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
#pragma unroll
            for (int n2 = 0; n2 < 2; ++n2) c[u][n2][0] = c[u][n2][1] = 0.0;
            const int mt = pw + G::NPW * (2 * h + u);
            if (mt < NMT) {
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {
                const double av = sA[(mt * L2 + 4 * ks + fk) * Q1 + fr];
#pragma unroll
                for (int n2 = 0; n2 < 2; ++n2) rxws_pdmma(c[u][n2][0], c[u][n2][1], av, bIy[n2][ks]);
              }
            }
          }
          if (h == 0 && i >= 2) mbar_wait(&emptyB[bb], (unsigned)(((i >> 1) - 1) & 1));
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int mt = pw + G::NPW * (2 * h + u);
            if (mt < NMT) {
#pragma unroll
              for (int n2 = 0; n2 < 2; ++n2) {
                const int n0 = 8 * n2 + 2 * fk;
                out[mt * BJ + n0 * BS1 + fr] = c[u][n2][0];
                out[mt * BJ + (n0 + 1) * BS1 + fr] = c[u][n2][1];
              }
            }
          }
        }
        mbar_arrive(&fullB[bb]);
      }
      if (has_fq) {
        // y projection of function fq: lines (j3, q1), K = q2, N = j2: sC[fq & 1] -> sD
        const int cb = fq & 1;
        mbar_wait(&fullC[cb], (unsigned)((fq >> 1) & 1));
        const double* in = sC + cb * G::SC;
        double c[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          c[u][0] = c[u][1] = 0.0;
          const int mt = pw + G::NPW * u;            // = j3
          if (mt < L3) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) rxws_pdmma(c[u][0], c[u][1], in[mt * CS + (4 * ks + fk) * Q1 + fr], bPy[ks]);
          }
        }
        mbar_arrive(&emptyC[cb]);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int mt = pw + G::NPW * u, n0 = 2 * fk;
          if (mt < L3) {
            if (n0 < L2) sD[(mt * L2 + n0) * DS1 + fr] = c[u][0];
            if (n0 + 1 < L2) sD[(mt * L2 + n0 + 1) * DS1 + fr] = c[u][1];
          }
        }
      }
      rxws_bar_producers();
      if (has_fq) {
        // x projection of function fq: lines (j3, j2), K = q1, N = j1 -> y (fire-and-forget reductions:
        // one writer per y entry per colour launch, stream-ordered launches: deterministic)
        const int ct = fq + r.rowoff;
        const long long row = (ct >= 0 && ct < r.ntc) ? (long long)ct * ns : -1;
        constexpr int NMT = (L3 * L2 + 7) / 8;       // 35 lines, 5 tiles
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int mt = pw + G::NPW * u;
          if (mt < NMT) {
            const int xline = 8 * mt + fr;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) rxws_pdmma(c0, c1, sD[xline * DS1 + 4 * ks + fk], bPx[ks]);
            if (row >= 0) {
              if (yidx[u][0] >= 0) atomicAdd(r.y + row + yidx[u][0], c0);
              if (yidx[u][1] >= 0) atomicAdd(r.y + row + yidx[u][1], c1);
            }
          }
        }
      }
    }
  }
}

// all colour classes of the warp-specialised kernel (d = 3, p = p_t = 3, fused mode)
static int reaction_ws_launch(mi_ctx* c, RxArgs r) {
  using G = RxWS;
  MI_DEV_FLAG(attr);
  if (!attr) {
    MI_CUDA(cudaFuncSetAttribute(reaction_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
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
    reaction_ws<<<(unsigned)nb, G::NTH, G::SMEM, c->stream>>>(r);
    MI_CHECK_LAUNCH("reaction_ws");
  }
  return MI_OK;
}

}  // namespace mi
