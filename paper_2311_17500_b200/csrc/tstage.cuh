// Fused time stage of the fast-diagonalisation preconditioner (reference
// FastDiagPreconditioner.apply, linalg.py:329-346: the time mode product,
// the arrowhead solve of _diag_blocks / linalg.py:335-345, and the inverse
// time mode product), one kernel per column tile:
//
//   Y[:, s] <- Q (C_m T + mu_s I)^-1 Q^T Y[:, s]      for every spatial eigen-index s
//
// A block owns NC consecutive columns (s) of the time-major (nt x ncols)
// tensor and keeps the whole 8*MB x NC tile in shared memory, so Y crosses
// HBM once each way (separate Q^T / arrowhead / Q passes: 3 reads + 3 writes).
//  - Tile load: 8-byte cp.async (the row stride ncols is odd at the BASELINE
//    sizes, so rows are not 16-byte aligned), issued up front in 8-row chunks,
//    each completing on its own mbarrier; the first product starts on chunk 0
//    while the rest is in flight.
//  - Products: FP64 tensor cores (DMMA m8n8k4).  A warp owns 16 columns and
//    half of the row blocks; its accumulators stay in registers.  Q^T and Q
//    are the A operands, prebuilt fragment-major and streamed by the TMA bulk
//    engine through an NST-stage shared-memory ring (KC k-steps x all MB row
//    blocks per stage, full/empty mbarriers), so every fragment is read from
//    L2 once per block and shared by all warps.
//  - Arrowhead: on the tile in shared memory, parallel over rows (the two
//    border sums are per-column reductions), mu_s formed on the fly.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "ptx.cuh"

#ifndef MI_TS_WM
#define MI_TS_WM 4
#endif
#ifndef MI_TS_KC
#define MI_TS_KC 2
#endif
#ifndef MI_TS_NST
#define MI_TS_NST 4
#endif

namespace mi {

struct TStageArgs {
  double* y;                       // (nt x ncols), row stride ncols, in place
  const double* frag;              // [2 products][KSP][MB][32]: Q^T then Q
  const double *lam1, *lam2, *lam3;
  const double *diag, *off, *gb, *gl;
  const int* partner;
  double sigma, cm, react;
  int n1, n2, nt, ksp;             // ksp = k-steps padded to a multiple of KC
  long long ncols, col0;
};

template <int MB, int NC, int WM>
struct TStage {
  static constexpr int KC = MI_TS_KC;               // k-steps per ring stage (2 = 8 tile rows)
  static constexpr int NST = MI_TS_NST;             // ring stages
  static constexpr int NP = NC / 16;                // column pairs of 8-column blocks
  static constexpr int MH = (MB + WM - 1) / WM;     // row blocks per warp (rows split in WM groups)
  static constexpr int WARPS = WM * NP;
  static constexpr int THREADS = 32 * WARPS;        // = 2 WM NC: the arrowhead uses 2 WM row groups x NC columns
  static constexpr int RG = 2 * WM;
  static constexpr int LD = NC + 4;                 // = 4 (mod 16) doubles: conflict-free B fragment reads
  static constexpr int ROWS = 8 * MB;
  static constexpr int RCH = MB;                    // 8-row load chunks
  static constexpr int STAGE = KC * MB * 32;        // doubles per ring stage
  static constexpr size_t SMEM = ((size_t)ROWS * LD + (size_t)NST * STAGE + 2 * RG * NC) * 8 +
                                 (size_t)(2 * NST + RCH) * 8;
};

template <int MB, int NC, int WM>
__global__ void __launch_bounds__(TStage<MB, NC, WM>::THREADS, 1) time_stage_fused(TStageArgs a) {
  using G = TStage<MB, NC, WM>;
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;                                 // [NST][KC][MB][32]   (16-byte aligned for the bulk copies)
  double* Ys = ring + G::NST * G::STAGE;             // [ROWS][LD]
  double* red = Ys + G::ROWS * G::LD;                // [2][RG][NC] border-sum partials
  unsigned long long* full = reinterpret_cast<unsigned long long*>(red + 2 * G::RG * NC);
  unsigned long long* empty = full + G::NST;
  unsigned long long* ybar = empty + G::NST;         // [RCH]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  const long long c0 = (long long)blockIdx.x * NC;
  const int nt = a.nt;
  const int nchk = a.ksp / G::KC;                    // ring chunks per product
  const int total = 2 * nchk;

  if (tid == 0) {
    for (int s = 0; s < G::NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::WARPS);
    }
    for (int r = 0; r < G::RCH; ++r) mbar_init(&ybar[r], G::THREADS);
    mbar_fence_init();
  }
  __syncthreads();

  // ring producer (thread 0): chunk f of the 2 x nchk sequence into stage f % NST
  auto produce = [&](int f) {
    if (f >= total) return;
    const int s = f % G::NST;
    if (f >= G::NST) mbar_wait(&empty[s], (unsigned)(((f / G::NST) - 1) & 1));
    mbar_expect_tx(&full[s], G::STAGE * 8);
    bulk_g2s(ring + s * G::STAGE, a.frag + (long long)f * G::STAGE, G::STAGE * 8, &full[s]);
  };
  if (tid == 0)
    for (int f = 0; f < G::NST - 1; ++f) produce(f);

  // ---- tile load, 8-row chunks (rows >= nt and columns >= ncols are zero-filled)
  for (int r = 0; r < G::RCH; ++r) {
    for (int e = tid; e < 8 * NC; e += G::THREADS) {
      const int row = 8 * r + e / NC, c = e % NC;
      const bool v = row < nt && c0 + c < a.ncols;
      cp_async8(Ys + row * G::LD + c, v ? a.y + (long long)row * a.ncols + c0 + c : a.y, v);
    }
    cp_async_mbar_arrive_noinc(&ybar[r]);
  }

  const int h = warp / G::NP, q = warp % G::NP;
  const int nmine = min(G::MH, MB - h * G::MH);     // row blocks of this warp's group (the last may be short)
  double acc[G::MH][2][2];

  // one product: acc = A * Ys over ring chunks [f0, f0 + nchk)
  auto product = [&](int f0, bool wait_rows) {
#pragma unroll
    for (int i = 0; i < G::MH; ++i) acc[i][0][0] = acc[i][0][1] = acc[i][1][0] = acc[i][1][1] = 0.0;
    const double* bp = Ys + t4 * G::LD + 16 * q + gq;
    for (int k = 0; k < nchk; ++k) {
      const int f = f0 + k;
      if (tid == 0) produce(f + G::NST - 1);
      if (wait_rows)                                 // tile rows [4 KC k, 4 KC (k + 1)) have landed
        for (int j = (4 * G::KC * k) / 8; j < G::RCH && j < (4 * G::KC * (k + 1) + 7) / 8; ++j) mbar_wait(&ybar[j], 0);
      mbar_wait(&full[f % G::NST], (unsigned)((f / G::NST) & 1));
      const double* st = ring + (f % G::NST) * G::STAGE + (h * G::MH) * 32 + lane;
#pragma unroll
      for (int kk = 0; kk < G::KC; ++kk) {
        const int row = 4 * (k * G::KC + kk);
        const double b0 = bp[row * G::LD], b1 = bp[row * G::LD + 8];
#pragma unroll
        for (int i = 0; i < G::MH; ++i) {
          if (i < nmine) {
            const double av = st[(kk * MB + i) * 32];
            dmma(acc[i][0][0], acc[i][0][1], av, b0);
            dmma(acc[i][1][0], acc[i][1][1], av, b1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[f % G::NST]);
    }
  };

  // ---- Q^T Y
  product(0, true);
  __syncthreads();                                   // every warp has finished reading Ys
#pragma unroll
  for (int i = 0; i < G::MH; ++i) {
    if (i < nmine) {
      double* d = Ys + (8 * (h * G::MH + i) + gq) * G::LD + 16 * q + 2 * t4;
      d[0] = acc[i][0][0];
      d[1] = acc[i][0][1];
      d[8] = acc[i][1][0];
      d[9] = acc[i][1][1];
    }
  }
  __syncthreads();

  // ---- arrowhead solve per column (reference _diag_blocks, linalg.py:309-315, 335-345):
  // interior 2x2 blocks [[a, b], [c, e]] = C_m T_block + mu I, border column C_m g,
  // border row C_m glow, corner C_m sigma + mu.  Thread = (column c, row group rg).
  {
    const int c = tid % NC, rg = tid / NC;           // RG row groups
    const long long sg = a.col0 + c0 + c;
    const int i1 = (int)(sg % a.n1), i2 = (int)((sg / a.n1) % a.n2), i3 = (int)(sg / ((long long)a.n1 * a.n2));
    const double mu = a.react + __ldg(a.lam1 + i1) + __ldg(a.lam2 + i2) + __ldg(a.lam3 + i3);
    const double cm = a.cm;
    const int m = nt - 1;
    double sy = 0.0, sb = 0.0;
    for (int i = rg; i < m; i += G::RG) {
      const int j = __ldg(a.partner + i);
      const double di = fma(cm, __ldg(a.diag + i), mu), dj = fma(cm, __ldg(a.diag + j), mu);
      const double b = cm * __ldg(a.off + i), cc = cm * __ldg(a.off + j);
      const double inv = 1.0 / (di * dj - b * cc);
      const double yi = Ys[i * G::LD + c], yj = Ys[j * G::LD + c];
      const double gli = __ldg(a.gl + i);
      sy = fma(gli, (dj * yi - b * yj) * inv, sy);
      sb = fma(gli, cm * (dj * __ldg(a.gb + i) - b * __ldg(a.gb + j)) * inv, sb);
    }
    red[rg * NC + c] = sy;
    red[(G::RG + rg) * NC + c] = sb;
    __syncthreads();
    double syt = 0.0, sbt = 0.0;
#pragma unroll
    for (int g = 0; g < G::RG; ++g) {
      syt += red[g * NC + c];
      sbt += red[(G::RG + g) * NC + c];
    }
    const double xl = (Ys[m * G::LD + c] - cm * syt) / (fma(cm, a.sigma, mu) - cm * sbt);
    __syncthreads();                                 // all reads of the pre-solve row m are done
    // second sweep: rows of a 2x2 block are written together by the thread of the smaller index
    for (int i = rg; i < m; i += G::RG) {
      const int j = __ldg(a.partner + i);
      if (j < i) continue;
      const double di = fma(cm, __ldg(a.diag + i), mu), dj = fma(cm, __ldg(a.diag + j), mu);
      const double b = cm * __ldg(a.off + i), cc = cm * __ldg(a.off + j);
      const double inv = 1.0 / (di * dj - b * cc);
      const double ri = Ys[i * G::LD + c] - cm * __ldg(a.gb + i) * xl;
      const double rj = Ys[j * G::LD + c] - cm * __ldg(a.gb + j) * xl;
      Ys[i * G::LD + c] = (dj * ri - b * rj) * inv;
      if (j != i) Ys[j * G::LD + c] = (di * rj - cc * ri) * inv;
    }
    if (rg == 0) Ys[m * G::LD + c] = xl;
  }
  __syncthreads();

  // ---- Q Y, straight from the accumulators to HBM
  product(nchk, false);
#pragma unroll
  for (int i = 0; i < G::MH; ++i) {
    const int r = 8 * (h * G::MH + i) + gq;
    if (i < nmine && r < nt) {
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const long long col = c0 + 16 * q + 8 * n + 2 * t4;
        double* d = a.y + (long long)r * a.ncols + col;
        if (col < a.ncols) d[0] = acc[i][n][0];
        if (col + 1 < a.ncols) d[1] = acc[i][n][1];
      }
    }
  }
}

// Fragment-major DMMA A operands of Q^T and Q (nt x nt, row-major Q), padded to 8 mb x 4 ksp:
// f[((g * ksp + k) * mb + b) * 32 + lane] = A_g[8 b + lane / 4][4 k + lane % 4], A_0 = Q^T, A_1 = Q.
inline void build_tstage_frags(const double* Q, int nt, int mbn, int ksp, std::vector<double>& f) {
  f.assign((size_t)2 * ksp * mbn * 32, 0.0);
  for (int g = 0; g < 2; ++g)
    for (int k = 0; k < ksp; ++k)
      for (int b = 0; b < mbn; ++b)
        for (int l = 0; l < 32; ++l) {
          const int r = 8 * b + l / 4, c = 4 * k + l % 4;
          if (r < nt && c < nt)
            f[(((size_t)g * ksp + k) * mbn + b) * 32 + l] = g == 0 ? Q[(size_t)c * nt + r] : Q[(size_t)r * nt + c];
        }
}

// The smallest instantiated MB >= ceil(nt / 8) (0: nt beyond the fused range).
inline int tstage_mb(int nt) {
  const int need = (nt + 7) / 8;
  const int mbs[] = {4, 8, 13, 17, 25, 33, 41, 49};
  for (int m : mbs)
    if (m >= need) return m;
  return 0;
}

template <int MB, int NC, int WM>
inline cudaError_t launch_tstage_t(const TStageArgs& a, cudaStream_t st) {
  using G = TStage<MB, NC, WM>;
  static_assert(G::SMEM <= 232448, "tile does not fit in shared memory");
  MI_DEV_FLAG(attr);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(time_stage_fused<MB, NC, WM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long nb = (a.ncols + NC - 1) / NC;
  time_stage_fused<MB, NC, WM><<<(unsigned)nb, G::THREADS, G::SMEM, st>>>(a);
  return cudaGetLastError();
}

// Column-tile width per MB: the widest multiple of 16 whose tile + ring fit in shared memory.
inline cudaError_t launch_tstage(int mb, const TStageArgs& a, cudaStream_t st) {
  switch (mb) {
    case 4: return launch_tstage_t<4, 160, 2>(a, st);
    case 8: return launch_tstage_t<8, 160, 2>(a, st);
    case 13: return launch_tstage_t<13, 160, 2>(a, st);
    case 17: return launch_tstage_t<17, 160, 2>(a, st);
    case 25: return launch_tstage_t<25, 96, MI_TS_WM>(a, st);
    case 33: return launch_tstage_t<33, 64, 2>(a, st);
    case 41: return launch_tstage_t<41, 48, 2>(a, st);
    case 49: return launch_tstage_t<49, 32, 2>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace mi
