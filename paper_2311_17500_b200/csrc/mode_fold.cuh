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
// holds g_a[k]).
//
// One block per SM, warp-specialised over a ring of three panel buffers:
// 2 (n > 80) or 8 producer warps load tile j+2 (cp.async, completion on the buffer's
// mbarrier) and store tile j (coalesced rows) while 8 consumer warps run the
// DMMAs of tile j+1.  Each consumer warp owns 8 columns (rows) of the panel
// and writes its results back over them in place, so the store of a tile
// needs no staging copy and overlaps the next tile's tensor-core work.  Both
// half factors stay resident in shared memory as DMMA fragments.
// (Loads, stores and DMMAs serialised in one warp set measured additive:
// 2.4 + 2.5 + 4.3 ms for the six cfg-4 transforms.)  Contiguous-mode tiles are
// one contiguous HBM range: ONE bulk copy (TMA engine) in and one out, driven by a single
// producer thread.  (Strided tiles with 16-byte cp.async per column pair, each panel row shifted
// by the parity of its HBM start, measured slower than 8-byte copies: 7.4 vs 4.5 ms producer-only.)
#pragma once
#include <cuda_runtime.h>

#include "ptx.cuh"

#ifndef MI_MF_NPW
#define MI_MF_NPW 0    // > 0: fixed number of producer warps (timing experiments)
#endif

namespace mi {

template <int TH>
struct ModeFold {
  // consumer / producer warps.  The producers' 8-byte copies share the MIO queue with the consumers'
  // operand loads: at n = 99 (TH = 7) two producer warps keep up and beat 4 / 8 / 12 (pc_spatial 5.57 /
  // 5.70 / 5.94 / 6.91 ms at cfg 4); the shorter DMMA phase of smaller n needs the copies done faster
  static constexpr int NCW = 8, NPW = MI_MF_NPW > 0 ? MI_MF_NPW : (TH >= 7 ? 2 : 8);
  static constexpr int NTH = 32 * (NCW + NPW);
  static constexpr int NPT = 32 * NPW;              // producer threads
  static constexpr int NB = 3;                      // panel ring
  static constexpr int KS = 2 * TH;                 // k-steps per half block: K padded to 8 * TH >= hs
  static constexpr int KP = 16 * TH < 104 ? 16 * TH : 104;   // panel depth: n <= KP
  static constexpr int FH = TH * KS * 32;           // fragments of one half factor (doubles)
  static constexpr int BLD = 68;                    // COLS panel row stride (= 4 mod 16: conflict-free B reads)
  static constexpr int ALD = (KP % 16 == 4 || KP % 16 == 12) ? KP : KP + ((4 - KP % 16) + 16) % 16;
  // panel sizes (doubles).  ROWS tiles are contiguous in HBM and move as ONE bulk copy each way, so
  // their panel is dense (row stride n)
  static constexpr int PCOLS = KP * BLD, PROWS = 64 * KP;
  static constexpr size_t SMEM_COLS = (size_t)(2 * FH + NB * PCOLS) * 8 + 64;
  static constexpr size_t SMEM_ROWS = (size_t)(2 * FH + NB * PROWS) * 8 + 64;
  static_assert(SMEM_COLS <= 227 * 1024 && SMEM_ROWS <= 227 * 1024, "folded mode product exceeds shared memory");
};

// U: n x n row-major eigenvector matrix (columns = modes, symmetric first).  INV = false applies
// U^T (into mode space), INV = true applies U.  ROWS: the mode is the contiguous index
// (out[r][.] from in[r][.], `outer` rows); COLS: out[o][.][c] from in[o][.][c] (stride `inner`).
// Tiles: 64 flattened columns (COLS) or 64 rows (ROWS).
// COLS addressing maps (nullable, 2n int64 each): element (o, r, c) of the input / output sits at
// map[2r] + o * map[2r + 1] + c instead of (o * n + r) * inner + c.  The space-sharded P^-1
// (sharded.py) uses them to read and write the all-to-all send / receive layouts directly.
template <int TH, bool ROWS, bool INV>
__global__ void __launch_bounds__(ModeFold<TH>::NTH, 1) mode_fold(const double* __restrict__ U,
                                                                   const double* __restrict__ in,
                                                                   double* __restrict__ out, int n,
                                                                   long long inner, long long outer,
                                                                   const long long* __restrict__ imap,
                                                                   const long long* __restrict__ omap) {
  using G = ModeFold<TH>;
  constexpr int KS = G::KS, NB = G::NB;
  constexpr int PS = ROWS ? G::PROWS : G::PCOLS;    // panel size
  const int LD = ROWS ? n : G::BLD;                 // panel row stride
  extern __shared__ __align__(16) double smem[];
  double* frag = smem;                               // [half][TH][KS][32]
  double* pan = smem + 2 * G::FH;                    // [NB][panel]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(pan + NB * PS);   // [NB]
  unsigned long long* done = full + NB;                                              // [NB] computed
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  const int h = n >> 1, hs = n - h;
  const bool odd = (n & 1) != 0;
  // Half factor b (0 = symmetric, 1 = skew): C_b[m][k] = U[k][b * hs + m], m < size_b, k < size_b
  // (size_0 = hs, size_1 = h).  Tile index i / k-step ks select
  //   COLS fwd : A[m = 8 i + q][k = 4 ks + t]      COLS inv : A[k = 8 i + q][m = 4 ks + t]
  //   ROWS fwd : B[k = 4 ks + t][m = 8 i + q]      ROWS inv : B[m = 4 ks + t][k = 8 i + q]
  for (int e = tid; e < 2 * G::FH; e += G::NTH) {
    const int l = e & 31, ks = (e >> 5) % KS, i = ((e >> 5) / KS) % TH, b = (e >> 5) / (KS * TH);
    const int q = l >> 2, t = l & 3;
    const int r8 = 8 * i + q, c4 = 4 * ks + t;
    const int m = INV ? c4 : r8, k = INV ? r8 : c4;  // the forward tiles run over modes, the inverse over k
    const int sz = b == 0 ? hs : h;
    frag[e] = (m < sz && k < sz) ? __ldg(U + (long long)k * n + b * hs + m) : 0.0;
  }
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], ROWS ? 1 : G::NPT);        // COLS: one cp.async-completion arrival per producer thread
      mbar_init(&done[b], 32 * G::NCW);              // every consumer thread arrives after its write-back
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long total = ROWS ? outer : outer * inner;
  const long long ntiles = (total + 63) / 64;
  const long long nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp >= G::NCW) {
    // ================= producers: loads of tile j + 2, stores of tile j =================
    const int p = tid - 32 * G::NCW;
    // COLS: thread -> column c = p & 63, rows (p >> 6) + 2 m; ROWS: flat element stride
    // flattened column g -> (outer index o, inner index cc)
    auto col_pos = [&](long long tile, int c, long long& o, long long& cc) -> bool {
      const long long g = tile * 64 + c;
      if (g >= total) return false;
      o = g / inner;
      cc = g - o * inner;
      return true;
    };
    auto load = [&](long long j) {
      const int b = (int)(j % NB);
      const long long tile = blockIdx.x + j * gridDim.x;
      double* dst = pan + b * PS;
      if constexpr (!ROWS) {
        const int c = p & 63;
        long long o, cc;
        if (col_pos(tile, c, o, cc)) {
          if (imap != nullptr) {
            for (int r = p >> 6; r < n; r += G::NPT / 64)
              cp_async8(dst + r * LD + c, in + __ldg(imap + 2 * r) + o * __ldg(imap + 2 * r + 1) + cc, true);
          } else {
            const long long base = o * n * inner + cc;
            for (int r = p >> 6; r < n; r += G::NPT / 64) cp_async8(dst + r * LD + c, in + base + (long long)r * inner, true);
          }
        }
        cp_async_mbar_arrive_noinc(&full[b]);
      } else {
        // one thread: the tile's nel = nrow * n doubles start 16-byte aligned (tile * 64 * n is even); an
        // odd tail element is copied by hand before the arrive
        const long long r0 = tile * 64;
        const int nel = (int)(total - r0 < 64 ? total - r0 : 64) * n, nb = nel & ~1;
        const double* src = in + r0 * n;
        if (nel & 1) dst[nel - 1] = src[nel - 1];
        mbar_expect_tx(&full[b], (unsigned)nb * 8);
        if (nb) bulk_g2s(dst, src, (unsigned)nb * 8, &full[b]);
      }
    };
    auto store = [&](long long j) {
      const int b = (int)(j % NB);
      const long long tile = blockIdx.x + j * gridDim.x;
      const double* sp = pan + b * PS;
      if constexpr (!ROWS) {
        const int c = p & 63;
        long long o, cc;
        if (col_pos(tile, c, o, cc)) {
          if (omap != nullptr) {
            for (int r = p >> 6; r < n; r += G::NPT / 64)
              out[__ldg(omap + 2 * r) + o * __ldg(omap + 2 * r + 1) + cc] = sp[r * LD + c];
          } else {
            const long long base = o * n * inner + cc;
            for (int r = p >> 6; r < n; r += G::NPT / 64) out[base + (long long)r * inner] = sp[r * LD + c];
          }
        }
      } else {
        const long long r0 = tile * 64;
        const int nel = (int)(total - r0 < 64 ? total - r0 : 64) * n, nb = nel & ~1;
        double* dst = out + r0 * n;
        if (nel & 1) dst[nel - 1] = sp[nel - 1];
        if (nb) bulk_s2g(dst, sp, (unsigned)nb * 8);
        bulk_commit();
      }
    };
    if (ROWS && p != 0) return;                      // ROWS: one thread drives the bulk copies
    if (nloc > 0) load(0);
    if (nloc > 1) load(1);
    for (long long j = 0; j < nloc; ++j) {
      // buffer (j + 2) % NB held tile j - 1, stored by every producer in the previous iteration
      if constexpr (ROWS)
        bulk_wait_read0();                           // the bulk store of tile j - 1 has read its buffer
      else
        asm volatile("bar.sync 1, %0;\n" ::"n"(G::NPT) : "memory");
      if (j + 2 < nloc) load(j + 2);
      mbar_wait(&done[j % NB], (unsigned)((j / NB) & 1));
      store(j);
    }
    if constexpr (ROWS) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // before the block's smem goes away
  } else {
    // ================= consumers: DMMAs of tile j, results written over the panel =================
    const int own = 8 * warp + gq;                   // COLS: column; ROWS: row of this lane's operand
    const int ksn = (hs + 3) >> 2;
    for (long long j = 0; j < nloc; ++j) {
      const int b = (int)(j % NB);
      mbar_wait(&full[b], (unsigned)((j / NB) & 1));
      double* P = pan + b * PS;
      double as_[TH][2], aa_[TH][2];
#pragma unroll
      for (int i = 0; i < TH; ++i) as_[i][0] = as_[i][1] = aa_[i][0] = aa_[i][1] = 0.0;
      // operand element v(k): COLS panel row k of column `own`; ROWS row `own`, column k
      const double* src = ROWS ? P + own * LD : P + own;
      constexpr int ST = ROWS ? 1 : LD;
#pragma unroll 2
      for (int ks = 0; ks < ksn; ++ks) {            // K = hs (>= h) padded to 4, not to 8 * TH
        const int k = 4 * ks + t4;
        double vs, va;
        if constexpr (!INV) {
          const double xk = src[k * ST];
          const double xr = src[(k < h ? n - 1 - k : k) * ST];
          vs = k < h ? xk + xr : ((odd && k == h) ? xk : 0.0);
          va = k < h ? xk - xr : 0.0;
        } else {
          vs = k < hs ? src[k * ST] : 0.0;
          va = k < h ? src[(hs + k) * ST] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < TH; ++i) {
          if constexpr (!ROWS) {
            dmma(as_[i][0], as_[i][1], frag[(i * KS + ks) * 32 + lane], vs);
            dmma(aa_[i][0], aa_[i][1], frag[G::FH + (i * KS + ks) * 32 + lane], va);
          } else {
            dmma(as_[i][0], as_[i][1], vs, frag[(i * KS + ks) * 32 + lane]);
            dmma(aa_[i][0], aa_[i][1], va, frag[G::FH + (i * KS + ks) * 32 + lane]);
          }
        }
      }
      __syncwarp();                                  // every lane's operand reads precede the write-back
      // this lane's results: index r = 8 i + gq (COLS: panel row, columns 8 warp + 2 t4 + e) or
      // r = 8 i + 2 t4 + e (ROWS: panel column of row 8 warp + gq)
#pragma unroll
      for (int i = 0; i < TH; ++i)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = ROWS ? 8 * i + 2 * t4 + e : 8 * i + gq;
          double* d = ROWS ? P + (8 * warp + gq) * LD : P + 8 * warp + 2 * t4 + e;
          if constexpr (!INV) {
            if (r < hs) d[r * ST] = as_[i][e];
            if (r < h) d[(hs + r) * ST] = aa_[i][e];
          } else {
            if (r < h) {
              d[r * ST] = as_[i][e] + aa_[i][e];
              d[(n - 1 - r) * ST] = as_[i][e] - aa_[i][e];
            } else if (odd && r == h) {
              d[r * ST] = as_[i][e];
            }
          }
        }
      if constexpr (ROWS) fence_proxy_async_smem();   // the write-back is read by the bulk store (async proxy)
      mbar_arrive(&done[b]);
    }
  }
}

// Launch for hs = n - n/2 <= 8 * TH and n <= KP; returns false (nothing launched) outside the
// instantiated range.
template <bool ROWS>
inline bool launch_mode_fold(const double* U, const double* in, double* out, int n, bool inverse, long long inner,
                             long long outer, int nsm, cudaStream_t st, cudaError_t* err,
                             const long long* imap = nullptr, const long long* omap = nullptr) {
  const int hs = n - n / 2;
#define MI_MF(THV)                                                                                       \
  if (hs <= 8 * THV && n <= ModeFold<THV>::KP) {                                                         \
    constexpr size_t sm = ROWS ? ModeFold<THV>::SMEM_ROWS : ModeFold<THV>::SMEM_COLS;                    \
    constexpr int nth = ModeFold<THV>::NTH;                                                              \
    MI_DEV_FLAG(attr);                                                                            \
    if (!attr) {                                                                                         \
      cudaFuncSetAttribute(mode_fold<THV, ROWS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
      cudaFuncSetAttribute(mode_fold<THV, ROWS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);  \
      attr = true;                                                                                       \
    }                                                                                                    \
    const long long total = ROWS ? outer : outer * inner;                                                \
    const long long ntiles = (total + 63) / 64;                                                          \
    const int grid = (int)(ntiles < nsm ? ntiles : nsm);                                                 \
    if (inverse)                                                                                         \
      mode_fold<THV, ROWS, true><<<grid > 0 ? grid : 1, nth, sm, st>>>(U, in, out, n, inner, outer, imap, omap);  \
    else                                                                                                 \
      mode_fold<THV, ROWS, false><<<grid > 0 ? grid : 1, nth, sm, st>>>(U, in, out, n, inner, outer, imap, omap); \
    *err = cudaGetLastError();                                                                           \
    return true;                                                                                         \
  }
  MI_MF(1) MI_MF(2) MI_MF(3) MI_MF(5) MI_MF(7)
#undef MI_MF
  return false;
}

}  // namespace mi
