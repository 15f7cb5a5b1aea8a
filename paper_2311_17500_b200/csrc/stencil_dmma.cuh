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
// double-buffered halo tile; two warps per point split K.  W is written
// time-innermost and the banded time filter is a separate kernel
// (tfilter.cuh).  (Fusing the filter into this kernel with a 3-chunk W ring in
// shared memory measured 65.6 ms against 38.4 + 3.65 ms: with one 229 KB block
// per SM nothing overlaps the filter phase, whose band loads sit on its
// critical path; profiles/r02_optimisation_log.md S1.)
#pragma once
#include "common.cuh"
#include "ptx.cuh"
#include <cuda.h>

#ifndef MI_STEN_B1
#define MI_STEN_B1 1
#endif
#ifndef MI_STEN_B2
#define MI_STEN_B2 4
#endif
#ifndef MI_STEN_PERSIST
#define MI_STEN_PERSIST 1   // persistent CTAs with cross-cube prefetch (stencil_dmma)
#endif
#ifndef MI_STEN_DECOUPLED
#define MI_STEN_DECOUPLED 1 // no block barrier in the chunk loop: the two warps of a point meet on a named barrier,
                            // the halo buffers are recycled by whichever warp finishes a chunk last
#endif
#ifndef MI_STEN_L2PF
#define MI_STEN_L2PF 1      // persistent CTAs also prefetch the next cube's fragments into L2
#endif

namespace mi {

template <int D, int P>
struct DmmaSten {
  static constexpr int W = 2 * P + 1;
  static constexpr int S = D == 3 ? W * W * W : (D == 2 ? W * W : W);
  // K order: the S stencil points in (a3, a2, a1) order, 4 per k-step (unpadded);
  // a k-step's 4 points span at most one stencil-row boundary (W >= 4 for p >= 2)
  static constexpr int KS = (S + 3) / 4;            // k-steps per point
  static constexpr int KH = (KS + 1) / 2;           // k-steps per warp (2 warps / point)
  // point block of one CTA: 1 x 4 x 2 points in 3D.  With B1 = 1 the halo rows are exactly the stencil
  // width, so k-steps that cross an x-row read consecutive halo points (no shared-memory bank
  // conflicts; only plane crossings still conflict), with the same 8 points per block as the 2x2x2 cube
  // it replaced (cfg 4: 38.68 -> 38.27 ms).  (A 1x1x6 column was 0.7 ms SLOWER: 33% more blocks, each
  // paying the start-up.)
  static constexpr int B1 = D == 3 ? MI_STEN_B1 : (D == 2 ? 4 : 8);
  static constexpr int B2 = D == 3 ? MI_STEN_B2 : (D == 2 ? 2 : 1);
  static constexpr int B3 = D == 3 ? 8 / (MI_STEN_B1 * MI_STEN_B2) : 1;
  static constexpr int PPB = B1 * B2 * B3;          // points per block
  static constexpr int H1 = B1 + 2 * P;
  static constexpr int H2 = D >= 2 ? B2 + 2 * P : 1;
  static constexpr int H3 = D >= 3 ? B3 + 2 * P : 1;
  static constexpr int HS = H1 * H2 * H3;
  static constexpr int MT = 2;                      // M-tiles (8 time rows each) per chunk
  static constexpr int TT = 8 * MT;                 // time rows per chunk
  static constexpr int TSTR = TT + 4;               // smem stride per halo point (= 4 mod 16)
  static constexpr int PTMAX = 4;
  static constexpr int BW = 2 * PTMAX + 1;
  static constexpr int WL = 2 * TT;                 // W partial rows: this chunk + the previous one
  static constexpr int PSTR = 8 * WL + 4;           // point stride in the W buffer (= 4 mod 16)
  static constexpr int THREADS = 64 * PPB;          // two warps per point
  static constexpr int FK = 8 * 16;                 // filter K: 8 channels x 16 time taps
  static constexpr size_t SMEM = (size_t)2 * HS * TSTR * 8       // X halo [buf][h][t]
                                 + (size_t)2 * PPB * PSTR * 8     // W partials [half][pt][ch*WL + row]
                                 + 16                             // TMA mbarriers
                                 + 16;                            // buffer-release counters
  // halo offset of stencil point s (0 beyond S)
  static constexpr __host__ __device__ int offs(int s) {
    return s >= S ? 0 : ((D >= 3 ? s / (W * W) : 0) * H2 + (D >= 2 ? (s / W) % W : 0)) * H1 + s % W;
  }
  // lane kl of k-step ks reads offs(4 ks) + kl + (kl >= cut(ks) ? jump(ks) : 0)
  static constexpr __host__ __device__ int cut(int ks) {
    return (4 * ks + 1 < S && offs(4 * ks + 1) != offs(4 * ks) + 1) ? 1
         : (4 * ks + 2 < S && offs(4 * ks + 2) != offs(4 * ks) + 2) ? 2
         : (4 * ks + 3 < S && offs(4 * ks + 3) != offs(4 * ks) + 3) ? 3 : 4;
  }
  static constexpr __host__ __device__ int jump(int ks) {
    return cut(ks) < 4 ? offs(4 * ks + cut(ks)) - offs(4 * ks) - cut(ks) : 0;
  }
};

struct DmmaArgs {
  const double* xt;     // time-innermost copy of x: xt[i * ntp + t]
  double* wout;         // W_c of all channels, time-innermost (nchan, ns, ntp): the time filter is a separate kernel
  const double* frag;   // fragment-major coefficients of this channel group
  const double* band;   // time bands (nchan_total, nt, 2pt+1)
  double* y;
  int c0, nc;           // channel group [c0, c0+nc)
  int pt, accumulate;
  int n1, n2, n3, nt, ntp;
  int C1, C2, C3;       // cube grid
  long long ns;
  int zoff;             // halo planes below the owned ones in xt (z-slab contexts; 0 unsharded)
  int cube_lo, cube_hi; // cubes of this launch (a z range: cubes are numbered z-slowest)
};

// x (nt, ns) -> xt (ns, ntp), zero padded in time; 32x32 smem tiles.  Columns [0, ns) of x and rows
// [0, ns) of xt, both given already offset to the first spatial index of the range; x_ld = x's row
// stride (the full N_s when a range of spatial points is transposed).
__global__ void transpose_time_inner(const double* __restrict__ x, double* __restrict__ xt, int nt, int ntp,
                                     long long ns, long long x_ld) {
  __shared__ double tile[32][33];
  const long long s0 = (long long)blockIdx.x * 32;
  const int t0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int t = t0 + r;
    const long long s = s0 + threadIdx.x;
    tile[r][threadIdx.x] = (t < nt && s < ns) ? x[(long long)t * x_ld + s] : 0.0;
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
template <class G, int HALF, int MTV>
__device__ __forceinline__ void dmma_sweep(const double* X, int kl, const double (&breg)[G::KH],
                                           double (&acc)[G::MT][2]) {
  const bool ge1 = kl >= 1, ge2 = kl >= 2, ge3 = kl >= 3;
#pragma unroll
  for (int j = 0; j < G::KH; ++j) {
    const int ks = HALF * G::KH + j;
    if (ks < G::KS) {
      constexpr int dummy = 0;
      (void)dummy;
      const int ct = G::cut(ks);
      const bool past = ct == 1 ? ge1 : (ct == 2 ? ge2 : (ct == 3 ? ge3 : false));
      const double* xa = X + (G::offs(4 * ks) + (past ? G::jump(ks) : 0)) * G::TSTR;
#pragma unroll
      for (int m = 0; m < MTV; ++m) dmma(acc[m][0], acc[m][1], xa[m * 8], breg[j]);
    }
  }
}

template <int D, int P>
__global__ void __launch_bounds__(DmmaSten<D, P>::THREADS, 1) stencil_dmma(DmmaArgs a,
                                                                          const __grid_constant__ CUtensorMap tmap) {
  using G = DmmaSten<D, P>;
  extern __shared__ __align__(128) double sm[];
  double* Xs = sm;                                   // [2][HS][TSTR]
  double* Wp = Xs + 2 * G::HS * G::TSTR;             // [2 half][8 pt][PSTR]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(Wp + 2 * G::PPB * G::PSTR);   // 2 mbarriers

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pt = warp >> 1, half = warp & 1;
  const int ncubes = a.cube_hi;                      // this launch sweeps cubes [cube_lo, cube_hi)
  // Persistent CTAs (MI_STEN_PERSIST): block b sweeps cubes b, b + grid, ...  The first halo tile of the
  // next cube is loaded by TMA during the current cube's last chunk and the next cube's coefficient
  // fragments are prefetched into L2 during its sweep, so a cube's start-up (fragment loads, first
  // tile) no longer runs with the tensor cores idle.  Without persistence: one cube per block.
  const int cstep = MI_STEN_PERSIST ? (int)gridDim.x : ncubes - a.cube_lo;

  for (int e = tid; e < 2 * G::PPB * G::PSTR; e += G::THREADS) Wp[e] = 0.0;

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
  auto origin = [&](int cube, int& o1, int& o2, int& o3) {
    const int c1 = cube % a.C1, c2 = (cube / a.C1) % a.C2, c3 = cube / (a.C1 * a.C2);
    o1 = c1 * G::B1;
    o2 = c2 * G::B2;
    o3 = c3 * G::B3;
  };
  auto load_chunk = [&](int cube, int buf, int t0) {
    if (tid == 0 && t0 < a.nt) {
      int q1, q2, q3;
      origin(cube, q1, q2, q3);
      mbar_expect_tx(&bars[buf], TILE_BYTES);
      tma_load_4d(Xs + buf * G::HS * G::TSTR, &tmap, &bars[buf], t0, q1 - P, D >= 2 ? q2 - P : 0,
                  D >= 3 ? q3 - P + a.zoff : 0);
    }
  };
  constexpr long long FRAG_CUBE = (long long)G::PPB * G::KS * 32;   // doubles of one cube's fragments
  const int base = ((pt / (G::B1 * G::B2)) * G::H2 + (pt / G::B1) % G::B2) * G::H1 + pt % G::B1;
  const int kl = lane & 3, mrow = lane >> 2;
  double* wmine = Wp + (half * G::PPB + pt) * G::PSTR + 2 * kl * G::WL;   // channels 2kl, 2kl+1
  const int nchunks = (a.nt + G::TT - 1) / G::TT;
  int gc = 0;                                        // chunks consumed by this block: buffer gc & 1, phase (gc >> 1) & 1

#if MI_STEN_DECOUPLED
  {
    // ---- decoupled sweep.  The block's chunk sequence g = 0, 1, ... runs over its cubes (nchunks
    // chunks each); chunk g lives in halo buffer g & 1 and in W ring half g & 1.  No block barrier:
    //   * a warp that has finished the sweep of chunk g bumps cnt[g & 1]; the LAST of the block's warps
    //     to do so re-arms the buffer with the TMA load of chunk g + 2 (nobody waits for a free buffer);
    //   * the two warps of a point (the K halves) meet on a named barrier once per chunk, after which
    //     the pair writes the point's 8 channels x 16 rows of W out.
    // A warp that is done with chunk g starts on g + 1 at once, so the write-out, the barrier skew and
    // the accumulator drains of some warps overlap the DMMA sweeps of the others.
    int* cnt = reinterpret_cast<int*>(bars + 2);
    constexpr int NWARP = G::THREADS / 32;
    const int first = a.cube_lo + (int)blockIdx.x;
    const int ncb = first < ncubes ? (ncubes - first + cstep - 1) / cstep : 0;     // cubes of this block
    const long long gtot = (long long)ncb * nchunks;
    auto load_g = [&](long long g) {                 // one thread: TMA load of chunk g into buffer g & 1
      if (g < gtot) {
        const int cube = first + (int)(g / nchunks) * cstep, t0 = (int)(g % nchunks) * G::TT;
        int q1, q2, q3;
        origin(cube, q1, q2, q3);
        const int buf = (int)(g & 1);
        mbar_expect_tx(&bars[buf], TILE_BYTES);
        tma_load_4d(Xs + buf * G::HS * G::TSTR, &tmap, &bars[buf], t0, q1 - P, D >= 2 ? q2 - P : 0,
                    D >= 3 ? q3 - P + a.zoff : 0);
      }
    };
    if (tid == 0) {
      cnt[0] = cnt[1] = 0;
      load_g(0);
      load_g(1);
    }
    __syncthreads();                                 // Wp zeroed, counters set
    const int tp = half * 32 + lane;                 // thread of the point's warp pair
    long long g = 0;
    for (int ci = 0; ci < ncb; ++ci) {
      const int cube = first + ci * cstep;
      int o1, o2, o3;
      origin(cube, o1, o2, o3);
      double breg[G::KH];
      {
        const double* f = a.frag + ((long long)cube * G::PPB + pt) * G::KS * 32 + lane;
#pragma unroll
        for (int j = 0; j < G::KH; ++j) {
          const int ks = half * G::KH + j;
          breg[j] = ks < G::KS ? __ldg(f + ks * 32) : 0.0;
        }
      }
      if (MI_STEN_L2PF && ci + 1 < ncb && warp == 0) {
        const char* nf = reinterpret_cast<const char*>(a.frag + (long long)(cube + cstep) * FRAG_CUBE);
        constexpr long long BYTES = FRAG_CUBE * 8;
        for (long long off = (long long)lane * 16384; off < BYTES; off += 32LL * 16384) {
          const unsigned sz = (unsigned)(BYTES - off < 16384 ? BYTES - off : 16384);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(nf + off), "r"(sz) : "memory");
        }
      }
      // this point's output position
      const int q1 = o1 + pt % G::B1, q2 = o2 + (pt / G::B1) % G::B2, q3 = o3 + pt / (G::B1 * G::B2);
      const bool pvalid = q1 < a.n1 && q2 < a.n2 && q3 < a.n3;
      const long long gi = ((long long)q3 * a.n2 + q2) * a.n1 + q1;
      for (int ch = 0; ch < nchunks; ++ch, ++g) {
        const int t0 = ch * G::TT, buf = (int)(g & 1), rb = buf * G::TT;   // W ring half of this chunk
        mbar_wait(&bars[buf], (unsigned)((g >> 1) & 1));                   // X(g) landed
        double acc[G::MT][2];
#pragma unroll
        for (int m = 0; m < G::MT; ++m) acc[m][0] = acc[m][1] = 0.0;
        {
          const double* X = Xs + buf * G::HS * G::TSTR + (base + kl) * G::TSTR + mrow;
          if (t0 + 8 * (G::MT - 1) < a.nt) {
            if (half == 0)
              dmma_sweep<G, 0, G::MT>(X, kl, breg, acc);
            else
              dmma_sweep<G, 1, G::MT>(X, kl, breg, acc);
          } else {
            if (half == 0)
              dmma_sweep<G, 0, 1>(X, kl, breg, acc);
            else
              dmma_sweep<G, 1, 1>(X, kl, breg, acc);
          }
        }
        // the sweep's operand loads have returned (their DMMAs have issued): release the halo buffer
        __syncwarp();
        if (lane == 0) {
          if (atomicAdd(&cnt[buf], 1) == NWARP - 1) {
            cnt[buf] = 0;
            load_g(g + 2);
          }
        }
#pragma unroll
        for (int m = 0; m < G::MT; ++m) {
          wmine[rb + m * 8 + mrow] = acc[m][0];
          wmine[G::WL + rb + m * 8 + mrow] = acc[m][1];
        }
        asm volatile("bar.sync %0, 64;\n" ::"r"(1 + pt) : "memory");      // both K halves of this point are in
        // W of this chunk: thread -> (row pair rp, channel c); 8 consecutive threads write 16 rows (128 B)
        {
          const int rp = tp & 7, c = tp >> 3;
          if (c < a.nc && pvalid) {
            const double* w0 = Wp + pt * G::PSTR + c * G::WL + rb + 2 * rp;
            const double* w1 = w0 + G::PPB * G::PSTR;
            double2 v;
            v.x = w0[0] + w1[0];
            v.y = w0[1] + w1[1];
            *reinterpret_cast<double2*>(a.wout + ((long long)(a.c0 + c) * a.ns + gi) * a.ntp + t0 + 2 * rp) = v;
          }
        }
      }
    }
    return;
  }
#endif
  if (a.cube_lo + (int)blockIdx.x < ncubes) load_chunk(a.cube_lo + blockIdx.x, 0, 0);
  for (int cube = a.cube_lo + blockIdx.x; cube < ncubes; cube += cstep) {
    int o1, o2, o3;
    origin(cube, o1, o2, o3);
    const int next = cube + cstep;
    double breg[G::KH];
    {
      const double* f = a.frag + ((long long)cube * G::PPB + pt) * G::KS * 32 + lane;
#pragma unroll
      for (int j = 0; j < G::KH; ++j) {
        const int ks = half * G::KH + j;
        breg[j] = ks < G::KS ? __ldg(f + ks * 32) : 0.0;
      }
    }
    // the next cube's fragments into L2 while this one sweeps (one bulk prefetch per 16 KB piece)
    if (MI_STEN_PERSIST && MI_STEN_L2PF && next < ncubes && warp == 0) {
      const char* nf = reinterpret_cast<const char*>(a.frag + (long long)next * FRAG_CUBE);
      constexpr long long BYTES = FRAG_CUBE * 8;
      for (long long off = (long long)lane * 16384; off < BYTES; off += 32LL * 16384) {
        const unsigned sz = (unsigned)(BYTES - off < 16384 ? BYTES - off : 16384);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(nf + off), "r"(sz) : "memory");
      }
    }

    // write-out of W of a finished chunk (both K-halves summed) to the time-innermost layout:
    // thread -> (row pair rp, point q, channel c); 8 consecutive threads write 16 consecutive rows (128 B)
    auto write_w = [&](int tc0) {
      const int rp = tid & 7, q = (tid >> 3) % G::PPB, c = tid / (8 * G::PPB);
      const int q1 = o1 + q % G::B1, q2 = o2 + (q / G::B1) % G::B2, q3 = o3 + q / (G::B1 * G::B2);
      if (c >= a.nc || q1 >= a.n1 || q2 >= a.n2 || q3 >= a.n3) return;
      const long long gi = ((long long)q3 * a.n2 + q2) * a.n1 + q1;
      const double* w0 = Wp + q * G::PSTR + c * G::WL;
      const double* w1 = w0 + G::PPB * G::PSTR;
      const int t = tc0 + 2 * rp;                    // tc0 is a multiple of TT; ntp a multiple of TT
      const int r = t % G::WL;
      double2 v;
      v.x = w0[r] + w1[r];
      v.y = w0[r + 1] + w1[r + 1];
      *reinterpret_cast<double2*>(a.wout + ((long long)(a.c0 + c) * a.ns + gi) * a.ntp + t) = v;
    };

    for (int ch = 0; ch < nchunks; ++ch, ++gc) {
      const int t0 = ch * G::TT;
      if (t0 < a.nt) mbar_wait(&bars[gc & 1], (gc >> 1) & 1);   // X(ch) landed (k-th use of buffer -> parity k&1)
      __syncthreads();                // other buffer free; W rows of chunk ch-1 complete
      if (ch + 1 < nchunks)
        load_chunk(cube, (gc + 1) & 1, t0 + G::TT);
      else if (next < ncubes)
        load_chunk(next, (gc + 1) & 1, 0);           // the next cube's first tile
      // ---- W of chunk ch-1 to HBM (its partials were completed before the barrier)
      if (ch >= 1) write_w(t0 - G::TT);
      // ---- DMMA sweep of chunk ch into this half's W partial rows
      {
        double acc[G::MT][2];
#pragma unroll
        for (int m = 0; m < G::MT; ++m) acc[m][0] = acc[m][1] = 0.0;
        if (t0 < a.nt) {
          const double* X = Xs + (gc & 1) * G::HS * G::TSTR + (base + kl) * G::TSTR + mrow;
          // the last chunk skips M-tiles that lie wholly past nt (warp-uniform)
          if (t0 + 8 * (G::MT - 1) < a.nt) {
            if (half == 0)
              dmma_sweep<G, 0, G::MT>(X, kl, breg, acc);
            else
              dmma_sweep<G, 1, G::MT>(X, kl, breg, acc);
          } else {
            if (half == 0)
              dmma_sweep<G, 0, 1>(X, kl, breg, acc);
            else
              dmma_sweep<G, 1, 1>(X, kl, breg, acc);
          }
        }
#pragma unroll
        for (int m = 0; m < G::MT; ++m) {
          const int r = (t0 + m * 8 + mrow) % G::WL;
          wmine[r] = acc[m][0];
          wmine[G::WL + r] = acc[m][1];
        }
      }
    }
    // W of the last chunk
    __syncthreads();
    write_w((nchunks - 1) * G::TT);
  }
}

// y[t, i] (+)= sum_c sum_k band_c[t, k] W_c[t - pt + k, i] with W time-innermost
// (nchan, ns, ntp): thread = one spatial point x TR time rows; per channel it reads
// TR + 2 pt contiguous values (16-byte loads), the band rows of the block's TR rows
// are staged in smem (shared by all points).  Writes y coalesced along i.
template <int TR, int PT>
__global__ void __launch_bounds__(128) time_filter_ti(const double* __restrict__ w, const double* __restrict__ band,
                                                      double* __restrict__ y, int nchan, int nt, int ntp,
                                                      long long ns, int accumulate) {
  constexpr int PX = PT + (PT & 1), BWX = 2 * PT + 1;   // PX even: 16-byte aligned pairs
  extern __shared__ double bs[];                     // [nchan][TR][BWX]
  const long long i = blockIdx.x * 128LL + threadIdx.x;
  const int t0 = blockIdx.y * TR;
  constexpr int W = 2 * PT + 1;
  for (int e = threadIdx.x; e < nchan * TR * W; e += blockDim.x) {
    const int k = e % W, r = (e / W) % TR, c = e / (W * TR);
    const int t = t0 + r;
    bs[(c * TR + r) * BWX + k] = t < nt ? band[((long long)c * nt + t) * W + k] : 0.0;
  }
  __syncthreads();
  if (i >= ns) return;
  double acc[TR];
#pragma unroll
  for (int r = 0; r < TR; ++r) acc[r] = 0.0;
  for (int c = 0; c < nchan; ++c) {
    const double* wc = w + ((long long)c * ns + i) * ntp;
    double v[TR + 2 * PX];
#pragma unroll
    for (int r = 0; r < TR + 2 * PX; r += 2) {
      const int t = t0 - PX + r;                     // even: t0, PX even -> 16-byte aligned pairs
      if (t >= 0 && t + 1 < ntp) {
        const double2 q = __ldg(reinterpret_cast<const double2*>(wc + t));
        v[r] = q.x;
        v[r + 1] = q.y;
      } else {
        v[r] = (t >= 0 && t < ntp) ? __ldg(wc + t) : 0.0;
        v[r + 1] = (t + 1 >= 0 && t + 1 < ntp) ? __ldg(wc + t + 1) : 0.0;
      }
    }
    const double* bc = bs + c * TR * BWX;
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int k = 0; k < W; ++k) acc[r] = fma(bc[r * BWX + k], v[r + PX - PT + k], acc[r]);
  }
#pragma unroll
  for (int r = 0; r < TR; ++r) {
    const int t = t0 + r;
    if (t < nt) {
      double* dst = y + (long long)t * ns + i;
      if (accumulate) *dst += acc[r]; else *dst = acc[r];
    }
  }
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
  const int pt = (int)(pid % G::PPB);
  const long long cube = pid / G::PPB;
  const int cc1 = (int)(cube % C1), cc2 = (int)((cube / C1) % C2), cc3 = (int)(cube / ((long long)C1 * C2));
  const int i1 = cc1 * G::B1 + pt % G::B1, i2 = cc2 * G::B2 + (pt / G::B1) % G::B2,
            i3 = cc3 * G::B3 + pt / (G::B1 * G::B2);
  const int ch = lane >> 2;
  const int s = ks * 4 + (lane & 3);              // stencil index (unpadded K order)
  double v = 0.0;
  if (ch < nc && s < G::S && i1 < n1 && i2 < n2 && i3 < n3) {
    const long long i = ((long long)i3 * n2 + i2) * n1 + i1;
    v = sten[((long long)(c0 + ch) * G::S + s) * ns + i];
  }
  frag[e] = v;
}

}  // namespace mi
