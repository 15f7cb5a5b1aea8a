// Banded time filter of the operator on the FP64 tensor cores (HBM-bound):
//
//   y[t][i] = sum_c sum_k band_c[t][k] W_c[i][t - p_t + k]
//
// W (the per-channel spatial stencil partials, stencil_dmma.cuh) is stored
// time-innermost: W[c][i][ntp].  A block owns one block of TR = 56 output
// time rows (7 DMMA m-tiles) and walks point tiles of 64 points; per channel
// it streams the (64 points x 64 times) W window by TMA -- four 16 x 64 boxes
// with 128-byte swizzle, so the B-fragment reads are conflict-free -- through
// a 6-stage mbarrier pipeline, and accumulates Band_c (8 rows x 16 times per
// k-window, from a compact copy in shared memory) x W_c on the tensor cores.
// The time halo over-read is 64 / 56; everything else is read once.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace mi {

struct TFilterCfg {
  static constexpr int MT = 7, TR = 8 * MT;         // output time rows per block
  static constexpr int PX = 4, TW = TR + 2 * PX;    // window (= 64): times t0 - PX .. t0 + TR + PX - 1
  static constexpr int NP = 64;                      // points per tile
  static constexpr int STAGE = NP * TW;              // doubles per stage (4 boxes of 16 x 64)
  // FRAG: the band A fragments stored fragment-major [c][m][j][lane] (conflict-free LDS; 5 stages so
  // 8 channels fit); else the compact band rows [c][row][k] (6 stages; 2-way bank conflicts)
  static constexpr __host__ __device__ int nst(bool frag) { return frag ? 5 : 6; }
  static __host__ __device__ size_t bands(int pt, int nchan, bool frag) {
    return frag ? (size_t)nchan * MT * 4 * 32 : (size_t)nchan * TR * (2 * pt + 1);
  }
  static size_t smem(int pt, int nchan, bool frag) {
    return 1024 + (size_t)nst(frag) * STAGE * 8 + bands(pt, nchan, frag) * 8 + 128;
  }
};

template <int PT, bool FRAG>
__global__ void __launch_bounds__(256, 1) time_filter_dmma(const __grid_constant__ CUtensorMap tmap,
                                                           const double* __restrict__ band, double* __restrict__ y,
                                                           int nchan, int nt, long long ns, int ntb, int accumulate) {
  using F = TFilterCfg;
  constexpr int BW = 2 * PT + 1;
  constexpr int NST = F::nst(FRAG);
  static_assert(PT <= F::PX, "time degree too large for the filter window");
  extern __shared__ __align__(1024) unsigned char raw[];
  // 1024-byte aligned stage buffers (128-byte swizzle atoms)
  double* stages = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  double* bands = stages + NST * F::STAGE;                      // [nchan][TR][BW]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bands + F::bands(PT, nchan, FRAG));   // full[NST]
  unsigned long long* empty = bars + NST;                                                        // empty[NST]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, fk = lane & 3;
  const int tb = blockIdx.x % ntb;
  const int t0 = tb * F::TR;
  const long long npt = (ns + F::NP - 1) / F::NP;
  const long long p_first = blockIdx.x / ntb, p_step = gridDim.x / ntb;
  if constexpr (FRAG) {
    // A fragment of (channel c, m-tile m, k-step j) for lane (g, f): band row 8 m + g, column 4 j + f - g - PX + PT
    for (int e = tid; e < nchan * F::MT * 128; e += 256) {
      const int ln = e & 31, j = (e >> 5) & 3, m = (e >> 7) % F::MT, c = e / (F::MT * 128);
      const int g = ln >> 2, f = ln & 3, k = 4 * j + f - g - F::PX + PT, t = t0 + 8 * m + g;
      bands[e] = (t < nt && k >= 0 && k < BW) ? band[((long long)c * nt + t) * BW + k] : 0.0;
    }
  } else {
    // compact band rows of this time block
    for (int e = tid; e < nchan * F::TR * BW; e += 256) {
      const int k = e % BW, r = (e / BW) % F::TR, c = e / (BW * F::TR);
      const int t = t0 + r;
      bands[e] = t < nt ? band[((long long)c * nt + t) * BW + k] : 0.0;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&empty[s], 8);                       // one arrival per warp when it is done with the stage
    }
    mbar_fence_init();
  }
  __syncthreads();
  // steps: (point tile, channel); step s of this block -> tile p_first + (s / nchan) * p_step, channel s % nchan
  const long long ntiles = p_first < npt ? (npt - 1 - p_first) / p_step + 1 : 0;
  const long long nsteps = ntiles * nchan;
  auto issue = [&](long long s) {
    const long long p = p_first + (s / nchan) * p_step;
    const int c = (int)(s % nchan);
    double* dst = stages + (s % NST) * F::STAGE;
    unsigned long long* bar = &bars[s % NST];
    mbar_expect_tx(bar, F::STAGE * 8);
    const int row = (int)((long long)c * ns + p * F::NP);
#pragma unroll
    for (int q = 0; q < F::TW / 16; ++q) tma_load_2d(dst + q * (F::NP * 16), &tmap, bar, t0 - F::PX + 16 * q, row);
  };
  if (tid == 0)
    for (long long s = 0; s < NST - 1 && s < nsteps; ++s) issue(s);
  // per-lane band offsets of the 4 k-steps of an m-tile: band column kk = 4 j + fk - gq - PX + PT
  int kk[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) kk[j] = 4 * j + fk - gq - F::PX + PT;
  const int r8 = 8 * warp + gq;                          // this lane's B row (point within the tile)
  // swizzled byte offsets of this lane's B elements: window time tk = C + fk with C = 8 m + 4 j
  // (compile-time): box C >> 4, 16-byte unit ((C & 15) >> 1) + (fk >> 1) XOR (r8 & 7), half fk & 1
  int pb[4];
#pragma unroll
  for (int v = 0; v < 4; ++v)
    pb[v] = r8 * 128 + ((((2 * v) ^ (r8 & 6)) + ((fk >> 1) ^ (r8 & 1))) << 4) + ((fk & 1) << 3);
  bool kv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) kv[j] = kk[j] >= 0 && kk[j] < BW;
  double acc[F::MT][2];
#pragma unroll
  for (int m = 0; m < F::MT; ++m) acc[m][0] = acc[m][1] = 0.0;
  const bool pair = (ns & 1) == 0;                      // y rows 16-byte aligned at even points
  for (long long s = 0; s < nsteps; ++s) {
    if (tid == 0 && s + NST - 1 < nsteps) {
      // refill the stage step s - 1 used, once all 8 warps have released it
      const long long f = s + NST - 1;
      if (f >= NST) mbar_wait(&empty[f % NST], (unsigned)(((f / NST) - 1) & 1));
      issue(f);
    }
    mbar_wait(&bars[s % NST], (unsigned)((s / NST) & 1));
    const int c = (int)(s % nchan);
    const unsigned char* st = reinterpret_cast<const unsigned char*>(stages + (s % NST) * F::STAGE);
    const double* bc = bands + c * (FRAG ? F::MT * 128 : F::TR * BW);
#pragma unroll
    for (int m = 0; m < F::MT; ++m) {
      const double* brow = bc + (8 * m + gq) * BW;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double av = FRAG ? bc[(m * 4 + j) * 32 + lane] : (kv[j] ? brow[kk[j]] : 0.0);
        const int C = 8 * m + 4 * j;
        const double bv = *reinterpret_cast<const double*>(st + pb[((C & 15) >> 2)] + (C >> 4) * (F::NP * 128));
        dmma(acc[m][0], acc[m][1], av, bv);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s % NST]);
    if (c == nchan - 1) {
      const long long p = p_first + (s / nchan) * p_step;
      const long long i0 = p * F::NP + 8 * warp + 2 * fk;
#pragma unroll
      for (int m = 0; m < F::MT; ++m) {
        const int t = t0 + 8 * m + gq;
        if (t < nt) {
          double* dst = y + (long long)t * ns + i0;
          if (accumulate) {
            if (i0 < ns) dst[0] += acc[m][0];
            if (i0 + 1 < ns) dst[1] += acc[m][1];
          } else if (pair && i0 + 1 < ns) {
            *reinterpret_cast<double2*>(dst) = make_double2(acc[m][0], acc[m][1]);
          } else {
            if (i0 < ns) dst[0] = acc[m][0];
            if (i0 + 1 < ns) dst[1] = acc[m][1];
          }
        }
        acc[m][0] = acc[m][1] = 0.0;
      }
    }
  }
}

}  // namespace mi
