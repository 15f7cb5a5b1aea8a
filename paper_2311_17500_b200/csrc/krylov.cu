// Krylov vector kernels for the device GMRES (reference gmres, linalg.py:367-447:
// CGS2 dots/updates 405-411, basis append 434, solution update 444).
// Deterministic reductions: a fixed grid of KB blocks writes per-block
// partials, a second kernel adds them in a fixed tree order.
#include "common.cuh"

namespace mi {

#ifndef MI_KRY_KB
#define MI_KRY_KB 296
#endif
#ifndef MI_KRY_KU
#define MI_KRY_KU 1
#endif
constexpr int KB = MI_KRY_KB;   // reduction blocks: 2 x 148 SMs, one wave at <= 128 registers
constexpr int KT = 256;
constexpr int KG = 8;     // vectors per pass
constexpr int KU = MI_KRY_KU;   // elements per thread per loop trip (independent loads in flight)

// Every reduction below walks its block's chunk [lo, hi) in the same order -- thread t takes
// j = lo + t + u KT for u < KU, then advances by KU KT -- so the fused and the two-pass kernels sum
// in the same order and agree bit for bit.

template <int G>
__global__ void __launch_bounds__(KT, 2) dots_partial(const double* __restrict__ V, long long ldv,
                                                   const double* __restrict__ w, long long n, int k0,
                                                   int k, double* __restrict__ part) {
  __shared__ double red[G][KT / 32];
  double acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = 0.0;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  for (long long b = lo + threadIdx.x; b < hi; b += KU * KT) {
    double wv[KU], vv[KU][G];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const long long i = b + (long long)u * KT;
      const bool ok = i < hi;
      wv[u] = ok ? w[i] : 0.0;
#pragma unroll
      for (int g = 0; g < G; ++g) vv[u][g] = (ok && k0 + g < k) ? V[(long long)(k0 + g) * ldv + i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u)
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (b + (long long)u * KT < hi && k0 + g < k) acc[g] = fma(vv[u][g], wv[u], acc[g]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double v = acc[g];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[g][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < G && k0 + threadIdx.x < k) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < KT / 32; ++q) v += red[threadIdx.x][q];
    part[(long long)(k0 + threadIdx.x) * gridDim.x + blockIdx.x] = v;
  }
}

__global__ void dots_final(const double* __restrict__ part, int nb, double* __restrict__ h, int hstride) {
  __shared__ double s[1024];
  const int k = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += part[(long long)k * nb + b];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) h[(long long)k * hstride] = s[0];
}

__global__ void sub_comb(const double* __restrict__ V, long long ldv, const double* __restrict__ h, int k,
                         double* __restrict__ w, long long n) {
  extern __shared__ double hs[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc = fma(hs[i], V[(long long)i * ldv + j], acc);
    w[j] -= acc;
  }
}

__global__ void comb(const double* __restrict__ V, long long ldv, const double* __restrict__ y, int k,
                     const double* __restrict__ x0, double* __restrict__ out, long long n) {
  extern __shared__ double ys[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc = fma(ys[i], V[(long long)i * ldv + j], acc);
    out[j] = (x0 ? x0[j] : 0.0) + acc;
  }
}

__global__ void scale_div(const double* __restrict__ x, const double* __restrict__ s, double* __restrict__ out,
                          long long n, int take_sqrt) {
  const double d = take_sqrt ? sqrt(*s) : *s;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < n; b += KU * stride) {
    double v[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) v[u] = b + u * stride < n ? x[b + u * stride] : 0.0;
#pragma unroll
    for (int u = 0; u < KU; ++u)
      if (b + u * stride < n) out[b + u * stride] = v[u] / d;
  }
}

// Fused CGS2 pass (k <= KM basis vectors): w -= V h, then h_out = V^T w (the second classical
// Gram-Schmidt pass's dots); each V entry streams from HBM once (the reduction re-reads it from L1).
// Per-block partials in a fixed partition, reduced by dots_final, in the same order as
// sub_comb + dots_partial: the two agree bit for bit.
template <int KM>
__global__ void __launch_bounds__(KT, 2) sub_reduce(const double* __restrict__ V, long long ldv,
                                                    const double* __restrict__ h, int k, double* __restrict__ w,
                                                    long long n, double* __restrict__ part) {
  __shared__ double hs[KM];
  __shared__ double red[KM][KT / 32];
  if (threadIdx.x < KM) hs[threadIdx.x] = threadIdx.x < k ? h[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[KM];
#pragma unroll
  for (int g = 0; g < KM; ++g) acc[g] = 0.0;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  for (long long b = lo + threadIdx.x; b < hi; b += KU * KT) {
    double wn[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const long long j = b + (long long)u * KT;
      double sacc = 0.0;
      if (j < hi) {
#pragma unroll
        for (int i = 0; i < KM; ++i)
          if (i < k) sacc = fma(hs[i], V[(long long)i * ldv + j], sacc);
        wn[u] = w[j] - sacc;
        w[j] = wn[u];
      }
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const long long j = b + (long long)u * KT;
      if (j < hi) {
#pragma unroll
        for (int i = 0; i < KM; ++i)
          if (i < k) acc[i] = fma(V[(long long)i * ldv + j], wn[u], acc[i]);   // second read: L1
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < KM; ++g) {
    double x = acc[g];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[g][warp] = x;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < k; g += KT) {
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < KT / 32; ++q) x += red[g][q];
    part[(long long)g * gridDim.x + blockIdx.x] = x;
  }
}

static int grid_for(long long n) {
  long long b = (n + 255) / 256;
  return (int)(b < 148LL * 16 ? b : 148LL * 16);
}

}  // namespace mi

using namespace mi;

extern "C" {

int mi_dots(mi_ctx* c, long long n, int k, const double* V, long long ldv, const double* w, double* h) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr && k >= 0, MI_ERR_ARG, "bad arguments to mi_dots");
  if (k == 0) return MI_OK;
  int rc;
  if ((rc = dalloc(c->partials, (size_t)k * KB))) return rc;
  ProfScope ps(c, PROF_KRYLOV, (k + KG - 1) / KG + 1);
  for (int k0 = 0; k0 < k; k0 += KG) {
    dots_partial<KG><<<KB, KT, 0, c->stream>>>(V, ldv, w, n, k0, k, c->partials.p);
    MI_CHECK_LAUNCH("dots_partial");
  }
  dots_final<<<k, 512, 0, c->stream>>>(c->partials.p, KB, h, 1);
  MI_CHECK_LAUNCH("dots_final");
  return MI_OK;
}

int mi_sub_combination(mi_ctx* c, long long n, int k, const double* V, long long ldv, const double* h, double* w) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr && k >= 0, MI_ERR_ARG, "bad arguments to mi_sub_combination");
  if (k == 0) return MI_OK;
  ProfScope ps(c, PROF_KRYLOV);
  sub_comb<<<grid_for(n), 256, sizeof(double) * k, c->stream>>>(V, ldv, h, k, w, n);
  MI_CHECK_LAUNCH("sub_comb");
  return MI_OK;
}

int mi_combination(mi_ctx* c, long long n, int k, const double* V, long long ldv, const double* y,
                   const double* x0, double* out) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr && k >= 0, MI_ERR_ARG, "bad arguments to mi_combination");
  ProfScope ps(c, PROF_KRYLOV);
  comb<<<grid_for(n), 256, sizeof(double) * (k > 0 ? k : 1), c->stream>>>(V, ldv, y, k, x0, out, n);
  MI_CHECK_LAUNCH("comb");
  return MI_OK;
}

int mi_scale_inv(mi_ctx* c, long long n, const double* x, const double* hnorm, double* out) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  ProfScope ps(c, PROF_KRYLOV);
  scale_div<<<grid_for(n), 256, 0, c->stream>>>(x, hnorm, out, n, 0);
  MI_CHECK_LAUNCH("scale_div");
  return MI_OK;
}

int mi_normalize(mi_ctx* c, long long n, const double* x, const double* nrm2, double* out) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  ProfScope ps(c, PROF_KRYLOV);
  scale_div<<<grid_for(n), 256, 0, c->stream>>>(x, nrm2, out, n, 1);
  MI_CHECK_LAUNCH("scale_div");
  return MI_OK;
}

int mi_cgs_pass(mi_ctx* c, long long n, int k, const double* V, long long ldv, const double* h_in, double* w,
                double* h_out) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr && k >= 0, MI_ERR_ARG, "bad arguments to mi_cgs_pass");
  if (k == 0) return MI_OK;
  // fused for k <= 8 (one read of V: 0.70 vs 0.90 ms at N = 37 M); beyond, the elementwise subtraction
  // plus the 8-row reductions stream at ~6 TB/s and tie or beat the fused kernel, whose per-thread row
  // count limits its loads in flight (tools/time_krylov.py, profiles/r02_optimisation_log.md K3)
  if (k > 8) {
    int rc = mi_sub_combination(c, n, k, V, ldv, h_in, w);
    if (rc) return rc;
    return mi_dots(c, n, k, V, ldv, w, h_out);
  }
  int rc;
  if ((rc = dalloc(c->partials, (size_t)k * KB))) return rc;
  ProfScope ps(c, PROF_KRYLOV, 2);
  sub_reduce<8><<<KB, KT, 0, c->stream>>>(V, ldv, h_in, k, w, n, c->partials.p);
  MI_CHECK_LAUNCH("sub_reduce");
  dots_final<<<k, 512, 0, c->stream>>>(c->partials.p, KB, h_out, 1);
  MI_CHECK_LAUNCH("dots_final");
  return MI_OK;
}

int mi_cgs_norm_pass(mi_ctx* c, long long n, int k, const double* V, long long ldv, const double* h_in, double* w,
                     double* nrm2) {
  // the last CGS2 subtraction and |w|^2 as two streaming passes: measured faster than a fused kernel
  // at every k (0.54 vs 0.74 ms at k = 8, N = 37 M)
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr && k >= 0, MI_ERR_ARG, "bad arguments to mi_cgs_norm_pass");
  int rc = mi_sub_combination(c, n, k, V, ldv, h_in, w);
  if (rc) return rc;
  return mi_dots(c, n, 1, w, n, w, nrm2);
}

}  // extern "C"
