// Operator A = sum_c T_c (x) S_c  (reference: KroneckerOperator.matvec,
// assembly.py:430-444, with the terms of _Workspace.operator, solver.py:213-236,
// and the Spline Upwind terms of StabilizationMatrices.terms, stabilization.py:439-445).
//
// Every Kronecker term of the reference is one "channel": a banded time
// factor T_c and a spatial factor S_c.  Spatial factors are (2p+1)^d
// stencils generated on the device:
//   * Kronecker channels (M_s, K_s, K_sigma: assembly.py:222-238) from 1D bands,
//   * Spline Upwind channels (S^s_r: the theta_r-weighted spatial mass,
//     stabilization.py:469-488) from theta_r and 1D hat triple products.
// Apply: W_c = S_c x (one stencil sweep per channel group), then
// y = sum_c T_c W_c along time (banded), plus the reaction correction.
#include "common.cuh"
#include "dispatch.cuh"
#include "stencil_dmma.cuh"
#include "tfilter.cuh"

typedef CUresult (*mi_encode_tiled_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                       CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                       CUtensorMapFloatOOBfill);

namespace mi {

struct Dims {
  int n1, n2, n3, nt;
  long long ns, N;
  int z_lo, n3g;        // global plane of local z = 0, global n_3 (z-slab contexts)
};

static Dims dims_of(const mi_ctx* c) {
  return Dims{c->n[0], c->n[1], c->n[2], c->nt, c->ns, c->N, c->z_lo, c->n3g};
}

// rows of the host 1D tables (bands, hat triple products): global in every direction
static int table_rows(const mi_ctx* c) { return std::max(c->n[0], std::max(c->n[1], c->n3g)); }

template <int D, int P>
struct Sten {
  static constexpr int W = 2 * P + 1;
  static constexpr int W1 = W;
  static constexpr int W2 = D >= 2 ? W : 1;
  static constexpr int W3 = D >= 3 ? W : 1;
  static constexpr int S = W1 * W2 * W3;
};

// ---------------------------------------------------------------- build
template <int D, int P>
__global__ void build_kron_channel(double* __restrict__ out, const double* __restrict__ coef,
                                   const double* __restrict__ bands, int nterms, int nmax, Dims g) {
  using ST = Sten<D, P>;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (i >= g.ns) return;
  const int a1 = s % ST::W1, a2 = (s / ST::W1) % ST::W2, a3 = s / (ST::W1 * ST::W2);
  const int i1 = (int)(i % g.n1), i2 = (int)((i / g.n1) % g.n2),
            i3 = (int)(i / ((long long)g.n1 * g.n2)) + g.z_lo;     // global plane
  const int ii[3] = {i1, i2, i3};
  const int aa[3] = {a1, a2, a3};
  const int nn[3] = {g.n1, g.n2, g.n3g};
  bool inside = true;
#pragma unroll
  for (int l = 0; l < D; ++l) {
    int j = ii[l] + aa[l] - P;
    inside = inside && j >= 0 && j < nn[l];
  }
  double v = 0.0;
  if (inside) {
    const int W = 2 * P + 1;
    for (int t = 0; t < nterms; ++t) {
      double prod = coef[t];
#pragma unroll
      for (int l = 0; l < D; ++l)
        prod *= bands[(((long long)t * D + l) * nmax + ii[l]) * W + aa[l]];
      v += prod;
    }
  }
  out[(long long)s * g.ns + i] = v;
}

template <int D, int P>
__global__ void build_su_channel(double* __restrict__ out, const double* __restrict__ theta,
                                 const double* __restrict__ H, int ko, int nmax, Dims g) {
  using ST = Sten<D, P>;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (i >= g.ns) return;
  const int a1 = s % ST::W1, a2 = (s / ST::W1) % ST::W2, a3 = s / (ST::W1 * ST::W2);
  const int i1 = (int)(i % g.n1), i2 = (int)((i / g.n1) % g.n2),
            i3 = (int)(i / ((long long)g.n1 * g.n2)) + g.z_lo;     // global plane (theta, H are global)
  const int ii[3] = {i1, i2, i3};
  const int aa[3] = {a1, a2, a3};
  const int nn[3] = {g.n1, g.n2, g.n3g};
  const int W = 2 * P + 1;
  const int KW = 2 * ko + 1;
  bool inside = true;
#pragma unroll
  for (int l = 0; l < D; ++l) {
    int j = ii[l] + aa[l] - P;
    inside = inside && j >= 0 && j < nn[l];
  }
  double v = 0.0;
  if (inside) {
    // H_l row pointers for (i_l, a_l)
    const double* h[3];
#pragma unroll
    for (int l = 0; l < D; ++l) h[l] = H + (((long long)l * nmax + ii[l]) * W + aa[l]) * KW;
    const int b3n = D >= 3 ? KW : 1, b2n = D >= 2 ? KW : 1;
    for (int b3 = 0; b3 < b3n; ++b3) {
      int k3 = D >= 3 ? i3 + b3 - ko : 0;
      if (k3 < 0 || k3 >= g.n3g) continue;
      double h3 = D >= 3 ? h[2][b3] : 1.0;
      if (h3 == 0.0) continue;
      for (int b2 = 0; b2 < b2n; ++b2) {
        int k2 = D >= 2 ? i2 + b2 - ko : 0;
        if (k2 < 0 || k2 >= g.n2) continue;
        double h23 = h3 * (D >= 2 ? h[1][b2] : 1.0);
        if (h23 == 0.0) continue;
        const double* th = theta + ((long long)k3 * g.n2 + k2) * g.n1;
        double acc = 0.0;
        for (int b1 = 0; b1 < KW; ++b1) {
          int k1 = i1 + b1 - ko;
          if (k1 < 0 || k1 >= g.n1) continue;
          acc += th[k1] * h[0][b1];
        }
        v += h23 * acc;
      }
    }
  }
  out[(long long)s * g.ns + i] = v;
}

// Mapped-geometry spatial factors (SpatialQuadratureData.mass / .stiffness, assembly.py:197-219):
//   S[i, j] = sum_t coef_t sum_k theta_t[k] prod_l T_{t,l}[i_l, j_l - i_l + p, k_l - (i_l - p) q_l]
// over the tensor Gauss grid k (q_l points per element, Q_l in total).  theta_t = w |det J| (mass) or
// w |det J| (J^-1 J^-T)_ab (stiffness term a, b); T_{t,l}[i, a, b] = B^(o)_i(x_k) B^(o')_j(x_k) with the
// derivative orders of the term.  Function i's support covers the Gauss points
// [(i - p) q_l, (i + 1) q_l): KW_l = (p + 1) q_l window entries.
struct QuadSpec {
  int q[3], Q[3];       // Gauss points per element / in total, per direction (1 beyond d)
  int kw;               // window length (max over directions) = row stride of the T tables
  long long nq;         // Q_1 Q_2 Q_3
  int kwl[3];           // window length per direction
  const int* kst;       // device [3][nmax]: first Gauss point of function i's window (null: (i - p) q)
  int nmax;
  __device__ int k0(int l, int i, int P) const { return kst ? kst[l * nmax + i] : (i - P) * q[l]; }
};

template <int D, int P>
__global__ void build_quad_channel(double* __restrict__ out, const double* __restrict__ coef,
                                   const double* __restrict__ theta, const double* __restrict__ T, int nterms,
                                   int nmax, QuadSpec qs, Dims g) {
  using ST = Sten<D, P>;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (i >= g.ns) return;
  const int a1 = s % ST::W1, a2 = (s / ST::W1) % ST::W2, a3 = s / (ST::W1 * ST::W2);
  const int i1 = (int)(i % g.n1), i2 = (int)((i / g.n1) % g.n2), i3 = (int)(i / ((long long)g.n1 * g.n2)) + g.z_lo;
  const int ii[3] = {i1, i2, i3};
  const int aa[3] = {a1, a2, a3};
  const int nn[3] = {g.n1, g.n2, g.n3g};
  const int W = 2 * P + 1;
  bool inside = true;
#pragma unroll
  for (int l = 0; l < D; ++l) {
    int j = ii[l] + aa[l] - P;
    inside = inside && j >= 0 && j < nn[l];
  }
  double v = 0.0;
  if (inside) {
    const int kw1 = qs.kwl[0];
    const int kw2 = D >= 2 ? qs.kwl[1] : 1, kw3 = D >= 3 ? qs.kwl[2] : 1;
    const int s1 = qs.k0(0, i1, P), s2 = D >= 2 ? qs.k0(1, i2, P) : 0, s3 = D >= 3 ? qs.k0(2, i3, P) : 0;
    for (int t = 0; t < nterms; ++t) {
      const double* th = theta + (long long)t * qs.nq;
      const double* h[3];
#pragma unroll
      for (int l = 0; l < D; ++l) h[l] = T + ((((long long)t * D + l) * nmax + ii[l]) * W + aa[l]) * qs.kw;
      double vt = 0.0;
      for (int b3 = 0; b3 < kw3; ++b3) {
        const int k3 = D >= 3 ? s3 + b3 : 0;
        if (k3 < 0 || k3 >= qs.Q[2]) continue;
        const double h3 = D >= 3 ? h[2][b3] : 1.0;
        if (h3 == 0.0) continue;
        for (int b2 = 0; b2 < kw2; ++b2) {
          const int k2 = D >= 2 ? s2 + b2 : 0;
          if (k2 < 0 || k2 >= qs.Q[1]) continue;
          const double h23 = h3 * (D >= 2 ? h[1][b2] : 1.0);
          if (h23 == 0.0) continue;
          const double* tr = th + ((long long)k3 * qs.Q[1] + k2) * qs.Q[0];
          double acc = 0.0;
          for (int b1 = 0; b1 < kw1; ++b1) {
            const int k1 = s1 + b1;
            if (k1 < 0 || k1 >= qs.Q[0]) continue;
            acc += tr[k1] * h[0][b1];
          }
          vt += h23 * acc;
        }
      }
      v += coef[t] * vt;
    }
  }
  out[(long long)s * g.ns + i] = v;
}

// Sum-factorised form of build_quad_channel for d = 3: one block per point i, the term's Gauss-weight
// window theta[k3][k2][k1] (KW^3) staged in shared memory, then contracted one direction at a time
// (k1 -> a1, k2 -> a2, k3 -> a3): ~KW^3 W + KW^2 W^2 + KW W^3 multiply-adds per term instead of
// W^3 KW^3.
template <int P, int KW>
__global__ void __launch_bounds__(256) build_quad_channel_sf(double* __restrict__ out, const double* __restrict__ coef,
                                                            const double* __restrict__ theta,
                                                            const double* __restrict__ T, int nterms, int nmax,
                                                            QuadSpec qs, Dims g) {
  constexpr int W = 2 * P + 1, S = W * W * W;
  extern __shared__ double smq[];
  double* th = smq;                                  // [KW^3] Gauss-weight window
  double* a1s = th + KW * KW * KW;                   // [KW][KW][W]
  double* a2s = a1s + KW * KW * W;                   // [KW][W][W]
  double (*h)[W * KW] = reinterpret_cast<double (*)[W * KW]>(a2s + KW * W * W);   // [3][W * KW]
  const long long i = blockIdx.x;
  const int tid = threadIdx.x;
  const int i1 = (int)(i % g.n1), i2 = (int)((i / g.n1) % g.n2), i3 = (int)(i / ((long long)g.n1 * g.n2)) + g.z_lo;
  const int ii[3] = {i1, i2, i3};
  const int k0[3] = {qs.k0(0, i1, P), qs.k0(1, i2, P), qs.k0(2, i3, P)};
  const int kw[3] = {qs.kwl[0], qs.kwl[1], qs.kwl[2]};
  double acc[(S + 255) / 256];
#pragma unroll
  for (int r = 0; r < (S + 255) / 256; ++r) acc[r] = 0.0;
  for (int t = 0; t < nterms; ++t) {
    __syncthreads();                                 // previous term's stages are done with th / h
    for (int e = tid; e < KW * KW * KW; e += 256) {
      const int b1 = e % KW, b2 = (e / KW) % KW, b3 = e / (KW * KW);
      const int k1 = k0[0] + b1, k2 = k0[1] + b2, k3 = k0[2] + b3;
      const bool ok = b1 < kw[0] && b2 < kw[1] && b3 < kw[2] && k1 >= 0 && k1 < qs.Q[0] && k2 >= 0 &&
                      k2 < qs.Q[1] && k3 >= 0 && k3 < qs.Q[2];
      th[e] = ok ? __ldg(theta + (long long)t * qs.nq + ((long long)k3 * qs.Q[1] + k2) * qs.Q[0] + k1) : 0.0;
    }
    for (int e = tid; e < 3 * W * KW; e += 256) {
      const int l = e / (W * KW), r = e % (W * KW), a = r / KW, b = r % KW;
      h[l][r] = b < qs.kw ? __ldg(T + ((((long long)t * 3 + l) * nmax + ii[l]) * W + a) * qs.kw + b) : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < KW * KW * W; e += 256) {    // a1s[b3][b2][a1] = sum_b1 h1[a1][b1] th[b3][b2][b1]
      const int a1 = e % W, b23 = e / W;
      const double* tr = th + b23 * KW;
      const double* hr = h[0] + a1 * KW;
      double v = 0.0;
#pragma unroll
      for (int b = 0; b < KW; ++b) v = fma(hr[b], tr[b], v);
      a1s[e] = v;
    }
    __syncthreads();
    for (int e = tid; e < KW * W * W; e += 256) {     // a2s[b3][a2][a1] = sum_b2 h2[a2][b2] a1s[b3][b2][a1]
      const int a1 = e % W, a2 = (e / W) % W, b3 = e / (W * W);
      const double* hr = h[1] + a2 * KW;
      double v = 0.0;
#pragma unroll
      for (int b = 0; b < KW; ++b) v = fma(hr[b], a1s[(b3 * KW + b) * W + a1], v);
      a2s[e] = v;
    }
    __syncthreads();
    const double ct = __ldg(coef + t);
#pragma unroll
    for (int r = 0; r < (S + 255) / 256; ++r) {       // S[a3][a2][a1] += coef sum_b3 h3[a3][b3] a2s[b3][a2][a1]
      const int s = tid + 256 * r;
      if (s < S) {
        const int a12 = s % (W * W), a3 = s / (W * W);
        const double* hr = h[2] + a3 * KW;
        double v = 0.0;
#pragma unroll
        for (int b = 0; b < KW; ++b) v = fma(hr[b], a2s[b * W * W + a12], v);
        acc[r] = fma(ct, v, acc[r]);
      }
    }
  }
  const int nn[3] = {g.n1, g.n2, g.n3g};
#pragma unroll
  for (int r = 0; r < (S + 255) / 256; ++r) {
    const int s = tid + 256 * r;
    if (s < S) {
      const int a1 = s % W, a2 = (s / W) % W, a3 = s / (W * W);
      const int aa[3] = {a1, a2, a3};
      bool inside = true;
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const int j = ii[l] + aa[l] - P;
        inside = inside && j >= 0 && j < nn[l];
      }
      out[(long long)s * g.ns + i] = inside ? acc[r] : 0.0;
    }
  }
}

// ---------------------------------------------------------------- apply
// W_c[t, i] = sum_s S_c[s, i] x[t, i + off(s)], channels in groups of CG,
// TC time slices per thread.
template <int D, int P, int CG, int TC>
__global__ void __launch_bounds__(128) stencil_apply(const double* __restrict__ x,
                                                     const double* __restrict__ sten,
                                                     double* __restrict__ wout, int c0, int nc,
                                                     Dims g) {
  using ST = Sten<D, P>;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int t0 = blockIdx.y * TC;
  if (i >= g.ns) return;
  const int i1 = (int)(i % g.n1), i2 = (int)((i / g.n1) % g.n2), i3 = (int)(i / ((long long)g.n1 * g.n2));
  double acc[CG][TC];
#pragma unroll
  for (int c = 0; c < CG; ++c)
#pragma unroll
    for (int t = 0; t < TC; ++t) acc[c][t] = 0.0;
  const double* xt = x + (long long)t0 * g.ns;
  int s = 0;
  for (int a3 = 0; a3 < ST::W3; ++a3) {
    int j3 = D >= 3 ? min(max(i3 + a3 - P, 0), g.n3 - 1) : 0;
    for (int a2 = 0; a2 < ST::W2; ++a2) {
      int j2 = D >= 2 ? min(max(i2 + a2 - P, 0), g.n2 - 1) : 0;
      const long long row = ((long long)j3 * g.n2 + j2) * g.n1;
#pragma unroll
      for (int a1 = 0; a1 < ST::W1; ++a1, ++s) {
        int j1 = min(max(i1 + a1 - P, 0), g.n1 - 1);
        const long long j = row + j1;
        double xv[TC];
#pragma unroll
        for (int t = 0; t < TC; ++t) xv[t] = (t0 + t < g.nt) ? __ldg(xt + (long long)t * g.ns + j) : 0.0;
#pragma unroll
        for (int c = 0; c < CG; ++c) {
          if (c < nc) {
            double cf = __ldg(sten + ((long long)(c0 + c) * ST::S + s) * g.ns + i);
#pragma unroll
            for (int t = 0; t < TC; ++t) acc[c][t] = fma(cf, xv[t], acc[c][t]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CG; ++c) {
    if (c < nc) {
#pragma unroll
      for (int t = 0; t < TC; ++t)
        if (t0 + t < g.nt) wout[(long long)(c0 + c) * g.N + (long long)(t0 + t) * g.ns + i] = acc[c][t];
    }
  }
}

// y[t, i] = sum_c sum_k band_c[t, k] W_c[t - pt + k, i]
__global__ void time_filter(const double* __restrict__ w, const double* __restrict__ band,
                            double* __restrict__ y, int nchan, int pt, Dims g) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (i >= g.ns) return;
  const int W = 2 * pt + 1;
  double acc = 0.0;
  for (int c = 0; c < nchan; ++c) {
    const double* b = band + ((long long)c * g.nt + t) * W;
    const double* wc = w + (long long)c * g.N;
    for (int k = 0; k < W; ++k) {
      int tt = t - pt + k;
      if (tt < 0 || tt >= g.nt) continue;
      acc = fma(__ldg(b + k), __ldg(wc + (long long)tt * g.ns + i), acc);
    }
  }
  y[(long long)t * g.ns + i] = acc;
}

int reaction_apply(mi_ctx* c, const double* x, double* y, const double* x0);  // reaction.cu

}  // namespace mi

using namespace mi;

extern "C" {

int mi_op_setup(mi_ctx* c, int nchan) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  MI_REQUIRE(nchan >= 1 && nchan <= MI_MAX_CHAN, MI_ERR_ARG, "nchan must be in [1, 64]");
  c->nchan = nchan;
  int rc;
  if ((rc = dalloc(c->tband, (size_t)nchan * c->nt * (2 * c->pt + 1)))) return rc;
  if ((rc = dalloc(c->stencil, (size_t)nchan * c->nsten * c->ns))) return rc;
  c->stencil_released = false;
  c->use_dmma = c->p <= 3 && c->pt <= 4;
  MI_REQUIRE(c->use_dmma || (c->n3g == c->n[2] && c->ns_in == c->ns), MI_ERR_ARG,
             "z-slab contexts need the tensor-core operator (p <= 3)");
  if (!c->use_dmma && (rc = dalloc(c->wbuf, (size_t)nchan * c->N))) return rc;
  c->frag_dirty = true;
  MI_CUDA(cudaMemsetAsync(c->stencil.p, 0, sizeof(double) * nchan * c->nsten * c->ns, c->stream));
  MI_CUDA(cudaMemsetAsync(c->tband.p, 0, sizeof(double) * nchan * c->nt * (2 * c->pt + 1), c->stream));
  c->op_ready = true;
  return MI_OK;
}

int mi_op_set_time_bands(mi_ctx* c, const double* bands) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_CUDA(cudaMemcpyAsync(c->tband.p, bands, sizeof(double) * c->nchan * c->nt * (2 * c->pt + 1),
                          cudaMemcpyHostToDevice, c->stream));
  MI_CUDA(cudaStreamSynchronize(c->stream));
  return MI_OK;
}

int mi_op_set_kron_channel(mi_ctx* c, int ch, int nterms, const double* coef, const double* bands) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(!c->stencil_released, MI_ERR_STATE, "channel stencils were packed and released (mi_op_finalize); call mi_op_setup again");
  MI_REQUIRE(ch >= 0 && ch < c->nchan, MI_ERR_ARG, "channel out of range");
  MI_REQUIRE(nterms >= 1, MI_ERR_ARG, "nterms must be >= 1");
  const int nmax = table_rows(c);
  const size_t nb = (size_t)nterms * c->d * nmax * (2 * c->p + 1);
  DeviceBuf dc, db;
  int rc;
  if ((rc = dalloc(dc, nterms)) || (rc = dalloc(db, nb))) return rc;
  MI_CUDA(cudaMemcpyAsync(dc.p, coef, sizeof(double) * nterms, cudaMemcpyHostToDevice, c->stream));
  MI_CUDA(cudaMemcpyAsync(db.p, bands, sizeof(double) * nb, cudaMemcpyHostToDevice, c->stream));
  Dims g = dims_of(c);
  dim3 grid((unsigned)((c->ns + 127) / 128), c->nsten);
  double* out = c->stencil.p + (size_t)ch * c->nsten * c->ns;
  MI_DISPATCH_DP(c->d, c->p, (build_kron_channel<D_, P_><<<grid, 128, 0, c->stream>>>(out, dc.p, db.p, nterms, nmax, g)));
  MI_CHECK_LAUNCH("build_kron_channel");
  c->frag_dirty = true;
  MI_CUDA(cudaStreamSynchronize(c->stream));
  dfree(dc);
  dfree(db);
  return MI_OK;
}

int mi_op_set_su_channel(mi_ctx* c, int ch, const double* theta, const double* H, int ko) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(!c->stencil_released, MI_ERR_STATE, "channel stencils were packed and released (mi_op_finalize); call mi_op_setup again");
  MI_REQUIRE(ch >= 0 && ch < c->nchan, MI_ERR_ARG, "channel out of range");
  MI_REQUIRE(ko >= 0 && ko <= 8, MI_ERR_ARG, "ko out of range");
  const int nmax = table_rows(c);
  const size_t nh = (size_t)c->d * nmax * (2 * c->p + 1) * (2 * ko + 1);
  const size_t nth = (size_t)c->n[0] * c->n[1] * c->n3g;      // theta on the global spatial grid
  DeviceBuf dt, dh;
  int rc;
  if ((rc = dalloc(dt, nth)) || (rc = dalloc(dh, nh))) return rc;
  MI_CUDA(cudaMemcpyAsync(dt.p, theta, sizeof(double) * nth, cudaMemcpyHostToDevice, c->stream));
  MI_CUDA(cudaMemcpyAsync(dh.p, H, sizeof(double) * nh, cudaMemcpyHostToDevice, c->stream));
  Dims g = dims_of(c);
  dim3 grid((unsigned)((c->ns + 127) / 128), c->nsten);
  double* out = c->stencil.p + (size_t)ch * c->nsten * c->ns;
  MI_DISPATCH_DP(c->d, c->p, (build_su_channel<D_, P_><<<grid, 128, 0, c->stream>>>(out, dt.p, dh.p, ko, nmax, g)));
  MI_CHECK_LAUNCH("build_su_channel");
  c->frag_dirty = true;
  MI_CUDA(cudaStreamSynchronize(c->stream));
  dfree(dt);
  dfree(dh);
  return MI_OK;
}

static int quad_channel(mi_ctx* c, int ch, int nterms, const double* coef, const double* theta, const double* T,
                        const int* q, const int* kstart, const int* kwin, const int* Q) {
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(!c->stencil_released, MI_ERR_STATE, "channel stencils were packed and released (mi_op_finalize); call mi_op_setup again");
  MI_REQUIRE(ch >= 0 && ch < c->nchan, MI_ERR_ARG, "channel out of range");
  MI_REQUIRE(nterms >= 1 && coef && theta && T && Q && (q || (kstart && kwin)), MI_ERR_ARG,
             "bad quadrature channel arguments");
  QuadSpec qs{};
  qs.nq = 1;
  int kw = 1;
  for (int l = 0; l < 3; ++l) {
    qs.q[l] = l < c->d && q ? q[l] : 1;
    qs.Q[l] = l < c->d ? Q[l] : 1;
    qs.kwl[l] = l < c->d ? (q ? (c->p + 1) * q[l] : kwin[l]) : 1;
    MI_REQUIRE(qs.q[l] >= 1 && qs.Q[l] >= 1 && qs.kwl[l] >= 1, MI_ERR_ARG, "quadrature sizes must be positive");
    kw = max(kw, qs.kwl[l]);
    qs.nq *= qs.Q[l];
  }
  qs.kw = kw;
  const int nmax = table_rows(c);
  const size_t nT = (size_t)nterms * c->d * nmax * (2 * c->p + 1) * kw;
  DeviceBuf dc, dth, dT;
  int rc;
  if ((rc = dalloc(dc, nterms)) || (rc = dalloc(dth, (size_t)nterms * qs.nq)) || (rc = dalloc(dT, nT))) return rc;
  qs.nmax = nmax;
  int* dks = nullptr;
  if (kstart) {
    std::vector<int> ks((size_t)3 * nmax, 0);
    for (int l = 0; l < c->d; ++l)
      for (int i = 0; i < nmax; ++i) ks[(size_t)l * nmax + i] = kstart[(size_t)l * nmax + i];
    MI_CUDA(cudaMalloc(&dks, sizeof(int) * ks.size()));
    MI_CUDA(cudaMemcpyAsync(dks, ks.data(), sizeof(int) * ks.size(), cudaMemcpyHostToDevice, c->stream));
    qs.kst = dks;
  }
  // host or device arrays (unified addressing picks the copy direction)
  MI_CUDA(cudaMemcpyAsync(dc.p, coef, sizeof(double) * nterms, cudaMemcpyDefault, c->stream));
  MI_CUDA(cudaMemcpyAsync(dth.p, theta, sizeof(double) * nterms * qs.nq, cudaMemcpyDefault, c->stream));
  MI_CUDA(cudaMemcpyAsync(dT.p, T, sizeof(double) * nT, cudaMemcpyDefault, c->stream));
  Dims g = dims_of(c);
  double* out = c->stencil.p + (size_t)ch * c->nsten * c->ns;
  const bool sf = c->d == 3 && ((c->p == 3 && kw <= 25) || (c->p == 2 && kw <= 24) || (c->p == 1 && kw <= 6));
  if (sf) {
    // sum-factorised generator (d = 3): q = p + 1 windows, or the refined (Greville-split, p + 2 point)
    // rules of the mapped Spline Upwind factors
#define MI_QSF(PV, KWV)                                                                                   \
  if (c->p == PV && kw <= KWV) {                                                                        \
    constexpr int Wv = 2 * PV + 1;                                                                      \
    constexpr size_t sm = (size_t)(KWV * KWV * KWV + KWV * KWV * Wv + KWV * Wv * Wv + 3 * Wv * KWV) * 8; \
    MI_CUDA(cudaFuncSetAttribute(build_quad_channel_sf<PV, KWV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)sm));                                                             \
    build_quad_channel_sf<PV, KWV><<<(unsigned)c->ns, 256, sm, c->stream>>>(out, dc.p, dth.p, dT.p, nterms, nmax, \
                                                                            qs, g);                     \
  }
    MI_QSF(3, 16) else MI_QSF(3, 25) else MI_QSF(2, 9) else MI_QSF(2, 24) else MI_QSF(1, 4) else MI_QSF(1, 6)
#undef MI_QSF
  } else {
    dim3 grid((unsigned)((c->ns + 127) / 128), c->nsten);
    MI_DISPATCH_DP(c->d, c->p, (build_quad_channel<D_, P_><<<grid, 128, 0, c->stream>>>(out, dc.p, dth.p, dT.p, nterms,
                                                                                        nmax, qs, g)));
  }
  MI_CHECK_LAUNCH("build_quad_channel");
  c->frag_dirty = true;
  MI_CUDA(cudaStreamSynchronize(c->stream));
  dfree(dc);
  dfree(dth);
  dfree(dT);
  if (dks) cudaFree(dks);
  return MI_OK;
}

int mi_op_set_quad_channel(mi_ctx* c, int ch, int nterms, const double* coef, const double* theta,
                           const double* T, const int* q, const int* Q) {
  MI_DEVICE_GUARD(c);
  return quad_channel(c, ch, nterms, coef, theta, T, q, nullptr, nullptr, Q);
}

int mi_op_set_quad_channel_k(mi_ctx* c, int ch, int nterms, const double* coef, const double* theta,
                             const double* T, const int* kstart, const int* kw, const int* Q) {
  MI_DEVICE_GUARD(c);
  return quad_channel(c, ch, nterms, coef, theta, T, nullptr, kstart, kw, Q);
}

int mi_op_set_channel_stencil(mi_ctx* c, int ch, const double* sten) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(!c->stencil_released, MI_ERR_STATE, "channel stencils were packed and released (mi_op_finalize); call mi_op_setup again");
  MI_REQUIRE(ch >= 0 && ch < c->nchan && sten != nullptr, MI_ERR_ARG, "channel out of range");
  MI_CUDA(cudaMemcpyAsync(c->stencil.p + (size_t)ch * c->nsten * c->ns, sten, sizeof(double) * c->nsten * c->ns,
                          cudaMemcpyDeviceToDevice, c->stream));
  c->frag_dirty = true;
  return MI_OK;
}

int mi_op_get_channel_stencil(mi_ctx* c, int ch, double* sten) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(!c->stencil_released, MI_ERR_STATE, "channel stencils were packed and released (mi_op_finalize); call mi_op_setup again");
  MI_REQUIRE(ch >= 0 && ch < c->nchan && sten != nullptr, MI_ERR_ARG, "channel out of range");
  MI_CUDA(cudaMemcpyAsync(sten, c->stencil.p + (size_t)ch * c->nsten * c->ns, sizeof(double) * c->nsten * c->ns,
                          cudaMemcpyDeviceToDevice, c->stream));
  return MI_OK;
}

static int dmma_prepare(mi_ctx* c) {
  int rc = MI_OK;
  MI_DISPATCH_DP(c->d, c->p, {
    using G = DmmaSten<D_, P_>;
    c->C[0] = (c->n[0] + G::B1 - 1) / G::B1;
    c->C[1] = (c->n[1] + G::B2 - 1) / G::B2;
    c->C[2] = (c->n[2] + G::B3 - 1) / G::B3;
    const long long ncubes = (long long)c->C[0] * c->C[1] * c->C[2];
    const long long per_group = ncubes * G::PPB * G::KS * 32;
    const int ngroups = (c->nchan + 7) / 8;
    if ((rc = dalloc(c->frag, (size_t)per_group * ngroups))) return rc;
    const int ntp = ((c->nt + G::TT - 1) / G::TT) * G::TT;
    if ((rc = dalloc(c->xt, (size_t)ntp * c->ns_in))) return rc;
    {
      // TMA descriptor of the time-innermost copy: dims (ntp, n1, n2, n3), box (TSTR, H1, H2, H3)
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      MI_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      MI_REQUIRE(fn != nullptr && q == cudaDriverEntryPointSuccess, MI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      // (the input slab: owned planes plus the z halo)
      cuuint64_t dims[4] = {(cuuint64_t)ntp, (cuuint64_t)c->n[0], (cuuint64_t)c->n[1],
                            (cuuint64_t)(c->n[2] + c->hz_lo + c->hz_hi)};
      cuuint64_t strides[3] = {(cuuint64_t)ntp * 8, (cuuint64_t)ntp * c->n[0] * 8,
                               (cuuint64_t)ntp * c->n[0] * c->n[1] * 8};
      cuuint32_t box[4] = {(cuuint32_t)G::TSTR, (cuuint32_t)G::H1, (cuuint32_t)G::H2, (cuuint32_t)G::H3};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = ((mi_encode_tiled_fn)fn)(&c->tmap_xt, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, c->xt.p, dims, strides,
                                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      MI_REQUIRE(r == CUDA_SUCCESS, MI_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    }
    for (int gi = 0; gi < ngroups; ++gi) {
      const int c0 = gi * 8, nc = min(8, c->nchan - c0);
      repack_frag<D_, P_><<<(unsigned)((per_group + 255) / 256), 256, 0, c->stream>>>(
          c->stencil.p, c->frag.p + gi * per_group, c0, nc, c->n[0], c->n[1], c->n[2], c->C[0], c->C[1],
          c->ns, per_group);
      MI_CHECK_LAUNCH("repack_frag");
    }
    if ((rc = dalloc(c->wbuf, (size_t)c->nchan * c->ns * ntp))) return rc;
    MI_CUDA(cudaMemsetAsync(c->wbuf.p, 0, sizeof(double) * c->nchan * c->ns * ntp, c->stream));
    {
      // TMA descriptor of W for the tensor-core time filter: 2D (ntp times, nchan*ns rows), box 16 x 64,
      // 128-byte swizzle (conflict-free B-fragment reads)
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      MI_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      MI_REQUIRE(fn != nullptr && q == cudaDriverEntryPointSuccess, MI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      cuuint64_t dims[2] = {(cuuint64_t)ntp, (cuuint64_t)c->nchan * c->ns};
      cuuint64_t strides[1] = {(cuuint64_t)ntp * 8};
      cuuint32_t box[2] = {16, (cuuint32_t)TFilterCfg::NP};
      cuuint32_t es[2] = {1, 1};
      CUresult r = ((mi_encode_tiled_fn)fn)(&c->tmap_w, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, c->wbuf.p, dims, strides,
                                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      MI_REQUIRE(r == CUDA_SUCCESS, MI_ERR_CUDA, "cuTensorMapEncodeTiled (W) failed");
    }
    MI_CUDA(cudaFuncSetAttribute(stencil_dmma<D_, P_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)G::SMEM));
  });
  MI_CUDA(cudaStreamSynchronize(c->stream));
  c->frag_dirty = false;
  return rc;
}

// y = sum_c T_c (x) along time of the time-innermost W buffer (HBM-bound)
static int launch_time_filter(mi_ctx* c, double* y) {
  MI_REQUIRE(c->nchan <= 64, MI_ERR_ARG, "too many channels for the time filter");
#ifndef MI_TF_FRAG
#define MI_TF_FRAG 1
#endif
  const bool frag = MI_TF_FRAG && TFilterCfg::smem(c->pt, c->nchan, true) <= 232448;
  if (TFilterCfg::smem(c->pt, c->nchan, frag) <= 232448 && c->pt <= TFilterCfg::PX) {
    // tensor-core filter: persistent blocks, one time block of 56 rows each
    const int nsm = mi::num_sms();
    const int ntb = (c->nt + TFilterCfg::TR - 1) / TFilterCfg::TR;
    const int grid = ntb * std::max(1, nsm / ntb);
    const size_t sm = TFilterCfg::smem(c->pt, c->nchan, frag);
#define MI_TFD(PTV)                                                                                            \
  case PTV: {                                                                                                  \
    MI_DEV_FLAG(attr);                                                                                  \
    if (!attr) {                                                                                               \
      MI_CUDA(cudaFuncSetAttribute(time_filter_dmma<PTV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448)); \
      MI_CUDA(cudaFuncSetAttribute(time_filter_dmma<PTV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448)); \
      attr = true;                                                                                             \
    }                                                                                                          \
    if (frag)                                                                                                  \
      time_filter_dmma<PTV, true><<<grid, 256, sm, c->stream>>>(c->tmap_w, c->tband.p, y, c->nchan, c->nt, c->ns, ntb, 0); \
    else                                                                                                       \
      time_filter_dmma<PTV, false><<<grid, 256, sm, c->stream>>>(c->tmap_w, c->tband.p, y, c->nchan, c->nt, c->ns, ntb, 0); \
  } break;
    switch (c->pt) {
      MI_TFD(1) MI_TFD(2) MI_TFD(3) MI_TFD(4)
      default:
        set_error("time degree > 4");
        return MI_ERR_ARG;
    }
#undef MI_TFD
    MI_CHECK_LAUNCH("time_filter_dmma");
    return MI_OK;
  }
  dim3 fg((unsigned)((c->ns + 127) / 128), (c->nt + 15) / 16);
  const int ntp = ((c->nt + 15) / 16) * 16;
  const size_t fsm = (size_t)c->nchan * 16 * (2 * c->pt + 1) * sizeof(double);
#define MI_TF(PTV)                                                                                       \
  case PTV:                                                                                              \
    if (fsm > 48 * 1024)                                                                                 \
      MI_CUDA(cudaFuncSetAttribute(time_filter_ti<16, PTV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                   (int)fsm));                                                           \
    time_filter_ti<16, PTV><<<fg, 128, fsm, c->stream>>>(c->wbuf.p, c->tband.p, y, c->nchan, c->nt, ntp, \
                                                         c->ns, 0);                                      \
    break;
  switch (c->pt) {
    MI_TF(1) MI_TF(2) MI_TF(3) MI_TF(4)
    default:
      set_error("time degree > 4");
      return MI_ERR_ARG;
  }
#undef MI_TF
  MI_CHECK_LAUNCH("time_filter_ti");
  return MI_OK;
}

// The DMMA operator in stages: transpose spatial points [s_lo, s_hi) of x into xt, run the stencil over
// cubes [cube_lo, cube_hi) (z-slowest numbering), then the time filter over everything.  dmma_apply runs
// them once over the whole domain; mi_op_apply_from_host interleaves them with the H2D copy of x.
static int dmma_transpose(mi_ctx* c, const double* x, long long s_lo, long long s_hi) {
  const int ntp = ((c->nt + 15) / 16) * 16;          // = DmmaSten<.,.>::TT multiple (TT = 16)
  if (s_hi <= s_lo) return MI_OK;
  ProfScope ps(c, PROF_OP_STENCIL);
  dim3 tg((unsigned)((s_hi - s_lo + 31) / 32), (ntp + 31) / 32);
  transpose_time_inner<<<tg, dim3(32, 8), 0, c->stream>>>(x + s_lo, c->xt.p + s_lo * ntp, c->nt, ntp, s_hi - s_lo,
                                                          c->ns_in);
  MI_CHECK_LAUNCH("transpose_time_inner");
  return MI_OK;
}

static int dmma_stencil(mi_ctx* c, double* y, int cube_lo, int cube_hi) {
  MI_DISPATCH_DP(c->d, c->p, {
    using G = DmmaSten<D_, P_>;
    static_assert(G::TT == 16, "dmma_transpose pads time to multiples of 16");
    const long long ncubes = (long long)c->C[0] * c->C[1] * c->C[2];
    const long long per_group = ncubes * G::PPB * G::KS * 32;
    const int ngroups = (c->nchan + 7) / 8;
    const int ntp = ((c->nt + G::TT - 1) / G::TT) * G::TT;
    for (int gi = 0; gi < ngroups && cube_hi > cube_lo; ++gi) {
      DmmaArgs a{c->xt.p, c->wbuf.p, c->frag.p + gi * per_group, c->tband.p, y, gi * 8, min(8, c->nchan - gi * 8), c->pt,
                 gi > 0 ? 1 : 0, c->n[0], c->n[1], c->n[2], c->nt, ntp, c->C[0], c->C[1], c->C[2], c->ns, c->hz_lo,
                 cube_lo, cube_hi};
      ProfScope ps(c, PROF_OP_STENCIL);
      // persistent: one CTA per SM (the kernel is sized for 1 CTA / SM), each sweeping cubes b, b + grid, ...
      const long long nc = cube_hi - cube_lo;
      const long long grid = MI_STEN_PERSIST ? std::min<long long>(nc, mi::num_sms()) : nc;
      stencil_dmma<D_, P_><<<(unsigned)grid, G::THREADS, G::SMEM, c->stream>>>(a, c->tmap_xt);
      MI_CHECK_LAUNCH("stencil_dmma");
    }
  });
  return MI_OK;
}

static int dmma_apply(mi_ctx* c, const double* x, double* y) {
  int rc;
  if ((rc = dmma_transpose(c, x, 0, c->ns_in))) return rc;
  if ((rc = dmma_stencil(c, y, 0, c->C[0] * c->C[1] * c->C[2]))) return rc;
  ProfScope ps(c, PROF_OP_TFILTER);
  return launch_time_filter(c, y);
}

// y = sum_c T_c (x) S_c x (every Kronecker / SU / quadrature channel; no reaction)
static int channels_apply(mi_ctx* c, const double* x, double* y) {
  if (c->use_dmma) {
    int rc;
    if (c->frag_dirty && (rc = dmma_prepare(c))) return rc;
    return dmma_apply(c, x, y);
  }
  Dims g = dims_of(c);
  constexpr int CG = 4, TC = 8;
  dim3 grid((unsigned)((c->ns + 127) / 128), (c->nt + TC - 1) / TC);
  for (int c0 = 0; c0 < c->nchan; c0 += CG) {
    int nc = min(CG, c->nchan - c0);
    ProfScope ps(c, PROF_OP_STENCIL);
    MI_DISPATCH_DP(c->d, c->p, (stencil_apply<D_, P_, CG, TC><<<grid, 128, 0, c->stream>>>(x, c->stencil.p, c->wbuf.p, c0, nc, g)));
    MI_CHECK_LAUNCH("stencil_apply");
  }
  dim3 g2((unsigned)((c->ns + 255) / 256), c->nt);
  ProfScope ps(c, PROF_OP_TFILTER);
  time_filter<<<g2, 256, 0, c->stream>>>(c->wbuf.p, c->tband.p, y, c->nchan, c->pt, g);
  MI_CHECK_LAUNCH("time_filter");
  return MI_OK;
}

int mi_op_apply(mi_ctx* c, const double* x, double* y) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "operator not set up");
  MI_REQUIRE(x != y, MI_ERR_ARG, "x and y must not alias");
  int rc = channels_apply(c, x, y);
  if (rc) return rc;
  if (c->reaction_on) {
    ProfScope ps(c, PROF_OP_REACTION);
    return reaction_apply(c, x, y, nullptr);
  }
  return MI_OK;
}

int mi_op_apply_from_host(mi_ctx* c, const double* x_host, double* x_dev, double* y, int nparts) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "operator not set up");
  MI_REQUIRE(x_host && x_dev && y && x_dev != y, MI_ERR_ARG, "bad pointers to mi_op_apply_from_host");
  const long long plane = (long long)c->n[0] * c->n[1];
  if (!c->use_dmma || c->d != 3 || c->ns_in != c->ns || nparts <= 1) {
    MI_CUDA(cudaMemcpyAsync(x_dev, x_host, sizeof(double) * c->N, cudaMemcpyHostToDevice, c->stream));
    return mi_op_apply(c, x_dev, y);
  }
  int rc;
  if (c->frag_dirty && (rc = dmma_prepare(c))) return rc;
  if (!c->copy_stream) MI_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  while ((int)c->copy_events.size() < nparts + 1) {
    cudaEvent_t e;
    MI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->copy_events.push_back(e);
  }
  // part p: the stencil over cube layers [cz_p, cz_{p+1}) (cube z size B3 = 2 planes); H2D chunk p holds
  // planes [b_p, b_{p+1}) with b_p = cz_p B3 + p_s (the stencil of part p reads up to p_s planes past its
  // layers).  Chunk p+1 copies while part p's stencil runs.
  const int C3 = c->C[2], B3 = (int)((c->n[2] + C3 - 1) / C3);
  nparts = std::min(nparts, C3);
  std::vector<int> cz(nparts + 1), b(nparts + 1);
  for (int q = 0; q <= nparts; ++q) cz[q] = (int)((long long)q * C3 / nparts);
  for (int q = 0; q <= nparts; ++q) b[q] = q == 0 ? 0 : (q == nparts ? c->n[2] : std::min(c->n[2], cz[q] * B3 + c->p));
  // x_dev is free once the compute stream reaches this point
  MI_CUDA(cudaEventRecord(c->copy_events[nparts], c->stream));
  MI_CUDA(cudaStreamWaitEvent(c->copy_stream, c->copy_events[nparts], 0));
  for (int q = 0; q < nparts; ++q) {
    const long long o = b[q] * plane, w = (long long)(b[q + 1] - b[q]) * plane;
    if (w > 0)
      MI_CUDA(cudaMemcpy2DAsync(x_dev + o, sizeof(double) * c->ns, x_host + o, sizeof(double) * c->ns,
                                sizeof(double) * w, c->nt, cudaMemcpyHostToDevice, c->copy_stream));
    MI_CUDA(cudaEventRecord(c->copy_events[q], c->copy_stream));
  }
  const int cubes_per_layer = c->C[0] * c->C[1];
  for (int q = 0; q < nparts; ++q) {
    MI_CUDA(cudaStreamWaitEvent(c->stream, c->copy_events[q], 0));
    if ((rc = dmma_transpose(c, x_dev, b[q] * plane, b[q + 1] * plane))) return rc;
    if ((rc = dmma_stencil(c, y, cz[q] * cubes_per_layer, cz[q + 1] * cubes_per_layer))) return rc;
  }
  {
    ProfScope ps(c, PROF_OP_TFILTER);
    if ((rc = launch_time_filter(c, y))) return rc;
  }
  if (c->reaction_on) {
    ProfScope ps(c, PROF_OP_REACTION);
    return reaction_apply(c, x_dev, y, nullptr);
  }
  return MI_OK;
}

int mi_op_finalize(mi_ctx* c, int release) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  if (!c->use_dmma || c->stencil_released) return MI_OK;
  int rc;
  if (c->frag_dirty && (rc = dmma_prepare(c))) return rc;
  if (release) {
    mi::dfree(c->stencil);        // only the fragment-major copy is read from now on
    c->stencil_released = true;
  }
  return MI_OK;
}

int mi_op_set_lift(mi_ctx* c, const double* column0, const double* u0) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  if (u0 == nullptr) {
    c->lift_on = false;
    c->rx_cw_dirty = true;
    return MI_OK;
  }
  MI_REQUIRE(column0 != nullptr, MI_ERR_ARG, "NULL lifting column");
  MI_REQUIRE(c->rx_rowoff == -1, MI_ERR_ARG, "lifting needs the whole time axis (not a time slab)");
  int rc;
  if ((rc = dalloc(c->lift_u0, (size_t)c->ns_in))) return rc;
  MI_CUDA(cudaMemcpyAsync(c->lift_u0.p, u0, sizeof(double) * c->ns_in, cudaMemcpyDeviceToDevice, c->stream));
  // the column-0 coupling v_c[t] = T_c,full[t + 1, 0] multiplies W_c at time row 0 (where mi_op_apply_lift
  // places u0): band entry k = pt - t of row t
  const int bw = 2 * c->pt + 1;
  std::vector<double> hb((size_t)c->nchan * c->nt * bw, 0.0);
  for (int ch = 0; ch < c->nchan; ++ch)
    for (int t = 0; t < std::min(c->pt, c->nt); ++t)
      hb[((size_t)ch * c->nt + t) * bw + (c->pt - t)] = column0[(size_t)ch * c->nt + t];
  for (int ch = 0; ch < c->nchan; ++ch)
    for (int t = c->pt; t < c->nt; ++t)
      MI_REQUIRE(column0[(size_t)ch * c->nt + t] == 0.0, MI_ERR_ARG, "lifting column beyond the time band");
  if ((rc = dalloc(c->lift_band, hb.size()))) return rc;
  MI_CUDA(cudaMemcpyAsync(c->lift_band.p, hb.data(), sizeof(double) * hb.size(), cudaMemcpyHostToDevice, c->stream));
  MI_CUDA(cudaStreamSynchronize(c->stream));
  c->lift_on = true;
  c->rx_cw_dirty = true;      // C_r sees the lifted iterate
  return MI_OK;
}

int mi_op_apply_lift(mi_ctx* c, double* y) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "operator not set up");
  MI_REQUIRE(c->lift_on, MI_ERR_STATE, "no lifting set (mi_op_set_lift)");
  int rc;
  if ((rc = dalloc(c->lift_x, (size_t)c->N_in))) return rc;
  // channels: x = u0 in time row 0, time bands = the column-0 couplings
  MI_CUDA(cudaMemsetAsync(c->lift_x.p, 0, sizeof(double) * c->N_in, c->stream));
  MI_CUDA(cudaMemcpyAsync(c->lift_x.p, c->lift_u0.p, sizeof(double) * c->ns_in, cudaMemcpyDeviceToDevice, c->stream));
  std::swap(c->tband, c->lift_band);
  rc = channels_apply(c, c->lift_x.p, y);
  std::swap(c->tband, c->lift_band);
  if (rc) return rc;
  if (c->reaction_on) {
    // reaction: x = 0 on the constrained rows, u0 on the lifted slab
    MI_CUDA(cudaMemsetAsync(c->lift_x.p, 0, sizeof(double) * c->ns_in, c->stream));
    ProfScope ps(c, PROF_OP_REACTION);
    return reaction_apply(c, c->lift_x.p, y, c->lift_u0.p);
  }
  return MI_OK;
}

}  // extern "C"
