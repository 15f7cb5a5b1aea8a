// Recovery-variable solve (reference solve_w_system, linalg.py:502-547, and
// the per-time-row PCG with the Kronecker mass preconditioner, linalg.py:
// 176-203 / 450-499):
//
//   ((W_t + b d_e M_t) (x) M_s) w = g
//
// Time: Y = K_t^{-1} G as one DMMA mode product with the host-factored
// inverse (K_t is N_t x N_t).  Space: every time row is solved with PCG
// (M_s = kron_l L_l M_l, preconditioner kron_l M_l^{-1}); all rows advance
// together (row-batched PCG), so the kernels here are the mass / inverse
// mass mode products and per-row dot products / axpys.
#include "common.cuh"
#include "gemm.cuh"

namespace mi {

__global__ void rowdots_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                               long long ncols) {
  // one block per row; fixed-order tree reduction (deterministic)
  __shared__ double s[256];
  const long long r = blockIdx.x;
  const double* ar = a + r * ncols;
  const double* br = b + r * ncols;
  double v = 0.0;
  for (long long j = threadIdx.x; j < ncols; j += blockDim.x) v = fma(ar[j], br[j], v);
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = s[0];
}

__global__ void row_axpy_kernel(const double* __restrict__ alpha, double sign, const double* __restrict__ x,
                                double* __restrict__ y, long long ncols, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(sign * alpha[i / ncols], x[i], y[i]);
}

__global__ void row_xpby_kernel(const double* __restrict__ beta, const double* __restrict__ z,
                                double* __restrict__ p, long long ncols, long long total) {
  // p = z + beta_row * p
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(beta[i / ncols], p[i], z[i]);
}

// spatial Kronecker product kron_l A_l on nrows rows (A_l: n_l x n_l row-major on the device)
static int kron_spatial(mi_ctx* c, const double* AT0, double* const* A, const double* in, double* out,
                        long long nrows) {
  cudaStream_t st = c->stream;
  const int n1 = c->n[0], n2 = c->n[1], n3 = c->n[2];
  const long long N = nrows * c->ns;
  const bool has[3] = {n1 > 1, n2 > 1, n3 > 1};
  const int nstage = has[0] + has[1] + has[2];
  if (nstage == 0) {
    // n = 1 in every direction: scale by A[0][0] of each (1x1) -- handled by the caller's tables
    MI_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    return MI_OK;
  }
  double* cand[3] = {c->ws_t1.p, c->ws_t2.p, c->ws_t3.p};
  double* bufs[2];
  int nb = 0;
  for (int i = 0; i < 3 && nb < 2; ++i)
    if (cand[i] != in && cand[i] != out) bufs[nb++] = cand[i];
  int k = 0, done = 0;
  const double* cur = in;
  for (int l = 0; l < 3; ++l) {
    if (!has[l]) continue;
    double* o;
    if (++done == nstage) {
      o = out;
    } else {
      o = bufs[k];
      k ^= 1;
    }
    const int nl = c->n[l];
    if (l == 0) {
      // out[r, i] = sum_j in[r, j] A[i, j]  ->  B = A^T
      GemmArgs g{cur, AT0, o, (int)(N / n1), n1, n1, n1, n1, n1, 0, 0, 0};
      MI_CUDA(launch_panel_n<false>(g, n1, 1, st));
    } else {
      const long long inner = l == 1 ? n1 : (long long)n1 * n2;
      const long long outer = N / (inner * nl);
      GemmArgs g{A[l], cur, o, nl, (int)inner, nl, nl, inner, inner, 0, (long long)nl * inner, (long long)nl * inner};
      MI_CUDA(launch_panel_n<true>(g, nl, (int)outer, st));
    }
    cur = o;
  }
  return MI_OK;
}

}  // namespace mi

using namespace mi;

extern "C" {

int mi_ws_setup(mi_ctx* c, const double* Kinv, const double* Mmat, const double* Minv) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  const int nmax = max(c->n[0], max(c->n[1], c->n[2]));
  int rc;
  if ((rc = dalloc(c->ws_Kinv, (size_t)c->nt * c->nt))) return rc;
  MI_CUDA(cudaMemcpy(c->ws_Kinv.p, Kinv, sizeof(double) * c->nt * c->nt, cudaMemcpyHostToDevice));
  for (int l = 0; l < 3; ++l) {
    const int nl = c->n[l];
    std::vector<double> m(nl * nl), mi_(nl * nl), mt(nl * nl), mit(nl * nl);
    for (int i = 0; i < nl; ++i)
      for (int j = 0; j < nl; ++j) {
        const double a = l < c->d ? Mmat[((size_t)l * nmax + i) * nmax + j] : 1.0;
        const double b = l < c->d ? Minv[((size_t)l * nmax + i) * nmax + j] : 1.0;
        m[i * nl + j] = a;
        mi_[i * nl + j] = b;
        mt[j * nl + i] = a;
        mit[j * nl + i] = b;
      }
    if ((rc = dalloc(c->ws_M[l], nl * nl)) || (rc = dalloc(c->ws_Mi[l], nl * nl))) return rc;
    MI_CUDA(cudaMemcpy(c->ws_M[l].p, m.data(), sizeof(double) * nl * nl, cudaMemcpyHostToDevice));
    MI_CUDA(cudaMemcpy(c->ws_Mi[l].p, mi_.data(), sizeof(double) * nl * nl, cudaMemcpyHostToDevice));
    if (l == 0) {
      if ((rc = dalloc(c->ws_MT0, nl * nl)) || (rc = dalloc(c->ws_MiT0, nl * nl))) return rc;
      MI_CUDA(cudaMemcpy(c->ws_MT0.p, mt.data(), sizeof(double) * nl * nl, cudaMemcpyHostToDevice));
      MI_CUDA(cudaMemcpy(c->ws_MiT0.p, mit.data(), sizeof(double) * nl * nl, cudaMemcpyHostToDevice));
    }
  }
  if ((rc = dalloc(c->ws_t1, c->N)) || (rc = dalloc(c->ws_t2, c->N)) || (rc = dalloc(c->ws_t3, c->N))) return rc;
  c->ws_ready = true;
  return MI_OK;
}

/* out = (K_t^{-1} (x) I) in */
int mi_ws_time(mi_ctx* c, const double* in, double* out) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->ws_ready, MI_ERR_STATE, "w-solve not set up");
  MI_REQUIRE(in != out, MI_ERR_ARG, "in and out must not alias");
  GemmArgs g{c->ws_Kinv.p, in, out, c->nt, (int)c->ns, c->nt, c->nt, c->ns, c->ns, 0, 0, 0};
  MI_CUDA(launch_dgemm(g, 1, c->stream));
  return MI_OK;
}

/* out = (I (x) kron_l M_l) in  (inverse != 0: kron_l M_l^{-1}) on nrows time rows */
int mi_ws_mass(mi_ctx* c, const double* in, double* out, long long nrows, int inverse) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->ws_ready, MI_ERR_STATE, "w-solve not set up");
  MI_REQUIRE(in != out, MI_ERR_ARG, "in and out must not alias");
  double* A[3] = {nullptr, inverse ? c->ws_Mi[1].p : c->ws_M[1].p, inverse ? c->ws_Mi[2].p : c->ws_M[2].p};
  return kron_spatial(c, inverse ? c->ws_MiT0.p : c->ws_MT0.p, A, in, out, nrows);
}

/* out[r] = <a[r, :], b[r, :]> for r < nrows (device) */
int mi_rowdots(mi_ctx* c, long long nrows, long long ncols, const double* a, const double* b, double* out) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr && nrows >= 0, MI_ERR_ARG, "bad arguments to mi_rowdots");
  if (nrows == 0) return MI_OK;
  rowdots_kernel<<<(unsigned)nrows, 256, 0, c->stream>>>(a, b, out, ncols);
  MI_CHECK_LAUNCH("rowdots_kernel");
  return MI_OK;
}

/* y[r, :] += sign * alpha[r] * x[r, :] */
int mi_row_axpy(mi_ctx* c, long long nrows, long long ncols, const double* alpha, double sign, const double* x,
                double* y) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  const long long total = nrows * ncols;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  row_axpy_kernel<<<grid, 256, 0, c->stream>>>(alpha, sign, x, y, ncols, total);
  MI_CHECK_LAUNCH("row_axpy_kernel");
  return MI_OK;
}

/* p[r, :] = z[r, :] + beta[r] * p[r, :] */
int mi_row_xpby(mi_ctx* c, long long nrows, long long ncols, const double* beta, const double* z, double* p) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  const long long total = nrows * ncols;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  row_xpby_kernel<<<grid, 256, 0, c->stream>>>(beta, z, p, ncols, total);
  MI_CHECK_LAUNCH("row_xpby_kernel");
  return MI_OK;
}

}  // extern "C"
