// Fast-diagonalisation preconditioner (reference FastDiagPreconditioner.apply,
// linalg.py:317-353; _diag_blocks, linalg.py:309-315).
//
//   z = (Q (x) U_d..U_1) (C_m Delta + mu_s I)^-1 (Q^T (x) U_d^T..U_1^T) r
//
// Dense mode products run on the FP64 tensor cores (DMMA, gemm.cuh).  The
// time basis Q is the REAL 2x2-block form of the reference's complex
// pencil (factors.RealTimePencil), so the whole apply is real arithmetic.
// The block-arrowhead core is solved per spatial eigen-index s with
// mu_s = react + sum_l sigma_l lam_l[i_l] formed on the fly (the
// reference materialises H_int as an (N_t-1) x N_s complex array).
#include "common.cuh"
#include "gemm.cuh"
#include "mode_fold.cuh"
#include "mode_resident.cuh"

#include <cstdlib>
#include "tstage.cuh"

#ifndef MI_TSTAGE
#define MI_TSTAGE 1   // fused time stage (tstage.cuh); 0 = separate Q^T / arrowhead / Q passes
#endif

namespace mi {

// Block-arrowhead solve, one thread per spatial column s, in place on Y
// (nt x ns).  Interior rows i < m = nt-1 carry 2x2 blocks
// [[a, b], [c, e]] = C_m T_block + mu I; border column C_m g, border row
// C_m glow, corner C_m sigma + mu.
__global__ void arrowhead_solve(double* __restrict__ Y, const double* __restrict__ lam1,
                                const double* __restrict__ lam2, const double* __restrict__ lam3,
                                const double* __restrict__ diag, const double* __restrict__ off,
                                const int* __restrict__ partner, const double* __restrict__ gb,
                                const double* __restrict__ gl, double sigma, double cm, double react,
                                int n1, int n2, int nt, long long ns, long long col0) {
  // Y is (nt x ns) with ns = number of columns handled; column j is global
  // spatial eigen-index col0 + j (a caller may hand in a column range).
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const long long sg = s + col0;
  const int i1 = (int)(sg % n1), i2 = (int)((sg / n1) % n2), i3 = (int)(sg / ((long long)n1 * n2));
  const double mu = react + lam1[i1] + lam2[i2] + lam3[i3];
  const int m = nt - 1;
  double sy = 0.0, sb = 0.0;
  for (int i = 0; i < m; ++i) {
    const int j = partner[i];
    const double a = fma(cm, diag[i], mu), e = fma(cm, diag[j], mu);
    const double b = cm * off[i], c = cm * off[j];
    const double inv = 1.0 / (a * e - b * c);
    const double yi = Y[(long long)i * ns + s], yj = Y[(long long)j * ns + s];
    const double dy = (e * yi - b * yj) * inv;
    const double db = cm * (e * gb[i] - b * gb[j]) * inv;
    sy = fma(gl[i], dy, sy);
    sb = fma(gl[i], db, sb);
  }
  const double xl = (Y[(long long)m * ns + s] - cm * sy) / (fma(cm, sigma, mu) - cm * sb);
  // second sweep: x_i = Dinv y - Dinv (C_m g) x_l ; rows of a 2x2 block are
  // written together (both read before either is overwritten).
  for (int i = 0; i < m; ++i) {
    const int j = partner[i];
    if (j < i) continue;
    const double a = fma(cm, diag[i], mu), e = fma(cm, diag[j], mu);
    const double b = cm * off[i], c = cm * off[j];
    const double inv = 1.0 / (a * e - b * c);
    const double yi = Y[(long long)i * ns + s], yj = Y[(long long)j * ns + s];
    const double gi = cm * gb[i] * xl, gj = cm * gb[j] * xl;
    const double ri = yi - gi, rj = yj - gj;
    // rows i (own diag a, partner diag e) and j (own diag e, partner diag a)
    Y[(long long)i * ns + s] = (e * ri - b * rj) * inv;
    if (j != i) Y[(long long)j * ns + s] = (a * rj - c * ri) * inv;
  }
  Y[(long long)m * ns + s] = xl;
}


static cudaError_t mode_strided(const double* A, const double* in, double* out, int n, long long inner,
                                long long outer, cudaStream_t st) {
  // out[o, i, c] = sum_j A[i, j] in[o, j, c]
  cudaError_t err;
  if (launch_mode_resident<false>(A, in, out, n, inner, outer, num_sms(), st, &err)) return err;
  GemmArgs g{A, in, out, n, (int)inner, n, n, inner, inner, 0, (long long)n * inner, (long long)n * inner};
  return launch_panel_n<true>(g, n, (int)outer, st);
}

static cudaError_t mode_contig(const double* Bm, const double* in, double* out, int n, long long rows,
                               cudaStream_t st) {
  // out[r, i] = sum_j in[r, j] Bm[j, i]
  cudaError_t err;
  if (launch_mode_resident<true>(Bm, in, out, n, 0, rows, num_sms(), st, &err)) return err;
  GemmArgs g{in, Bm, out, (int)rows, n, n, n, n, n, 0, 0, 0};
  return launch_panel_n<false>(g, n, 1, st);
}

// Spatial transform of direction l (forward U_l^T, inverse U_l) along a mode of extent n_l that is
// contiguous (inner == 1: `outer` rows) or strided.  Even/odd bases take the folded kernel.
static cudaError_t spatial_mode(mi_ctx* c, int l, bool inverse, const double* in, double* out, long long inner,
                                long long outer) {
  const int n = c->n[l];
  cudaError_t err;
  // the contiguous mode moves each tile as one bulk copy: 16-byte-aligned buffers only
  if (c->fold_hs[l] > 0 && (inner != 1 || ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0)) {
    const bool done = inner == 1
        ? launch_mode_fold<true>(c->Us[l].p, in, out, n, inverse, 1, outer, num_sms(), c->stream, &err)
        : launch_mode_fold<false>(c->Us[l].p, in, out, n, inverse, inner, outer, num_sms(), c->stream, &err);
    if (done) return err;
  }
  if (inner == 1) return mode_contig(inverse ? c->UsT[l].p : c->Us[l].p, in, out, n, outer, c->stream);
  return mode_strided(inverse ? c->Us[l].p : c->UsT[l].p, in, out, n, inner, outer, c->stream);
}

// hs (> 0) if the n x n row-major U is EXACTLY an even/odd basis with the symmetric modes first
// (U[n-1-k][m] = U[k][m] for m < hs, = -U[k][m] and U[n/2][m] = 0 (n odd) for m >= hs), else 0
static int exact_fold(const std::vector<double>& u, int n) {
  const int h = n / 2, hs = n - h;
  if (n < 4) return 0;
  for (int k = 0; k < h; ++k)
    for (int m = 0; m < n; ++m) {
      const double a = u[(size_t)k * n + m], b = u[(size_t)(n - 1 - k) * n + m];
      if (m < hs ? (a != b) : (a != -b)) return 0;
    }
  if (n & 1)
    for (int m = hs; m < n; ++m)
      if (u[(size_t)h * n + m] != 0.0) return 0;
  return hs;
}

}  // namespace mi

using namespace mi;

extern "C" {

int mi_pc_setup(mi_ctx* c, const double* U, const double* lam, double cm, double react, const double* Q,
                const double* diag, const double* off, const int* partner, const double* g,
                const double* glow, double sigma) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  const int nmax = max(c->n[0], max(c->n[1], c->n[2]));
  int rc;
  for (int l = 0; l < 3; ++l) {
    const int nl = c->n[l];
    if ((rc = dalloc(c->Us[l], (size_t)nl * nl)) || (rc = dalloc(c->UsT[l], (size_t)nl * nl)) ||
        (rc = dalloc(c->lam[l], nl)))
      return rc;
    std::vector<double> u(nl * nl), ut(nl * nl), lm(nl, 0.0);
    if (l < c->d) {
      for (int i = 0; i < nl; ++i)
        for (int j = 0; j < nl; ++j) {
          u[i * nl + j] = U[((size_t)l * nmax + i) * nmax + j];
          ut[j * nl + i] = u[i * nl + j];
        }
      for (int i = 0; i < nl; ++i) lm[i] = lam[(size_t)l * nmax + i];
    } else {
      u[0] = ut[0] = 1.0;
    }
    c->fold_hs[l] = (l < c->d && std::getenv("MI_NO_FOLD") == nullptr) ? exact_fold(u, nl) : 0;
    MI_CUDA(cudaMemcpy(c->Us[l].p, u.data(), sizeof(double) * nl * nl, cudaMemcpyHostToDevice));
    MI_CUDA(cudaMemcpy(c->UsT[l].p, ut.data(), sizeof(double) * nl * nl, cudaMemcpyHostToDevice));
    MI_CUDA(cudaMemcpy(c->lam[l].p, lm.data(), sizeof(double) * nl, cudaMemcpyHostToDevice));
  }
  const int nt = c->nt, m = nt - 1;
  std::vector<double> qt((size_t)nt * nt);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j < nt; ++j) qt[(size_t)j * nt + i] = Q[(size_t)i * nt + j];
  if ((rc = dalloc(c->Q, (size_t)nt * nt)) || (rc = dalloc(c->QT, (size_t)nt * nt)) ||
      (rc = dalloc(c->pen_diag, m)) || (rc = dalloc(c->pen_off, m)) || (rc = dalloc(c->pen_g, m)) ||
      (rc = dalloc(c->pen_glow, m)) || (rc = dalloc(c->pc_t1, c->N)) || (rc = dalloc(c->pc_t2, c->N)) ||
      (rc = dalloc(c->pc_t3, c->N)))
    return rc;
  for (int i = 0; i < m; ++i)
    MI_REQUIRE(partner[i] >= 0 && partner[i] < m && partner[partner[i]] == i, MI_ERR_ARG,
               "pencil partner table is not an involution");
  MI_CUDA(cudaMemcpy(c->Q.p, Q, sizeof(double) * nt * nt, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->QT.p, qt.data(), sizeof(double) * nt * nt, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->pen_diag.p, diag, sizeof(double) * m, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->pen_off.p, off, sizeof(double) * m, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->pen_g.p, g, sizeof(double) * m, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->pen_glow.p, glow, sizeof(double) * m, cudaMemcpyHostToDevice));
  if (!c->pen_partner) MI_CUDA(cudaMalloc(&c->pen_partner, sizeof(int) * m));
  MI_CUDA(cudaMemcpy(c->pen_partner, partner, sizeof(int) * m, cudaMemcpyHostToDevice));
  c->tq_mb = MI_TSTAGE ? tstage_mb(nt) : 0;
  if (c->tq_mb > 0) {
    c->tq_ksp = MI_TS_KC * (((nt + 3) / 4 + MI_TS_KC - 1) / MI_TS_KC);
    std::vector<double> f;
    build_tstage_frags(Q, nt, c->tq_mb, c->tq_ksp, f);
    if ((rc = dalloc(c->tq_frag, f.size()))) return rc;
    MI_CUDA(cudaMemcpy(c->tq_frag.p, f.data(), sizeof(double) * f.size(), cudaMemcpyHostToDevice));
  }
  c->pen_sigma = sigma;
  c->pc_cm = cm;
  c->pc_react = react;
  c->pc_ready = true;
  return MI_OK;
}

}  // extern "C"

namespace mi {

// spatial transforms of nrows time rows: forward U_1^T, U_2^T, U_3^T or inverse U_3, U_2, U_1.
// The result is written to out; scratch t1/t2 (>= nrows * ns each).
static int pc_spatial(mi_ctx* c, const double* in, double* out, long long nrows, bool inverse) {
  cudaStream_t st = c->stream;
  const int n1 = c->n[0], n2 = c->n[1], n3 = c->n[2];
  const long long ns = c->ns, N = nrows * ns;
  const bool has[3] = {n1 > 1, n2 > 1, n3 > 1};
  int nstage = has[0] + has[1] + has[2];
  if (nstage == 0) {
    if (out != in) MI_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    return MI_OK;
  }
  double* cand[3] = {c->pc_t1.p, c->pc_t2.p, c->pc_t3.p};
  double* bufs[2];
  int nb = 0;
  for (int i = 0; i < 3 && nb < 2; ++i)
    if (cand[i] != in && cand[i] != out) bufs[nb++] = cand[i];
  int k = 0, done = 0;
  const double* cur = in;
  auto dst = [&]() { ++done; if (done == nstage) return out; double* b = bufs[k]; k ^= 1; return b; };
  for (int step = 0; step < 3; ++step) {
    const int l = inverse ? 2 - step : step;
    if (!has[l]) continue;
    double* o = dst();
    ProfScope ps(c, PROF_PC_SPATIAL);
    if (l == 0) {
      MI_CUDA(spatial_mode(c, 0, inverse, cur, o, 1, N / n1));
    } else if (l == 1) {
      MI_CUDA(spatial_mode(c, 1, inverse, cur, o, n1, N / ((long long)n1 * n2)));
    } else {
      MI_CUDA(spatial_mode(c, 2, inverse, cur, o, (long long)n1 * n2, nrows));
    }
    cur = o;
  }
  return MI_OK;
}

// time stage on a (nt x ncols) column block (time-major): Q^T, arrowhead, Q.  In place.  Column j is
// the spatial eigen-index col0 + j of the grid (n1, n2c, *) whose direction-2 indices start at y_lo
// (unsharded / column ranges: n2c = n_2, y_lo = 0; z-sharded y-slabs: n2c = owned y range).
static int pc_time(mi_ctx* c, double* y, long long ncols, long long col0, int y_lo = 0, int n2c = -1) {
  cudaStream_t st = c->stream;
  const int nt = c->nt;
  if (n2c < 0) n2c = c->n[1];
  const double* lam2 = c->lam[1].p + y_lo;
  if (c->tq_mb > 0) {
    ProfScope ps(c, PROF_PC_TIME);
    TStageArgs a{y, c->tq_frag.p, c->lam[0].p, lam2, c->lam[2].p, c->pen_diag.p, c->pen_off.p,
                 c->pen_g.p, c->pen_glow.p, c->pen_partner, c->pen_sigma, c->pc_cm, c->pc_react, c->n[0], n2c,
                 nt, c->tq_ksp, ncols, col0};
    MI_CUDA(launch_tstage(c->tq_mb, a, st));
    return MI_OK;
  }
  double* t = c->pc_t2.p;
  {
    ProfScope ps(c, PROF_PC_TIME);
    MI_CUDA(mode_strided(c->QT.p, y, t, nt, ncols, 1, st));
  }
  {
    ProfScope ps(c, PROF_PC_ARROW);
    arrowhead_solve<<<(unsigned)((ncols + 127) / 128), 128, 0, st>>>(
        t, c->lam[0].p, lam2, c->lam[2].p, c->pen_diag.p, c->pen_off.p, c->pen_partner, c->pen_g.p,
        c->pen_glow.p, c->pen_sigma, c->pc_cm, c->pc_react, c->n[0], n2c, nt, ncols, col0);
    MI_CHECK_LAUNCH("arrowhead_solve");
  }
  {
    ProfScope ps(c, PROF_PC_TIME);
    MI_CUDA(mode_strided(c->Q.p, t, y, nt, ncols, 1, st));
  }
  return MI_OK;
}

}  // namespace mi

using namespace mi;

extern "C" {

int mi_pc_apply(mi_ctx* c, const double* r, double* z) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->pc_ready, MI_ERR_STATE, "preconditioner not set up");
  int rc;
  // forward spatial into pc_t1 (scratch t2 used internally), time stage in place, inverse into z
  double* y = c->pc_t1.p;
  if ((rc = pc_spatial(c, r, y, c->nt, false))) return rc;
  if ((rc = pc_time(c, y, c->ns, 0))) return rc;
  return pc_spatial(c, y, z, c->nt, true);
}

int mi_pc_apply_spatial(mi_ctx* c, const double* in, double* out, long long nrows, int inverse) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->pc_ready, MI_ERR_STATE, "preconditioner not set up");
  MI_REQUIRE(nrows >= 1 && nrows <= c->nt, MI_ERR_ARG, "nrows out of range");
  MI_REQUIRE(in != out, MI_ERR_ARG, "in and out must not alias");
  return pc_spatial(c, in, out, nrows, inverse != 0);
}

int mi_pc_apply_time(mi_ctx* c, double* y, long long ncols, long long col0) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->pc_ready, MI_ERR_STATE, "preconditioner not set up");
  MI_REQUIRE(ncols >= 1 && col0 >= 0 && col0 + ncols <= c->ns, MI_ERR_ARG, "column range out of range");
  return pc_time(c, y, ncols, col0);
}

int mi_pc_apply_time_yslab(mi_ctx* c, double* y, int y_lo, int y_hi) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->pc_ready, MI_ERR_STATE, "preconditioner not set up");
  MI_REQUIRE(c->d == 3 && 0 <= y_lo && y_lo < y_hi && y_hi <= c->n[1], MI_ERR_ARG, "y range out of range");
  const long long ncols = (long long)c->n[0] * (y_hi - y_lo) * c->n[2];
  return pc_time(c, y, ncols, 0, y_lo, y_hi - y_lo);
}

int mi_pc_fold(mi_ctx* c, int l) {
  MI_DEVICE_GUARD(c);
  if (c == nullptr || !c->pc_ready || l < 0 || l > 2) return 0;
  return c->fold_hs[l];
}

int mi_pc_mode_mapped(mi_ctx* c, int l, int inverse, const double* in, double* out, long long outer,
                      long long inner, const long long* imap, const long long* omap) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->pc_ready, MI_ERR_STATE, "preconditioner not set up");
  MI_REQUIRE(l >= 0 && l < c->d, MI_ERR_ARG, "direction out of range");
  MI_REQUIRE(outer >= 1 && inner >= 2 && in != out, MI_ERR_ARG, "bad mode-product shape or aliasing");
  MI_REQUIRE(c->fold_hs[l] > 0, MI_ERR_ARG, "addressing maps need a mirrored (folded) eigenbasis");
  ProfScope ps(c, PROF_PC_SPATIAL);
  cudaError_t err = cudaSuccess;
  const bool done = launch_mode_fold<false>(c->Us[l].p, in, out, c->n[l], inverse != 0, inner, outer, num_sms(),
                                            c->stream, &err, imap, omap);
  MI_REQUIRE(done, MI_ERR_ARG, "mode extent outside the folded kernel's range");
  MI_CUDA(err);
  return MI_OK;
}

int mi_pc_mode(mi_ctx* c, int l, int inverse, const double* in, double* out, long long outer, long long inner) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c && c->pc_ready, MI_ERR_STATE, "preconditioner not set up");
  MI_REQUIRE(l >= 0 && l < c->d, MI_ERR_ARG, "direction out of range");
  MI_REQUIRE(outer >= 1 && inner >= 1 && in != out, MI_ERR_ARG, "bad mode-product shape or aliasing");
  ProfScope ps(c, PROF_PC_SPATIAL);
  // forward applies U_l^T, inverse U_l (pc_spatial's convention)
  MI_CUDA(spatial_mode(c, l, inverse != 0, in, out, inner, outer));
  return MI_OK;
}

}  // extern "C"
