// Reaction correction y += M_R x with the Rogers-McCulloch linearisation
// (reference reaction_mass, assembly.py:287-347):
//
//   M_R[i, j] = int int C_r B_i B_j,   C_r = c1 (u - a)(u - 1) + c2 w,
//
// u, w = the frozen iterate, evaluated at q = p+1 Gauss points per element
// in every direction (space and time; assembly.py:313-318 -- the rule is
// parity-critical).  Matrix-free: a block owns a tile
// of p elements per direction (incl. time), loads the local coefficients of
// u, w, x, interpolates them to the tile's Gauss grid one time point at a
// time (sum factorisation: t, then x, y, z), evaluates the ionic
// linearisation pointwise, and projects back (z, y, x, t).  Tiles are
// processed in 2^(d+1) colour classes so concurrently running blocks never
// touch the same output DoF: no atomics, bitwise deterministic.
#include "common.cuh"
#include "dispatch.cuh"

namespace mi {

struct RxArgs {
  const double* u;
  const double* w;
  const double* x;
  double* y;
  // per direction l = 0 (x), 1 (y), 2 (z), 3 (t): basis values at Gauss points
  // B_l[(e * q + g) * (p_l + 1) + a] of function e + a, weights W_l[e * q + g]
  const double* B[4];
  const double* Wq[4];
  int q[4];            // Gauss points per element per direction (1 for absent dims)
  int pl[4];           // degree per direction (0 for absent dims)
  int nel[4];          // elements per direction (1 for absent dims)
  int n[4];            // functions per direction (time: FULL basis incl. removed first)
  int E[4];            // tile size in elements per direction
  int ntile[4];        // tiles per direction
  int color[4];        // colour class of this launch (tile parity)
  int ncol[4];         // tiles of this colour per direction
  int ntc;             // constrained time functions (= n[3] - 1)
  long long ns;
  double c1, a, c2;
};

// Interpolate along one direction: in[..., L] (coefficients) -> out[..., Q]
// (Gauss points of the tile's elements).  Layout: pre x dim x post.
__device__ __forceinline__ void interp_dir(const double* in, double* out, int pre, int L, int Q, int post,
                                           const double* B, int q, int p, int e0, int k0) {
  // out[pre][Qi][post] = sum_a B[(e*q+g)*(p+1)+a] in[pre][e - k0 + a][post], Qi = (e - e0)*q + g
  const int total = pre * Q * post;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int po = idx % post, r = idx / post;
    const int Qi = r % Q, pr = r / Q;
    const int e = e0 + Qi / q, g = Qi % q;
    const double* b = B + ((long long)e * q + g) * (p + 1);
    const double* src = in + ((long long)pr * L + (e - k0)) * post + po;
    double v = 0.0;
    for (int aa = 0; aa <= p; ++aa) v = fma(b[aa], src[aa * post], v);
    out[idx] = v;
  }
}

// Project (transpose of interp_dir): in[pre][Q][post] -> out[pre][L][post]
__device__ __forceinline__ void project_dir(const double* in, double* out, int pre, int L, int Q, int post,
                                            const double* B, int q, int p, int e0, int ne, int k0) {
  const int total = pre * L * post;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int po = idx % post, r = idx / post;
    const int li = r % L, pr = r / L;
    const int f = k0 + li;                       // function index
    double v = 0.0;
    // elements e in [e0, e0+ne) with f - e in [0, p]
    const int elo = max(e0, f - p), ehi = min(e0 + ne - 1, f);
    for (int e = elo; e <= ehi; ++e) {
      const int aa = f - e;
      for (int g = 0; g < q; ++g) {
        const double bv = B[((long long)e * q + g) * (p + 1) + aa];
        v = fma(bv, in[((long long)pr * Q + (e - e0) * q + g) * post + po], v);
      }
    }
    out[idx] = v;
  }
}

__global__ void reaction_tile(RxArgs r) {
  extern __shared__ double sm[];
  // tile coordinates of this colour
  int b = blockIdx.x;
  int k[4], e0[4], ne[4], L[4], Q[4];
  for (int l = 0; l < 4; ++l) {
    const int m = b % r.ncol[l];
    b /= r.ncol[l];
    k[l] = 2 * m + r.color[l];
    e0[l] = k[l] * r.E[l];
    ne[l] = min(r.E[l], r.nel[l] - e0[l]);
    L[l] = ne[l] + r.pl[l];                      // local functions [e0, e0 + L)
    Q[l] = ne[l] * r.q[l];
  }
  const int Ls = L[0] * L[1] * L[2];
  const int Qs = Q[0] * Q[1] * Q[2];
  // smem carve-up (sizes from the launch: worst case per block)
  double* cu = sm;                               // [Lt][Ls] x3 fields
  double* cw = cu + L[3] * Ls;
  double* cx = cw + L[3] * Ls;
  double* outc = cx + L[3] * Ls;                 // [Lt][Ls] output accumulation
  double* f0 = outc + L[3] * Ls;                 // time-interpolated fields [3][Ls]
  const int big = max(Qs, max(Q[0] * L[1] * L[2], Q[0] * Q[1] * L[2]));
  double* s1 = f0 + 3 * Ls;                      // [3][big]
  double* s2 = s1 + 3 * big;                     // [3][big]

  // load local coefficients (time index in the FULL basis: constrained = f - 1)
  for (int idx = threadIdx.x; idx < L[3] * Ls; idx += blockDim.x) {
    const int sl = idx % Ls, tl = idx / Ls;
    const int i1 = sl % L[0], i2 = (sl / L[0]) % L[1], i3 = sl / (L[0] * L[1]);
    const int ft = e0[3] + tl, ct = ft - 1;
    const long long gs = ((long long)(e0[2] + i3) * r.n[1] + (e0[1] + i2)) * r.n[0] + (e0[0] + i1);
    const bool v = ct >= 0 && ct < r.ntc;
    const long long gi = (long long)ct * r.ns + gs;
    cu[idx] = v ? r.u[gi] : 0.0;
    cw[idx] = v ? r.w[gi] : 0.0;
    cx[idx] = v ? r.x[gi] : 0.0;
    outc[idx] = 0.0;
  }
  __syncthreads();
  const int pt = r.pl[3], qt = r.q[3];
  for (int et = e0[3]; et < e0[3] + ne[3]; ++et) {
    for (int g = 0; g < qt; ++g) {
      const double* bt = r.B[3] + ((long long)et * qt + g) * (pt + 1);
      const double wt = r.Wq[3][et * qt + g];
      // time interpolation of u, w, x at this Gauss time
      for (int idx = threadIdx.x; idx < 3 * Ls; idx += blockDim.x) {
        const int fld = idx / Ls, sl = idx % Ls;
        const double* c = (fld == 0 ? cu : (fld == 1 ? cw : cx)) + (et - e0[3]) * Ls + sl;
        double v = 0.0;
        for (int aa = 0; aa <= pt; ++aa) v = fma(bt[aa], c[aa * Ls], v);
        f0[idx] = v;
      }
      __syncthreads();
      // spatial interpolation x -> y -> z for the 3 fields
      for (int fld = 0; fld < 3; ++fld)
        interp_dir(f0 + fld * Ls, s1 + fld * big, L[2] * L[1], L[0], Q[0], 1, r.B[0], r.q[0], r.pl[0], e0[0], e0[0]);
      __syncthreads();
      for (int fld = 0; fld < 3; ++fld)
        interp_dir(s1 + fld * big, s2 + fld * big, L[2], L[1], Q[1], Q[0], r.B[1], r.q[1], r.pl[1], e0[1], e0[1]);
      __syncthreads();
      for (int fld = 0; fld < 3; ++fld)
        interp_dir(s2 + fld * big, s1 + fld * big, 1, L[2], Q[2], Q[1] * Q[0], r.B[2], r.q[2], r.pl[2], e0[2], e0[2]);
      __syncthreads();
      // pointwise ionic linearisation and quadrature weights
      for (int idx = threadIdx.x; idx < Qs; idx += blockDim.x) {
        const int g1 = idx % Q[0], g2 = (idx / Q[0]) % Q[1], g3 = idx / (Q[0] * Q[1]);
        const double w1 = r.Wq[0][e0[0] * r.q[0] + g1];
        const double w2 = r.Wq[1][e0[1] * r.q[1] + g2];
        const double w3 = r.Wq[2][e0[2] * r.q[2] + g3];
        const double uu = s1[idx], ww = s1[big + idx], xx = s1[2 * big + idx];
        const double cr = r.c1 * (uu - r.a) * (uu - 1.0) + r.c2 * ww;
        s2[idx] = cr * xx * (wt * w1 * w2 * w3);
      }
      __syncthreads();
      // projection z -> y -> x
      project_dir(s2, s1, 1, L[2], Q[2], Q[1] * Q[0], r.B[2], r.q[2], r.pl[2], e0[2], ne[2], e0[2]);
      __syncthreads();
      project_dir(s1, s2, L[2], L[1], Q[1], Q[0], r.B[1], r.q[1], r.pl[1], e0[1], ne[1], e0[1]);
      __syncthreads();
      project_dir(s2, s1, L[2] * L[1], L[0], Q[0], 1, r.B[0], r.q[0], r.pl[0], e0[0], ne[0], e0[0]);
      __syncthreads();
      // time projection into the output block
      for (int idx = threadIdx.x; idx < (pt + 1) * Ls; idx += blockDim.x) {
        const int aa = idx / Ls, sl = idx % Ls;
        outc[(et - e0[3] + aa) * Ls + sl] += bt[aa] * s1[sl];
      }
      __syncthreads();
    }
  }
  // add to y (this colour's tiles own disjoint output DoFs)
  for (int idx = threadIdx.x; idx < L[3] * Ls; idx += blockDim.x) {
    const int sl = idx % Ls, tl = idx / Ls;
    const int i1 = sl % L[0], i2 = (sl / L[0]) % L[1], i3 = sl / (L[0] * L[1]);
    const int ct = e0[3] + tl - 1;
    if (ct < 0 || ct >= r.ntc) continue;
    const long long gs = ((long long)(e0[2] + i3) * r.n[1] + (e0[1] + i2)) * r.n[0] + (e0[0] + i1);
    r.y[(long long)ct * r.ns + gs] += outc[idx];
  }
}

static size_t rx_smem(const mi_ctx* c) {
  int L[4], Q[4];
  for (int l = 0; l < 4; ++l) {
    L[l] = c->rx_E[l] + c->rx_p[l];
    Q[l] = c->rx_E[l] * c->rx_q[l];
  }
  const size_t Ls = (size_t)L[0] * L[1] * L[2];
  const size_t Qs = (size_t)Q[0] * Q[1] * Q[2];
  const size_t big = std::max(Qs, std::max((size_t)Q[0] * L[1] * L[2], (size_t)Q[0] * Q[1] * L[2]));
  return (4 * L[3] * Ls + 3 * Ls + 6 * big) * sizeof(double);
}

int reaction_apply(mi_ctx* c, const double* x, double* y) {
  RxArgs r{};
  r.u = c->u_it.p;
  r.w = c->w_it.p;
  r.x = x;
  r.y = y;
  for (int l = 0; l < 4; ++l) {
    r.B[l] = c->rx_B.p + c->rx_Boff[l];
    r.Wq[l] = c->rx_W.p + c->rx_Woff[l];
    r.q[l] = c->rx_q[l];
    r.pl[l] = c->rx_p[l];
    r.nel[l] = c->rx_nel[l];
    r.E[l] = c->rx_E[l];
    r.ntile[l] = (c->rx_nel[l] + c->rx_E[l] - 1) / c->rx_E[l];
  }
  r.n[0] = c->n[0];
  r.n[1] = c->n[1];
  r.n[2] = c->n[2];
  r.n[3] = c->nt + 1;
  r.ntc = c->nt;
  r.ns = c->ns;
  r.c1 = c->c1;
  r.a = c->a;
  r.c2 = c->c2;
  const size_t smem = rx_smem(c);
  for (int col = 0; col < 16; ++col) {
    long long nb = 1;
    bool empty = false;
    for (int l = 0; l < 4; ++l) {
      r.color[l] = (col >> l) & 1;
      r.ncol[l] = (r.ntile[l] - r.color[l] + 1) / 2;
      if (r.ncol[l] <= 0) empty = true;
      nb *= r.ncol[l];
    }
    if (empty) continue;
    reaction_tile<<<(unsigned)nb, 256, smem, c->stream>>>(r);
    MI_CHECK_LAUNCH("reaction_tile");
  }
  return MI_OK;
}

}  // namespace mi

using namespace mi;

extern "C" {

int mi_op_set_reaction(mi_ctx* c, const double* u, const double* w, double c1, double a, double c2,
                       const int* q, const int* nel, const double* B, const double* Wq) {
  MI_REQUIRE(c && c->op_ready, MI_ERR_STATE, "mi_op_setup must be called first");
  MI_REQUIRE(u && w && q && nel && B && Wq, MI_ERR_ARG, "NULL argument to mi_op_set_reaction");
  int rc;
  if ((rc = dalloc(c->u_it, c->N)) || (rc = dalloc(c->w_it, c->N))) return rc;
  MI_CUDA(cudaMemcpyAsync(c->u_it.p, u, sizeof(double) * c->N, cudaMemcpyDeviceToDevice, c->stream));
  MI_CUDA(cudaMemcpyAsync(c->w_it.p, w, sizeof(double) * c->N, cudaMemcpyDeviceToDevice, c->stream));
  // per direction tables, direction order x, y, z, t; absent spatial dims get q=1, p=0
  size_t nb = 0, nw = 0;
  for (int l = 0; l < 4; ++l) {
    const bool present = l == 3 || l < c->d;
    const int src = l == 3 ? c->d : l;           // host arrays: x, y, ..., t
    c->rx_q[l] = present ? q[src] : 1;
    c->rx_p[l] = present ? (l == 3 ? c->pt : c->p) : 0;
    c->rx_nel[l] = present ? nel[src] : 1;
    c->rx_E[l] = present ? std::max(1, c->rx_p[l]) : 1;
    c->rx_Boff[l] = nb;
    c->rx_Woff[l] = nw;
    nb += (size_t)c->rx_nel[l] * c->rx_q[l] * (c->rx_p[l] + 1);
    nw += (size_t)c->rx_nel[l] * c->rx_q[l];
  }
  std::vector<double> hb(nb), hw(nw);
  size_t sb = 0, sw = 0;
  for (int l = 0; l < 4; ++l) {
    const bool present = l == 3 || l < c->d;
    const size_t cb = (size_t)c->rx_nel[l] * c->rx_q[l] * (c->rx_p[l] + 1);
    const size_t cw = (size_t)c->rx_nel[l] * c->rx_q[l];
    for (size_t i = 0; i < cb; ++i) hb[c->rx_Boff[l] + i] = present ? B[sb + i] : 1.0;
    for (size_t i = 0; i < cw; ++i) hw[c->rx_Woff[l] + i] = present ? Wq[sw + i] : 1.0;
    if (present) {
      sb += cb;
      sw += cw;
    }
  }
  if ((rc = dalloc(c->rx_B, nb)) || (rc = dalloc(c->rx_W, nw))) return rc;
  MI_CUDA(cudaMemcpy(c->rx_B.p, hb.data(), sizeof(double) * nb, cudaMemcpyHostToDevice));
  MI_CUDA(cudaMemcpy(c->rx_W.p, hw.data(), sizeof(double) * nw, cudaMemcpyHostToDevice));
  c->c1 = c1;
  c->a = a;
  c->c2 = c2;
  const size_t smem = rx_smem(c);
  MI_REQUIRE(smem <= 227 * 1024, MI_ERR_ARG, "reaction tile does not fit in shared memory");
  MI_CUDA(cudaFuncSetAttribute(reaction_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  c->reaction_on = true;
  return MI_OK;
}

int mi_op_clear_reaction(mi_ctx* c) {
  if (c) c->reaction_on = false;
  return MI_OK;
}

}  // extern "C"
