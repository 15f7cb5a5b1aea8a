/*
 * libmonoiga_b200 -- C ABI of the B200-native preconditioned space-time
 * Krylov solve (hot path of arxiv 2311.17500 / reference package `monoiga`).
 *
 * Plain C: opaque context, raw pointers and sizes, int status codes.  All
 * vector arguments named x/y/r/z/V/w/h are DEVICE pointers (fp64) in the
 * reference layout: C-order (N_t, n_d, ..., n_1), direction 1 fastest
 * (reference tensorops.py:1-7).  Table arguments marked "host" are copied
 * to the device by the call.  Every call is ordered on the context's
 * stream; none allocates after the corresponding *_setup call.
 *
 * Status: 0 ok; MI_ERR_ARG (bad argument / dimension mismatch, maps to the
 * reference's ValueError); MI_ERR_CUDA (device failure); MI_ERR_STATE (call
 * order); the message is in mi_last_error() (thread-local).
 */
#ifndef MONOIGA_B200_H
#define MONOIGA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MI_OK 0
#define MI_ERR_ARG 1
#define MI_ERR_CUDA 2
#define MI_ERR_STATE 3

typedef struct mi_ctx mi_ctx;

/* Library identity and last error of the calling thread. */
int mi_version(void);
const char* mi_last_error(void);

/* Measurement diagnostic (no reference counterpart): FP64 throughput on `device` of a DMMA-only
 * (kind 0, mma.sync m8n8k4 f64), DFMA-only (kind 1) or mixed DMMA+DFMA (kind 2) kernel, 8 blocks of
 * 256 threads per SM.  bench.py takes max(cuBLAS DGEMM, kind 0) as the FP64 tensor peak. */
int mi_diag_fp64_peak(int device, int kind, double* tflops, double* ms);

/* Context for one space-time tensor shape on one device.
 * Replaces the dimension bookkeeping of SpaceTimeSpace (bspline.py:311-420):
 * d spatial directions with n[0..d-1] = n_1..n_d functions, N_t = nt
 * (first time function removed), spatial degree p, time degree pt. */
int mi_ctx_create(int device, int d, const int* n, int nt, int p, int pt, mi_ctx** out);
int mi_ctx_destroy(mi_ctx* ctx);
int mi_ctx_set_stream(mi_ctx* ctx, void* cuda_stream);
/* z-slab context for the space-sharded solve (no reference
 * counterpart: the reference is single-process).  d = 3 only; call before
 * mi_op_setup.  The context's n[2] planes are the global planes
 * [z_lo, z_lo + n[2]) of n3g; mi_op_apply then takes x (and the reaction
 * iterate u, w) on the INPUT slab = hz_lo halo planes + the owned planes +
 * hz_hi halo planes (hz <= p), and writes y on the owned planes only.
 * Channel tables stay global: band / H tables have max(n_1, n_2, n3g) rows,
 * theta has n_1 n_2 n3g entries. */
int mi_ctx_set_zslab(mi_ctx* ctx, int z_lo, int n3g, int hz_lo, int hz_hi);

/* Per-kernel-class CUDA-event timing (bench/roofline support; no reference
 * counterpart).  Slots: 0 op stencil, 1 op time filter, 2 op reaction,
 * 3 pc spatial transforms, 4 pc time transforms, 5 pc arrowhead, 6 krylov,
 * 7 setup.  mi_prof_read syncs the stream and returns accumulated ms and
 * launch counts (arrays of 8); reset != 0 clears them. */
int mi_prof_enable(mi_ctx* ctx, int on);
int mi_prof_read(mi_ctx* ctx, double* ms, long long* launches, int reset);

/* ---------------------------------------------------------------------
 * Operator A  (replaces KroneckerOperator + two_factor_matvec,
 * assembly.py:401-444 / tensorops.py:45-56, with the term list of
 * _Workspace.operator, solver.py:213-236)
 *
 * A = sum_c T_c (x) S_c  over nchan channels.  T_c: banded N_t x N_t time
 * factor, host band (nchan, nt, 2pt+1) with band[c][i][k] = T_c[i, i-pt+k].
 * S_c: spatial factor, generated on the device as a (2p+1)^d stencil from
 * either a sum of Kronecker products of banded 1D factors
 * (mi_op_set_kron_channel: M_s, K_s, K_sigma of assembly.py:222-238) or a
 * multilinear-theta weighted mass (mi_op_set_su_channel: S^s_r of
 * stabilization.py:469-488).
 * ------------------------------------------------------------------- */
int mi_op_setup(mi_ctx* ctx, int nchan);
int mi_op_set_time_bands(mi_ctx* ctx, const double* bands /* host nchan*nt*(2pt+1) */);
/* channel c spatial factor = sum_t coef[t] * kron_l band[t][l]
 * bands: host (nterms, d, nmax, 2p+1), band[t][l][i][k] = F_{t,l}[i, i-p+k],
 * nmax = max_l n_l. */
int mi_op_set_kron_channel(mi_ctx* ctx, int c, int nterms, const double* coef, const double* bands);
/* channel c spatial factor = sum_k theta[k] prod_l H_l[i_l, j_l-i_l+p, k_l-i_l+ko]
 * theta: host N_s (flat spatial order); H: host (d, nmax, 2p+1, 2ko+1). */
int mi_op_set_su_channel(mi_ctx* ctx, int c, const double* theta, const double* H, int ko);
/* Mapped (non-affine) geometry: channel c spatial factor assembled by
 * tensor Gauss quadrature (replaces SpatialQuadratureData.mass/stiffness,
 * assembly.py:197-219):
 *   S[i, j] = sum_t coef[t] sum_k theta[t][k] prod_l T[t][l][i_l][j_l-i_l+p][k_l-(i_l-p) q_l]
 * theta: host nterms x (Q_d ... Q_1) Gauss-grid weights (w |det J|, times the
 * metric (J^-1 J^-T)_ab for stiffness terms); T: host nterms x d x nmax x
 * (2p+1) x kw products of basis values / derivatives, kw = max_l (p+1) q_l;
 * q[l] Gauss points per element, Q[l] in total (direction 1 first). */
int mi_op_set_quad_channel(mi_ctx* ctx, int c, int nterms, const double* coef, const double* theta,
                           const double* T, const int* q, const int* Q);
/* The same with an explicit window per basis function (the Spline Upwind
 * factors on mapped geometries, stabilization.py:469-488, integrate on cells
 * split at the spatial Greville abscissae with p+2 points, so the number of
 * Gauss points per element varies): function i of direction l covers the
 * Gauss points kstart[l][i] .. kstart[l][i] + kw[l] - 1 of that direction
 * (kstart: host d x nmax ints), and T's last index is relative to kstart. */
int mi_op_set_quad_channel_k(mi_ctx* ctx, int c, int nterms, const double* coef, const double* theta,
                             const double* T, const int* kstart, const int* kw, const int* Q);
/* Device-to-device copy of channel c's stencil ((2p+1)^d x N_s, point
 * fastest) in / out: a caller reuses generated spatial factors across
 * operator rebuilds (the reference keeps M_s, K_s in its _Workspace,
 * solver.py:167-175). */
int mi_op_set_channel_stencil(mi_ctx* ctx, int c, const double* stencil);
int mi_op_get_channel_stencil(mi_ctx* ctx, int c, double* stencil);
/* y = A x   (x, y device, length N, must not alias) */
int mi_op_apply(mi_ctx* ctx, const double* x, double* y);
/* y = A x for x in PINNED HOST memory (x_dev: a device buffer of N for the copy): the host-to-device copy
 * of x runs on the context's copy stream in nparts z-plane chunks, and the stencil over the cube layers
 * of chunk p runs while chunk p+1 is still on its way (d = 3 tensor-core operator; otherwise one copy
 * then mi_op_apply).  The reference-facing KroneckerOperator.matvec path for host input. */
int mi_op_apply_from_host(mi_ctx* ctx, const double* x_host, double* x_dev, double* y, int nparts);

/* Reaction correction y += M_R x (added by every subsequent mi_op_apply),
 * M_R = int int C_r B_i B_j with the Rogers-McCulloch linearisation
 * C_r = c1 (u - a)(u - 1) + c2 w evaluated at q = p+1 Gauss points per
 * element and direction (replaces reaction_mass + the CSR correction of
 * KroneckerOperator.matvec, assembly.py:287-347 / 442-443).
 * u, w: DEVICE iterate coefficients (length N, copied).  Host tables per
 * present direction in the order x, y, ..., t (spatial directions 1..d,
 * then time): q[l] Gauss points per element, nel[l] elements; B = concat_l
 * (nel_l, q_l, p_l + 1) values of functions e..e+p_l at the Gauss points of
 * element e (time: FULL basis incl. the removed first function); Wq = concat_l
 * (nel_l, q_l) weights (Gauss x half-length x box length, x T in time).
 * q, nel have d+1 entries. */
int mi_op_set_reaction(mi_ctx* ctx, const double* u, const double* w, double c1, double a, double c2,
                       const int* q, const int* nel, const double* B, const double* Wq);
int mi_op_clear_reaction(mi_ctx* ctx);

/* u0 lifting (no reference counterpart: the reference's trial space drops the first time function,
 * bspline.py:384-387, and fields.py:8-12 pads that slab with zeros, so it cannot take u0 != 0; SURVEY
 * Appendix B).  u = u0_h(x) b_0(t) + u~.  mi_op_set_lift stores the lifting coefficients u0 (device,
 * N_s of the input slab; NULL clears) and, per channel, the column of the channel's FULL time factor
 * that couples the constrained rows to b_0 (host, nchan x N_t, nonzero in the first p_t rows only).
 * While a lift is set the reaction's C_r sees the lifted iterate (the u0 slab is read for b_0).
 * mi_op_apply_lift writes y = A_{c,0} u0: the lifted column of every channel and of M_R applied to u0
 * (the sweep's right-hand side correction f - A_{c,0} u0). */
int mi_op_set_lift(mi_ctx* ctx, const double* column0, const double* u0);

/* Pack the channel stencils into the tensor-core layout now; with release != 0 also free the plain
 * stencil copy (the operator's largest table after the packed one: 21 GB at BASELINE cfg 4), after
 * which the channels are immutable until the next mi_op_setup (time bands, the reaction and the lift
 * may still change).  Contexts rebuilt every sweep keep it (release = 0): no per-sweep reallocation. */
int mi_op_finalize(mi_ctx* ctx, int release);
int mi_op_apply_lift(mi_ctx* ctx, double* y);
/* Mapped geometry: |det J| at the spatial Gauss points (host, C order
 * Q_d ... Q_1) multiplies the reaction's quadrature weights
 * (reaction_mass with spatial_data, assembly.py:320-326); NULL = box.
 * Call after mi_op_set_reaction. */
int mi_op_set_reaction_weight(mi_ctx* ctx, const double* jw);
/* Stored-coefficient mode of the reaction: the iterate is frozen for a
 * whole solve, so C_r times the spatial quadrature weight is evaluated once
 * at every space-time Gauss point (next apply after a change) and each
 * apply interpolates only x.  mode -1: when it fits in 40% of the free
 * device memory (default), 0: never, 1: always. */
int mi_op_set_reaction_store(mi_ctx* ctx, int mode);
/* Kernel of the fused (non-stored) reaction: -1 auto (the warp-specialised
 * reaction_ws at d = 3, p = p_t = 3, c1 >= 0; reaction_tile otherwise),
 * 0 reaction_tile, 1 reaction_ws.  Both evaluate reaction_mass's quadrature
 * (assembly.py:287-347); the switch exists for parity tests and timing. */
int mi_op_set_reaction_kernel(mi_ctx* ctx, int kernel);
/* Time slabs (KroneckerOperator(time_rows=...)): the reaction tables cover local time elements whose
 * full-basis function ft maps to local row ft + row_offset (default -1). */
int mi_op_set_reaction_rows(mi_ctx* ctx, int row_offset);

/* ---------------------------------------------------------------------
 * Fast-diagonalisation preconditioner  (replaces
 * FastDiagPreconditioner.apply / _diag_blocks, linalg.py:309-353, built
 * from FastDiagPreconditioner.build, linalg.py:264-307)
 *
 * P^-1 = (Q (x) U_s) (C_m Delta + mu I)^-1 (Q^T (x) U_s^T)
 * U: host (d, nmax, nmax) per-direction eigenvectors (row-major n_l x n_l);
 * lam: host (d, nmax) eigenvalues already multiplied by sigma_l;
 * Q: host nt x nt real time basis; Delta = real block arrowhead given by
 * diag/off/partner (2x2 blocks) + border g (upper), glow (lower), sigma.
 * ------------------------------------------------------------------- */
int mi_pc_setup(mi_ctx* ctx, const double* U, const double* lam, double cm, double react,
                const double* Q, const double* diag, const double* off, const int* partner,
                const double* g, const double* glow, double sigma);
/* z = P^-1 r  (r, z device; may alias) */
int mi_pc_apply(mi_ctx* ctx, const double* r, double* z);
/* Split preconditioner stages (a caller distributing the columns itself): spatial transforms
 * of nrows local time rows (inverse=0: U^T, inverse=1: U), and the time
 * stage (Q^T, block-arrowhead solve, Q) in place on a time-major (N_t x
 * ncols) block of spatial eigen-columns [col0, col0+ncols) after the
 * all-to-all transpose. */
int mi_pc_apply_spatial(mi_ctx* ctx, const double* in, double* out, long long nrows, int inverse);
int mi_pc_apply_time(mi_ctx* ctx, double* y, long long ncols, long long col0);
/* Stages for the z-sharded preconditioner (sharded.py; the reference's
 * mode_apply, tensorops.py:13-26, one direction at a time): out = the
 * direction-l mode product of in viewed as (outer, n_l, inner), with U_l^T
 * (inverse=0) or U_l (inverse=1); and the time stage on a y-slab
 * (N_t, n_3, y_hi - y_lo, n_1) holding spatial eigen-indices with
 * i_2 in [y_lo, y_hi). */
int mi_pc_mode(mi_ctx* ctx, int l, int inverse, const double* in, double* out, long long outer, long long inner);
/* mi_pc_mode along a strided direction (inner >= 2) with addressing maps (device int64, 2 n_l entries
 * each, nullable): element (o, r, c) of the input / output lives at map[2r] + o * map[2r+1] + c.  Lets
 * the space-sharded P^-1 read and write the all-to-all send / receive layouts without packing copies.
 * Needs a mirrored (folded) eigenbasis. */
int mi_pc_mode_mapped(mi_ctx* ctx, int l, int inverse, const double* in, double* out, long long outer,
                      long long inner, const long long* imap, const long long* omap);
int mi_pc_apply_time_yslab(mi_ctx* ctx, double* y, int y_lo, int y_hi);
/* Number of symmetric modes hs of direction l when its eigenbasis is an
 * exactly mirrored even/odd basis (uniform knots: factors._centro_eigh) and
 * the spatial transforms run as two half-size products (mode_fold.cuh);
 * 0 when the dense n_l x n_l product is used.  Same P^-1 either way. */
int mi_pc_fold(mi_ctx* ctx, int l);

/* ---------------------------------------------------------------------
 * Recovery-variable solve ((W_t + b d_e M_t) (x) M_s) w = g  (replaces
 * solve_w_system + pcg + KroneckerMassPreconditioner, linalg.py:176-203,
 * 450-547).  Host tables: Kinv (nt x nt) = (W_t + b d_e M_t)^{-1};
 * M, Minv (d, nmax, nmax): spatial mass factors (incl. box length) and the
 * preconditioner's inverse univariate masses.  The PCG over time rows is
 * driven by the caller with the row-batched primitives below.
 * ------------------------------------------------------------------- */
int mi_ws_setup(mi_ctx* ctx, const double* Kinv, const double* M, const double* Minv);
int mi_ws_time(mi_ctx* ctx, const double* in, double* out);
int mi_ws_mass(mi_ctx* ctx, const double* in, double* out, long long nrows, int inverse);
int mi_rowdots(mi_ctx* ctx, long long nrows, long long ncols, const double* a, const double* b, double* out);
int mi_row_axpy(mi_ctx* ctx, long long nrows, long long ncols, const double* alpha, double sign,
                const double* x, double* y);
int mi_row_xpby(mi_ctx* ctx, long long nrows, long long ncols, const double* beta, const double* z, double* p);

/* ---------------------------------------------------------------------
 * Krylov primitives (replace the numpy CGS2 / update steps of gmres,
 * linalg.py:404-444).  V is a device matrix of k rows of length n with
 * row stride ldv.  Reductions are deterministic (fixed partition, fixed
 * order, no atomics): repeated calls are bitwise identical.
 * ------------------------------------------------------------------- */
/* h[i] = <V_i, w>, i < k   (h device) */
int mi_dots(mi_ctx* ctx, long long n, int k, const double* V, long long ldv, const double* w, double* h);
/* w -= sum_i h[i] V_i   (h device) */
int mi_sub_combination(mi_ctx* ctx, long long n, int k, const double* V, long long ldv, const double* h, double* w);
/* out = x0 + sum_i y[i] V_i   (y device; x0 may be NULL for 0) */
int mi_combination(mi_ctx* ctx, long long n, int k, const double* V, long long ldv, const double* y,
                   const double* x0, double* out);
/* out = x * s  with s = 1 / *hnorm read on the device */
int mi_scale_inv(mi_ctx* ctx, long long n, const double* x, const double* hnorm, double* out);
/* out = x / sqrt(*nrm2)  (nrm2 device: squared norm from mi_dots) */
int mi_normalize(mi_ctx* ctx, long long n, const double* x, const double* nrm2, double* out);
/* fused CGS2 pass (linalg.py:405-411, one read of V): w -= sum_i h_in[i] V_i, then h_out[i] = V_i . w;
 * bitwise the same as mi_sub_combination followed by mi_dots (k <= 32 fused, two passes beyond) */
int mi_cgs_pass(mi_ctx* ctx, long long n, int k, const double* V, long long ldv, const double* h_in,
                double* w, double* h_out);
/* fused last CGS2 pass + norm (linalg.py:409-412): w -= sum_i h_in[i] V_i, then *nrm2 = w . w;
 * bitwise the same as mi_sub_combination followed by mi_dots(w, w) */
int mi_cgs_norm_pass(mi_ctx* ctx, long long n, int k, const double* V, long long ldv, const double* h_in,
                     double* w, double* nrm2);

/* ---------------------------------------------------------------------
 * Spline Upwind residual indicator (replaces compute_theta's grid work,
 * stabilization.py:235-339, with the strong residual of 148-174 and the
 * ionic current c1 u (u-a)(u-1) + c2 u w at the q = p+1 Gauss points).
 * ------------------------------------------------------------------- */
/* Element tables per present direction x, y, z (d of them) then t, each
   [nel][q][p+1] (value of function e + a at Gauss point g of element e):
   B0 values; B1 second parametric derivatives (space) / first (time).
   lengths: box edge lengths; diffusion: D_l per direction (the reference's
   scalar D repeated), so the diffusion term is sum_l D_l d2u/dx_l^2 / L_l^2. */
int mi_theta_setup(mi_ctx* ctx, const int* nel, const double* B0, const double* B1, const double* lengths,
                   const double* diffusion, double final_time, double C_m, double c1, double a, double c2);
/* Element maxima of |res| for time elements [et0, et1) into emax (device,
   [nel_t][nel_3][nel_2][nel_1]) and running maxima of |u|, |u_t| into
   maxes (device double[2], zeroed by the caller before the first call).
   src: NULL, or the source at the Gauss points of those elements,
   [(et - et0) * q_t + g][spatial Gauss index] (device). */
int mi_theta_elements(mi_ctx* ctx, const double* u, const double* w, const double* src, int et0, int et1,
                      double* emax, double* maxes);
/* out[o][i][r] = max over e in [w0[i], w1[i]) of in[o][e][r]   (w0, w1 host) */
/* Mapped geometries: the residual indicator's element maxima from
 * precomputed Gauss-point fields of time elements [et0, et1)
 * (stabilization.py:235-295 with the pulled-back Laplacian):
 * fields = [u, u_tau, w, d_i u (i < d), d_ab u (a = b first, then a < b)]
 * x rows x G_s, coef = [cg_i, cm_ab] x G_s (see theta.py MappedDeviceIndicator),
 * src = NULL or f at the same points; G[l] = nel[l] q spatial Gauss points.
 * emax / maxes as mi_theta_elements. */
/* Lifting for the indicator: the u field's dropped slab holds u0 (device, N_s) instead of zeros
 * (the lifted counterpart of _full_time_tensor, fields.py:8-12); NULL clears. */
int mi_theta_set_lift(mi_ctx* ctx, const double* u0);

int mi_theta_mapped_elements(mi_ctx* ctx, const double* fields, const double* coef, const double* src, int et0,
                             int et1, const int* G, int q, int qt, const int* nel, double D, double cmT, double c1,
                             double a, double c2, double* emax, double* maxes);
int mi_window_max(mi_ctx* ctx, const double* in, double* out, long long outer, int n_in, int n_out,
                  long long inner, const int* w0, const int* w1);
/* theta = min(numer / denom, 1)   (denom > 0) */
int mi_theta_ratio(mi_ctx* ctx, const double* numer, double* theta, long long n, double denom);

#ifdef __cplusplus
}
#endif
#endif
