// Shared definitions for libmonoiga_b200 (sm_100a).
//
// Tensor layout everywhere: C-order (N_t, n_3, n_2, n_1) fp64, direction 1
// fastest (reference tensorops.py:1-7, bspline.py:311-316).  Spatial
// directions beyond d have extent 1, so every kernel is written for d = 3.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/monoiga_b200.h"

#define MI_MAX_P 4
#define MI_MAX_CHAN 64

namespace mi {

void set_error(const std::string& msg);
int fail(const char* what, cudaError_t err);

#define MI_CUDA(call)                                                   \
  do {                                                                  \
    cudaError_t _e = (call);                                            \
    if (_e != cudaSuccess) return ::mi::fail(#call, _e);                \
  } while (0)

#define MI_CHECK_LAUNCH(name)                                           \
  do {                                                                  \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) return ::mi::fail(name, _e);                 \
  } while (0)

#define MI_REQUIRE(cond, code, msg)                                     \
  do {                                                                  \
    if (!(cond)) { ::mi::set_error(msg); return (code); }               \
  } while (0)

enum ProfSlot { PROF_OP_STENCIL = 0, PROF_OP_TFILTER, PROF_OP_REACTION, PROF_PC_SPATIAL, PROF_PC_TIME,
                PROF_PC_ARROW, PROF_KRYLOV, PROF_BUILD, PROF_NSLOTS };

// Records a CUDA event pair around the launches of one slot when profiling
// is on; always counts launches.
struct ProfScope {
  mi_ctx* c;
  int slot;
  cudaEvent_t e1 = nullptr;
  ProfScope(mi_ctx* ctx, int s, int nlaunch = 1);
  ~ProfScope();
};

// Makes the context's device current for one C-ABI call and restores the caller's device on return
// (every mi_* entry point that takes a context opens with MI_DEVICE_GUARD).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};
#define MI_DEVICE_GUARD(ctx) ::mi::DeviceGuard _mi_dev_guard((ctx) ? (ctx)->device : -1)

struct DeviceBuf {
  double* p = nullptr;
  size_t n = 0;
};

int dalloc(DeviceBuf& b, size_t n);
void dfree(DeviceBuf& b);

}  // namespace mi

struct mi_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int d = 1, p = 1, pt = 1;     // spatial dims, spatial degree, time degree
  int n[3] = {1, 1, 1};         // n_1, n_2, n_3 (1 beyond d)
  int nt = 0;                   // N_t (constrained)
  long long ns = 0, N = 0;      // N_s, N
  // z-slab (space-sharded runs, sharded.py): the points are the global planes [z_lo, z_lo + n[2]) of
  // n3g; operator inputs carry hz_lo / hz_hi halo planes before / after them.  Unsharded: z_lo = 0,
  // n3g = n[2], no halo, ns_in = ns.
  int z_lo = 0, n3g = 1, hz_lo = 0, hz_hi = 0;
  long long ns_in = 0, N_in = 0;  // operator input slab (owned + halo planes)

  // ---- operator A: channels c = 0..nchan-1, y = sum_c T_c (x)_t (S_c x)
  int nchan = 0;
  int nsten = 0;                // (2p+1)^d stencil points
  mi::DeviceBuf tband;          // nchan x nt x (2pt+1)
  mi::DeviceBuf stencil;        // nchan x nsten x ns
  mi::DeviceBuf wbuf;           // nchan x N  (S_c x per channel), fallback path only
  mi::DeviceBuf frag;           // fragment-major coefficients for the DMMA path
  mi::DeviceBuf xt;             // time-innermost copy of the operator input
  CUtensorMap tmap_xt;          // TMA descriptor of xt (DMMA path)
  CUtensorMap tmap_w;           // TMA descriptor of wbuf as (nchan*ns) rows x ntp times (time filter)
  mi::DeviceBuf afr;            // time-filter A fragments (DMMA path)
  int ntau = 0;
  bool op_ready = false;
  bool frag_dirty = true;
  bool stencil_released = false;  // mi_op_finalize freed `stencil` after packing it into `frag`
  bool use_dmma = false;
  int C[3] = {1, 1, 1};         // DMMA cube grid

  // ---- u0 lifting (initial data on the dropped first time function, DESIGN 7)
  bool lift_on = false;
  mi::DeviceBuf lift_u0;        // N_s_in lifting coefficients (input slab)
  mi::DeviceBuf lift_band;      // nchan x nt x (2pt+1): each channel's full-time column 0 as band entries
  mi::DeviceBuf lift_x;         // N_in scratch of mi_op_apply_lift

  // ---- reaction correction M_R (variant B)
  bool reaction_on = false;
  mi::DeviceBuf u_it, w_it;     // iterate coefficients (N_in each: input slab)
  mi::DeviceBuf y_in;           // reaction output on the input slab (z-slab contexts with a halo)
  double c1 = 0, a = 0, c2 = 0;
  mi::DeviceBuf rx_B, rx_W;     // Gauss tables, directions x, y, z, t
  size_t rx_Boff[4] = {0, 0, 0, 0}, rx_Woff[4] = {0, 0, 0, 0};
  int rx_rowoff = -1;          // constrained row of full time function ft = ft + rx_rowoff
  int rx_q[4] = {1, 1, 1, 1}, rx_p[4] = {0, 0, 0, 0}, rx_nel[4] = {1, 1, 1, 1}, rx_E[4] = {1, 1, 1, 1};
  mi::DeviceBuf rx_jw;          // mapped geometry: |det J| on the spatial Gauss grid (Q_d .. Q_1); empty = box
  bool rx_mapped = false;
  mi::DeviceBuf rx_cw;          // stored C_r x spatial weight at every Gauss point (reaction.cu RX_STORED)
  bool rx_cw_ok = false, rx_cw_dirty = true;
  bool rx_cw_ws = false;        // rx_cw is in reaction_ws's layout (else reaction_tile's)
  int rx_store_mode = -1;       // -1 auto (fits in 40% of free memory), 0 off, 1 on
  int rx_kernel = -1;           // fused mode: -1 auto (reaction_ws where it applies), 0 reaction_tile, 1 reaction_ws

  // ---- preconditioner
  bool pc_ready = false;
  mi::DeviceBuf Us[3], UsT[3];  // per direction n_l x n_l (U and U^T)
  int fold_hs[3] = {0, 0, 0};   // > 0: U_l is an exactly mirrored even/odd basis (mode_fold.cuh), hs symmetric modes first
  mi::DeviceBuf lam[3];         // per direction eigenvalues (already scaled by sigma_l)
  mi::DeviceBuf Q, QT;          // time basis nt x nt and transpose
  mi::DeviceBuf pen_diag, pen_off, pen_g, pen_glow;  // (nt-1)
  int* pen_partner = nullptr;   // (nt-1)
  double pen_sigma = 0, pc_cm = 1, pc_react = 0;
  mi::DeviceBuf pc_t1, pc_t2, pc_t3;   // N each
  mi::DeviceBuf tq_frag;        // fused time stage: Q^T and Q as fragment-major DMMA A operands
  int tq_mb = 0, tq_ksp = 0;    // row blocks (8 rows) and padded k-steps of the fused time stage (0 = unfused)

  // ---- recovery-variable solve (w-solve)
  bool ws_ready = false;
  mi::DeviceBuf ws_Kinv;        // (W_t + b d_e M_t)^{-1}, nt x nt
  mi::DeviceBuf ws_M[3], ws_Mi[3], ws_MT0, ws_MiT0;   // spatial mass factors, inverses (+ transposes, dir 1)
  mi::DeviceBuf ws_t1, ws_t2, ws_t3;

  // ---- SU residual indicator (compute_theta)
  bool th_ready = false;
  mi::DeviceBuf th_u0;          // lifting coefficients seen by the indicator (empty: no lifting)
  mi::DeviceBuf th_B0, th_B1;   // element tables, directions x, y, z, t (values; 2nd / 1st derivatives)
  size_t th_off[4] = {0, 0, 0, 0};
  int th_nel[4] = {1, 1, 1, 1};
  double th_il2[3] = {0, 0, 0};
  double th_cmT = 0, th_c1 = 0, th_a = 0, th_c2 = 0;
  int* th_win = nullptr;        // window tables of mi_window_max
  int th_nwin = 0;

  // ---- profiling: per-slot accumulated ms and launch counts
  bool prof_on = false;
  long long launches[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  struct EvRec { int slot; cudaEvent_t a, b; };
  std::vector<EvRec> prof_events;
  std::vector<cudaEvent_t> prof_pool;
  double prof_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};

  // ---- Krylov scratch
  mi::DeviceBuf partials;       // reduction partials

  // ---- host-input apply (mi_op_apply_from_host): H2D copy stream and per-chunk events
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> copy_events;
};
