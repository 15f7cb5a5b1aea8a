// Context lifetime, error reporting, device allocation.
#include "common.cuh"

#include <cstdio>

namespace mi {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(const char* what, cudaError_t err) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(err);
  return MI_ERR_CUDA;
}

int dalloc(DeviceBuf& b, size_t n) {
  if (b.p && b.n >= n) return MI_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.n = 0;
  if (n == 0) return MI_OK;
  cudaError_t e = cudaMalloc(&b.p, n * sizeof(double));
  if (e != cudaSuccess) {
    b.p = nullptr;
    char buf[128];
    snprintf(buf, sizeof(buf), "cudaMalloc(%zu doubles)", n);
    return fail(buf, e);
  }
  b.n = n;
  return MI_OK;
}

void dfree(DeviceBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.n = 0;
}

static cudaEvent_t take_event(mi_ctx* c) {
  if (!c->prof_pool.empty()) {
    cudaEvent_t e = c->prof_pool.back();
    c->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

ProfScope::ProfScope(mi_ctx* ctx, int s, int nlaunch) : c(ctx), slot(s) {
  c->launches[s] += nlaunch;
  if (c->prof_on) {
    e1 = take_event(c);
    cudaEventRecord(e1, c->stream);
  }
}

ProfScope::~ProfScope() {
  if (e1) {
    cudaEvent_t e2 = take_event(c);
    cudaEventRecord(e2, c->stream);
    c->prof_events.push_back({slot, e1, e2});
  }
}

DeviceGuard::DeviceGuard(int dev) {
  if (dev < 0) return;
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return;
  if (cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
}

DeviceGuard::~DeviceGuard() {
  if (prev >= 0) cudaSetDevice(prev);
}

}  // namespace mi

extern "C" {

int mi_prof_enable(mi_ctx* c, int on) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  c->prof_on = on != 0;
  return MI_OK;
}

int mi_prof_read(mi_ctx* c, double* ms, long long* launches, int reset) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  MI_CUDA(cudaStreamSynchronize(c->stream));
  for (auto& r : c->prof_events) {
    float t = 0.f;
    MI_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    c->prof_ms[r.slot] += t;
    c->prof_pool.push_back(r.a);
    c->prof_pool.push_back(r.b);
  }
  c->prof_events.clear();
  for (int s = 0; s < mi::PROF_NSLOTS; ++s) {
    if (ms) ms[s] = c->prof_ms[s];
    if (launches) launches[s] = c->launches[s];
    if (reset) {
      c->prof_ms[s] = 0;
      c->launches[s] = 0;
    }
  }
  return MI_OK;
}

int mi_version(void) { return 1; }

const char* mi_last_error(void) { return mi::g_last_error.c_str(); }

int mi_ctx_create(int device, int d, const int* n, int nt, int p, int pt, mi_ctx** out) {
  MI_REQUIRE(out != nullptr, MI_ERR_ARG, "out is NULL");
  MI_REQUIRE(d >= 1 && d <= 3, MI_ERR_ARG, "d must be 1, 2 or 3");
  MI_REQUIRE(p >= 1 && p <= MI_MAX_P, MI_ERR_ARG, "spatial degree must be in [1, 4]");
  MI_REQUIRE(pt >= 1 && pt <= MI_MAX_P, MI_ERR_ARG, "time degree must be in [1, 4]");
  MI_REQUIRE(nt >= 2, MI_ERR_ARG, "N_t must be >= 2");
  int ndev = 0;
  MI_CUDA(cudaGetDeviceCount(&ndev));
  MI_REQUIRE(device >= 0 && device < ndev, MI_ERR_ARG, "device ordinal out of range");
  mi::DeviceGuard guard(device);
  mi_ctx* c = new mi_ctx();
  c->device = device;
  c->d = d;
  c->p = p;
  c->pt = pt;
  c->nt = nt;
  long long ns = 1;
  for (int l = 0; l < 3; ++l) {
    c->n[l] = l < d ? n[l] : 1;
    if (c->n[l] < 1) {
      delete c;
      mi::set_error("spatial dimensions must be positive");
      return MI_ERR_ARG;
    }
    ns *= c->n[l];
  }
  c->ns = ns;
  c->N = ns * nt;
  c->n3g = c->n[2];
  c->ns_in = ns;
  c->N_in = c->N;
  int s = 1;
  for (int l = 0; l < d; ++l) s *= 2 * p + 1;
  c->nsten = s;
  int rc = mi::dalloc(c->partials, (size_t)1024 * 592);
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return MI_OK;
}

int mi_ctx_set_zslab(mi_ctx* c, int z_lo, int n3g, int hz_lo, int hz_hi) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  MI_REQUIRE(!c->op_ready, MI_ERR_STATE, "mi_ctx_set_zslab must precede mi_op_setup");
  MI_REQUIRE(c->d == 3, MI_ERR_ARG, "z-slab contexts need d = 3");
  MI_REQUIRE(z_lo >= 0 && z_lo + c->n[2] <= n3g, MI_ERR_ARG, "slab planes outside [0, n3g)");
  MI_REQUIRE(hz_lo >= 0 && hz_hi >= 0 && hz_lo <= c->p && hz_hi <= c->p, MI_ERR_ARG, "halo must be in [0, p]");
  MI_REQUIRE(z_lo - hz_lo >= 0 && z_lo + c->n[2] + hz_hi <= n3g, MI_ERR_ARG, "halo planes outside [0, n3g)");
  c->z_lo = z_lo;
  c->n3g = n3g;
  c->hz_lo = hz_lo;
  c->hz_hi = hz_hi;
  c->ns_in = (long long)c->n[0] * c->n[1] * (c->n[2] + hz_lo + hz_hi);
  c->N_in = c->ns_in * c->nt;
  return MI_OK;
}

int mi_ctx_destroy(mi_ctx* c) {
  MI_DEVICE_GUARD(c);
  if (!c) return MI_OK;
  mi::DeviceBuf* bufs[] = {&c->tband, &c->stencil, &c->wbuf, &c->frag, &c->xt, &c->afr, &c->u_it, &c->w_it, &c->rx_B,
                           &c->rx_W, &c->Q, &c->QT, &c->pen_diag, &c->pen_off,
                           &c->pen_g, &c->pen_glow, &c->pc_t1, &c->pc_t2, &c->pc_t3, &c->tq_frag, &c->y_in, &c->rx_jw, &c->rx_cw,
                           &c->partials, &c->lift_u0, &c->lift_band, &c->lift_x, &c->th_u0};
  for (auto* b : bufs) mi::dfree(*b);
  mi::DeviceBuf* wbufs[] = {&c->ws_Kinv, &c->ws_MT0, &c->ws_MiT0, &c->ws_t1, &c->ws_t2, &c->ws_t3,
                            &c->th_B0, &c->th_B1};
  for (auto* b : wbufs) mi::dfree(*b);
  for (int l = 0; l < 3; ++l) {
    mi::dfree(c->ws_M[l]);
    mi::dfree(c->ws_Mi[l]);
    mi::dfree(c->Us[l]);
    mi::dfree(c->UsT[l]);
    mi::dfree(c->lam[l]);
  }
  if (c->pen_partner) cudaFree(c->pen_partner);
  if (c->th_win) cudaFree(c->th_win);
  for (auto& r : c->prof_events) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->prof_pool) cudaEventDestroy(e);
  for (auto e : c->copy_events) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  delete c;
  return MI_OK;
}

int mi_ctx_set_stream(mi_ctx* c, void* stream) {
  MI_DEVICE_GUARD(c);
  MI_REQUIRE(c != nullptr, MI_ERR_ARG, "ctx is NULL");
  c->stream = static_cast<cudaStream_t>(stream);
  return MI_OK;
}

}  // extern "C"
