// lb_api.cu -- host runtime behind the C ABI of include/lb.h.
//
// Owns device memory, the CUDA stream, the halo transport (loopback copies or
// NCCL send/recv, "halo region populated using neighboring sub-domain
// data") and per-kernel CUDA-event timing.  One handle = one z-slab set on one
// GPU.  See DESIGN.md "Boundary" and "Multi-GPU".
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lb.h"
#include "lb_kernels.cuh"

using namespace lbk;

namespace {

thread_local std::string g_create_error;

enum KernelId { K_PHI = 0, K_STEP, K_INIT, K_PERMUTE, K_HALO_DIST, K_HALO_PHI, K_COUNT };
const char* const kKernelNames[K_COUNT] = {"k_phi", "k_step", "k_init_eq", "k_permute", "halo_dist", "halo_phi"};

struct Slab {
  int z0 = 0;  // global z of local plane 0
  double* A = nullptr;  // current state (pre-collision f, g)
  double* B = nullptr;  // next state / staging
  double* phi = nullptr;
  double* phi2 = nullptr;  // finite-difference Cahn-Hilliard handles: next phi
  ChMaps chA{}, chB{};     // and the TMA descriptors of their f box
  // liquid-crystal handles (NEXT-4): Q (5 components) and the stored velocity u
  // (3), current and next, plane-major [z][component][y][x]; f tile maps (32 x 8)
  double* q = nullptr;
  double* q2 = nullptr;
  double* u = nullptr;
  double* u2 = nullptr;
  StepMaps lcA{}, lcB{};
  StepMaps mapsA{}, mapsB{};        // TMA descriptors of A and B (swapped with them)
  unsigned long long* sync = nullptr;  // SW_WORDS sync words of the peer transport (slabs only)
};

struct Pending {
  int kid;
  cudaEvent_t e0, e1;
};

}  // namespace

struct lb_ctx {
  int nx = 0, ny = 0, nz = 0;
  int nzl = 0;            // planes per slab
  int nranks = 1, rank = 0;
  int nslabs = 1;         // slabs held by this handle (loopback > 1)
  lb_params prm{};
  DevParams dp{};
  Geom G{};
  std::vector<Slab> slabs;
  cudaStream_t stream = nullptr;
  int device = 0;
  int num_sms = 148;
  int zc = 1;             // z-chunk of the step kernel
  int ty = 8;             // tile rows of the step kernel
  TileOrder order{0, 1};  // block order of the step kernels (0: the kernel's occupancy)
  L2Pol l2{};             // L2 policies of the warp-specialised kernel's copies
  bool graphs_on = true;  // lb_debug_tune(LB_TUNE_GRAPHS)
  int variant = 0;        // lb_debug_tune(LB_TUNE_VARIANT): a kernel-internal alternative, for A/B
  bool ch = false;        // NEXT-2 handle: state (f, phi), lb_create_ch
  bool lc = false;        // NEXT-4 handle: state (f, Q, u), lb_create_lc
  int lczc = 1;           // z-chunk of the liquid-crystal step kernel
  int kernel_choice = 0;  // 0 default, 1 tile, 2 warp-specialised, 3 warp-specialised with the phi exchange
  double* xphi[2] = {nullptr, nullptr};  // phi exchange of the warp-specialised kernel (nx*ny*nzl), single slab
  bool xch_default = false;               // kernel 0 uses it (all blocks in one wave)
  bool xch_dirty = false;                 // a step since the last one that used it: refill before the next
  // R22 health words (device): [0] first offending (step << 40 | site), ~0 = clean;
  // [1] steps completed by the step kernels; d_done: CTAs finished in a launch
  unsigned long long* d_health = nullptr;
  unsigned* d_done = nullptr;
  int* d_check = nullptr;  // LB_CHECKED builds: first failed device bounds check
  unsigned long long* h_health = nullptr;  // pinned copy of d_health[0]
  long long steps_done = 0;                // host mirror of d_health[1]
  ncclComm_t comm = nullptr;
  // halo transport: 0 = exchange (ghost planes + copies / NCCL send-recv after the
  // kernels), 1 = peer (fused: the kernels store into the neighbours' buffers)
  int halo_mode = 0;
  // peer transport between ranks: the neighbours' A, B and phi buffers mapped by
  // CUDA IPC ([0] = slab below, [1] = slab above; the same mapping when nranks == 2)
  double* peerA[2] = {nullptr, nullptr};
  double* peerB[2] = {nullptr, nullptr};
  double* peerPhi[2] = {nullptr, nullptr};
  unsigned long long* peerSync[2] = {nullptr, nullptr};  // the neighbours' sync words
  std::vector<void*> ipc_opened;
  double* d_token = nullptr;  // 4 doubles: NCCL barrier tokens
  // external bootstrap (lb_create_slab_ext): the caller's all-gather, no NCCL
  lb_allgather_fn allgather = nullptr;
  void* allgather_ctx = nullptr;
  unsigned long long* h_sync = nullptr;  // pinned: SW_ERR of each slab, read by finish()
  std::vector<std::pair<double*, size_t>> guarded;  // buffers with guard zones (dev_alloc)
  bool have_state = false;
  bool broken = false;
  // CUDA graphs of kGraphSteps steps (single process, no per-launch profiling): one
  // per parity of the A/B buffers, keyed by the state buffer at capture; dropped by
  // every call that changes what a step launches
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    const double* A = nullptr;
    long long launches = 0;  // kernels per replay
    long long steps = 0;     // steps per replay
    bool dirty_after = true;  // xch_dirty after a replay
  } graphs[2];
  std::string err;
  long long launches = 0;
  // profiling
  bool prof_on = false;
  double prof_ms[K_COUNT] = {0};
  long long prof_n[K_COUNT] = {0};
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> ev_pool;
};

namespace {

int set_err(lb_ctx* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) {
    h->err = buf;
    if (code == LB_ECUDA || code == LB_ENCCL) h->broken = true;
  } else {
    g_create_error = buf;
  }
  return code;
}

#define CK(h, call)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return set_err((h), e_ == cudaErrorMemoryAllocation ? LB_ENOMEM : LB_ECUDA, "%s: %s (%s:%d)", #call, \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                            \
  } while (0)

#define NK(h, call)                                                                                 \
  do {                                                                                              \
    ncclResult_t r_ = (call);                                                                       \
    if (r_ != ncclSuccess)                                                                          \
      return set_err((h), LB_ENCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

bool finite(double v) { return std::isfinite(v); }

int check_params(const lb_params* p) {
  if (!p) return set_err(nullptr, LB_EINVAL, "params is NULL");
  if (!finite(p->tau_f) || !(p->tau_f > 0.5)) return set_err(nullptr, LB_EINVAL, "tau_f must be finite and > 0.5");
  if (!finite(p->tau_g) || !(p->tau_g > 0.5)) return set_err(nullptr, LB_EINVAL, "tau_g must be finite and > 0.5");
  if (!finite(p->A) || !finite(p->B)) return set_err(nullptr, LB_EINVAL, "A and B must be finite");
  if (!finite(p->kappa) || p->kappa < 0) return set_err(nullptr, LB_EINVAL, "kappa must be finite and >= 0");
  if (!finite(p->mobility) || p->mobility < 0) return set_err(nullptr, LB_EINVAL, "mobility must be finite and >= 0");
  return LB_OK;
}

DevParams derive(const lb_params& p) {
  DevParams d;
  d.A = p.A;
  d.B = p.B;
  d.kappa = p.kappa;
  d.inv_tau_f = 1.0 / p.tau_f;
  d.inv_tau_g = 1.0 / p.tau_g;
  d.guo_pref = 1.0 - 1.0 / (2.0 * p.tau_f);
  d.gamma = p.mobility / (p.tau_g - 0.5);
  d.coll = 0;
  d.inv_tau_s = d.inv_tau_b = d.inv_tau_ghost = d.inv_tau_f;
  d.mob = p.mobility;
  return d;
}

size_t dist_doubles(const Geom& G) { return (size_t)(G.nzl + 2 * GZ) * (size_t)G.plane; }
size_t phi_doubles(const Geom& G) { return (size_t)(G.nzl + 2 * GP) * (size_t)G.nxy; }
// liquid-crystal fields, plane-major [z][c][y][x] with ghost planes: Q (5 components,
// 2 ghost planes each side: the stress at z +- 1 needs Q at z +- 2), u (3, one)
constexpr int LC_GQ = 2, LC_GU = 1;
size_t lc_q_doubles(const Geom& G) { return (size_t)(G.nzl + 2 * LC_GQ) * 5 * (size_t)G.nxy; }
size_t lc_u_doubles(const Geom& G) { return (size_t)(G.nzl + 2 * LC_GU) * 3 * (size_t)G.nxy; }
double* lc_q0(const Geom& G, double* q) { return q + (size_t)LC_GQ * 5 * G.nxy; }  // plane 0
double* lc_u0(const Geom& G, double* u) { return u + (size_t)LC_GU * 3 * G.nxy; }
int exchange_lc(lb_ctx* h);  // Q / u halos of the liquid-crystal slabs (defined with the LC calls)
int exchange_fedge(lb_ctx* h);  // f edge planes of the Cahn-Hilliard slabs (defined with lb_create_ch)

// ---- profiling -------------------------------------------------------------
template <class Fn>
cudaError_t timed(lb_ctx* h, int kid, bool is_kernel, Fn&& fn) {
  if (!h->prof_on) {
    cudaError_t e = fn();
    if (is_kernel) ++h->launches;
    return e;
  }
  cudaEvent_t ev[2];
  for (int k = 0; k < 2; ++k) {
    if (h->ev_pool.empty()) {
      cudaError_t e = cudaEventCreate(&ev[k]);
      if (e != cudaSuccess) return e;
    } else {
      ev[k] = h->ev_pool.back();
      h->ev_pool.pop_back();
    }
  }
  cudaEventRecord(ev[0], h->stream);
  cudaError_t e = fn();
  cudaEventRecord(ev[1], h->stream);
  h->pending.push_back({kid, ev[0], ev[1]});
  if (is_kernel) ++h->launches;
  return e;
}

// after a stream sync: fold pending event pairs into the totals
void resolve_pending(lb_ctx* h) {
  for (auto& p : h->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.e0, p.e1) == cudaSuccess) {
      h->prof_ms[p.kid] += ms;
      h->prof_n[p.kid] += 1;
    }
    h->ev_pool.push_back(p.e0);
    h->ev_pool.push_back(p.e1);
  }
  h->pending.clear();
}

// ---- allocation ------------------------------------------------------------
// Every field buffer carries guard zones of kGuardBytes on both sides, filled
// with kGuardByte: lb_debug_guards finds any store that left its buffer (the
// out-of-bounds half of a memory checker, which this pool has no tool for).
constexpr size_t kGuardBytes = 64 * 1024;
constexpr unsigned char kGuardByte = 0xA5;

cudaError_t dev_alloc(lb_ctx* h, double** p, size_t bytes) {
  unsigned char* raw = nullptr;
  cudaError_t e = cudaMalloc(&raw, bytes + 2 * kGuardBytes);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(raw, kGuardByte, kGuardBytes, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(raw + kGuardBytes + bytes, kGuardByte, kGuardBytes, h->stream);
  *p = reinterpret_cast<double*>(raw + kGuardBytes);
  h->guarded.push_back({*p, bytes});
  return e;
}
void* raw_of(const void* p) { return p ? (void*)(static_cast<const unsigned char*>(p) - kGuardBytes) : nullptr; }
void dev_free(double* p) {
  if (p) cudaFree(raw_of(p));
}

// the two phi arrays of the phi-exchange kernel (kernel 5), filled with kXchEmpty
int ensure_xch(lb_ctx* h) {
  if (h->xphi[0]) return LB_OK;
  const long long n = h->G.nxy * h->G.nzl;
  for (int k = 0; k < 2; ++k) {
    CK(h, dev_alloc(h, &h->xphi[k], (size_t)n * sizeof(double)));
    CK(h, fill_xch_empty(h->xphi[k], n, h->stream));
  }
  h->xch_dirty = false;
  return LB_OK;
}

// A step without the phi exchange leaves the array of the next exchange step
// unreset (stale phi would pass for fresh): refill both before it.
int refresh_xch(lb_ctx* h) {
  if (!h->xphi[0] || !h->xch_dirty) return LB_OK;
  const long long n = h->G.nxy * h->G.nzl;
  for (int k = 0; k < 2; ++k) CK(h, fill_xch_empty(h->xphi[k], n, h->stream));
  h->xch_dirty = false;
  return LB_OK;
}

// the phi-exchange step kernel is the default where its blocks run in one wave
// (over several waves neighbouring tiles drift apart)
void choose_xch(lb_ctx* h) {
  h->xch_default = h->nslabs == 1 && step_xch_fits(h->G, &h->slabs[0].mapsA) && h->kernel_choice == 0 &&
                   ws_xch_blocks(h->G, h->zc) <= h->num_sms;
}

int alloc_slabs(lb_ctx* h) {
  h->slabs.resize(h->nslabs);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    s.z0 = (h->rank * h->nslabs + r) * h->nzl;
    CK(h, dev_alloc(h, &s.A, dist_doubles(h->G) * sizeof(double)));
    CK(h, dev_alloc(h, &s.B, dist_doubles(h->G) * sizeof(double)));
    CK(h, dev_alloc(h, &s.phi, phi_doubles(h->G) * sizeof(double)));
    // NaN-fill: a read of a plane nobody wrote shows up as a parity failure
    CK(h, cudaMemsetAsync(s.A, 0xff, dist_doubles(h->G) * sizeof(double), h->stream));
    CK(h, cudaMemsetAsync(s.B, 0xff, dist_doubles(h->G) * sizeof(double), h->stream));
    CK(h, cudaMemsetAsync(s.phi, 0xff, phi_doubles(h->G) * sizeof(double), h->stream));
    if (!make_step_maps(h->G, s.A, h->ty, &s.mapsA) || !make_step_maps(h->G, s.B, h->ty, &s.mapsB))
      return set_err(h, LB_ECUDA, "cuTensorMapEncodeTiled failed for the step kernel's TMA descriptors");
  }
  choose_xch(h);
  if (!h->G.zwrap) {  // sync words of the peer transport, one set per slab
    for (auto& s : h->slabs) {
      CK(h, cudaMalloc(&s.sync, SW_WORDS * sizeof(unsigned long long)));
      CK(h, cudaMemsetAsync(s.sync, 0, SW_WORDS * sizeof(unsigned long long), h->stream));
    }
    CK(h, cudaMallocHost(&h->h_sync, h->nslabs * sizeof(unsigned long long)));
  }
  CK(h, cudaMalloc(&h->d_health, 2 * sizeof(unsigned long long)));
  CK(h, cudaMemsetAsync(h->d_health, 0xff, sizeof(unsigned long long), h->stream));
  CK(h, cudaMemsetAsync(h->d_health + 1, 0, sizeof(unsigned long long), h->stream));
  CK(h, cudaMalloc(&h->d_done, sizeof(unsigned)));
  CK(h, cudaMemsetAsync(h->d_done, 0, sizeof(unsigned), h->stream));
  CK(h, cudaMalloc(&h->d_check, sizeof(int)));
  CK(h, cudaMemsetAsync(h->d_check, 0, sizeof(int), h->stream));
  CK(h, cudaMallocHost(&h->h_health, sizeof(unsigned long long)));
  CK(h, cudaStreamSynchronize(h->stream));
  return LB_OK;
}

// health words of slab r's launch in a step: only the last launch of a step ticks
Health health_of(const lb_ctx* h, int r, bool tick) {
  Health hl;
  hl.flag = h->d_health;
  hl.step = h->d_health + 1;
  hl.done = tick ? h->d_done : nullptr;
  hl.site0 = (long long)h->slabs[r].z0 * h->G.nxy;
  hl.check = h->d_check;
  return hl;
}

Launch launch_of(const lb_ctx* h) {
  Launch ln;
  ln.zc = h->zc;
  ln.order = h->order;
  ln.order.edge_last = h->halo_mode == 1 && !h->G.zwrap;
  ln.l2 = h->l2;
  return ln;
}

int create_common(int nx, int ny, int nz, const lb_params* params, int nranks, int rank, int nslabs, lb_t** out) {
  if (!out) return set_err(nullptr, LB_EINVAL, "out is NULL");
  *out = nullptr;
  int rc = check_params(params);
  if (rc) return rc;
  if (nx < 3 || ny < 3 || nz < 3) return set_err(nullptr, LB_EINVAL, "extents must be >= 3 (got %d x %d x %d)", nx, ny, nz);
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_err(nullptr, LB_EINVAL, "bad rank %d of %d", rank, nranks);
  if (nslabs < 1) return set_err(nullptr, LB_EINVAL, "nslabs must be >= 1");
  const int parts = nranks * nslabs;
  if (nz % parts != 0) return set_err(nullptr, LB_EINVAL, "nz = %d is not divisible by %d slabs", nz, parts);
  if (parts > 1 && nz / parts < 2) return set_err(nullptr, LB_EINVAL, "a slab needs >= 2 planes (nz/slabs = %d)", nz / parts);
  if ((long long)nx * ny > (1LL << 31)) return set_err(nullptr, LB_EINVAL, "nx*ny too large");

  lb_ctx* h = new lb_ctx;
  h->nx = nx;
  h->ny = ny;
  h->nz = nz;
  h->nranks = nranks;
  h->rank = rank;
  h->nslabs = nslabs;
  h->nzl = nz / parts;
  h->prm = *params;
  h->dp = derive(*params);
  h->G.nx = nx;
  h->G.ny = ny;
  h->G.nzl = h->nzl;
  h->G.zwrap = parts == 1 ? 1 : 0;
  h->G.nxy = (long long)nx * ny;
  h->G.plane = (long long)NSLOT * h->G.nxy;
  cudaError_t e = cudaGetDevice(&h->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    set_err(nullptr, LB_ECUDA, "CUDA init failed: %s", cudaGetErrorString(e));
    delete h;
    return LB_ECUDA;
  }
  h->halo_mode = (parts > 1 && nranks == 1) ? 1 : 0;  // ranks: after the IPC setup
  h->ty = step_tile_rows(h->G, h->num_sms);
  h->zc = step_zchunk(h->G, h->num_sms, h->ty);
  // every step kernel's per-device preparation now, never inside a graph capture
  e = prepare_step_kernels();
  if (e == cudaSuccess) e = prepare_ws_kernels();
  if (e == cudaSuccess) e = prepare_ch_kernels();
  if (e == cudaSuccess) e = prepare_lc_kernels();
  if (e != cudaSuccess) {
    set_err(nullptr, LB_ECUDA, "kernel preparation failed: %s", cudaGetErrorString(e));
    cudaStreamDestroy(h->stream);
    delete h;
    return LB_ECUDA;
  }
  rc = alloc_slabs(h);
  if (rc) {
    g_create_error = h->err;
    lb_destroy(h);
    return rc;
  }
  *out = h;
  return LB_OK;
}

int usable(lb_ctx* h) {
  if (!h) return set_err(nullptr, LB_EINVAL, "handle is NULL");
  if (h->broken) return set_err(h, LB_ECUDA, "handle unusable after an earlier CUDA/NCCL failure: %s", h->err.c_str());
  return LB_OK;
}

// ---- halo transport ---------------------------------------------------------
// Distribution halo after a step, on buffer B of every slab:
//   ghost plane nzl (cz=+1 run, slots [0,10)) -> plane 0 of the slab above, same slots
//   ghost plane -1  (cz=-1 run, slots [28,38)) -> plane nzl-1 of the slab below
// phi halo before a step:
//   planes [nzl-2, nzl) -> ghost planes [-2, 0) of the slab above
//   planes [0, 2)       -> ghost planes [nzl, nzl+2) of the slab below
int exchange_dist(lb_ctx* h) {
  const Geom& G = h->G;
  const size_t cnt = (size_t)HALO_COMPS * G.nxy;
  if (h->nranks > 1) {
    Slab& s = h->slabs[0];
    const int up = (h->rank + 1) % h->nranks, dn = (h->rank - 1 + h->nranks) % h->nranks;
    cudaError_t ce = timed(h, K_HALO_DIST, false, [&]() {
      ncclGroupStart();
      ncclSend(s.B + dist_index(G, G.nzl, SLOT_UP_FIRST, 0), cnt, ncclDouble, up, h->comm, h->stream);
      ncclRecv(s.B + dist_index(G, 0, SLOT_UP_FIRST, 0), cnt, ncclDouble, dn, h->comm, h->stream);
      ncclSend(s.B + dist_index(G, -1, SLOT_DOWN_FIRST, 0), cnt, ncclDouble, dn, h->comm, h->stream);
      ncclRecv(s.B + dist_index(G, G.nzl - 1, SLOT_DOWN_FIRST, 0), cnt, ncclDouble, up, h->comm, h->stream);
      return ncclGroupEnd() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
    });
    if (ce != cudaSuccess) return set_err(h, LB_ENCCL, "NCCL distribution halo exchange failed");
    return LB_OK;
  }
  if (h->nslabs == 1) return LB_OK;  // periodic single slab: kernels wrap
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    Slab& up = h->slabs[(r + 1) % h->nslabs];
    Slab& dn = h->slabs[(r - 1 + h->nslabs) % h->nslabs];
    CK(h, timed(h, K_HALO_DIST, false, [&]() {
      cudaError_t e = cudaMemcpyAsync(up.B + dist_index(G, 0, SLOT_UP_FIRST, 0), s.B + dist_index(G, G.nzl, SLOT_UP_FIRST, 0),
                                      cnt * sizeof(double), cudaMemcpyDeviceToDevice, h->stream);
      if (e != cudaSuccess) return e;
      return cudaMemcpyAsync(dn.B + dist_index(G, G.nzl - 1, SLOT_DOWN_FIRST, 0), s.B + dist_index(G, -1, SLOT_DOWN_FIRST, 0),
                             cnt * sizeof(double), cudaMemcpyDeviceToDevice, h->stream);
    }));
  }
  return LB_OK;
}

int halo_barrier(lb_ctx* h, int kid);

int exchange_phi(lb_ctx* h) {
  const Geom& G = h->G;
  const size_t cnt = (size_t)2 * G.nxy;
  if (h->nranks > 1 && !h->comm) {  // external bootstrap: copies into the mapped neighbours' ghost planes
    if (!h->peerPhi[0] || !h->peerPhi[1]) return set_err(h, LB_EINVAL, "no halo transport on this handle");
    Slab& s = h->slabs[0];
    int rc = halo_barrier(h, K_HALO_PHI);  // every rank's phi planes are in place
    if (rc) return rc;
    CK(h, cudaMemcpyAsync(h->peerPhi[1] + phi_plane_index(G, -2), s.phi + phi_plane_index(G, G.nzl - 2),
                          cnt * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    CK(h, cudaMemcpyAsync(h->peerPhi[0] + phi_plane_index(G, G.nzl), s.phi + phi_plane_index(G, 0),
                          cnt * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    return halo_barrier(h, K_HALO_PHI);  // (stream synchronised first) every rank's copies have landed
  }
  if (h->nranks > 1) {
    Slab& s = h->slabs[0];
    const int up = (h->rank + 1) % h->nranks, dn = (h->rank - 1 + h->nranks) % h->nranks;
    cudaError_t ce = timed(h, K_HALO_PHI, false, [&]() {
      ncclGroupStart();
      ncclSend(s.phi + phi_plane_index(G, G.nzl - 2), cnt, ncclDouble, up, h->comm, h->stream);
      ncclRecv(s.phi + phi_plane_index(G, -2), cnt, ncclDouble, dn, h->comm, h->stream);
      ncclSend(s.phi + phi_plane_index(G, 0), cnt, ncclDouble, dn, h->comm, h->stream);
      ncclRecv(s.phi + phi_plane_index(G, G.nzl), cnt, ncclDouble, up, h->comm, h->stream);
      return ncclGroupEnd() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
    });
    if (ce != cudaSuccess) return set_err(h, LB_ENCCL, "NCCL phi halo exchange failed");
    return LB_OK;
  }
  if (h->nslabs == 1) return LB_OK;
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    Slab& up = h->slabs[(r + 1) % h->nslabs];
    Slab& dn = h->slabs[(r - 1 + h->nslabs) % h->nslabs];
    CK(h, timed(h, K_HALO_PHI, false, [&]() {
      cudaError_t e = cudaMemcpyAsync(up.phi + phi_plane_index(G, -2), s.phi + phi_plane_index(G, G.nzl - 2),
                                      cnt * sizeof(double), cudaMemcpyDeviceToDevice, h->stream);
      if (e != cudaSuccess) return e;
      return cudaMemcpyAsync(dn.phi + phi_plane_index(G, G.nzl), s.phi + phi_plane_index(G, 0), cnt * sizeof(double),
                             cudaMemcpyDeviceToDevice, h->stream);
    }));
  }
  return LB_OK;
}

// ---- fused halo (peer transport) ----------------------------------------------
// Neighbour buffers of slab r: other slabs of this handle (loopback) or the IPC
// mappings of the neighbouring ranks' buffers.
Peers peers_of(const lb_ctx* h, int r) {
  Peers P;
  if (h->halo_mode != 1 || h->G.zwrap) return P;
  if (h->nranks > 1) {
    P.dn = h->peerB[0];
    P.up = h->peerB[1];
    P.phi_dn = h->peerPhi[0];
    P.phi_up = h->peerPhi[1];
    P.sync = h->slabs[0].sync;
    P.sync_dn = h->peerSync[0];
    P.sync_up = h->peerSync[1];
  } else {
    const Slab& dn = h->slabs[(r - 1 + h->nslabs) % h->nslabs];
    const Slab& up = h->slabs[(r + 1) % h->nslabs];
    P.dn = dn.B;
    P.up = up.B;
    P.phi_dn = dn.phi;
    P.phi_up = up.phi;
    P.sync = h->slabs[r].sync;
    P.sync_dn = dn.sync;
    P.sync_up = up.sync;
  }
  return P;
}

// Ordering point of the peer transport between ranks: a one-double NCCL send/recv
// with both neighbours on the stream.  A neighbour's send is issued after its
// kernel (which ended with __threadfence_system), so once both receives have
// completed, every P2P store the neighbours made into this rank's buffers is
// visible to the kernels that follow.  Loopback slabs share one stream: no-op.
int halo_barrier(lb_ctx* h, int kid) {
  if (h->nranks == 1) return LB_OK;
  if (h->allgather) {  // external bootstrap: the device work so far, then the caller's all-gather as a barrier
    CK(h, cudaStreamSynchronize(h->stream));
    const char mine = 1;
    std::vector<char> all(h->nranks);
    if (h->allgather(h->allgather_ctx, &mine, all.data(), 1) != 0) return set_err(h, LB_ENCCL, "the caller's all-gather failed");
    return LB_OK;
  }
  const int up = (h->rank + 1) % h->nranks, dn = (h->rank - 1 + h->nranks) % h->nranks;
  cudaError_t ce = timed(h, kid, false, [&]() {
    ncclGroupStart();
    ncclSend(h->d_token, 1, ncclDouble, up, h->comm, h->stream);
    ncclRecv(h->d_token + 1, 1, ncclDouble, dn, h->comm, h->stream);
    ncclSend(h->d_token, 1, ncclDouble, dn, h->comm, h->stream);
    ncclRecv(h->d_token + 2, 1, ncclDouble, up, h->comm, h->stream);
    return ncclGroupEnd() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
  });
  if (ce != cudaSuccess) return set_err(h, LB_ENCCL, "NCCL halo barrier failed");
  return LB_OK;
}

// The host side of the end of a step: the next state becomes the current one (the
// A/B buffers and their TMA maps; phi / Q / u fields of the Cahn-Hilliard and
// liquid-crystal handles; the mapped neighbour buffers, which swap in lockstep).
// fields = false: only the distributions (propagation only).
void swap_roles(lb_ctx* h, bool fields = true) {
  for (auto& s : h->slabs) {
    std::swap(s.A, s.B);
    std::swap(s.mapsA, s.mapsB);
    if (h->lc && fields) {
      std::swap(s.lcA, s.lcB);
      std::swap(s.q, s.q2);
      std::swap(s.u, s.u2);
    }
    if (h->ch && fields) {
      std::swap(s.chA, s.chB);
      std::swap(s.phi, s.phi2);
    }
  }
  for (int k = 0; k < 2; ++k) std::swap(h->peerA[k], h->peerB[k]);
}

// The step kernel of the binary fluid on one slab.  Default: the warp-specialised
// kernel for 32 x 8 tiles (large planes), the tile kernel for 32 x 4 tiles (two
// CTAs per SM) and odd nx; the phi exchange where all blocks
// run in one wave.
cudaError_t launch_bgk_step(lb_ctx* h, Slab& s, const Launch& ln, const Health& hl, const Peers& pr) {
  const Geom& G = h->G;
  const bool ws = step_ws_fits(&s.mapsA) && (h->kernel_choice >= 2 || (h->kernel_choice == 0 && s.mapsA.ty == 8));
  // (MRT launches the plain kernel, which leaves the exchange arrays alone: the
  // step must count as one without the exchange, or the next exchange step would
  // read the phi of two steps ago where an owner runs behind)
  const bool xch = ws && h->xphi[0] && h->dp.coll == 0 &&
                   (h->kernel_choice == 3 || (h->kernel_choice == 0 && h->xch_default)) && step_xch_fits(G, &s.mapsA);
  h->xch_dirty = !xch;
  if (xch) {  // the two phi buffers alternate with the A/B roles of the state buffers
    const int k = s.A < s.B ? 0 : 1;
    const XchArgs xa{h->xphi[k], h->xphi[1 - k], G.nxy * G.nzl <= (1LL << 20) ? 2 : 1};
    return launch_step_ws(G, h->dp, s.A, s.B, s.phi, ln, hl, &s.mapsA, h->stream, pr, &xa);
  }
  if (ws) return launch_step_ws(G, h->dp, s.A, s.B, s.phi, ln, hl, &s.mapsA, h->stream, pr);
  return launch_step(G, h->dp, s.A, s.B, s.phi, ln, hl, &s.mapsA, h->stream, pr);
}

// one timestep on every slab.  Single periodic slab: the fused step alone.
// Slabs: phi on the two edge planes at each end (K_phi), phi halo exchange, the
// fused step (A -> B), distribution halo exchange, swap.
// stream_only: propagation only (k_stream, lb_debug_stream)
int one_step(lb_ctx* h, bool stream_only = false) {
  const Geom& G = h->G;
  int rc;
  h->xch_dirty = true;  // until a phi-exchange launch below says otherwise
  const bool peer = h->halo_mode == 1 && !G.zwrap;
  const int last = h->nslabs - 1;
  if (h->lc && !stream_only) {  // Q, u halos; the step; f halo (the components that left each slab)
    if (!G.zwrap && (rc = exchange_lc(h))) return rc;
    for (int r = 0; r < h->nslabs; ++r) {
      Slab& s = h->slabs[r];
      CK(h, timed(h, K_STEP, true, [&]() {
           return launch_step_lc(G, h->dp, s.A, s.B, lc_q0(G, s.q), lc_q0(G, s.q2), lc_u0(G, s.u), lc_u0(G, s.u2),
                                 h->lczc, health_of(h, r, r == last), &s.lcA, h->stream);
         }));
    }
    if (!G.zwrap && (rc = exchange_dist(h))) return rc;
    swap_roles(h);
    ++h->steps_done;
    return LB_OK;
  }
  if (h->ch && !stream_only) {  // f edge planes and phi halos; the step; f halo
    if (!G.zwrap && ((rc = exchange_fedge(h)) || (rc = exchange_phi(h)))) return rc;
    for (int r = 0; r < h->nslabs; ++r) {
      Slab& s = h->slabs[r];
      CK(h, timed(h, K_STEP, true, [&]() {
           return launch_step_ch(G, h->dp, s.A, s.B, s.phi, s.phi2, h->zc, health_of(h, r, r == last), &s.chA,
                                 h->stream, h->kernel_choice != 1, h->variant);
         }));
    }
    if (!G.zwrap && (rc = exchange_dist(h))) return rc;
    swap_roles(h);
    ++h->steps_done;
    return LB_OK;
  }
  if (stream_only) {
    for (int r = 0; r < h->nslabs; ++r) {
      Slab& s = h->slabs[r];
      const Peers pr = peers_of(h, r);
      CK(h, timed(h, K_STEP, true, [&]() { return launch_stream(G, s.A, s.B, h->stream, pr); }));
    }
  } else {
    if (!G.zwrap) {
      for (int r = 0; r < h->nslabs; ++r) {
        Slab& s = h->slabs[r];
        const Peers pr = peers_of(h, r);
        if (peer) {  // edge phi into the neighbours' ghost planes, ordered by the sync words (NEXT-1)
          CK(h, timed(h, K_PHI, true, [&]() { return launch_phi_edges(G, s.A, s.phi, h->stream, pr); }));
          h->launches += 2;  // (the one-thread wait and publication around it)
        } else {
          CK(h, timed(h, K_PHI, true, [&]() { return launch_phi(G, s.A, s.phi, 0, 2, h->stream); }));
          CK(h, timed(h, K_PHI, true, [&]() { return launch_phi(G, s.A, s.phi, G.nzl - 2, G.nzl, h->stream); }));
        }
      }
      if (!peer && (rc = exchange_phi(h))) return rc;
    }
    const Launch ln = launch_of(h);
    for (int r = 0; r < h->nslabs; ++r) {
      Slab& s = h->slabs[r];
      const Peers pr = peers_of(h, r);
      const Health hl = health_of(h, r, r == last);
      CK(h, timed(h, K_STEP, true, [&]() { return launch_bgk_step(h, s, ln, hl, pr); }));
      if (peer && pr.sync) {  // the push epoch of this slab, after its step kernel
        CK(h, launch_publish_push(pr, h->stream));
        ++h->launches;
      }
    }
  }
  // peer transport: the step kernels published their pushes (device-side); only
  // propagation-only steps between ranks (test support) order by a host barrier
  if ((rc = peer ? (stream_only ? halo_barrier(h, K_HALO_DIST) : LB_OK) : exchange_dist(h))) return rc;
  swap_roles(h, !stream_only);
  if (!stream_only) ++h->steps_done;
  return LB_OK;
}

// ---- CUDA graphs of the step loop ---------------------------------------------
constexpr int kGraphSteps = 8;  // even: a replay returns the A/B buffers to their roles

void drop_graphs(lb_ctx* h) {
  for (auto& g : h->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g = lb_ctx::StepGraph{};
  }
}

// Anything that changes what a step launches: the graphs go (every kernel was
// prepared at lb_create, so a new one's first launch may be captured).
void steps_changed(lb_ctx* h) { drop_graphs(h); }

bool graphs_usable(const lb_ctx* h) {
  // ranks: with the peer transport a step is kernels only (device-side ordering);
  // the NCCL exchange transport stays outside graphs
  return h->graphs_on && (h->nranks == 1 || h->halo_mode == 1) && !h->prof_on;
}

// Everything one_step changes on the host: restored if a capture fails half way.
struct HostStepState {
  std::vector<Slab> slabs;
  double* peerA[2];
  double* peerB[2];
  bool xch_dirty;
  long long steps_done;
};
HostStepState save_state(const lb_ctx* h) {
  HostStepState st{h->slabs, {h->peerA[0], h->peerA[1]}, {h->peerB[0], h->peerB[1]}, h->xch_dirty, h->steps_done};
  return st;
}
void restore_state(lb_ctx* h, const HostStepState& st) {
  h->slabs = st.slabs;
  for (int k = 0; k < 2; ++k) h->peerA[k] = st.peerA[k], h->peerB[k] = st.peerB[k];
  h->xch_dirty = st.xch_dirty;
  h->steps_done = st.steps_done;
}

// Capture kGraphSteps steps from the current buffer roles into a graph slot (the
// host state is restored afterwards: capturing runs nothing).  Returns the slot,
// or nullptr when no graph could be made (the caller steps plainly).
lb_ctx::StepGraph* capture_graph(lb_ctx* h) {
  const double* A = h->slabs[0].A;
  for (auto& c : h->graphs)
    if (c.exec && c.A == A) return &c;
  lb_ctx::StepGraph* slot = !h->graphs[0].exec ? &h->graphs[0] : &h->graphs[1];
  if (slot->exec) cudaGraphExecDestroy(slot->exec), *slot = lb_ctx::StepGraph{};
  const long long n0 = h->launches;
  const HostStepState before = save_state(h);
  if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  int rc = LB_OK;
  for (int t = 0; t < kGraphSteps && !rc; ++t) rc = one_step(h);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(h->stream, &graph);
  const long long nk = h->launches - n0;
  h->launches = n0;  // captured, not launched
  // a replay leaves the buffers where the capture left them: kGraphSteps is even,
  // so that is where they started (checked, not assumed)
  const bool same = h->slabs[0].A == before.slabs[0].A;
  const long long nsteps = h->steps_done - before.steps_done;
  const bool dirty_after = h->xch_dirty;
  restore_state(h, before);
  if (rc || ec != cudaSuccess || !graph || !same) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    h->broken = false;  // a failed capture is not a device failure: step plainly
    h->err.clear();
    return nullptr;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  slot->exec = exec;
  slot->A = A;
  slot->launches = nk;
  slot->steps = nsteps;
  slot->dirty_after = dirty_after;
  return slot;
}

// Replay (capturing first if needed) kGraphSteps steps.  Returns LB_OK, or a
// negative code; *done = false when no graph could be made (the caller steps
// plainly, from the state as it was before the attempt).
int graph_steps(lb_ctx* h, bool* done) {
  *done = false;
  lb_ctx::StepGraph* g = capture_graph(h);
  if (!g) return LB_OK;
  CK(h, cudaGraphLaunch(g->exec, h->stream));
  h->launches += g->launches;
  h->steps_done += g->steps;
  h->xch_dirty = g->dirty_after;
  *done = true;
  return LB_OK;
}

// After a call's steps: wait, then the R22 report -- the first offending step and
// site since the call began (the flag is reset for the next call).
int finish(lb_ctx* h, long long step0 = -1) {
  const bool peer = h->halo_mode == 1 && !h->G.zwrap;
  // ranks: the neighbours' stores into this slab have landed before lb_step returns
  if (peer && h->nranks > 1) CK(h, launch_wait_inbound(peers_of(h, 0), h->stream));
  CK(h, cudaMemcpyAsync(h->h_health, h->d_health, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
  if (peer)
    for (int r = 0; r < h->nslabs; ++r)
      CK(h, cudaMemcpyAsync(h->h_sync + r, h->slabs[r].sync + SW_ERR, sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  if (peer)
    for (int r = 0; r < h->nslabs; ++r)
      if (h->h_sync[r]) {
        h->broken = true;
        return set_err(h, LB_ECUDA, "peer transport: a wait for a neighbour's epoch timed out (slab %d)", r);
      }
  const unsigned long long v = *h->h_health;
  if (v != ~0ULL) {
    CK(h, cudaMemsetAsync(h->d_health, 0xff, sizeof(unsigned long long), h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    const long long step = (long long)(v >> 40), site = (long long)(v & ((1ULL << 40) - 1));
    const long long x = site % h->nx, y = (site / h->nx) % h->ny, z = site / ((long long)h->nx * h->ny);
    return set_err(h, LB_ENUMERIC,
                   "numerical-domain error (R22): rho <= 0 or a non-finite value at site (x=%lld, y=%lld, z=%lld) "
                   "in step %lld of this call (step %lld since the handle was created)",
                   x, y, z, step0 >= 0 ? step - step0 : step, step);
  }
  return LB_OK;
}

__global__ void k_poke(double* p, double v) {
  *p = v;
  __threadfence_system();
}

void close_peers(lb_ctx* h) {
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  h->ipc_opened.clear();
  for (int k = 0; k < 2; ++k) h->peerA[k] = h->peerB[k] = h->peerPhi[k] = nullptr, h->peerSync[k] = nullptr;
}

// All-gather of `bytes` host bytes per rank (rank order) over the handle's
// bootstrap: NCCL (lb_create_slab) or the caller's callback (lb_create_slab_ext).
int allgather_host(lb_ctx* h, const void* mine, void* all, size_t bytes) {
  if (h->allgather) {
    if (h->allgather(h->allgather_ctx, mine, all, bytes) != 0)
      return set_err(h, LB_ENCCL, "the caller's all-gather failed");
    return LB_OK;
  }
  char* d_all = nullptr;
  CK(h, cudaMalloc(&d_all, bytes * h->nranks));
  CK(h, cudaMemcpyAsync(d_all + bytes * h->rank, mine, bytes, cudaMemcpyHostToDevice, h->stream));
  NK(h, ncclAllGather(d_all + bytes * h->rank, d_all, bytes, ncclChar, h->comm, h->stream));
  CK(h, cudaMemcpyAsync(all, d_all, bytes * h->nranks, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  cudaFree(d_all);
  return LB_OK;
}

// Peer transport between ranks (collective): exchange CUDA IPC handles of A, B,
// phi and the sync words over the bootstrap, map the neighbours' buffers, and
// check the mapping end to end -- each rank stores a token into both neighbours'
// phi ghost planes with a kernel and reads back what its neighbours stored.  On
// success halo_mode = 1; if the neighbours' memory cannot be mapped (no peer
// access) or the check fails on any rank, every rank keeps the NCCL exchange (the
// decision is agreed by an all-gather; an external bootstrap has no exchange
// transport, so there it is an error).  Only a NCCL/CUDA error on the way is an
// error otherwise.
int open_peers(lb_ctx* h) {
  const Geom& G = h->G;
  Slab& s = h->slabs[0];
  CK(h, cudaMalloc(&h->d_token, 4 * sizeof(double)));
  CK(h, cudaMemsetAsync(h->d_token, 0, 4 * sizeof(double), h->stream));
  struct Handles {
    cudaIpcMemHandle_t a, b, phi, sync;
  } mine{};
  int ok = 1;
  // (handles of whole allocations: the field buffers start kGuardBytes into theirs)
  if (cudaIpcGetMemHandle(&mine.a, raw_of(s.A)) != cudaSuccess || cudaIpcGetMemHandle(&mine.b, raw_of(s.B)) != cudaSuccess ||
      cudaIpcGetMemHandle(&mine.phi, raw_of(s.phi)) != cudaSuccess || cudaIpcGetMemHandle(&mine.sync, s.sync) != cudaSuccess)
    ok = 0;
  cudaGetLastError();
  std::vector<Handles> all(h->nranks);
  int rc = allgather_host(h, &mine, all.data(), sizeof(Handles));
  if (rc) return rc;
  const int nb[2] = {(h->rank - 1 + h->nranks) % h->nranks, (h->rank + 1) % h->nranks};
  for (int k = 0; k < 2 && ok; ++k) {
    if (k == 1 && nb[1] == nb[0]) {
      h->peerA[1] = h->peerA[0], h->peerB[1] = h->peerB[0], h->peerPhi[1] = h->peerPhi[0];
      h->peerSync[1] = h->peerSync[0];
      break;
    }
    const cudaIpcMemHandle_t* hs[4] = {&all[nb[k]].a, &all[nb[k]].b, &all[nb[k]].phi, &all[nb[k]].sync};
    void** dst[4] = {reinterpret_cast<void**>(&h->peerA[k]), reinterpret_cast<void**>(&h->peerB[k]),
                     reinterpret_cast<void**>(&h->peerPhi[k]), reinterpret_cast<void**>(&h->peerSync[k])};
    for (int j = 0; j < 4 && ok; ++j) {
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, *hs[j], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        ok = 0;
        cudaGetLastError();
      } else {
        h->ipc_opened.push_back(p);
        *dst[j] = j < 3 ? static_cast<unsigned char*>(p) + kGuardBytes : p;
      }
    }
  }
  // end-to-end check of the mapping with kernel stores (the barrier is collective:
  // every rank takes part, mapped or not)
  if (ok) {
    k_poke<<<1, 1, 0, h->stream>>>(h->peerPhi[1] + phi_plane_index(G, -GP), 1000.0 + h->rank);
    k_poke<<<1, 1, 0, h->stream>>>(h->peerPhi[0] + phi_plane_index(G, G.nzl) + 1, 2000.0 + h->rank);
    CK(h, cudaGetLastError());
  }
  if ((rc = halo_barrier(h, K_HALO_PHI))) return rc;
  double got[2] = {0, 0};
  CK(h, cudaMemcpyAsync(&got[0], s.phi + phi_plane_index(G, -GP), 8, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaMemcpyAsync(&got[1], s.phi + phi_plane_index(G, G.nzl) + 1, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  ok = ok && got[0] == 1000.0 + nb[0] && got[1] == 2000.0 + nb[1];
  // every rank must agree (a neighbour that could not map falls back with us)
  std::vector<int> oks(h->nranks);
  if ((rc = allgather_host(h, &ok, oks.data(), sizeof(int)))) return rc;
  for (int v : oks) ok = ok && v;
  if (!ok) close_peers(h);
  if (!ok && h->allgather) return set_err(h, LB_ENCCL, "peer mapping failed and an external bootstrap has no exchange transport");
  h->halo_mode = ok ? 1 : 0;
  return LB_OK;
}

// host (whole lattice for loopback, this rank's slab for NCCL) <-> canonical staging in B
size_t host_nloc(const lb_ctx* h) { return (size_t)h->G.nxy * h->nzl * h->nslabs; }

}  // namespace

namespace {

// Cahn-Hilliard slabs: f's edge planes (the 19 f slots of planes 0 and nzl-1 of the
// current state A) to the neighbours' ghost planes nzl and -1 of A, where the
// kernel's f box reads them for u = j / rho at z +- 1 (three slot runs each way).
int exchange_fedge(lb_ctx* h) {
  const Geom& G = h->G;
  const int run0[3] = {0, 10, 28}, rlen[3] = {5, 9, 5};
  if (h->nranks > 1) {
    Slab& s = h->slabs[0];
    const int up = (h->rank + 1) % h->nranks, dn = (h->rank - 1 + h->nranks) % h->nranks;
    cudaError_t ce = timed(h, K_HALO_DIST, false, [&]() {
      ncclGroupStart();
      for (int r = 0; r < 3; ++r) {
        const size_t cnt = (size_t)rlen[r] * G.nxy;
        ncclSend(s.A + dist_index(G, G.nzl - 1, run0[r], 0), cnt, ncclDouble, up, h->comm, h->stream);
        ncclRecv(s.A + dist_index(G, -1, run0[r], 0), cnt, ncclDouble, dn, h->comm, h->stream);
        ncclSend(s.A + dist_index(G, 0, run0[r], 0), cnt, ncclDouble, dn, h->comm, h->stream);
        ncclRecv(s.A + dist_index(G, G.nzl, run0[r], 0), cnt, ncclDouble, up, h->comm, h->stream);
      }
      return ncclGroupEnd() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
    });
    if (ce != cudaSuccess) return set_err(h, LB_ENCCL, "NCCL f edge-plane exchange failed");
    return LB_OK;
  }
  for (int i = 0; i < h->nslabs; ++i) {
    Slab& s = h->slabs[i];
    Slab& up = h->slabs[(i + 1) % h->nslabs];
    Slab& dn = h->slabs[(i - 1 + h->nslabs) % h->nslabs];
    CK(h, timed(h, K_HALO_DIST, false, [&]() {
      cudaError_t e = cudaSuccess;
      for (int r = 0; r < 3 && e == cudaSuccess; ++r) {
        const size_t bytes = (size_t)rlen[r] * G.nxy * 8;
        e = cudaMemcpyAsync(up.A + dist_index(G, -1, run0[r], 0), s.A + dist_index(G, G.nzl - 1, run0[r], 0), bytes,
                            cudaMemcpyDeviceToDevice, h->stream);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(dn.A + dist_index(G, G.nzl, run0[r], 0), s.A + dist_index(G, 0, run0[r], 0), bytes,
                              cudaMemcpyDeviceToDevice, h->stream);
      }
      return e;
    }));
  }
  return LB_OK;
}

int ch_create(int nx, int ny, int nz, const lb_params* params, double tau_shear, double tau_bulk, double tau_ghost,
              int nranks, int rank, int nslabs, const void* id128, lb_t** out) {
  if (out) *out = nullptr;
  if (nx % 2 != 0) return set_err(nullptr, LB_EINVAL, "the Cahn-Hilliard variant needs nx even (TMA rows)");
  for (double t : {tau_shear, tau_bulk, tau_ghost})
    if (!std::isfinite(t) || !(t > 0.5)) return set_err(nullptr, LB_EINVAL, "MRT relaxation times must be finite and > 0.5");
  if (nranks > 1 && !id128) return set_err(nullptr, LB_EINVAL, "id128 is NULL");
  int rc = create_common(nx, ny, nz, params, nranks, rank, nslabs, out);
  if (rc) return rc;
  lb_ctx* h = *out;
  h->ch = true;
  h->halo_mode = 0;  // ghost planes + copies / NCCL send-recv
  h->dp.coll = 1;
  h->dp.inv_tau_s = 1.0 / tau_shear;
  h->dp.inv_tau_b = 1.0 / tau_bulk;
  h->dp.inv_tau_ghost = 1.0 / tau_ghost;
  cudaError_t e = cudaSuccess;
  bool maps_ok = true;
  for (auto& s : h->slabs) {
    if (e == cudaSuccess) e = dev_alloc(h, &s.phi2, phi_doubles(h->G) * sizeof(double));
    if (e == cudaSuccess) e = cudaMemsetAsync(s.phi2, 0xff, phi_doubles(h->G) * sizeof(double), h->stream);
    maps_ok = maps_ok && make_ch_maps(h->G, s.A, s.phi, h->ty, &s.chA) && make_ch_maps(h->G, s.B, s.phi2, h->ty, &s.chB);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess || !maps_ok) {
    g_create_error = "Cahn-Hilliard handle: allocation or TMA descriptor failed";
    lb_destroy(h);
    *out = nullptr;
    return e == cudaErrorMemoryAllocation ? LB_ENOMEM : LB_ECUDA;
  }
  if (nranks > 1) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      g_create_error = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      h->comm = nullptr;
      lb_destroy(h);
      *out = nullptr;
      return LB_ENCCL;
    }
  }
  return LB_OK;
}

}  // namespace

// ============================================================================
extern "C" {

const char* lb_version(void) { return "lb-b200 0.1 (sm_100a, fp64 D3Q19 binary fluid)"; }

int lb_create(int nx, int ny, int nz, const lb_params* params, lb_t** out) {
  return create_common(nx, ny, nz, params, 1, 0, 1, out);
}

int lb_create_loopback(int nx, int ny, int nz, const lb_params* params, int nslabs, lb_t** out) {
  return create_common(nx, ny, nz, params, 1, 0, nslabs, out);
}

int lb_nccl_get_unique_id(void* id128) {
  if (!id128) return set_err(nullptr, LB_EINVAL, "id128 is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_err(nullptr, LB_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(id128, &id, sizeof id);
  return LB_OK;
}

int lb_create_slab(int nx, int ny, int nz, const lb_params* params, int nranks, int rank, const void* id128,
                   lb_t** out) {
  if (nranks > 1 && !id128) return set_err(nullptr, LB_EINVAL, "id128 is NULL");
  int rc = create_common(nx, ny, nz, params, nranks, rank, 1, out);
  if (rc || nranks == 1) return rc;
  lb_ctx* h = *out;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    g_create_error = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
    h->comm = nullptr;
    lb_destroy(h);
    *out = nullptr;
    return LB_ENCCL;
  }
  rc = open_peers(h);
  if (rc) {
    g_create_error = h->err;
    lb_destroy(h);
    *out = nullptr;
    return rc;
  }
  return LB_OK;
}

int lb_create_slab_ext(int nx, int ny, int nz, const lb_params* params, int nranks, int rank,
                       lb_allgather_fn allgather, void* ctx, lb_t** out) {
  if (!allgather) return set_err(nullptr, LB_EINVAL, "allgather is NULL");
  if (nranks < 2) return set_err(nullptr, LB_EINVAL, "an external bootstrap needs nranks >= 2");
  int rc = create_common(nx, ny, nz, params, nranks, rank, 1, out);
  if (rc) return rc;
  lb_ctx* h = *out;
  h->allgather = allgather;
  h->allgather_ctx = ctx;
  if ((rc = open_peers(h))) {
    g_create_error = h->err;
    lb_destroy(h);
    *out = nullptr;
    return rc;
  }
  return LB_OK;
}

int lb_debug_step_phase(lb_t* h, int phase) {
  int rc = usable(h);
  if (rc) return rc;
  if (phase < 0 || phase > 2) return set_err(h, LB_EINVAL, "phase must be 0 (K_phi), 1 (step) or 2 (finish)");
  if (h->ch || h->lc || h->G.zwrap || h->halo_mode != 1)
    return set_err(h, LB_EINVAL, "step phases exist for slab handles of the binary fluid with the peer transport");
  if (!h->have_state) return set_err(h, LB_ESTATE, "no state");
  const Geom& G = h->G;
  if (phase == 0) {
    for (int r = 0; r < h->nslabs; ++r)
      CK(h, launch_phi_edges(G, h->slabs[r].A, h->slabs[r].phi, h->stream, peers_of(h, r)));
    h->launches += 3;
    CK(h, cudaStreamSynchronize(h->stream));
    return LB_OK;
  }
  if (phase == 1) {
    const Launch ln = launch_of(h);
    for (int r = 0; r < h->nslabs; ++r) {
      Slab& s = h->slabs[r];
      const Health hl = health_of(h, r, r == h->nslabs - 1);
      CK(h, launch_bgk_step(h, s, ln, hl, peers_of(h, r)));
      CK(h, launch_publish_push(peers_of(h, r), h->stream));
      h->launches += 2;
    }
    swap_roles(h);
    ++h->steps_done;
    CK(h, cudaStreamSynchronize(h->stream));
    return LB_OK;
  }
  return finish(h);
}

size_t lb_local_sites(const lb_t* h) { return h ? host_nloc(h) : 0; }

int lb_set_state(lb_t* h, const double* f, const double* g) {
  int rc = usable(h);
  if (rc) return rc;
  if (h->ch) return set_err(h, LB_EINVAL, "a Cahn-Hilliard handle holds (f, phi): use lb_set_state_ch");
  if (h->lc) return set_err(h, LB_EINVAL, "a liquid-crystal handle holds (f, Q, u): use lb_set_state_lc");
  if (!f || !g) return set_err(h, LB_EINVAL, "f or g is NULL");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl, N = host_nloc(h);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    // 19 rows of nloc doubles, host row pitch N (whole lattice) -> staging rows of nloc
    CK(h, cudaMemcpy2DAsync(s.B, nloc * 8, f + r * nloc, N * 8, nloc * 8, Q, cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemcpy2DAsync(s.B + Q * nloc, nloc * 8, g + r * nloc, N * 8, nloc * 8, Q, cudaMemcpyHostToDevice, h->stream));
    CK(h, timed(h, K_PERMUTE, true, [&]() { return launch_canon_to_planes(G, s.B, s.A, h->stream); }));
  }
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  h->have_state = true;
  return LB_OK;
}

int lb_get_state(lb_t* h, double* f, double* g) {
  int rc = usable(h);
  if (rc) return rc;
  if (h->ch) return set_err(h, LB_EINVAL, "a Cahn-Hilliard handle holds (f, phi): use lb_get_state_ch");
  if (h->lc) return set_err(h, LB_EINVAL, "a liquid-crystal handle holds (f, Q, u): use lb_get_state_lc");
  if (!f || !g) return set_err(h, LB_EINVAL, "f or g is NULL");
  if (!h->have_state) return set_err(h, LB_ESTATE, "no state: call lb_set_state or lb_init_equilibrium first");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl, N = host_nloc(h);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    CK(h, timed(h, K_PERMUTE, true, [&]() { return launch_planes_to_canon(G, s.A, s.B, h->stream); }));
    CK(h, cudaMemcpy2DAsync(f + r * nloc, N * 8, s.B, nloc * 8, nloc * 8, Q, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpy2DAsync(g + r * nloc, N * 8, s.B + Q * nloc, nloc * 8, nloc * 8, Q, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  return LB_OK;
}

int lb_init_equilibrium(lb_t* h, const double* rho, const double* u, const double* phi) {
  int rc = usable(h);
  if (rc) return rc;
  if (h->lc) return set_err(h, LB_EINVAL, "a liquid-crystal handle is initialised by lb_init_lc");
  if (!phi) return set_err(h, LB_EINVAL, "phi is NULL");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl, N = host_nloc(h);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    CK(h, cudaMemcpyAsync(s.phi + phi_plane_index(G, 0), phi + r * nloc, nloc * 8, cudaMemcpyHostToDevice, h->stream));
    if (rho) CK(h, cudaMemcpyAsync(s.B, rho + r * nloc, nloc * 8, cudaMemcpyHostToDevice, h->stream));
    if (u) CK(h, cudaMemcpy2DAsync(s.B + nloc, nloc * 8, u + r * nloc, N * 8, nloc * 8, 3, cudaMemcpyHostToDevice, h->stream));
  }
  if ((rc = exchange_phi(h))) return rc;
  for (auto& s : h->slabs)
    CK(h, timed(h, K_INIT, true, [&]() {
         return launch_init_eq(G, h->dp, s.phi, rho ? s.B : nullptr, u ? s.B + nloc : nullptr, s.A, h->stream);
       }));
  // ranks with the peer transport: a neighbour's first K_phi stores into this
  // rank's phi ghost planes, which the init kernel above reads -- nobody steps
  // before every rank's init has finished
  if (h->nranks > 1 && h->halo_mode == 1 && !h->G.zwrap && (rc = halo_barrier(h, K_HALO_PHI))) return rc;
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  h->have_state = true;
  return LB_OK;
}

int lb_step(lb_t* h, int nsteps) {
  int rc = usable(h);
  if (rc) return rc;
  if (nsteps < 0) return set_err(h, LB_EINVAL, "nsteps must be >= 0");
  if (!h->have_state) return set_err(h, LB_ESTATE, "no state: call lb_set_state or lb_init_equilibrium first");
  if (nsteps > 0 && h->xch_default && !h->ch && !h->lc && (rc = ensure_xch(h))) return rc;  // (never inside a capture)
  if (nsteps > 0 && (rc = refresh_xch(h))) return rc;
  const long long step0 = h->steps_done;
  int t = 0;
  while (nsteps - t >= kGraphSteps && graphs_usable(h)) {
    bool done = false;
    if ((rc = graph_steps(h, &done))) return rc;
    if (!done) break;
    t += kGraphSteps;
  }
  for (; t < nsteps; ++t)
    if ((rc = one_step(h))) return rc;
  return finish(h, step0);
}

int lb_prepare(lb_t* h) {
  int rc = usable(h);
  if (rc) return rc;
  if (h->xch_default && !h->ch && !h->lc && (rc = ensure_xch(h))) return rc;
  if ((rc = refresh_xch(h))) return rc;
  if (!graphs_usable(h)) return LB_OK;
  for (int parity = 0; parity < 2; ++parity) {  // the graphs of both buffer roles
    capture_graph(h);
    swap_roles(h);
  }
  CK(h, cudaStreamSynchronize(h->stream));
  return LB_OK;
}

int lb_debug_step_kernel(lb_t* h, int which) {
  if (h && h->lc && which != 0) return set_err(h, LB_EINVAL, "a liquid-crystal handle has one step kernel");
  if (h && h->ch) {  // 0 auto (warp-specialised for 32 x 8 tiles), 1 tile kernel, 2 warp-specialised
    if (which < 0 || which > 2) return set_err(h, LB_EINVAL, "a Cahn-Hilliard handle: which must be 0, 1 or 2");
    h->kernel_choice = which;
    steps_changed(h);
    return LB_OK;
  }
  if (!h || which < 0 || which > 3)
    return set_err(h, LB_EINVAL,
                   "which must be 0 (auto), 1 (tile), 2 (warp-specialised) or 3 (warp-specialised with the phi exchange)");
  if (which == 3 && (h->nslabs != 1 || h->slabs.empty() || !step_xch_fits(h->G, &h->slabs[0].mapsA)))
    return set_err(h, LB_EINVAL, "the phi exchange needs one periodic slab, nx %% 32 == 0 and ny %% 8 == 0 (TMA rows)");
  if (which == 3) {
    const int rc = ensure_xch(h);
    if (rc) return rc;
  }
  if (which == 2 && !h->slabs.empty() && !step_ws_fits(&h->slabs[0].mapsA))
    return set_err(h, LB_EINVAL, "the warp-specialised kernel needs nx even (TMA rows)");
  h->kernel_choice = which;
  choose_xch(h);
  steps_changed(h);
  return LB_OK;
}

int lb_debug_tune(lb_t* h, int key, int value) {
  if (!h) return set_err(nullptr, LB_EINVAL, "handle is NULL");
  switch (key) {
    case LB_TUNE_ZCHUNK:
      if (value < 0) return set_err(h, LB_EINVAL, "z-chunk must be >= 0 (0: automatic)");
      if (value == 0) {
        h->zc = step_zchunk(h->G, h->num_sms, h->ty);
        h->lczc = lc_zchunk(h->G, h->num_sms);
      } else {
        h->zc = h->lczc = value < h->nzl ? value : h->nzl;
      }
      if (!h->slabs.empty()) choose_xch(h);
      break;
    case LB_TUNE_TILE_ROWS: {  // 4 or 8 (0: automatic); the TMA maps are re-encoded for it
      const int ty = value == 0 ? step_tile_rows(h->G, h->num_sms) : value;
      if (ty != 4 && ty != 8) return set_err(h, LB_EINVAL, "tile rows must be 4 or 8 (0: automatic)");
      if (h->lc && ty != 8) return set_err(h, LB_EINVAL, "the liquid-crystal kernel has 32 x 8 tiles");
      bool ok = true;
      for (auto& s : h->slabs) {
        ok = ok && make_step_maps(h->G, s.A, ty, &s.mapsA) && make_step_maps(h->G, s.B, ty, &s.mapsB);
        if (h->ch) ok = ok && make_ch_maps(h->G, s.A, s.phi, ty, &s.chA) && make_ch_maps(h->G, s.B, s.phi2, ty, &s.chB);
      }
      if (!ok) return set_err(h, LB_ECUDA, "cuTensorMapEncodeTiled failed");
      h->ty = ty;
      h->zc = step_zchunk(h->G, h->num_sms, h->ty);
      if (!h->slabs.empty()) choose_xch(h);
      break;
    }
    case LB_TUNE_BAND_ROWS:
      if (value < 1) return set_err(h, LB_EINVAL, "band rows must be >= 1");
      h->order.band = value;
      break;
    case LB_TUNE_RESID:
      if (value < 0) return set_err(h, LB_EINVAL, "resident CTAs must be >= 0 (0: the kernel's occupancy)");
      h->order.resid = value;
      break;
    case LB_TUNE_GRAPHS:
      h->graphs_on = value != 0;
      break;
    case LB_TUNE_VARIANT:
      if (value < 0 || value > 1) return set_err(h, LB_EINVAL, "variant must be 0 or 1");
      h->variant = value;
      break;
    case LB_TUNE_L2_BOX:
    case LB_TUNE_L2_FTILE:
    case LB_TUNE_L2_GTILE:
      if (value < 0 || value > 3) return set_err(h, LB_EINVAL, "L2 policy must be 0 (normal), 1 (first), 2 (last) or 3 (unchanged)");
      (key == LB_TUNE_L2_BOX ? h->l2.box : key == LB_TUNE_L2_FTILE ? h->l2.ftile : h->l2.gtile) = value;
      break;
    default:
      return set_err(h, LB_EINVAL, "unknown tuning key %d", key);
  }
  steps_changed(h);
  return LB_OK;
}

int lb_debug_stream(lb_t* h, int nsteps) {
  int rc = usable(h);
  if (rc) return rc;
  if (nsteps < 0) return set_err(h, LB_EINVAL, "nsteps must be >= 0");
  if (!h->have_state) return set_err(h, LB_ESTATE, "no state");
  for (int t = 0; t < nsteps; ++t)
    if ((rc = one_step(h, true))) return rc;
  return finish(h);
}

int lb_get_phi(lb_t* h, double* phi) {
  int rc = usable(h);
  if (rc) return rc;
  if (!phi) return set_err(h, LB_EINVAL, "phi is NULL");
  if (h->lc) return set_err(h, LB_EINVAL, "a liquid-crystal handle has no phi (use lb_get_state_lc)");
  if (!h->have_state) return set_err(h, LB_ESTATE, "no state: call lb_set_state or lb_init_equilibrium first");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl;
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    if (!h->ch)  // phi = sum g; a Cahn-Hilliard handle holds phi itself
      CK(h, timed(h, K_PHI, true, [&]() { return launch_phi(G, s.A, s.phi, 0, G.nzl, h->stream); }));
    CK(h, cudaMemcpyAsync(phi + r * nloc, s.phi + phi_plane_index(G, 0), nloc * 8, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  return LB_OK;
}

void lb_destroy(lb_t* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  drop_graphs(h);
  close_peers(h);
  cudaFree(h->d_token);
  if (h->comm) ncclCommDestroy(h->comm);
  for (auto& s : h->slabs) {
    for (double* b : {s.A, s.B, s.phi, s.phi2, s.q, s.q2, s.u, s.u2}) dev_free(b);
  }
  cudaFree(h->d_health);
  cudaFree(h->d_done);
  cudaFree(h->d_check);
  for (auto& s : h->slabs) cudaFree(s.sync);
  if (h->h_sync) cudaFreeHost(h->h_sync);
  dev_free(h->xphi[0]);
  dev_free(h->xphi[1]);
  if (h->h_health) cudaFreeHost(h->h_health);
  for (auto& p : h->pending) {
    cudaEventDestroy(p.e0);
    cudaEventDestroy(p.e1);
  }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

const char* lb_last_error(const lb_t* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

void* lb_stream(const lb_t* h) { return h ? (void*)h->stream : nullptr; }

long long lb_launch_count(const lb_t* h) { return h ? h->launches : 0; }

int lb_profile_enable(lb_t* h, int on) {
  if (!h) return set_err(nullptr, LB_EINVAL, "handle is NULL");
  h->prof_on = on != 0;  // (graphs are not used while per-launch events are on)
  return LB_OK;
}

int lb_profile_reset(lb_t* h) {
  if (!h) return set_err(nullptr, LB_EINVAL, "handle is NULL");
  for (int k = 0; k < K_COUNT; ++k) h->prof_ms[k] = 0, h->prof_n[k] = 0;
  return LB_OK;
}

int lb_profile_count(const lb_t* h) { return h ? K_COUNT : 0; }

int lb_profile_entry(const lb_t* h, int i, const char** name, double* total_ms, long long* launches) {
  if (!h || i < 0 || i >= K_COUNT) return LB_EINVAL;
  if (name) *name = kKernelNames[i];
  if (total_ms) *total_ms = h->prof_ms[i];
  if (launches) *launches = h->prof_n[i];
  return LB_OK;
}

double lb_bytes_per_site(void) { return 2.0 * NSLOT * sizeof(double); }

// Host-only: the composition of the kernels' push addressing (push_target) and
// the halo plan, inverted into a pull map over the GLOBAL lattice:
// out[p*N + s_dst] = canonical global index of the site whose component p
// streams into s_dst.  N = nx*ny*nz.  Exercises exactly the integer maps the
// device code uses, for any slab count.
int lb_debug_propagation_map(int nx, int ny, int nz, int nslabs, int64_t* out) {
  if (!out || nx < 3 || ny < 3 || nz < 3 || nslabs < 1 || nz % nslabs || (nslabs > 1 && nz / nslabs < 2))
    return LB_EINVAL;
  Geom G;
  G.nx = nx;
  G.ny = ny;
  G.nzl = nz / nslabs;
  G.zwrap = nslabs == 1;
  G.nxy = (long long)nx * ny;
  G.plane = (long long)NSLOT * G.nxy;
  const long long N = G.nxy * nz;
  for (long long k = 0; k < (long long)Q * N; ++k) out[k] = -1;
  for (int r = 0; r < nslabs; ++r)
    for (int z = 0; z < G.nzl; ++z)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x)
          for (int i = 0; i < Q; ++i) {
            const long long d = push_target(G, i, x, y, z);  // plane-relative address without slot
            const int zz = (int)(d / G.plane) - GZ;          // local destination plane
            const long long xy = d - (long long)(zz + GZ) * G.plane;
            int rdst = r, zdst = zz;
            if (zz == G.nzl) {  // ghost above: halo run goes to plane 0 of slab r+1
              if (slot(0, i) < SLOT_UP_FIRST || slot(0, i) >= SLOT_UP_FIRST + HALO_COMPS) return LB_EINVAL;
              rdst = (r + 1) % nslabs, zdst = 0;
            } else if (zz == -1) {  // ghost below: goes to plane nzl-1 of slab r-1
              if (slot(0, i) < SLOT_DOWN_FIRST || slot(0, i) >= SLOT_DOWN_FIRST + HALO_COMPS) return LB_EINVAL;
              rdst = (r - 1 + nslabs) % nslabs, zdst = G.nzl - 1;
            }
            const long long sdst = xy + G.nxy * ((long long)rdst * G.nzl + zdst);
            const long long ssrc = x + (long long)nx * (y + (long long)ny * ((long long)r * G.nzl + z));
            if (out[(long long)i * N + sdst] != -1) return LB_EINVAL;  // not a permutation
            out[(long long)i * N + sdst] = ssrc;
          }
  return LB_OK;
}

int lb_create_ch(int nx, int ny, int nz, const lb_params* params, double tau_shear, double tau_bulk, double tau_ghost,
                 lb_t** out) {
  return ch_create(nx, ny, nz, params, tau_shear, tau_bulk, tau_ghost, 1, 0, 1, nullptr, out);
}

int lb_create_ch_loopback(int nx, int ny, int nz, const lb_params* params, double tau_shear, double tau_bulk,
                          double tau_ghost, int nslabs, lb_t** out) {
  return ch_create(nx, ny, nz, params, tau_shear, tau_bulk, tau_ghost, 1, 0, nslabs, nullptr, out);
}

int lb_create_ch_slab(int nx, int ny, int nz, const lb_params* params, double tau_shear, double tau_bulk,
                      double tau_ghost, int nranks, int rank, const void* id128, lb_t** out) {
  return ch_create(nx, ny, nz, params, tau_shear, tau_bulk, tau_ghost, nranks, rank, 1, id128, out);
}

int lb_set_state_ch(lb_t* h, const double* f, const double* phi) {
  int rc = usable(h);
  if (rc) return rc;
  if (!h->ch) return set_err(h, LB_EINVAL, "not a Cahn-Hilliard handle");
  if (!f || !phi) return set_err(h, LB_EINVAL, "f or phi is NULL");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl, N = host_nloc(h);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    CK(h, cudaMemcpy2DAsync(s.B, nloc * 8, f + r * nloc, N * 8, nloc * 8, Q, cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemsetAsync(s.B + Q * nloc, 0, Q * nloc * 8, h->stream));  // the g slots are not used
    CK(h, timed(h, K_PERMUTE, true, [&]() { return launch_canon_to_planes(G, s.B, s.A, h->stream); }));
    CK(h, cudaMemcpyAsync(s.phi + phi_plane_index(G, 0), phi + r * nloc, nloc * 8, cudaMemcpyHostToDevice, h->stream));
  }
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  h->have_state = true;
  return LB_OK;
}

int lb_get_state_ch(lb_t* h, double* f, double* phi) {
  int rc = usable(h);
  if (rc) return rc;
  if (!h->ch) return set_err(h, LB_EINVAL, "not a Cahn-Hilliard handle");
  if (!f || !phi) return set_err(h, LB_EINVAL, "f or phi is NULL");
  if (!h->have_state) return set_err(h, LB_ESTATE, "no state: call lb_set_state_ch or lb_init_equilibrium first");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl, N = host_nloc(h);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    CK(h, timed(h, K_PERMUTE, true, [&]() { return launch_planes_to_canon(G, s.A, s.B, h->stream); }));
    CK(h, cudaMemcpy2DAsync(f + r * nloc, N * 8, s.B, nloc * 8, nloc * 8, Q, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpyAsync(phi + r * nloc, s.phi + phi_plane_index(G, 0), nloc * 8, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  return LB_OK;
}

int lb_set_collision(lb_t* h, int model, double tau_shear, double tau_bulk, double tau_ghost) {
  int rc = usable(h);
  if (rc) return rc;
  if (h->ch) return set_err(h, LB_EINVAL, "a Cahn-Hilliard handle's collision is fixed at lb_create_ch");
  if (h->lc) return set_err(h, LB_EINVAL, "a liquid-crystal handle's collision is fixed at lb_create_lc");
  steps_changed(h);
  if (model == 0) {
    h->dp.coll = 0;
    return LB_OK;
  }
  if (model != 1) return set_err(h, LB_EINVAL, "model must be 0 (BGK + force) or 1 (stress in f^eq, MRT)");
  for (double t : {tau_shear, tau_bulk, tau_ghost})
    if (!std::isfinite(t) || !(t > 0.5)) return set_err(h, LB_EINVAL, "MRT relaxation times must be finite and > 0.5");
  h->dp.coll = 1;
  h->dp.inv_tau_s = 1.0 / tau_shear;
  h->dp.inv_tau_b = 1.0 / tau_bulk;
  h->dp.inv_tau_ghost = 1.0 / tau_ghost;
  return LB_OK;
}

int lb_debug_halo_mode(lb_t* h, int mode) {
  if (!h) return set_err(nullptr, LB_EINVAL, "handle is NULL");
  if (mode == -1) return h->halo_mode;
  if (mode != 0 && mode != 1) return set_err(h, LB_EINVAL, "mode must be -1 (query), 0 (exchange) or 1 (peer)");
  if (mode == 1 && h->nranks > 1 && !h->peerB[0]) return set_err(h, LB_EINVAL, "no peer mapping on this handle");
  if (mode == 1 && h->G.zwrap) return set_err(h, LB_EINVAL, "a single periodic slab has no halo");
  h->halo_mode = mode;
  steps_changed(h);
  return LB_OK;
}

int lb_debug_propagation_map_peers(int nx, int ny, int nz, int nslabs, int64_t* out) {
  if (!out || nx < 3 || ny < 3 || nz < 3 || nslabs < 1 || nz % nslabs || (nslabs > 1 && nz / nslabs < 2))
    return LB_EINVAL;
  Geom G;
  G.nx = nx;
  G.ny = ny;
  G.nzl = nz / nslabs;
  G.zwrap = nslabs == 1;
  G.nxy = (long long)nx * ny;
  G.plane = (long long)NSLOT * G.nxy;
  const long long N = G.nxy * nz, per = (long long)(G.nzl + 2 * GZ) * G.plane;
  // the slabs' next-state buffers as one host array: the kernels' own address
  // arithmetic (push_plane with the neighbours' buffers) decides the destination
  std::vector<double> buf((size_t)(per * nslabs));
  for (long long k = 0; k < (long long)Q * N; ++k) out[k] = -1;
  for (int r = 0; r < nslabs; ++r) {
    Peers P;
    if (!G.zwrap) {
      P.dn = buf.data() + per * ((r - 1 + nslabs) % nslabs);
      P.up = buf.data() + per * ((r + 1) % nslabs);
    }
    double* B = buf.data() + per * r;
    for (int z = 0; z < G.nzl; ++z)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x)
          for (int i = 0; i < Q; ++i) {
            const double* d = push_plane(G, B, P, z + cz(i)) + push_in_plane(G, i, x, y) + (long long)slot(0, i) * G.nxy;
            const long long off = d - buf.data();
            const int rdst = (int)(off / per);
            const long long in = off - per * rdst;
            const int zz = (int)(in / G.plane) - GZ;
            if (zz < 0 || zz >= G.nzl) return LB_EINVAL;  // a ghost plane: the fused halo must not use them
            const long long rem = in - (long long)(zz + GZ) * G.plane;
            if (rem / G.nxy != slot(0, i)) return LB_EINVAL;
            const long long xy = rem - (long long)slot(0, i) * G.nxy;
            const long long sdst = xy + G.nxy * ((long long)rdst * G.nzl + zz);
            const long long ssrc = x + (long long)nx * (y + (long long)ny * ((long long)r * G.nzl + z));
            if (out[(long long)i * N + sdst] != -1) return LB_EINVAL;  // not a permutation
            out[(long long)i * N + sdst] = ssrc;
          }
  }
  return LB_OK;
}

int lb_debug_check(lb_t* h) {
  if (!h) return set_err(nullptr, LB_EINVAL, "handle is NULL");
  int line = 0;
  if (cudaMemcpy(&line, h->d_check, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_err(h, LB_ECUDA, "check word read-back failed");
  return line;
}

int lb_debug_checked(void) {
#ifdef LB_CHECKED
  return 1;
#else
  return 0;
#endif
}

long long lb_debug_guards(lb_t* h) {
  if (!h) return set_err(nullptr, LB_EINVAL, "handle is NULL");
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return set_err(h, LB_ECUDA, "stream synchronisation failed");
  std::vector<unsigned char> g(kGuardBytes);
  long long bad = 0;
  for (const auto& b : h->guarded) {
    const unsigned char* raw = static_cast<const unsigned char*>(raw_of(b.first));
    for (const unsigned char* z : {raw, raw + kGuardBytes + b.second}) {
      if (cudaMemcpy(g.data(), z, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        return set_err(h, LB_ECUDA, "guard read-back failed");
      for (unsigned char c : g) bad += c != kGuardByte;
    }
  }
  return bad;
}

int lb_debug_tile_order(int ntx, int nty, int nch, int resid, int band, int* out) {
  if (!out || ntx < 1 || nty < 1 || nch < 1 || resid < 1 || band == 0 || band < -ntx * nty) return LB_EINVAL;
  const int n = ntx * nty * nch;
  TileOrder o{resid, band < 0 ? -band : band};
  o.edge_last = band < 0;  // (negative band: the order of a z-slab with the peer transport)
  for (int L = 0; L < n; ++L) {
    const TileId t = tile_of_block(L, ntx, nty, nch, o);
    out[3 * L] = t.bx, out[3 * L + 1] = t.by, out[3 * L + 2] = t.bz;
  }
  return LB_OK;
}

int lb_halo_plan(int nx, int ny, int nz, int nranks, int rank, int64_t out[4]) {
  if (!out || nx < 3 || ny < 3 || nz < 3 || nranks < 1 || rank < 0 || rank >= nranks || nz % nranks ||
      (nranks > 1 && nz / nranks < 2))
    return LB_EINVAL;
  out[0] = (rank + 1) % nranks;
  out[1] = (rank - 1 + nranks) % nranks;
  out[2] = (int64_t)HALO_COMPS * nx * ny;
  out[3] = (int64_t)2 * nx * ny;
  return LB_OK;
}

}  // extern "C"

// ============================================================================
// NEXT-4: the liquid-crystal workload (R34-R45)
namespace {

lb_ctx* lc_handle(lb_t* h, int* rc) {
  *rc = usable(h);
  if (*rc) return nullptr;
  if (!h->lc) {
    *rc = set_err(h, LB_EINVAL, "not a liquid-crystal handle");
    return nullptr;
  }
  return h;
}

// canonical host field a[c*N + s] (ncomp components, N = host sites, this slab's
// sites starting at site0) <-> device plane-major [z][c][y][x] starting at plane 0
int lc_field_h2d(lb_ctx* h, double* dev0, const double* host, int ncomp, size_t site0) {
  const Geom& G = h->G;
  const size_t nxy = (size_t)G.nxy, N = host_nloc(h);
  for (int c = 0; c < ncomp; ++c)
    CK(h, cudaMemcpy2DAsync(dev0 + c * nxy, ncomp * nxy * 8, host + c * N + site0, nxy * 8, nxy * 8, G.nzl,
                            cudaMemcpyHostToDevice, h->stream));
  return LB_OK;
}
int lc_field_d2h(lb_ctx* h, double* host, const double* dev0, int ncomp, size_t site0) {
  const Geom& G = h->G;
  const size_t nxy = (size_t)G.nxy, N = host_nloc(h);
  for (int c = 0; c < ncomp; ++c)
    CK(h, cudaMemcpy2DAsync(host + c * N + site0, nxy * 8, dev0 + c * nxy, ncomp * nxy * 8, nxy * 8, G.nzl,
                            cudaMemcpyDeviceToHost, h->stream));
  return LB_OK;
}

// Q and u halos of z-slabs before a step: Q planes [nzl-2, nzl) -> ghost planes
// [-2, 0) of the slab above, [0, 2) -> [nzl, nzl+2) of the slab below; u likewise
// with one plane.  Each message is one contiguous run (plane-major layout).
int exchange_lc(lb_ctx* h) {
  const Geom& G = h->G;
  const size_t qp = (size_t)5 * G.nxy, up_ = (size_t)3 * G.nxy;  // doubles per plane
  auto qat = [&](Slab& s, int z) { return lc_q0(G, s.q) + (long long)z * qp; };
  auto uat = [&](Slab& s, int z) { return lc_u0(G, s.u) + (long long)z * up_; };
  if (h->nranks > 1) {
    Slab& s = h->slabs[0];
    const int up = (h->rank + 1) % h->nranks, dn = (h->rank - 1 + h->nranks) % h->nranks;
    cudaError_t ce = timed(h, K_HALO_PHI, false, [&]() {
      ncclGroupStart();
      ncclSend(qat(s, G.nzl - LC_GQ), LC_GQ * qp, ncclDouble, up, h->comm, h->stream);
      ncclRecv(qat(s, -LC_GQ), LC_GQ * qp, ncclDouble, dn, h->comm, h->stream);
      ncclSend(qat(s, 0), LC_GQ * qp, ncclDouble, dn, h->comm, h->stream);
      ncclRecv(qat(s, G.nzl), LC_GQ * qp, ncclDouble, up, h->comm, h->stream);
      ncclSend(uat(s, G.nzl - 1), up_, ncclDouble, up, h->comm, h->stream);
      ncclRecv(uat(s, -1), up_, ncclDouble, dn, h->comm, h->stream);
      ncclSend(uat(s, 0), up_, ncclDouble, dn, h->comm, h->stream);
      ncclRecv(uat(s, G.nzl), up_, ncclDouble, up, h->comm, h->stream);
      return ncclGroupEnd() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
    });
    if (ce != cudaSuccess) return set_err(h, LB_ENCCL, "NCCL Q / u halo exchange failed");
    return LB_OK;
  }
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    Slab& up = h->slabs[(r + 1) % h->nslabs];
    Slab& dn = h->slabs[(r - 1 + h->nslabs) % h->nslabs];
    CK(h, timed(h, K_HALO_PHI, false, [&]() {
      const cudaMemcpyKind k = cudaMemcpyDeviceToDevice;
      cudaError_t e = cudaMemcpyAsync(qat(up, -LC_GQ), qat(s, G.nzl - LC_GQ), LC_GQ * qp * 8, k, h->stream);
      if (e == cudaSuccess) e = cudaMemcpyAsync(qat(dn, G.nzl), qat(s, 0), LC_GQ * qp * 8, k, h->stream);
      if (e == cudaSuccess) e = cudaMemcpyAsync(uat(up, -1), uat(s, G.nzl - 1), up_ * 8, k, h->stream);
      if (e == cudaSuccess) e = cudaMemcpyAsync(uat(dn, G.nzl), uat(s, 0), up_ * 8, k, h->stream);
      return e;
    }));
  }
  return LB_OK;
}

int lc_create(int nx, int ny, int nz, const lb_lc_params* lp, int nranks, int rank, int nslabs, const void* id128,
              lb_t** out) {
  if (!out) return set_err(nullptr, LB_EINVAL, "out is NULL");
  *out = nullptr;
  if (!lp) return set_err(nullptr, LB_EINVAL, "params is NULL");
  if (nx % 2 != 0) return set_err(nullptr, LB_EINVAL, "the liquid-crystal workload needs nx even (16-byte rows)");
  if (!std::isfinite(lp->A0) || !std::isfinite(lp->gamma) || !std::isfinite(lp->xi))
    return set_err(nullptr, LB_EINVAL, "A0, gamma and xi must be finite");
  if (!std::isfinite(lp->Gamma) || lp->Gamma < 0) return set_err(nullptr, LB_EINVAL, "Gamma must be finite and >= 0");
  if (nranks > 1 && !id128) return set_err(nullptr, LB_EINVAL, "id128 is NULL");
  lb_params base{};
  base.tau_f = lp->tau_f;
  base.tau_g = 1.0;  // unused
  base.kappa = lp->kappa;
  int rc = create_common(nx, ny, nz, &base, nranks, rank, nslabs, out);
  if (rc) return rc;
  lb_ctx* h = *out;
  h->lc = true;
  h->halo_mode = 0;  // ghost planes + copies / NCCL send-recv
  h->dp.lc_a0 = lp->A0;
  h->dp.lc_gamma = lp->gamma;
  h->dp.lc_xi = lp->xi;
  h->dp.lc_Gamma = lp->Gamma;
  h->lczc = lc_zchunk(h->G, h->num_sms);
  const size_t nq = lc_q_doubles(h->G), nu = lc_u_doubles(h->G);
  cudaError_t e = cudaSuccess;
  bool maps_ok = true;
  for (auto& s : h->slabs) {
    for (double** b : {&s.q, &s.q2})
      if (e == cudaSuccess && (e = dev_alloc(h, b, nq * sizeof(double))) == cudaSuccess)
        e = cudaMemsetAsync(*b, 0xff, nq * sizeof(double), h->stream);
    for (double** b : {&s.u, &s.u2})
      if (e == cudaSuccess && (e = dev_alloc(h, b, nu * sizeof(double))) == cudaSuccess)
        e = cudaMemsetAsync(*b, 0xff, nu * sizeof(double), h->stream);
    maps_ok = maps_ok && make_step_maps(h->G, s.A, 8, &s.lcA) && make_step_maps(h->G, s.B, 8, &s.lcB);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess || !maps_ok) {
    g_create_error = "liquid-crystal handle: allocation or TMA descriptor failed";
    lb_destroy(h);
    *out = nullptr;
    return e == cudaErrorMemoryAllocation ? LB_ENOMEM : LB_ECUDA;
  }
  if (nranks > 1) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      g_create_error = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      h->comm = nullptr;
      lb_destroy(h);
      *out = nullptr;
      return LB_ENCCL;
    }
  }
  return LB_OK;
}

}  // namespace

extern "C" {

int lb_create_lc(int nx, int ny, int nz, const lb_lc_params* lp, lb_t** out) {
  return lc_create(nx, ny, nz, lp, 1, 0, 1, nullptr, out);
}

int lb_create_lc_loopback(int nx, int ny, int nz, const lb_lc_params* lp, int nslabs, lb_t** out) {
  return lc_create(nx, ny, nz, lp, 1, 0, nslabs, nullptr, out);
}

int lb_create_lc_slab(int nx, int ny, int nz, const lb_lc_params* lp, int nranks, int rank, const void* id128,
                      lb_t** out) {
  return lc_create(nx, ny, nz, lp, nranks, rank, 1, id128, out);
}

int lb_set_state_lc(lb_t* h_, const double* f, const double* q, const double* u) {
  int rc;
  lb_ctx* h = lc_handle(h_, &rc);
  if (!h) return rc;
  if (!f || !q || !u) return set_err(h, LB_EINVAL, "f, q or u is NULL");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl, N = host_nloc(h);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    CK(h, cudaMemcpy2DAsync(s.B, nloc * 8, f + r * nloc, N * 8, nloc * 8, Q, cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemsetAsync(s.B + Q * nloc, 0, Q * nloc * 8, h->stream));  // the g slots are not used
    CK(h, timed(h, K_PERMUTE, true, [&]() { return launch_canon_to_planes(G, s.B, s.A, h->stream); }));
    if ((rc = lc_field_h2d(h, lc_q0(G, s.q), q, 5, r * nloc)) || (rc = lc_field_h2d(h, lc_u0(G, s.u), u, 3, r * nloc)))
      return rc;
  }
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  h->have_state = true;
  return LB_OK;
}

int lb_get_state_lc(lb_t* h_, double* f, double* q, double* u) {
  int rc;
  lb_ctx* h = lc_handle(h_, &rc);
  if (!h) return rc;
  if (!f || !q || !u) return set_err(h, LB_EINVAL, "f, q or u is NULL");
  if (!h->have_state) return set_err(h, LB_ESTATE, "no state: call lb_set_state_lc or lb_init_lc first");
  const Geom& G = h->G;
  const size_t nloc = (size_t)G.nxy * G.nzl, N = host_nloc(h);
  for (int r = 0; r < h->nslabs; ++r) {
    Slab& s = h->slabs[r];
    CK(h, timed(h, K_PERMUTE, true, [&]() { return launch_planes_to_canon(G, s.A, s.B, h->stream); }));
    CK(h, cudaMemcpy2DAsync(f + r * nloc, N * 8, s.B, nloc * 8, nloc * 8, Q, cudaMemcpyDeviceToHost, h->stream));
    if ((rc = lc_field_d2h(h, q, lc_q0(G, s.q), 5, r * nloc)) || (rc = lc_field_d2h(h, u, lc_u0(G, s.u), 3, r * nloc)))
      return rc;
  }
  CK(h, cudaStreamSynchronize(h->stream));
  resolve_pending(h);
  return LB_OK;
}

int lb_init_lc(lb_t* h_, const double* rho, const double* u, const double* n) {
  int rc;
  lb_ctx* h = lc_handle(h_, &rc);
  if (!h) return rc;
  if (!n) return set_err(h, LB_EINVAL, "n is NULL");
  const double gam = h->dp.lc_gamma;
  if (!(gam > 8.0 / 3.0)) return set_err(h, LB_EINVAL, "lb_init_lc needs gamma > 8/3 (a nematic bulk minimum)");
  const size_t nloc = host_nloc(h);
  // R45: f = f^eq(rho, u) (R8), Q = S0 (n n - I/3), the stored velocity = u
  const double S0 = 0.25 + 0.75 * std::sqrt(1.0 - 8.0 / (3.0 * gam));
  std::vector<double> f(Q * nloc), q(5 * nloc), uu(3 * nloc, 0.0);
  for (size_t s = 0; s < nloc; ++s) {
    const double r = rho ? rho[s] : 1.0;
    double v[3] = {0, 0, 0};
    if (u)
      for (int a = 0; a < 3; ++a) v[a] = uu[a * nloc + s] = u[a * nloc + s];
    const double u2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    for (int i = 0; i < Q; ++i) {
      const double cu = cx(i) * v[0] + cy(i) * v[1] + cz(i) * v[2];
      f[i * nloc + s] = wgt(i) * r * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * u2);
    }
    const double d[3] = {n[s], n[nloc + s], n[2 * nloc + s]};
    const int ab[5][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}};
    for (int k = 0; k < 5; ++k)
      q[k * nloc + s] = S0 * (d[ab[k][0]] * d[ab[k][1]] - (ab[k][0] == ab[k][1] ? 1.0 / 3.0 : 0.0));
  }
  return lb_set_state_lc(h, f.data(), q.data(), uu.data());
}

}  // extern "C"
