// lb_kernels.cuh -- internal (C++) interface between the host runtime and the
// sm_100a kernels.  Not part of the C ABI (include/lb.h is).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "d3q19.cuh"

namespace lbk {

// LB_CHECKED builds (liblb_checked.so, test support): device-side bounds checks of
// the kernels' computed indices.  A failed check records its source line in the
// handle's check word (Health::check, read by lb_debug_check) and execution goes
// on -- no trap, no fault; in the product build the checks compile to nothing.
#ifdef LB_CHECKED
#define LB_CHECK(hl, cond)                                  \
  do {                                                      \
    if (!(cond) && (hl).check) atomicCAS((hl).check, 0, __LINE__); \
  } while (0)
#else
#define LB_CHECK(hl, cond) \
  do {                     \
  } while (0)
#endif

// Constants of the step derived once on the host from lb_params (R2, R7-R10).
struct DevParams {
  double A, B, kappa;
  double inv_tau_f;   // 1 / tau_f
  double inv_tau_g;   // 1 / tau_g
  double guo_pref;    // 1 - 1/(2 tau_f)   (R7)
  double gamma;       // M / (tau_g - 1/2) (R10)
  // collision of f: 0 = BGK with the Guo force F = -div P (R5, R7; the paper path),
  // 1 = chemical stress in f^eq + three-rate MRT (NEXT-3, R23-R26)
  int coll;
  double inv_tau_s, inv_tau_b, inv_tau_ghost;  // MRT rates (coll 1)
  double mob;  // M itself: the finite-difference Cahn-Hilliard variant (R30)
  // liquid-crystal workload (NEXT-4, R35-R42): Landau-de Gennes A0, gamma; flow-aligning
  // xi; rotational diffusion Gamma (kappa above is the elastic constant)
  double lc_a0, lc_gamma, lc_xi, lc_Gamma;
};

// Geometry of one z-slab as the kernels see it.
struct Geom {
  int nx, ny, nzl;  // local extents
  int zwrap;        // 1: this slab is the whole periodic z extent (no ghosts used)
  long long nxy;    // nx * ny
  long long plane;  // NSLOT * nxy doubles per distribution plane
};

// Buffer addressing.  dist buffer: (nzl + 2*GZ) planes; phi buffer: (nzl + 2*GP) planes.
__host__ __device__ inline long long dist_index(const Geom& G, int z, int s, long long xy) {
  return (long long)(z + GZ) * G.plane + (long long)s * G.nxy + xy;
}
__host__ __device__ inline long long phi_plane_index(const Geom& G, int z) {
  return (long long)(z + GP) * G.nxy;
}
__host__ __device__ inline int wrap_n(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// Where the kernels PUSH the post-collision component i of local site (x,y,z):
// (x + cx, y + cy) periodic in the plane; z + cz wraps when G.zwrap, otherwise
// z + cz in [-1, nzl] (planes -1 and nzl are the ghost planes sent to the
// neighbouring slabs).  Shared by the step kernel and the host-side map check.
__host__ __device__ inline long long push_plane_offset(const Geom& G, int zd) {
  if (G.zwrap) zd = wrap_n(zd, G.nzl);
  return (long long)(zd + GZ) * G.plane;
}
__host__ __device__ inline long long push_in_plane(const Geom& G, int i, int x, int y) {
  return (long long)wrap_n(x + cx(i), G.nx) + (long long)G.nx * wrap_n(y + cy(i), G.ny);
}
__host__ __device__ inline long long push_target(const Geom& G, int i, int x, int y, int z) {
  return push_plane_offset(G, z + cz(i)) + push_in_plane(G, i, x, y);  // + slot*nxy by caller
}

// Tile and z-chunk of a step-kernel block.  Blocks start in launch order, about
// `resid` of them resident at a time, each taking about as long as the others.
// The order is: groups of `resid` tiles; inside a group, all tiles of chunk 0,
// then all of chunk 1, ...  So chunk c of a tile starts when chunk c-1 of the
// same tile ends, and its first planes (the box loads of planes zA-2 .. zA+1,
// which the previous chunk loaded last) are still in L2 -- with chunks in
// separate waves they were read from DRAM twice.  Tiles are numbered row-major
// (band = 1), or in bands of `band` tile rows walked column by column (tile t of
// a band: column t / band, row t % band), which puts the y neighbours of a tile
// next to it in launch order.  Whole rows (or bands of rows) keep the CTAs
// resident at one time on whole 4 KB rows (narrow strips of tile columns, tried
// to bring y neighbours closer in launch order, lost more in DRAM locality than
// they gained in L2 reuse).
struct TileId {
  int bx, by, bz;
};
struct TileOrder {
  int resid = 148;  // CTAs resident at a time
  int band = 1;     // tile rows per band
  // z-slab with the peer transport: the chunks that read a neighbour's phi planes
  // (the first and the last) run after the interior ones -- chunk c of the launch
  // order is chunk (c + 1) % nch for nch >= 3 -- so the CTAs that may wait for a
  // neighbour's K_phi come last and the interior work runs meanwhile
  bool edge_last = false;
};
__host__ __device__ inline TileId tile_of_block(int L, int ntx, int nty, int nch, TileOrder o) {
  const int ntiles = ntx * nty;
  int resid = o.resid;
  if (resid > ntiles || resid < 1) resid = ntiles;
  const int per_group = resid * nch;
  const int grp = L / per_group;
  const int r = L - grp * per_group;
  const int rg = ntiles - grp * resid < resid ? ntiles - grp * resid : resid;
  const int cl = r / rg;
  const int c = o.edge_last && nch >= 3 ? (cl + 1 == nch ? 0 : cl + 1) : cl;
  const int t = grp * resid + (r - cl * rg);
  if (o.band <= 1) return TileId{t % ntx, t / ntx, c};
  const int per_band = o.band * ntx;  // tiles of a full band
  const int b = t / per_band, u = t - b * per_band;
  const int rows = nty - b * o.band < o.band ? nty - b * o.band : o.band;  // (last band may be partial)
  return TileId{u / rows, b * o.band + u % rows, c};
}

// R22 numerical-domain report: the first offending site of a call.  The
// step kernels fold (step << 40 | global site) into *flag with atomicMin (~0 =
// clean); *step counts the steps the handle's step kernels completed (the last
// CTA of the last launch of a step advances it, after every CTA's reports).
struct Health {
  unsigned long long* flag = nullptr;
  unsigned long long* step = nullptr;
  unsigned* done = nullptr;  // CTAs finished in this launch; nullptr: this launch does not tick
  long long site0 = 0;       // global site index of local site 0 (slab z0 * nx * ny)
  int* check = nullptr;      // LB_CHECKED builds: first failed bounds check (source line)
};

// Fused halo ("peer" transport): the buffers of the
// neighbouring slabs, on this GPU (loopback) or mapped from a peer GPU over
// NVLink (CUDA IPC).  With them the step kernel stores the components it pushes
// out of the slab straight into the neighbour's next state, and K_phi its edge
// planes straight into the neighbour's phi ghost planes -- no separate exchange.
// nullptr: ghost planes here + a copy / NCCL exchange afterwards.
//
// Ordering is device-side (NEXT-1): each slab owns a few 64-bit sync words; a
// neighbour WRITES its epochs into them (st.release.sys, remote) and the owner
// POLLS them (ld.acquire.sys, local).  Per step t, with epochs counted per slab:
//   K_phi(t)  is preceded by a one-thread wait for push(dn), push(up) >= its own
//             push epoch (the neighbours' step t-1 has stored into this slab's
//             state and stopped reading its phi ghost planes), stores its edge phi
//             planes, and is followed by a one-thread publication of phi epoch t+1
//             (a system fence, then the release stores);
//   step(t)   CTAs whose z-chunk reads a ghost phi plane wait for phi(dn) or
//             phi(up) >= its own phi epoch; interior chunks never wait; a one-thread
//             kernel after it publishes push epoch t+1.
// Waits are bounded (kSyncTimeoutNs): a timeout sets SW_ERR and lb_step fails.
enum SyncWord {
  SW_PHI_FROM_DN = 0,   // phi epoch of the slab below (it wrote our ghost planes -2, -1)
  SW_PHI_FROM_UP = 1,   // phi epoch of the slab above (ghost planes nzl, nzl+1)
  SW_PUSH_FROM_DN = 2,  // push epoch of the slab below (its step stored into our plane 0)
  SW_PUSH_FROM_UP = 3,  // push epoch of the slab above (our plane nzl-1)
  SW_PHI_EPOCH = 4,     // own K_phi launches completed
  SW_PUSH_EPOCH = 5,    // own step launches completed
  SW_ERR = 8,           // a wait timed out
  SW_WORDS = 16
};
constexpr unsigned long long kSyncTimeoutNs = 20ULL * 1000 * 1000 * 1000;
struct Peers {
  double* dn = nullptr;      // next-state buffer (B) of the slab below
  double* up = nullptr;      // next-state buffer (B) of the slab above
  double* phi_dn = nullptr;  // phi buffer of the slab below
  double* phi_up = nullptr;  // phi buffer of the slab above
  unsigned long long* sync = nullptr;     // this slab's sync words (nullptr: no device-side ordering)
  unsigned long long* sync_dn = nullptr;  // the neighbours' sync words
  unsigned long long* sync_up = nullptr;
};
// Base of the distribution plane that local plane zd in [-1, nzl] is pushed to:
// this slab's plane (wrapping when G.zwrap, else its ghost planes -1 / nzl), or,
// with peers, plane nzl-1 of the slab below / plane 0 of the slab above -- the
// very slots the exchange would have copied the ghost planes to.
__host__ __device__ inline double* push_plane(const Geom& G, double* B, const Peers& P, int zd) {
  if (!G.zwrap && zd < 0 && P.dn) return P.dn + push_plane_offset(G, G.nzl - 1);
  if (!G.zwrap && zd >= G.nzl && P.up) return P.up + push_plane_offset(G, 0);
  return B + push_plane_offset(G, zd);
}

// ---- launchers (lb_kernels.cu) -------------------------------------------
// All launch on `st`, return cudaGetLastError().
// K_phi on local planes [z0, z1) (lb_get_phi; the exchange transport's edges)
cudaError_t launch_phi(const Geom& G, const double* A, double* phi, int z0, int z1, cudaStream_t st,
                       const Peers& pr = Peers{});
// K_phi of the peer transport: the two edge planes at each end, stored here and
// into the neighbours' ghost planes, ordered by the sync words (pr.sync required):
// a one-thread wait for the neighbours' pushes, the edges, a one-thread publication
cudaError_t launch_phi_edges(const Geom& G, const double* A, double* phi, cudaStream_t st, const Peers& pr);
// after a slab's step kernel: one thread publishes its push epoch (pr.sync or nothing)
cudaError_t launch_publish_push(const Peers& pr, cudaStream_t st);
// one thread: wait until both neighbours' step launches up to this slab's push
// epoch have completed (all their stores into this slab have landed)
cudaError_t launch_wait_inbound(const Peers& pr, cudaStream_t st);
// Per-device kernel preparation (dynamic shared memory attribute above 48 KB, and
// the CTAs resident at a time): once per (kernel, device), thread-safe.
cudaError_t prepare_kernel(const void* fn, size_t smem, int threads, int* resid);
// every step kernel variant of lb_step.cu, lb_step_ws.cu, lb_step_ch.cu, lb_step_lc.cu
// (at handle creation: no first-launch preparation ever happens inside a graph capture)
cudaError_t prepare_step_kernels();
cudaError_t prepare_ws_kernels();
cudaError_t prepare_ch_kernels();
cudaError_t prepare_lc_kernels();
// the fused step (lb_step.cu): collide planes [0, nzl) of A into B; phig = phi
// buffer whose ghost planes are read when !G.zwrap; zc = z-chunk per CTA
int step_tile_rows(const Geom& G, int num_sms);  // 4 or 8
int step_zchunk(const Geom& G, int num_sms, int ty);
// TMA descriptors of one distribution buffer (four CUtensorMap, opaque here):
// tile boxes TX x TY x {5, 9} components, halo boxes (TX+4) x (TY+4) x {5, 9}.
struct alignas(64) StepMaps {
  unsigned char m[4][128];
  int ty;  // tile rows of the kernel these maps were made for
  bool ok;
};
bool make_step_maps(const Geom& G, const double* buf, int ty, StepMaps* out);
// Launch knobs of the step kernels: block order (tile_of_block; resid 0 = the
// occupancy of the kernel on this device)
// L2 eviction policy of a copy: 0 evict_normal, 1 evict_first, 2 evict_last, 3 evict_unchanged
struct L2Pol {
  int box = 2;    // g box (tile + 2-site halo) of plane j+2: re-read as the g tile two planes later
  int ftile = 1;  // f tile of plane j: its last use
  int gtile = 1;  // g tile of plane j
};
struct Launch {
  int zc = 1;
  TileOrder order{0, 1};
  L2Pol l2{};  // warp-specialised kernel
};
cudaError_t launch_step(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                        const Launch& ln, const Health& hl, const StepMaps* mapsA, cudaStream_t st,
                        const Peers& pr = Peers{});
// the warp-specialised variant of the step (lb_step_ws.cu): same maps, nx even.
bool step_ws_fits(const StepMaps* maps);
// phi exchange (xch, single periodic slab): the stencil warps load only the g tile
// and take the phi halo from the neighbouring tiles' CTAs through an L2-resident
// phi array (nx*ny*nzl doubles) whose unwritten sites hold kXchEmpty: `cur` is
// written (and read) in this step, `old` (last step's) is reset to kXchEmpty for
// the next.
// depth: g tiles of the stencil in flight (1 or 2; 2 pays where the state is
// about L2-sized and the step latency-bound, 64^3 +10%, and loses where it is
// HBM-bound, 128^3 -6%: the earlier loads queue in front of the collision's).
struct XchArgs {
  double* cur = nullptr;
  double* old = nullptr;
  int depth = 1;
};
int ws_xch_blocks(const Geom& G, int zc);  // blocks of the step (tiles x z-chunks)
constexpr unsigned long long kXchEmpty = 0xFFF4DEADBEEF0001ULL;  // a NaN no arithmetic produces
bool step_xch_fits(const Geom& G, const StepMaps* maps);
cudaError_t fill_xch_empty(double* buf, long long n, cudaStream_t st);
cudaError_t launch_step_ws(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                           const Launch& ln, const Health& hl, const StepMaps* mapsA, cudaStream_t st, const Peers& pr,
                           const XchArgs* xch = nullptr);
// the finite-difference Cahn-Hilliard variant (lb_step_ch.cu, NEXT-2): state f and
// a phi field; one TMA map (f box of one component, (32+4) x (ty+2)); one slab
// m[0]: f box of one component ((32+4) x (ty+2)); m[1], m[2]: the same box over 5
// and 9 components (the f slot runs); m[3]: the phi box (32+4) x (ty+4) of the phi
// buffer paired with this distribution buffer (they swap together)
struct alignas(64) ChMaps {
  unsigned char m[4][128];
  int ty;
  bool ok;
};
bool make_ch_maps(const Geom& G, const double* buf, const double* phibuf, int ty, ChMaps* out);
// ws: the warp-specialised kernel (32 x 8 tiles; same bits), else the tile kernel;
// variant (LB_TUNE_VARIANT, measurement): 1 = the ws kernel with a 5-plane phi ring
cudaError_t launch_step_ch(const Geom& G, const DevParams& p, const double* A, double* B, const double* phiA,
                           double* phiB, int zc, const Health& hl, const ChMaps* mapsA, cudaStream_t st, bool ws,
                           int variant = 0);
// the liquid-crystal workload (lb_step_lc.cu, NEXT-4): state f (dist buffer, f slots),
// Q (five components, q[z][c][y][x]) and u (q[z][a][y][x]); 32 x 8 tiles, the f tile
// by TMA through maps m[0] (5 components) and m[1] (9) of make_step_maps(.., 8, ..)
int lc_zchunk(const Geom& G, int num_sms);
cudaError_t launch_step_lc(const Geom& G, const DevParams& p, const double* A, double* B, const double* qA,
                           double* qB, const double* uA, double* uB, int zc, const Health& hl, const StepMaps* mapsA,
                           cudaStream_t st);
cudaError_t launch_stream(const Geom& G, const double* A, double* B, cudaStream_t st, const Peers& pr = Peers{});
cudaError_t launch_init_eq(const Geom& G, const DevParams& p, const double* phi, const double* rho,
                           const double* u, double* A, cudaStream_t st);
// canonical [2][19][nloc] (f block then g block) <-> plane-major buffer
cudaError_t launch_canon_to_planes(const Geom& G, const double* canon, double* buf, cudaStream_t st);
cudaError_t launch_planes_to_canon(const Geom& G, const double* buf, double* canon, cudaStream_t st);

}  // namespace lbk
