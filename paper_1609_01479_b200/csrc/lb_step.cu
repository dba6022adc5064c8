// lb_step.cu -- the fused single-pass D3Q19 binary-fluid step for sm_100a.
//
// One kernel does every row of the hot path for a z-slab (
// "Order Parameter Gradients", "Chemical Stress", force =
// "divergence of the 'Chemical stress'", "Collision", "Propagation"):
//
//   CTA   = a TX x TY tile of (x, y) columns marching in z over a chunk of planes
//           (2.5-D blocking); one thread per column.
//   smem  = sT : f and g of the tile on the plane being collided   (TMA, 1 op)
//           sG : g on the tile + 2-site halo, two planes ahead      (TMA, 3 ops;
//                1-D bulk row copies where the halo wraps the periodic edge)
//           sPhi: ring of 5 phi planes on the halo box (phi = sum_i g_i is
//                 recomputed for the halo: single pass, no phi round trip to HBM)
//           sP : chemical stress P_ab of one plane on the tile + 1-site halo
//   regs  = the z-column pieces of F = -div P: P_az on planes k-1, k, k+1 and the
//           in-plane divergence of plane k+1.
//
// Loads never occupy registers or LSU slots while in flight: both streams are
// asynchronous (TMA / bulk copies completing on an mbarrier each), issued one
// stage ahead by one thread, so the SM always has one of them outstanding while
// it computes on the other.  Odd nx (rows not 16-byte
// aligned) falls back to per-thread 8-byte cp.async with the same schedule.
//
// Iteration k (collide plane k):
//   wait sG = g(k+2) box     -> phi(k+2) into the ring; issue sG = g(k+3)
//   P(k+1) on the P box      -> own P_az(k+1), in-plane div P(k+1)
//   wait sT = f, g(k) tile   -> collide, push f*, g* to x + c_i (A.8); issue sT = f, g(k+1)
// HBM traffic per site: f and g read once, written once = 608 B;
// the halo part of sG and the re-read of g(k) hit L2.
// Slab edges (z < 0 or z >= nzl, multi-slab only) take phi from the ghost planes
// of the phi buffer, filled by K_phi + the halo exchange.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <utility>

#include "lb_device.cuh"
#include "lb_tma.cuh"

namespace lbk {
namespace {

// Tile 32 x 8 (256 threads, ~177 KB smem, one CTA per SM) or 32 x 4 (two CTAs per
// SM, odd nx on small planes): the halo box is 1.69x the tile (2.25x for 32 x 4).
constexpr int kTX = 32;
constexpr int kStepWaves = 8;  // 32 x 4 tiles: z-chunks for ~8 waves of CTAs

__device__ __forceinline__ int slot5(int z) {
  const int s = z % 5;
  return s < 0 ? s + 5 : s;
}

template <int TX, int TY>
struct alignas(128) StepSmem {
  static constexpr int BX = TX + 4, BY = TY + 4, NB = BX * BY;  // phi box: tile + 2 halo
  static constexpr int PX = TX + 2, PY = TY + 2, NP = PX * PY;  // P box: tile + 1 halo
  static constexpr int NTILE = TX * TY;
  alignas(128) double sTf[Q][NTILE];  // f of the tile, f-slot order   (TMA boxes TX x TY x 5|9|5)
  alignas(128) double sTg[Q][NTILE];  // g of the tile, g-slot order   (TMA boxes TX x TY x 5|9|5)
  alignas(128) double sG[Q][NB];      // g on the box, g-slot order     (TMA boxes BX x BY x 5|9|5)
  double sPhi[5][NB];
  double sP[6][NP];
  unsigned long long bar_f, bar_g, bar_box;
};

// USE_TMA: nx even (16-byte rows): TMA + bulk copies.  Otherwise 8-byte cp.async.
// The tile's f and g are separate streams: f (from HBM) is consumed first and
// re-issued for the next plane at the top of an iteration, so it has a whole
// iteration of lead time; g (an L2 hit: the box brought it in two planes ago)
// follows.
template <int TX, int TY, bool USE_TMA, int COLL>
__global__ void __launch_bounds__(TX* TY, 1)
    k_step_async(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B,
                 const double* __restrict__ phig, int zc, TileOrder ord, Health hl, Peers pr,
                 const __grid_constant__ CUtensorMap tm_t5, const __grid_constant__ CUtensorMap tm_t9,
                 const __grid_constant__ CUtensorMap tm_g5, const __grid_constant__ CUtensorMap tm_g9) {
  using S = StepSmem<TX, TY>;
  constexpr int NT = TX * TY;
  constexpr int BX = S::BX, BY = S::BY, NB = S::NB, PX = S::PX, NP = S::NP;
  constexpr unsigned TILE_BYTES = Q * NT * 8, BOX_BYTES = Q * NB * 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const int tid = threadIdx.x;
  const int lx = tid % TX, ly = tid / TX;
  const TileId tb = tile_of_block(blockIdx.x, (G.nx + TX - 1) / TX, (G.ny + TY - 1) / TY, (G.nzl + zc - 1) / zc, ord);
  const int x0 = tb.bx * TX, y0 = tb.by * TY;
  const int x = x0 + lx, y = y0 + ly;
  const bool active = (x < G.nx) && (y < G.ny);
  const int zA = tb.bz * zc;
  const int zB = min(zA + zc, G.nzl);
  const long long nxy = G.nxy;
  // box fully inside the plane: TMA tensor copies; else per-thread cp.async
  const bool box_interior = x0 >= 2 && x0 + TX + 2 <= G.nx && y0 >= 2 && y0 + TY + 2 <= G.ny;

  auto wrapx = [&](int v) { v %= G.nx; return v < 0 ? v + G.nx : v; };
  auto wrapy = [&](int v) { v %= G.ny; return v < 0 ? v + G.ny : v; };

  // per-thread copy plan of the halo box (fixed over z): units of VEC doubles
  constexpr int VEC = USE_TMA ? 2 : 1;
  constexpr int BROWU = BX / VEC, BOXU = BY * BROWU, BOXR = (BOXU + NT - 1) / NT;
  long long box_src[BOXR];
  int box_dst[BOXR];
#pragma unroll
  for (int r = 0; r < BOXR; ++r) {
    const int u = tid + r * NT;
    const int row = u / BROWU, cu = u - row * BROWU;
    box_src[r] = (long long)wrapy(y0 - 2 + row) * G.nx + wrapx(x0 - 2 + cu * VEC);
    box_dst[r] = u < BOXU ? row * BX + cu * VEC : -1;
    LB_CHECK(hl, box_dst[r] < 0 || (box_dst[r] + VEC - 1 < NB && box_src[r] >= 0 && box_src[r] + VEC - 1 < nxy));
  }
  auto zsrc = [&](int zp, bool& ghost) {
    ghost = false;
    if (G.zwrap) {  // one unsigned compare in the common case; a modulo only for slabs of < 3 planes
      const int n = G.nzl;
      if ((unsigned)zp >= (unsigned)n) {
        zp += zp < 0 ? n : -n;
        if ((unsigned)zp >= (unsigned)n) { zp %= n; zp += zp < 0 ? n : 0; }
      }
      return zp;
    }
    ghost = zp < 0 || zp >= G.nzl;
    return zp;
  };

  unsigned long long pol_first = 0, pol_last = 0;
  if (USE_TMA && tid < 32) pol_first = policy_evict_first(), pol_last = policy_evict_last();
  if (USE_TMA && tid == 0) {
    mbar_init(&sm.bar_f, 1);
    mbar_init(&sm.bar_g, 1);
    mbar_init(&sm.bar_box, 1);
    fence_barrier_init();
  }
  if (tid == 0) sync_wait_ghost_phi(G, pr, zA, zB);  // peer transport: slab-edge chunks wait for the neighbours' K_phi
  __syncthreads();
  unsigned ph_f = 0, ph_g = 0, ph_box = 0;  // mbarrier parities

  // ---- copy issue: g box of plane zp into sm.sG (returns false for a ghost plane)
  auto issue_box = [&](int zp) -> bool {
    bool ghost;
    const int zs = zsrc(zp, ghost);
    if (ghost) return false;
    if (USE_TMA && box_interior) {
      // three TMA boxes (g slots 5..9, 19..27, 33..37), one thread
      if (tid == 0) {
        const int cpl = (zs + GZ) * NSLOT;  // component-plane index of slot 0
        fence_proxy_async();
        mbar_expect_tx(&sm.bar_box, BOX_BYTES);
        tma_load_3d(&sm.sG[0][0], &tm_g5, x0 - 2, y0 - 2, cpl + 5, &sm.bar_box, pol_last);
        tma_load_3d(&sm.sG[5][0], &tm_g9, x0 - 2, y0 - 2, cpl + 19, &sm.bar_box, pol_last);
        tma_load_3d(&sm.sG[14][0], &tm_g5, x0 - 2, y0 - 2, cpl + 33, &sm.bar_box, pol_last);
      }
    } else {
      // the halo wraps the periodic edge (or odd nx): every thread copies its
      // fixed box positions of all 19 components (cp.async, one group)
      const double* base = A + (long long)(zs + GZ) * G.plane;
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const double* bj = base + (long long)gslot_of_rank(j) * nxy;
#pragma unroll
        for (int r = 0; r < BOXR; ++r)
          if (box_dst[r] >= 0) cp_async_v<VEC>(&sm.sG[j][box_dst[r]], bj + box_src[r]);
      }
      cp_commit();
    }
    return true;
  };
  auto wait_box = [&](bool issued) {
    if (!issued) return;
    if (USE_TMA && box_interior) {
      mbar_wait(&sm.bar_box, ph_box);
      ph_box ^= 1;
    } else {
      cp_wait<0>();  // only box copies use cp.async groups
    }
  };
  // ---- copy issue: f, g of the tile at plane zp (always a local plane) into sm.sT
  // dist 0: f slots 0..4 | 10..18 | 28..32 -> sTf;  dist 1: g slots 5..9 | 19..27 | 33..37 -> sTg
  auto issue_tile = [&](int zp, int dist) {
    double(*dst)[NT] = dist == 0 ? sm.sTf : sm.sTg;
    if constexpr (USE_TMA) {
      if (zp < zB && tid == 0) {
        unsigned long long* bar = dist == 0 ? &sm.bar_f : &sm.bar_g;
        const int cp0 = (zp + GZ) * NSLOT + (dist == 0 ? 0 : 5);
        fence_proxy_async();
        mbar_expect_tx(bar, TILE_BYTES);
        tma_load_3d(&dst[0][0], &tm_t5, x0, y0, cp0, bar, pol_first);
        tma_load_3d(&dst[5][0], &tm_t9, x0, y0, cp0 + (dist == 0 ? 10 : 14), bar, pol_first);
        tma_load_3d(&dst[14][0], &tm_t5, x0, y0, cp0 + 28, bar, pol_first);
      }
    } else {
      // odd nx: one 8-byte copy per (component, site), wrap only for partial tiles
      if (zp < zB) {
        const double* base =
            A + (long long)(zp + GZ) * G.plane + (long long)wrapy(y0 + ly) * G.nx + wrapx(x0 + lx);
#pragma unroll
        for (int j = 0; j < Q; ++j)
          cp_async_v<1>(&dst[j][tid], base + (long long)(dist == 0 ? fslot_of_rank(j) : gslot_of_rank(j)) * nxy);
      }
      cp_commit();
    }
  };
  auto wait_tile = [&](int dist) {
    if constexpr (USE_TMA) {
      if (dist == 0) {
        mbar_wait(&sm.bar_f, ph_f);
        ph_f ^= 1;
      } else {
        mbar_wait(&sm.bar_g, ph_g);
        ph_g ^= 1;
      }
    } else {
      cp_wait<0>();
    }
  };
  // ---- phi of plane zp on the box -> ring (from sG, or from the ghost phi planes)
  auto make_phi = [&](int zp) {
    bool ghost;
    const int zs = zsrc(zp, ghost);
    double* ring = sm.sPhi[slot5(zp)];
    for (int b = tid; b < NB; b += NT) {
      double v;
      if (ghost) {
        const int gx = wrapx(x0 - 2 + b % BX), gy = wrapy(y0 - 2 + b / BX);
        LB_CHECK(hl, zs >= -GP && zs < G.nzl + GP && gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny);
        v = ldg(phig + phi_plane_index(G, zs) + (long long)gy * G.nx + gx);
      } else {
        v = sm.sG[grank(0)][b];  // A.3, canonical order (same as phi_sum)
#pragma unroll
        for (int i = 1; i < Q; ++i) v += sm.sG[grank(i)][b];
      }
      ring[b] = v;
    }
  };
  // ---- chemical stress on plane zp over the P box (needs phi planes zp-1..zp+1)
  auto compute_P = [&](int zp) {
    const double* f0 = sm.sPhi[slot5(zp - 1)];
    const double* f1 = sm.sPhi[slot5(zp)];
    const double* f2 = sm.sPhi[slot5(zp + 1)];
    for (int e = tid; e < NP; e += NT) {
      const int c = (e / PX + 1) * BX + (e % PX + 1);
      const double ph = f1[c];
      const double xp = f1[c + 1], xm = f1[c - 1];
      const double yp = f1[c + BX], ym = f1[c - BX];
      const double zp_ = f2[c], zm = f0[c];
      const double lap = (xp + xm) + (yp + ym) + (zp_ + zm) - 6.0 * ph;  // A.2
      double P[6];
      stress6(p, ph, 0.5 * (xp - xm), 0.5 * (yp - ym), 0.5 * (zp_ - zm), lap, P);
#pragma unroll
      for (int q = 0; q < 6; ++q) sm.sP[q][e] = P[q];
    }
  };
  // ---- own-site pieces of F = -div P (A.5): P_az, and the b = x, y terms
  auto own_P = [&](double Pz[3], double Fxy[3]) {
    const int e = (ly + 1) * PX + (lx + 1);
    const auto& P = sm.sP;
    Pz[0] = P[PXZ][e];
    Pz[1] = P[PYZ][e];
    Pz[2] = P[PZZ][e];
    Fxy[0] = -0.5 * (P[PXX][e + 1] - P[PXX][e - 1]) - 0.5 * (P[PXY][e + PX] - P[PXY][e - PX]);
    Fxy[1] = -0.5 * (P[PXY][e + 1] - P[PXY][e - 1]) - 0.5 * (P[PYY][e + PX] - P[PYY][e - PX]);
    Fxy[2] = -0.5 * (P[PXZ][e + 1] - P[PXZ][e - 1]) - 0.5 * (P[PYZ][e + PX] - P[PYZ][e - PX]);
  };

  // ---- own-site P (all six components), for the stress-in-equilibrium collision
  auto own_P6 = [&](double P6[6]) {
    const int e = (ly + 1) * PX + (lx + 1);
#pragma unroll
    for (int q = 0; q < 6; ++q) P6[q] = sm.sP[q][e];
  };

  // ---- prologue: phi on zA-2 .. zA+1; P on zA-1, zA; then prime the streams
  issue_tile(zA, 0);
  for (int zp = zA - 2; zp <= zA + 1; ++zp) {
    wait_box(issue_box(zp));
    __syncthreads();
    make_phi(zp);
    __syncthreads();
  }
  double Pz_prev[3] = {0, 0, 0}, Pz_cur[3] = {0, 0, 0}, Fxy_cur[3] = {0, 0, 0};
  double P6_cur[6] = {0, 0, 0, 0, 0, 0};  // COLL 1: P at this site, plane k
  {
    compute_P(zA - 1);
    __syncthreads();
    double unused[3];
    own_P(Pz_prev, unused);
    __syncthreads();
    compute_P(zA);
    __syncthreads();
    own_P(Pz_cur, Fxy_cur);
    if (COLL == 1) own_P6(P6_cur);
  }
  bool box_issued = issue_box(zA + 2);
  issue_tile(zA, 1);

  // push targets: wrapped neighbour columns/rows of this thread's site
  const int xm1 = wrapx(x - 1), xp1 = wrapx(x + 1), ym1 = wrapy(y - 1), yp1 = wrapy(y + 1);
  const int cbox = (ly + 2) * BX + (lx + 2);

  for (int k = zA; k < zB; ++k) {
    // f(k) to registers, then free sTf for f(k+1): a whole iteration of lead time
    double f[Q], g[Q];
    wait_tile(0);
#pragma unroll
    for (int i = 0; i < Q; ++i) f[i] = sm.sTf[frank(i)][tid];
    wait_box(box_issued);  // g(k+2) box landed
    __syncthreads();       // sTf consumed by all threads; sG visible
    issue_tile(k + 1, 0);
    double Pz_next[3] = {0, 0, 0}, Fxy_next[3] = {0, 0, 0};
    double P6_next[6] = {0, 0, 0, 0, 0, 0};
    make_phi(k + 2);
    __syncthreads();  // sG consumed, ring written
    box_issued = k + 1 < zB ? issue_box(k + 3) : false;
    compute_P(k + 1);
    __syncthreads();
    own_P(Pz_next, Fxy_next);
    if (COLL == 1) own_P6(P6_next);
    wait_tile(1);  // g(k) tile landed
#pragma unroll
    for (int i = 0; i < Q; ++i) g[i] = sm.sTg[grank(i)][tid];
    __syncthreads();  // sTg consumed
    issue_tile(k + 1, 1);
    double* const zb[3] = {push_plane(G, B, pr, k - 1), push_plane(G, B, pr, k), push_plane(G, B, pr, k + 1)};
    if (active) {
      const double* r0 = sm.sPhi[slot5(k)];
      const double ph = r0[cbox];
      const double lap = (r0[cbox + 1] + r0[cbox - 1]) + (r0[cbox + BX] + r0[cbox - BX]) +
                         (sm.sPhi[slot5(k + 1)][cbox] + sm.sPhi[slot5(k - 1)][cbox]) - 6.0 * ph;
      const double mu = chem_pot(p, ph, lap);
      auto push = [&](int i, double fs, double gs) {
        const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
        const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
        LB_CHECK(hl, xd >= 0 && xd < G.nx && yd >= 0 && yd < G.ny);
        double* d = zb[cz(i) + 1] + (long long)yd * G.nx + xd;  // A.8 push
        __stcs(d + (long long)slot(0, i) * nxy, fs);
        __stcs(d + (long long)slot(1, i) * nxy, gs);
      };
      double rho;
      if constexpr (COLL == 1) {
        rho = collide_mrt(p, f, g, ph, mu, P6_cur, push);
      } else {
        double F[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) F[a] = Fxy_cur[a] - 0.5 * (Pz_next[a] - Pz_prev[a]);
        rho = collide(p, f, g, ph, mu, F, push);
      }
      if (!(rho > 0.0) || !isfinite(rho) || !isfinite(ph)) health_report(hl, G, x, y, k);  // R22
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Pz_prev[a] = Pz_cur[a];
      Pz_cur[a] = Pz_next[a];
      Fxy_cur[a] = Fxy_next[a];
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) P6_cur[q] = P6_next[q];
  }
  cp_wait<0>();
  __syncthreads();  // every thread's pushes before the CTA's publication
  if (tid == 0) {
    health_tick(hl);
  }
}

template <int TY, bool USE_TMA, int COLL>
cudaError_t launch_t(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                     const Launch& ln, const Health& hl, const StepMaps* maps, cudaStream_t st, const Peers& pr) {
  constexpr size_t smem = sizeof(StepSmem<kTX, TY>);
  auto kern = k_step_async<kTX, TY, USE_TMA, COLL>;
  int resid = 0;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), smem, kTX * TY, &resid);
  if (e != cudaSuccess) return e;
  TileOrder ord = ln.order;
  if (ord.resid <= 0) ord.resid = resid;
  static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  const int zc = ln.zc;
  const unsigned nblk = (unsigned)(((G.nx + kTX - 1) / kTX) * ((G.ny + TY - 1) / TY) * ((G.nzl + zc - 1) / zc));
  kern<<<nblk, kTX * TY, smem, st>>>(G, p, A, B, phig, zc, ord, hl, pr, m[0], m[1], m[2], m[3]);
  return cudaGetLastError();
}

template <int TY, bool USE_TMA>
cudaError_t launch_coll(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                        const Launch& ln, const Health& hl, const StepMaps* maps, cudaStream_t st, const Peers& pr) {
  return p.coll == 1 ? launch_t<TY, USE_TMA, 1>(G, p, A, B, phig, ln, hl, maps, st, pr)
                     : launch_t<TY, USE_TMA, 0>(G, p, A, B, phig, ln, hl, maps, st, pr);
}

}  // namespace

cudaError_t prepare_kernel(const void* fn, size_t smem, int threads, int* resid) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> CTAs resident at a time
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({fn, dev});
  if (it != done.end()) {
    *resid = it->second;
    return cudaSuccess;
  }
  if (smem > 48 * 1024 && (e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return e;
  int sms = 0, per_sm = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem)) != cudaSuccess) return e;
  *resid = sms * (per_sm > 0 ? per_sm : 1);
  done[{fn, dev}] = *resid;
  return cudaSuccess;
}

// L2 promotion of the TMA copies (the fill granularity of a miss): tiles and halo boxes
#ifndef LB_TMA_PROMO_TILE
#define LB_TMA_PROMO_TILE CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
#ifndef LB_TMA_PROMO_BOX
#define LB_TMA_PROMO_BOX CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

// buffer viewed as a 3-D fp64 tensor {x: nx, y: ny, component-plane: (nzl+2GZ)*38}
bool encode_dist_map(CUtensorMap* m, const Geom& G, const double* buf, unsigned bx, unsigned by, unsigned bz) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)G.nx, (cuuint64_t)G.ny, (cuuint64_t)(G.nzl + 2 * GZ) * NSLOT};
  cuuint64_t strides[2] = {(cuuint64_t)G.nx * 8, (cuuint64_t)G.nxy * 8};
  cuuint32_t box[3] = {bx, by, bz};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapL2promotion promo = bx % 32 == 0 ? LB_TMA_PROMO_TILE : LB_TMA_PROMO_BOX;  // (tile rows: 32 sites)
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(buf), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// a phi buffer as a 3-D fp64 tensor {x: nx, y: ny, plane: nzl + 2GP} (ghost planes included)
bool encode_phi_map(CUtensorMap* m, const Geom& G, const double* phi, unsigned bx, unsigned by) {
  auto fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)G.nx, (cuuint64_t)G.ny, (cuuint64_t)(G.nzl + 2 * GP)};
  cuuint64_t strides[2] = {(cuuint64_t)G.nx * 8, (cuuint64_t)G.nxy * 8};
  cuuint32_t box[3] = {bx, by, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(phi), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tile rows of the step kernel.  Even nx (TMA rows): 32 x 8 tiles and the
// warp-specialised kernel for every plane size -- measured in round 1 against
// 32 x 4 tiles of the tile kernel (two CTAs per SM): +12% at 128^3, +17% at 64^3,
// +30% at 256^3, +7% at 256 x 256 x 32 (the 8-GPU slab of 256^3), equal at
// 512 x 512 x 64.  Odd nx (per-thread copies): 32 x 4 tiles
// unless the plane has >= 4 x SMs tiles of 32 x 8.
int step_tile_rows(const Geom& G, int num_sms) {
  if (G.nx % 2 == 0) return 8;
  const long long tiles8 = (long long)((G.nx + kTX - 1) / kTX) * ((G.ny + 7) / 8);
  return tiles8 >= 4LL * num_sms ? 8 : 4;
}

bool make_step_maps(const Geom& G, const double* buf, int ty, StepMaps* out) {
  out->ok = false;
  out->ty = ty;
  if (G.nx % 2 != 0) return true;  // odd rows: the cp.async path needs no maps
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(out->m);
  const unsigned BX = kTX + 4, BY = ty + 4;
  if (!encode_dist_map(&m[0], G, buf, kTX, ty, 5)) return false;
  if (!encode_dist_map(&m[1], G, buf, kTX, ty, 9)) return false;
  if (!encode_dist_map(&m[2], G, buf, BX, BY, 5)) return false;
  if (!encode_dist_map(&m[3], G, buf, BX, BY, 9)) return false;
  out->ok = true;
  return true;
}

// Planes per z-chunk (one CTA = one tile x one z-chunk).
// 32 x 8 tiles (one CTA per SM), from round-1 sweeps:
//  * fewer tiles than SMs: one wave -- as many chunks as fit beside each other on
//    the SMs (>= 8 planes each): 128^3 -> 2 x 64 planes, 64^3 -> 8 x 8;
//  * otherwise chunks of 32 planes (best at 512 x 512 x 64 and 256^3: more planes
//    per chunk lost up to 8%), or 16 when 32 leaves fewer than 4 waves of CTAs
//    (256 x 256 x 64: +2%).
// 32 x 4 tiles (odd nx): enough CTAs to fill the GPU several times, chunks >= 8.
int step_zchunk(const Geom& G, int num_sms, int ty) {
  const long long tiles = (long long)((G.nx + kTX - 1) / kTX) * ((G.ny + ty - 1) / ty);
  const long long maxchunks = G.nzl >= 16 ? G.nzl / 8 : 1;
  long long nchunks;
  if (ty == 8) {
    if (tiles < num_sms) {
      nchunks = num_sms / tiles;
    } else {
      int zc = G.nzl < 32 ? G.nzl : 32;
      if (zc == 32 && tiles * ((G.nzl + 31) / 32) < 4LL * num_sms) zc = 16;
      nchunks = (G.nzl + zc - 1) / zc;
    }
  } else {
    const long long target = (long long)kStepWaves * num_sms;
    nchunks = (target + tiles - 1) / tiles;
  }
  if (nchunks > maxchunks) nchunks = maxchunks;
  if (nchunks < 1) nchunks = 1;
  return (int)((G.nzl + nchunks - 1) / nchunks);
}

cudaError_t prepare_step_kernels() {
  int r = 0;
  cudaError_t e = cudaSuccess;
  auto prep = [&](const void* fn, size_t smem, int threads) {
    if (e == cudaSuccess) e = prepare_kernel(fn, smem, threads, &r);
  };
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 8, true, 0>), sizeof(StepSmem<kTX, 8>), kTX * 8);
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 8, true, 1>), sizeof(StepSmem<kTX, 8>), kTX * 8);
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 8, false, 0>), sizeof(StepSmem<kTX, 8>), kTX * 8);
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 8, false, 1>), sizeof(StepSmem<kTX, 8>), kTX * 8);
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 4, true, 0>), sizeof(StepSmem<kTX, 4>), kTX * 4);
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 4, true, 1>), sizeof(StepSmem<kTX, 4>), kTX * 4);
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 4, false, 0>), sizeof(StepSmem<kTX, 4>), kTX * 4);
  prep(reinterpret_cast<const void*>(k_step_async<kTX, 4, false, 1>), sizeof(StepSmem<kTX, 4>), kTX * 4);
  return e;
}

cudaError_t launch_step(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                        const Launch& ln, const Health& hl, const StepMaps* maps, cudaStream_t st, const Peers& pr) {
  if (!maps) return cudaErrorInvalidValue;
  const bool tma = maps->ok;
  if (maps->ty == 8)
    return tma ? launch_coll<8, true>(G, p, A, B, phig, ln, hl, maps, st, pr)
               : launch_coll<8, false>(G, p, A, B, phig, ln, hl, maps, st, pr);
  return tma ? launch_coll<4, true>(G, p, A, B, phig, ln, hl, maps, st, pr)
             : launch_coll<4, false>(G, p, A, B, phig, ln, hl, maps, st, pr);
}

}  // namespace lbk
