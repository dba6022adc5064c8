// lb_step.cu -- the fused single-pass D3Q19 binary-fluid step for sm_100a.
//
// One kernel does every row of the hot path for a z-slab (
// "Order Parameter Gradients", "Chemical Stress", force =
// "divergence of the 'Chemical stress'", "Collision", "Propagation"):
//
//   CTA   = a TX x TY tile of (x, y) columns marching in z over a chunk of
//           planes (2.5-D blocking); one thread per column.
//   smem  = sT : f and g of the tile on the plane being collided      (async-copied)
//           sG : g on the tile + 2-site halo, two planes ahead         (async-copied)
//           sPhi: ring of 5 phi planes on the halo box (phi = sum_i g_i recomputed
//                 for the halo: single pass, no phi round trip through HBM)
//           sP : chemical stress P_ab of one plane on the tile + 1-site halo
//   regs  = the z-column pieces of F = -div P: P_az on planes k-1, k, k+1 and the
//           in-plane divergence of plane k+1.
//
// Loads never occupy registers while in flight: both streams (sT, sG) are
// cp.async copies issued one stage ahead, so every SM always has one of them
// outstanding while it computes on the other.
//
// Iteration k (collide plane k), cp.async groups in commit order:
//   wait sG = g(k+2) box           -> phi(k+2) into the ring; issue sG = g(k+3)
//   P(k+1) on the P box            -> own P_az(k+1), in-plane div P(k+1)
//   wait sT = f, g(k) tile         -> collide, push f*, g* to x + c_i (A.8);
//                                     issue sT = f, g(k+1)
// HBM traffic per site: f and g read once, written once = 608 B;
// the halo part of sG and the re-read of g(k) hit L2.
// Slab edges (z < 0 or z >= nzl, multi-slab only) take phi from the ghost planes
// of the phi buffer, filled by K_phi + the halo exchange.
#include <cuda_runtime.h>

#include "lb_device.cuh"

namespace lbk {
namespace {

__device__ __forceinline__ int slot5(int z) {
  const int s = z % 5;
  return s < 0 ? s + 5 : s;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int VEC>
__device__ __forceinline__ void cp_async(void* dst, const double* src) {
  if constexpr (VEC == 2)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// slots of the 19 g components in canonical order
__device__ __forceinline__ constexpr int gslot(int i) { return slot(1, i); }

template <int TX, int TY>
struct StepSmem {
  static constexpr int BX = TX + 4, BY = TY + 4, NB = BX * BY;  // phi box: tile + 2 halo
  static constexpr int PX = TX + 2, PY = TY + 2, NP = PX * PY;  // P box: tile + 1 halo
  static constexpr int NTILE = TX * TY;
  double sT[NSLOT][NTILE];  // f, g of the tile, slot order
  double sG[Q][NB];         // g on the box, canonical order
  double sPhi[5][NB];
  double sP[6][NP];
};

template <int TX, int TY, int VEC>
__global__ void __launch_bounds__(TX* TY, 1)
    k_step_async(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B,
                 const double* __restrict__ phig, int zc, int* __restrict__ flag) {
  using S = StepSmem<TX, TY>;
  constexpr int NT = TX * TY;
  constexpr int BX = S::BX, NB = S::NB, PX = S::PX, NP = S::NP;
  constexpr int NBR = (NB + NT - 1) / NT;
  constexpr int NPR = (NP + NT - 1) / NT;
  // copy work: units of VEC doubles along x
  constexpr int TROWU = TX / VEC;                  // units per tile row
  constexpr int BROWU = BX / VEC;                  // units per box row
  constexpr int NTU = NSLOT * TY * TROWU;          // tile units
  constexpr int NBU = Q * S::BY * BROWU;           // box units
  static_assert(TX % VEC == 0 && BX % VEC == 0, "tile width must be a multiple of VEC");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const int tid = threadIdx.x;
  const int lx = tid % TX, ly = tid / TX;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int x = x0 + lx, y = y0 + ly;
  const bool active = (x < G.nx) && (y < G.ny);
  const int zA = blockIdx.z * zc;
  const int zB = min(zA + zc, G.nzl);
  const long long nxy = G.nxy;

  auto wrapx = [&](int v) { v %= G.nx; return v < 0 ? v + G.nx : v; };
  auto wrapy = [&](int v) { v %= G.ny; return v < 0 ? v + G.ny : v; };
  auto zsrc = [&](int zp, bool& ghost) {
    ghost = false;
    if (G.zwrap) { zp %= G.nzl; return zp < 0 ? zp + G.nzl : zp; }
    ghost = zp < 0 || zp >= G.nzl;
    return zp;
  };

  // Copy plans, fixed over z: each thread copies the same (row, column-unit)
  // positions of every component; only the component (slot) changes.
  //   box : per component BY*BROWU units, thread takes units tid + r*NT
  //   tile: per slot TY*TROWU units; NT is a multiple of it, so a thread's
  //         position is fixed and it covers slots s0, s0 + NT/(TY*TROWU), ...
  constexpr int BOXU = S::BY * BROWU;
  constexpr int BOXR = (BOXU + NT - 1) / NT;
  constexpr int TILEU = TY * TROWU;
  static_assert(NT % TILEU == 0, "tile copy plan needs NT % (TY * TX/VEC) == 0");
  constexpr int TSTEP = NT / TILEU;
  long long box_src[BOXR];
  int box_dst[BOXR];
#pragma unroll
  for (int r = 0; r < BOXR; ++r) {
    const int u = tid + r * NT;
    const int row = u / BROWU, cu = u - row * BROWU;
    box_src[r] = (long long)wrapy(y0 - 2 + row) * G.nx + wrapx(x0 - 2 + cu * VEC);
    box_dst[r] = u < BOXU ? row * BX + cu * VEC : -1;
  }
  const int t_unit = tid % TILEU, t_s0 = tid / TILEU;
  const long long tile_src =
      (long long)wrapy(y0 + t_unit / TROWU) * G.nx + wrapx(x0 + (t_unit % TROWU) * VEC);  // wrap: partial tiles
  const int tile_dst = (t_unit / TROWU) * TX + (t_unit % TROWU) * VEC;

  // ---- async copy issue: g box of plane zp into sm.sG (nothing if ghost plane)
  auto issue_box = [&](int zp) {
    bool ghost;
    const int zs = zsrc(zp, ghost);
    if (!ghost) {
      const double* base = A + (long long)(zs + GZ) * G.plane;
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const double* bi = base + (long long)gslot(i) * nxy;
#pragma unroll
        for (int r = 0; r < BOXR; ++r)
          if (box_dst[r] >= 0) cp_async<VEC>(&sm.sG[i][box_dst[r]], bi + box_src[r]);
      }
    }
    cp_commit();
  };
  // ---- async copy issue: f, g of the tile at plane zp (always interior) into sm.sT
  auto issue_tile = [&](int zp) {
    if (zp < zB) {
      const double* base = A + (long long)(zp + GZ) * G.plane + tile_src;
#pragma unroll
      for (int s = t_s0; s < NSLOT; s += TSTEP) cp_async<VEC>(&sm.sT[s][tile_dst], base + (long long)s * nxy);
    }
    cp_commit();
  };
  // ---- phi of plane zp on the box -> ring (from sG, or from the ghost phi planes)
  auto make_phi = [&](int zp) {
    bool ghost;
    const int zs = zsrc(zp, ghost);
    double* ring = sm.sPhi[slot5(zp)];
#pragma unroll
    for (int r = 0; r < NBR; ++r) {
      const int b = tid + r * NT;
      if (b < NB) {
        double v;
        if (ghost) {
          const int gx = wrapx(x0 - 2 + b % BX), gy = wrapy(y0 - 2 + b / BX);
          v = ldg(phig + phi_plane_index(G, zs) + (long long)gy * G.nx + gx);
        } else {
          v = sm.sG[0][b];  // A.3, canonical order (same as phi_sum)
#pragma unroll
          for (int i = 1; i < Q; ++i) v += sm.sG[i][b];
        }
        ring[b] = v;
      }
    }
  };
  // ---- chemical stress on plane zp over the P box (needs phi planes zp-1..zp+1)
  auto compute_P = [&](int zp) {
    const double* f0 = sm.sPhi[slot5(zp - 1)];
    const double* f1 = sm.sPhi[slot5(zp)];
    const double* f2 = sm.sPhi[slot5(zp + 1)];
#pragma unroll
    for (int r = 0; r < NPR; ++r) {
      const int e = tid + r * NT;
      if (e < NP) {
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

  // ---- prologue: phi on zA-2 .. zA+1; P on zA-1, zA; then prime both streams
  for (int zp = zA - 2; zp <= zA + 1; ++zp) {
    issue_box(zp);
    cp_wait<0>();
    __syncthreads();
    make_phi(zp);
    __syncthreads();
  }
  compute_P(zA - 1);
  __syncthreads();
  double Pz_prev[3], Pz_cur[3], Fxy_cur[3], unused[3];
  own_P(Pz_prev, unused);
  __syncthreads();
  compute_P(zA);
  __syncthreads();
  own_P(Pz_cur, Fxy_cur);
  issue_box(zA + 2);
  issue_tile(zA);

  // push targets: wrapped neighbour columns/rows of this thread's site
  const int xm1 = wrapx(x - 1), xp1 = wrapx(x + 1), ym1 = wrapy(y - 1), yp1 = wrapy(y + 1);
  const int ct = ly * TX + lx;
  const int cbox = (ly + 2) * BX + (lx + 2);

  for (int k = zA; k < zB; ++k) {
    // pending groups: [box(k+2), tile(k)]
    cp_wait<1>();
    __syncthreads();
    make_phi(k + 2);
    __syncthreads();  // sG consumed, ring written
    if (k + 1 < zB)
      issue_box(k + 3);  // pending: [tile(k), box(k+3)]
    else
      cp_commit();
    compute_P(k + 1);
    __syncthreads();
    double Pz_next[3], Fxy_next[3];
    own_P(Pz_next, Fxy_next);
    cp_wait<1>();  // tile(k) landed
    __syncthreads();
    if (active) {
      const double* r0 = sm.sPhi[slot5(k)];
      const double ph = r0[cbox];
      const double lap = (r0[cbox + 1] + r0[cbox - 1]) + (r0[cbox + BX] + r0[cbox - BX]) +
                         (sm.sPhi[slot5(k + 1)][cbox] + sm.sPhi[slot5(k - 1)][cbox]) - 6.0 * ph;
      const double mu = chem_pot(p, ph, lap);
      double F[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) F[a] = Fxy_cur[a] - 0.5 * (Pz_next[a] - Pz_prev[a]);
      double f[Q], g[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        f[i] = sm.sT[slot(0, i)][ct];
        g[i] = sm.sT[slot(1, i)][ct];
      }
      const long long zoff[3] = {(long long)(G.zwrap ? wrap_n(k - 1, G.nzl) : k - 1) + GZ,
                                 (long long)k + GZ,
                                 (long long)(G.zwrap ? wrap_n(k + 1, G.nzl) : k + 1) + GZ};
      const double rho = collide(p, f, g, ph, mu, F, [&](int i, double fs, double gs) {
        const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
        const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
        double* d = B + zoff[cz(i) + 1] * G.plane + (long long)yd * G.nx + xd;  // A.8 push
        __stcs(d + (long long)slot(0, i) * nxy, fs);
        __stcs(d + (long long)slot(1, i) * nxy, gs);
      });
      if (!(rho > 0.0) || !isfinite(rho) || !isfinite(ph)) *flag = 1;  // R22
    }
    __syncthreads();  // sT consumed
    issue_tile(k + 1);  // pending: [box(k+3), tile(k+1)]
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Pz_prev[a] = Pz_cur[a];
      Pz_cur[a] = Pz_next[a];
      Fxy_cur[a] = Fxy_next[a];
    }
  }
  cp_wait<0>();
}

#ifndef LB_STEP_TX
#define LB_STEP_TX 32
#endif
#ifndef LB_STEP_TY
#define LB_STEP_TY 8
#endif
constexpr int kTX = LB_STEP_TX, kTY = LB_STEP_TY;

template <int VEC>
cudaError_t launch_t(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig, int zc,
                     int* flag, cudaStream_t st) {
  constexpr size_t smem = sizeof(StepSmem<kTX, kTY>);
  auto kern = k_step_async<kTX, kTY, VEC>;
  static bool attr = false;  // per-process, per-instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((G.nx + kTX - 1) / kTX, (G.ny + kTY - 1) / kTY, (G.nzl + zc - 1) / zc);
  kern<<<grid, kTX * kTY, smem, st>>>(G, p, A, B, phig, zc, flag);
  return cudaGetLastError();
}

}  // namespace

// number of z-chunks: enough CTAs to fill the GPU several times, chunks >= 8 planes
int step_zchunk(const Geom& G, int num_sms) {
  const long long tiles = (long long)((G.nx + kTX - 1) / kTX) * ((G.ny + kTY - 1) / kTY);
  const long long target = 4LL * num_sms;
  long long nchunks = (target + tiles - 1) / tiles;
  const long long maxchunks = G.nzl >= 16 ? G.nzl / 8 : 1;
  if (nchunks > maxchunks) nchunks = maxchunks;
  if (nchunks < 1) nchunks = 1;
  return (int)((G.nzl + nchunks - 1) / nchunks);
}

cudaError_t launch_step(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig, int zc,
                        int* flag, cudaStream_t st) {
  // 16-byte copies need even rows (every row start then 16-byte aligned)
  if (G.nx % 2 == 0) return launch_t<2>(G, p, A, B, phig, zc, flag, st);
  return launch_t<1>(G, p, A, B, phig, zc, flag, st);
}

}  // namespace lbk
