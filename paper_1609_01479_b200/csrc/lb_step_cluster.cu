// lb_step_cluster.cu -- the fused single-pass step with phi halos shared through
// distributed shared memory inside a thread-block cluster (sm_90+/sm_100a).
//
// Same step and same arithmetic as lb_step.cu (rows a1-a7 of SURVEY 8(a); PAPER.md
// P:168-190), but the order-parameter halo is not recomputed from a halo box of g:
//
//   cluster = CLX x CLY CTAs (2 x 4) tiling a 64 x 16 region of the plane; each CTA
//             owns a 32 x 4 tile and marches in z (2.5-D blocking).
//   per plane, each CTA computes phi = sum_i g_i only for its own tile and for the
//             part of the region's 2-site halo ring that lies in its own box
//             (strips at the region edge), publishes it in its shared-memory phi
//             ring, passes one cluster barrier, and gathers the rest of its
//             (TX+4) x (TY+4) phi box from the owning CTAs' rings (ld.shared::cluster).
//   loads   = f tile (TMA, 3 boxes), g tile two planes ahead into a 3-plane ring
//             (TMA, 3 boxes), edge strips of g (cp.async, ~10% of a tile): every g
//             value crosses L2 -> SM about 1.3 times instead of 2.25 times.
//
// Sums, stencils and the collision are the same device functions as every other
// kernel (lb_device.cuh), so results are bitwise identical to lb_step.cu's kernel.
// Used when nx % 64 == 0, ny % 16 == 0 and nx even; otherwise lb_step.cu.
#include "lb_device.cuh"
#include "lb_tma.cuh"

namespace lbk {
namespace {

constexpr int CTX = 32, CTY = 4;  // tile
constexpr int CLX = 2, CLY = 4;   // cluster (portable size 8)
constexpr int NT = CTX * CTY;
constexpr int BX = CTX + 4, BY = CTY + 4, NB = BX * BY;  // phi box
constexpr int PX = CTX + 2, PY = CTY + 2, NP = PX * PY;  // P box
constexpr int NBR = (NB + NT - 1) / NT;

struct alignas(128) ClusterSmem {
  alignas(128) double sF[Q][NT];      // f of the tile, f-rank order (TMA)
  alignas(128) double sGr[3][Q][NT];  // g of the tile, planes k, k+1, k+2 (ring), g-rank order (TMA)
  alignas(16) double sLR[Q][CTY][2];  // g of the left/right halo strip (region edge), g-rank order
  alignas(16) double sC[Q][2][2];     // g of the region-corner 2 x 2 piece
  alignas(16) double sTB[Q][2][CTX];  // g of the top/bottom halo strip
  double sPhi[5][NB];                 // phi box ring
  double sP[6][NP];
  unsigned long long bar_f, bar_g;
};

__device__ __forceinline__ int mod_n(int v, int n) {
  v %= n;
  return v < 0 ? v + n : v;
}

template <int MODE>
__global__ void __launch_bounds__(NT, 2)
    k_step_cluster(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B,
                   const double* __restrict__ phig, int zc, int* __restrict__ flag, Peers pr,
                   const __grid_constant__ CUtensorMap tm_t5, const __grid_constant__ CUtensorMap tm_t9) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ClusterSmem& sm = *reinterpret_cast<ClusterSmem*>(smem_raw);
  constexpr unsigned TILE_BYTES = Q * NT * 8;

  const int tid = threadIdx.x;
  const int lx = tid % CTX, ly = tid / CTX;
  const int x0 = blockIdx.x * CTX, y0 = blockIdx.y * CTY;
  const int x = x0 + lx, y = y0 + ly;
  const int zA = blockIdx.z * zc;
  const int zB = min(zA + zc, G.nzl);
  const long long nxy = G.nxy;
  const unsigned myrank = cluster_ctarank();
  const int cxi = (int)(myrank % CLX), cyi = (int)(myrank / CLX);  // position in the cluster
  const int rx0 = x0 - CTX * cxi, ry0 = y0 - CTY * cyi;            // region origin

  auto zsrc = [&](int zp, bool& ghost) {
    ghost = !G.zwrap && (zp < 0 || zp >= G.nzl);
    return G.zwrap ? mod_n(zp, G.nzl) : zp;
  };

  // ---- ownership of this CTA's phi-box positions (fixed over z): the owner of a
  // position (u, v) relative to the region is the tile containing it, clamped to
  // the region (outside positions belong to the nearest edge CTA).
  int own_b[NBR], src_rank[NBR], src_b[NBR];
#pragma unroll
  for (int r = 0; r < NBR; ++r) {
    const int b = tid + r * NT;
    own_b[r] = 0;
    src_rank[r] = 0;
    src_b[r] = -1;
    if (b < NB) {
      const int u = x0 - 2 + b % BX - rx0, v = y0 - 2 + b / BX - ry0;
      const int px = u < 0 ? 0 : (u >= CLX * CTX ? CLX - 1 : u / CTX);
      const int py = v < 0 ? 0 : (v >= CLY * CTY ? CLY - 1 : v / CTY);
      if (px == cxi && py == cyi) {
        own_b[r] = 1;
      } else {
        src_rank[r] = px + CLX * py;
        src_b[r] = (v - CTY * py + 2) * BX + (u - CTX * px + 2);
      }
    }
  }
  // strips this CTA owns (region edge): left/right columns, top/bottom rows, corner
  const bool has_lr = true;  // CLX == 2: every CTA touches the left or the right region edge
  const int lr_x = cxi == 0 ? x0 - 2 : x0 + CTX;  // first of the 2 strip columns (unwrapped)
  const bool has_tb = cyi == 0 || cyi == CLY - 1;
  const int tb_y = cyi == 0 ? y0 - 2 : y0 + CTY;  // first of the 2 strip rows (unwrapped)

  unsigned long long pol_first = 0, pol_last = 0;
  if (tid == 0) {
    pol_first = policy_evict_first();
    pol_last = policy_evict_last();
    mbar_init(&sm.bar_f, 1);
    mbar_init(&sm.bar_g, 1);
    fence_barrier_init();
  }
  __syncthreads();
  unsigned ph_f = 0, ph_g = 0;

  // ---- copies
  auto issue_f = [&](int zp) {
    if (zp < zB && tid == 0) {
      const int cp0 = (zp + GZ) * NSLOT;
      fence_proxy_async();
      mbar_expect_tx(&sm.bar_f, TILE_BYTES);
#pragma unroll
      for (int r = 0; r < 3; ++r)
        tma_load_3d(&sm.sF[run_rank0(r)][0], r == 1 ? &tm_t9 : &tm_t5, x0, y0, cp0 + run_first(0, r), &sm.bar_f,
                    pol_first);
    }
  };
  // g tile of plane zp into ring slot zp % 3 (TMA) and the strips (cp.async);
  // returns false for a ghost plane
  auto issue_g = [&](int zp) -> bool {
    bool ghost;
    const int zs = zsrc(zp, ghost);
    if (ghost) return false;
    if (tid == 0) {
      const int cp0 = (zs + GZ) * NSLOT;
      fence_proxy_async();
      mbar_expect_tx(&sm.bar_g, TILE_BYTES);
#pragma unroll
      for (int r = 0; r < 3; ++r)
        tma_load_3d(&sm.sGr[mod_n(zp, 3)][run_rank0(r)][0], r == 1 ? &tm_t9 : &tm_t5, x0, y0,
                    cp0 + run_first(1, r), &sm.bar_g, pol_last);
    }
    const double* base = A + (long long)(zs + GZ) * G.plane;
    // left/right strip: 19 comps x CTY rows x 1 pair (16 B)
    for (int u = tid; u < Q * CTY; u += NT) {
      const int j = u / CTY, row = u % CTY;
      cp_async_v<2>(&sm.sLR[j][row][0], base + (long long)gslot_of_rank(j) * nxy +
                                             (long long)mod_n(y0 + row, G.ny) * G.nx + mod_n(lr_x, G.nx));
    }
    if (has_tb) {
      // top/bottom strip: 19 comps x 2 rows x CTX/2 pairs; corner: 19 x 2 rows x 1 pair
      for (int u = tid; u < Q * 2 * (CTX / 2); u += NT) {
        const int j = u / (CTX), rem = u % CTX, row = rem / (CTX / 2), pr = rem % (CTX / 2);
        cp_async_v<2>(&sm.sTB[j][row][2 * pr], base + (long long)gslot_of_rank(j) * nxy +
                                                   (long long)mod_n(tb_y + row, G.ny) * G.nx + (x0 + 2 * pr));
      }
      for (int u = tid; u < Q * 2; u += NT) {
        const int j = u / 2, row = u % 2;
        cp_async_v<2>(&sm.sC[j][row][0], base + (long long)gslot_of_rank(j) * nxy +
                                             (long long)mod_n(tb_y + row, G.ny) * G.nx + mod_n(lr_x, G.nx));
      }
    }
    cp_commit();
    return true;
  };
  auto wait_g = [&](bool issued) {
    if (!issued) return;
    mbar_wait(&sm.bar_g, ph_g);
    ph_g ^= 1;
    cp_wait<0>();
  };

  // ---- phi of plane zp at the positions this CTA owns -> its box ring slot
  auto own_phi = [&](int zp) {
    bool ghost;
    const int zs = zsrc(zp, ghost);
    double* ring = sm.sPhi[mod_n(zp, 5)];
    const double* gt = &sm.sGr[mod_n(zp, 3)][0][0];
#pragma unroll
    for (int r = 0; r < NBR; ++r) {
      const int b = tid + r * NT;
      if (b < NB && own_b[r]) {
        const int bx = b % BX, by = b / BX;
        double v;
        if (ghost) {
          v = ldg(phig + phi_plane_index(G, zs) + (long long)mod_n(y0 - 2 + by, G.ny) * G.nx +
                  mod_n(x0 - 2 + bx, G.nx));
        } else {
          // the g source of box position (bx, by): tile, left/right strip, top/bottom strip or corner
          const bool in_x = bx >= 2 && bx < CTX + 2, in_y = by >= 2 && by < CTY + 2;
          const double* src;
          int stride;
          if (in_x && in_y) {
            src = gt + (by - 2) * CTX + (bx - 2);
            stride = NT;
          } else if (in_y) {
            src = &sm.sLR[0][by - 2][bx < 2 ? bx : bx - CTX - 2];
            stride = CTY * 2;
          } else if (in_x) {
            src = &sm.sTB[0][by < 2 ? by : by - CTY - 2][bx - 2];
            stride = 2 * CTX;
          } else {
            src = &sm.sC[0][by < 2 ? by : by - CTY - 2][bx < 2 ? bx : bx - CTX - 2];
            stride = 4;
          }
          v = src[grank(0) * stride];  // A.3, canonical order (same as phi_sum)
#pragma unroll
          for (int i = 1; i < Q; ++i) v += src[grank(i) * stride];
        }
        ring[b] = v;
      }
    }
  };
  // ---- the rest of the box from the owners' rings (after a cluster barrier)
  auto gather_phi = [&](int zp) {
    double* ring = sm.sPhi[mod_n(zp, 5)];
#pragma unroll
    for (int r = 0; r < NBR; ++r) {
      const int b = tid + r * NT;
      if (b < NB && !own_b[r]) ring[b] = ld_dsmem(dsmem_addr(&ring[src_b[r]], (unsigned)src_rank[r]));
    }
  };
  // ---- chemical stress on plane zp over the P box (needs phi planes zp-1..zp+1)
  auto compute_P = [&](int zp) {
    const double* f0 = sm.sPhi[mod_n(zp - 1, 5)];
    const double* f1 = sm.sPhi[mod_n(zp, 5)];
    const double* f2 = sm.sPhi[mod_n(zp + 1, 5)];
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

  // ---- prologue: phi on zA-2 .. zA+1 (g of zA, zA+1 stay in the ring); P on zA-1, zA
  cluster_sync();  // every CTA of the cluster has started (its shared memory exists)
  issue_f(zA);
  for (int zp = zA - 2; zp <= zA + 1; ++zp) {
    wait_g(issue_g(zp));
    __syncthreads();
    own_phi(zp);
    __syncthreads();
    cluster_sync_smem();
    gather_phi(zp);
    __syncthreads();
  }
  double Pz_prev[3], Pz_cur[3], Fxy_cur[3], unused[3];
  compute_P(zA - 1);
  __syncthreads();
  own_P(Pz_prev, unused);
  __syncthreads();
  compute_P(zA);
  __syncthreads();
  own_P(Pz_cur, Fxy_cur);
  bool g_issued = issue_g(zA + 2);

  const int xm1 = mod_n(x - 1, G.nx), xp1 = mod_n(x + 1, G.nx), ym1 = mod_n(y - 1, G.ny), yp1 = mod_n(y + 1, G.ny);
  const int cbox = (ly + 2) * BX + (lx + 2);

  for (int k = zA; k < zB; ++k) {
    double f[Q], g[Q];
    mbar_wait(&sm.bar_f, ph_f);  // f(k)
    ph_f ^= 1;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      f[i] = sm.sF[frank(i)][tid];
      g[i] = sm.sGr[mod_n(k, 3)][grank(i)][tid];
    }
    wait_g(g_issued);  // g(k+2) tile and strips
    __syncthreads();   // sF and ring slot k consumed; g(k+2) visible
    issue_f(k + 1);
    own_phi(k + 2);
    __syncthreads();  // strips consumed
    g_issued = (k + 1 < zB) ? issue_g(k + 3) : false;  // into ring slot k % 3
    cluster_sync_smem();  // every CTA published phi(k+2) (its writes completed at the bar.sync above)
    gather_phi(k + 2);
    __syncthreads();
    double Pz_next[3], Fxy_next[3];
    compute_P(k + 1);
    __syncthreads();
    own_P(Pz_next, Fxy_next);
    if (x < G.nx && y < G.ny) {
      double* const zb[3] = {push_plane(G, B, pr, k - 1), push_plane(G, B, pr, k), push_plane(G, B, pr, k + 1)};
      auto emit = [&](int i, double fs, double gs) {
        const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
        const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
        double* d = zb[cz(i) + 1] + (long long)yd * G.nx + xd;  // A.8 push
        __stcs(d + (long long)slot(0, i) * nxy, fs);
        __stcs(d + (long long)slot(1, i) * nxy, gs);
      };
      const double* r0 = sm.sPhi[mod_n(k, 5)];
      const double ph = r0[cbox];
      const double lap = (r0[cbox + 1] + r0[cbox - 1]) + (r0[cbox + BX] + r0[cbox - BX]) +
                         (sm.sPhi[mod_n(k + 1, 5)][cbox] + sm.sPhi[mod_n(k - 1, 5)][cbox]) - 6.0 * ph;
      const double mu = chem_pot(p, ph, lap);
      double F[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) F[a] = Fxy_cur[a] - 0.5 * (Pz_next[a] - Pz_prev[a]);
      const double rho = collide(p, f, g, ph, mu, F, emit);
      if (!(rho > 0.0) || !isfinite(rho) || !isfinite(ph)) *flag = 1;  // R22
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Pz_prev[a] = Pz_cur[a];
      Pz_cur[a] = Pz_next[a];
      Fxy_cur[a] = Fxy_next[a];
    }
  }
  cp_wait<0>();
  if (pr.dn || pr.up) __threadfence_system();  // P2P stores visible before the halo barrier
  cluster_sync();  // no CTA leaves while a peer may still read its shared memory
}

}  // namespace

bool encode_dist_map(CUtensorMap* m, const Geom& G, const double* buf, unsigned bx, unsigned by, unsigned bz) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)G.nx, (cuuint64_t)G.ny, (cuuint64_t)(G.nzl + 2 * GZ) * NSLOT};
  cuuint64_t strides[2] = {(cuuint64_t)G.nx * 8, (cuuint64_t)G.nxy * 8};
  cuuint32_t box[3] = {bx, by, bz};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(buf), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool cluster_step_fits(const Geom& G) { return G.nx % (CLX * CTX) == 0 && G.ny % (CLY * CTY) == 0; }

bool make_cluster_maps(const Geom& G, const double* buf, ClusterMaps* out) {
  out->ok = false;
  if (!cluster_step_fits(G)) return true;
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(out->m);
  if (!encode_dist_map(&m[0], G, buf, CTX, CTY, 5)) return false;
  if (!encode_dist_map(&m[1], G, buf, CTX, CTY, 9)) return false;
  out->ok = true;
  return true;
}

int cluster_zchunk(const Geom& G, int num_sms) {
  if (!cluster_step_fits(G)) return G.nzl;
  const long long tiles = (long long)(G.nx / CTX) * (G.ny / CTY);
  const long long target = 8LL * num_sms;
  long long nchunks = (target + tiles - 1) / tiles;
  const long long maxchunks = G.nzl >= 16 ? G.nzl / 8 : 1;
  if (nchunks > maxchunks) nchunks = maxchunks;
  if (nchunks < 1) nchunks = 1;
  return (int)((G.nzl + nchunks - 1) / nchunks);
}

cudaError_t launch_step_cluster(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                                int zc, int* flag, const ClusterMaps* maps, cudaStream_t st, const Peers& pr) {
  if (!maps || !maps->ok) return cudaErrorInvalidValue;
  constexpr size_t smem = sizeof(ClusterSmem);
  auto kern = k_step_cluster<0>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G.nx / CTX, G.ny / CTY, (G.nzl + zc - 1) / zc);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CLX;
  at[0].val.clusterDim.y = CLY;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, G, p, A, B, phig, zc, flag, pr, m[0], m[1]);
}

}  // namespace lbk
