// lb_step_gr.cu -- the "g ring" variant of the warp-specialised binary-fluid step
// (the default for 32 x 8 tiles of the BGK + force path; lb_step_ws.cu keeps the
// halo-box kernel).  Same arithmetic in the same order as k_step_ws -- the same
// bits -- with a leaner data flow:
//
//   k_step_ws, per plane: f tile + g tile (collision) and the g box = tile + 2-site
//       halo (stencil): 39 + 39 + 66 KB through L2 into shared memory; the g tile
//       of plane j is the interior of the box of plane j two planes earlier.
//   k_step_gr, per plane: the stencil loads the g TILE of plane j+2 (kept in a
//       4-slot ring until the collision of plane j has read it) and only the
//       176-site halo RING (top, bottom 36 x 2, left, right 2 x 8 boxes); the
//       collision reads g from the ring and f of its site straight from global
//       memory (coalesced 256-byte rows, in flight while it waits for the
//       hand-off) -- 39 + 39 + 27 KB per plane (-27% through L2), and the f tile
//       buffer pays for the ring.
//
// Roles (512 threads, setmaxnreg 176 / 80 as k_step_ws):
//   stencil warps: iteration nn (box nn = plane zA - 2 + nn): wait for the g tile
//     and ring of box nn, phi on the box (tile sites from the tile slot, ring
//     sites from the ring buffer; A.3, canonical order), issue the ring of box
//     nn+1, the stress P(plane - 1) on the P box (A.4), F and mu of plane - 2
//     (A.5) handed over through sQ; then wait until the collision has read the g
//     tile of box nn-2 and issue the g tile of box nn+2 into its slot (a plane and
//     a half of lead).  Boxes that are no collision plane (the 2 below zA and
//     the 2 at zB, zB+1) release their slot themselves.
//   collision warps: f of the site (loads), the hand-off (mu, F), g from the tile
//     slot -- then release the slot -- phi = sum g (the same sum as the
//     stencil's), collide (A.6, A.7) and push (A.8).
// Shared memory: 4 g tiles 155,648 B + ring 27,136 + phi ring (4 planes) 13,824 +
// P 16,320 + hand-off 16,384 = 229 KB.  Periodic slabs and z-slabs (ghost planes
// of phi and the peer transport) as k_step_ws; tiles whose halo wraps the lattice
// edge load the ring by per-thread 16-byte cp.async.  nx even (TMA rows).
#include "lb_device.cuh"
#include "lb_tma.cuh"

namespace lbk {
namespace {

constexpr int kGX = 32, kGY = 8, kGT = kGX * kGY;  // tile; collision threads
constexpr int kGS = 256;                            // stencil threads
constexpr int kGBX = kGX + 4, kGBY = kGY + 4, kGNB = kGBX * kGBY;  // phi box: tile + 2
constexpr int kGPX = kGX + 2, kGPY = kGY + 2, kGNP = kGPX * kGPY;  // P box: tile + 1
constexpr int kGNR = 4 * kGBX + 4 * kGY;                             // ring sites (176)
constexpr int kGNPHI = 4;  // phi ring: planes j-1 .. j+2 live while plane j+2 is made

template <int R>
__device__ __forceinline__ int wslot(int z) {
  const int s = z % R;
  return s < 0 ? s + R : s;
}

// ---- the halo ring in shared memory: per f/g slot run r (5, 9, 5 components) the
// four TMA pieces top (36 x 2), bottom (36 x 2), left (2 x 8), right (2 x 8), each
// [component][row][col], each starting 128-byte aligned
__host__ __device__ constexpr int al16(int v) { return (v + 15) / 16 * 16; }
__host__ __device__ constexpr int rlen(int r) { return r == 1 ? 9 : 5; }
__host__ __device__ constexpr int rrank0(int r) { return r == 0 ? 0 : (r == 1 ? 5 : 14); }
__host__ __device__ constexpr int psites(int p) { return p < 2 ? 2 * kGBX : 2 * kGY; }  // sites of piece p
__host__ __device__ constexpr int psize(int r, int p) { return al16(rlen(r) * psites(p)); }
__host__ __device__ constexpr int run_size(int r) { return psize(r, 0) + psize(r, 1) + psize(r, 2) + psize(r, 3); }
__host__ __device__ constexpr int run_base(int r) { return r == 0 ? 0 : (r == 1 ? run_size(0) : run_size(0) + run_size(1)); }
__host__ __device__ constexpr int piece_base(int r, int p) {
  return run_base(r) + (p > 0 ? psize(r, 0) : 0) + (p > 1 ? psize(r, 1) : 0) + (p > 2 ? psize(r, 2) : 0);
}
constexpr int kGRing = run_size(0) + run_size(1) + run_size(2);
// ring site s (0..175: top rows 0-1, bottom rows TY+2, TY+3 (36 each), left columns
// 0-1 and right columns TX+2, TX+3 of box rows 2..TY+1) -> piece, index in piece, box index
__host__ __device__ constexpr int rpiece(int s) { return s < 72 ? 0 : (s < 144 ? 1 : (s < 160 ? 2 : 3)); }
__host__ __device__ constexpr int rlocal(int s) { return s < 72 ? s : (s < 144 ? s - 72 : (s < 160 ? s - 144 : s - 160)); }
__host__ __device__ constexpr int rbox(int s) {
  return s < 72 ? s : (s < 144 ? (kGY + 2) * kGBX + (s - 72)
                                : (2 + (rlocal(s) >> 1)) * kGBX + (s < 160 ? 0 : kGX + 2) + (rlocal(s) & 1));
}
// component rank j (g-slot order) of ring site s
__host__ __device__ constexpr int ring_at(int j, int s) {
  const int r = j < 5 ? 0 : (j < 14 ? 1 : 2);
  return piece_base(r, rpiece(s)) + (j - rrank0(r)) * psites(rpiece(s)) + rlocal(s);
}

struct alignas(128) GrSmem {
  alignas(128) double sGt[4][Q][kGT];  // g tiles of boxes n .. n+3 (slot n & 3), g-slot order
  alignas(128) double sRing[kGRing];   // g on the halo ring of one box
  alignas(16) double sPhi[kGNPHI][kGNB];
  double sP[6][kGNP];
  double sQ[2][4][kGT];  // hand-off: mu, Fx, Fy, Fz
  unsigned long long gt_full[4], gt_empty[4], ring_full, q_full[2], q_empty[2];
};
static_assert(sizeof(GrSmem) <= 232448, "shared memory per CTA exceeds 227 KB");

__device__ __forceinline__ void gr_named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void gr_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void gr_cp_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kGT + kGS, 1)
    k_step_gr(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B,
              const double* __restrict__ phig, int zc, TileOrder ord, L2Pol l2, Health hl, Peers pr,
              const __grid_constant__ CUtensorMap tm_t5, const __grid_constant__ CUtensorMap tm_t9,
              const __grid_constant__ CUtensorMap tm_h5, const __grid_constant__ CUtensorMap tm_h9,
              const __grid_constant__ CUtensorMap tm_v5, const __grid_constant__ CUtensorMap tm_v9) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  GrSmem& sm = *reinterpret_cast<GrSmem*>(smem_raw);
  constexpr int TX = kGX, TY = kGY, NT = kGT, BX = kGBX, NB = kGNB, PX = kGPX, NP = kGNP;
  constexpr unsigned TILE_BYTES = Q * NT * 8, RING_BYTES = Q * kGNR * 8;
  const int tid = threadIdx.x;
  const TileId tb = tile_of_block(blockIdx.x, (G.nx + TX - 1) / TX, (G.ny + TY - 1) / TY, (G.nzl + zc - 1) / zc, ord);
  const int x0 = tb.bx * TX, y0 = tb.by * TY;
  const int zA = tb.bz * zc, zB = min(zA + zc, G.nzl);
  const int nlast = zB - zA + 3;  // box n = plane zA - 2 + n, n = 0 .. nlast
  const long long nxy = G.nxy;
  // the halo ring inside the plane: TMA pieces; else per-thread copies (wrapping)
  const bool ring_tma = x0 >= 2 && x0 + TX + 2 <= G.nx && y0 >= 2 && y0 + TY + 2 <= G.ny;
  auto wrapx = [&](int v) { v %= G.nx; return v < 0 ? v + G.nx : v; };
  auto wrapy = [&](int v) { v %= G.ny; return v < 0 ? v + G.ny : v; };
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
  // a collision plane's box: its g tile slot is released by the collision
  auto is_coll = [&](int n) { return n >= 2 && n <= nlast - 2; };

  if (tid == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(&sm.gt_full[s], 1);
      mbar_init(&sm.gt_empty[s], 1);
    }
    mbar_init(&sm.ring_full, ring_tma ? 1 : kGS);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.q_full[s], kGS);
      mbar_init(&sm.q_empty[s], NT);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (tid >= NT) {
    // ============================ stencil warps ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;");
    const int a = tid - NT;
    const unsigned long long pol_g = policy_rt(l2.box);  // the g tile and the ring are read again
    if (pr.sync && !G.zwrap && (zA - 2 < 0 || zB + 1 >= G.nzl)) {  // peer transport: a slab-edge chunk
      if (a == 0) sync_wait_ghost_phi(G, pr, zA, zB);
      gr_named_sync(2, kGS);
    }
    // per-thread copy plan of a wrapping ring: 88 units of 2 sites (16 bytes) per
    // component -- top and bottom rows 18 each, left and right columns 8 each
    int ru_dst = -1;          // ring site of this thread's unit (its first site)
    long long ru_src = 0;     // xy offset in the plane
    if (!ring_tma && a < 88) {
      int s;
      if (a < 72) {  // rows: 4 rows x 18 units
        const int row = a / 18, c = a - row * 18;
        s = (row < 2 ? row * BX : 72 + (row - 2) * BX) + 2 * c;
        const int by = row < 2 ? row : TY + row;
        ru_src = (long long)wrapy(y0 - 2 + by) * G.nx + wrapx(x0 - 2 + 2 * c);
      } else {  // columns: left / right x 8 rows
        const int q = a - 72, side = q >> 3, row = q & 7;
        s = 144 + side * 16 + 2 * row;
        ru_src = (long long)wrapy(y0 + row) * G.nx + wrapx(side ? x0 + TX : x0 - 2);
      }
      ru_dst = s;
      LB_CHECK(hl, ru_src >= 0 && ru_src + 1 < nxy);
    }
    auto issue_tile = [&](int n) {  // g tile of box n (a collision or a phi-only plane) into slot n & 3
      if (a != 0) return;
      bool ghost;
      const int zs = zsrc(zA - 2 + n, ghost);
      unsigned long long* bar = &sm.gt_full[n & 3];
      if (ghost) {  // no tile: complete the slot's phase without bytes
        gr_arrive(bar);
        return;
      }
      const int cpl = (zs + GZ) * NSLOT;
      double* dst = &sm.sGt[n & 3][0][0];
      fence_proxy_async();
      mbar_expect_tx(bar, TILE_BYTES);
      tma_load_3d(dst, &tm_t5, x0, y0, cpl + 5, bar, pol_g);
      tma_load_3d(dst + 5 * NT, &tm_t9, x0, y0, cpl + 19, bar, pol_g);
      tma_load_3d(dst + 14 * NT, &tm_t5, x0, y0, cpl + 33, bar, pol_g);
    };
    auto issue_ring = [&](int n) -> bool {  // halo ring of box n into sRing
      bool ghost;
      const int zs = zsrc(zA - 2 + n, ghost);
      if (ghost) return false;
      const int cpl = (zs + GZ) * NSLOT;
      if (ring_tma) {
        if (a == 0) {
          fence_proxy_async();
          mbar_expect_tx(&sm.ring_full, RING_BYTES);
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const CUtensorMap* h = r == 1 ? &tm_h9 : &tm_h5;
            const CUtensorMap* v = r == 1 ? &tm_v9 : &tm_v5;
            const int c = cpl + (r == 0 ? 5 : (r == 1 ? 19 : 33));
            tma_load_3d(sm.sRing + piece_base(r, 0), h, x0 - 2, y0 - 2, c, &sm.ring_full, pol_g);
            tma_load_3d(sm.sRing + piece_base(r, 1), h, x0 - 2, y0 + TY, c, &sm.ring_full, pol_g);
            tma_load_3d(sm.sRing + piece_base(r, 2), v, x0 - 2, y0, c, &sm.ring_full, pol_g);
            tma_load_3d(sm.sRing + piece_base(r, 3), v, x0 + TX, y0, c, &sm.ring_full, pol_g);
          }
        }
      } else {
        if (ru_dst >= 0) {
          const double* base = A + (long long)(zs + GZ) * G.plane + ru_src;
#pragma unroll
          for (int j = 0; j < Q; ++j) cp_async_v<2>(&sm.sRing[ring_at(j, ru_dst)], base + (long long)gslot_of_rank(j) * nxy);
        }
        gr_cp_arrive(&sm.ring_full);
      }
      return true;
    };
    unsigned ring_ph = 0;
    auto make_phi = [&](int zp, int n, bool ring_issued) {
      bool ghost;
      const int zs = zsrc(zp, ghost);
      double* ring = sm.sPhi[wslot<kGNPHI>(zp)];
      if (ghost) {
        for (int b = a; b < NB; b += kGS) {
          const int gx = wrapx(x0 - 2 + b % BX), gy = wrapy(y0 - 2 + b / BX);
          LB_CHECK(hl, zs >= -GP && zs < G.nzl + GP && gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny);
          ring[b] = ldg(phig + phi_plane_index(G, zs) + (long long)gy * G.nx + gx);
        }
        return;
      }
      if (ring_issued) {
        mbar_wait(&sm.ring_full, ring_ph);
        ring_ph ^= 1;
      }
      mbar_wait(&sm.gt_full[n & 3], (unsigned)((n >> 2) & 1));
      // tile sites (A.3, canonical order, the same sum as phi_sum and the collision's);
      // a ragged tile's positions beyond the lattice hold the wrapped sites, summed
      // from global memory (the TMA tile has zeros there)
      {
        const double(*gt)[NT] = sm.sGt[n & 3];
        const int s = a;  // kGS == NT: one tile site per thread
        const int sx = x0 + s % TX, sy = y0 + s / TX;
        double v;
        if (sx < G.nx && sy < G.ny) {
          v = gt[grank(0)][s];
#pragma unroll
          for (int i = 1; i < Q; ++i) v += gt[grank(i)][s];
        } else {
          v = phi_sum(A + (long long)(zs + GZ) * G.plane + (long long)wrapy(sy) * G.nx + wrapx(sx), nxy);
        }
        ring[(s / TX + 2) * BX + s % TX + 2] = v;
      }
      if (a < kGNR) {  // ring sites
        double v = sm.sRing[ring_at(grank(0), a)];
#pragma unroll
        for (int i = 1; i < Q; ++i) v += sm.sRing[ring_at(grank(i), a)];
        ring[rbox(a)] = v;
      }
    };
    auto compute_P = [&](int zp) {
      const double* f0 = sm.sPhi[wslot<kGNPHI>(zp - 1)];
      const double* f1 = sm.sPhi[wslot<kGNPHI>(zp)];
      const double* f2 = sm.sPhi[wslot<kGNPHI>(zp + 1)];
      for (int e = a; e < NP; e += kGS) {
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
      const int e = (a / TX + 1) * PX + (a % TX + 1);
      const auto& P = sm.sP;
      Pz[0] = P[PXZ][e];
      Pz[1] = P[PYZ][e];
      Pz[2] = P[PZZ][e];
      Fxy[0] = -0.5 * (P[PXX][e + 1] - P[PXX][e - 1]) - 0.5 * (P[PXY][e + PX] - P[PXY][e - PX]);
      Fxy[1] = -0.5 * (P[PXY][e + 1] - P[PXY][e - 1]) - 0.5 * (P[PYY][e + PX] - P[PYY][e - PX]);
      Fxy[2] = -0.5 * (P[PXZ][e + 1] - P[PXZ][e - 1]) - 0.5 * (P[PYZ][e + PX] - P[PYZ][e - PX]);
    };
    double Pz_prev[3], Pz_cur[3], Fxy_cur[3];
    unsigned seq = 0;
    // prologue: the g tiles of boxes 0 and 1 (slots free), the ring of box 0
    issue_tile(0);
    if (1 <= nlast) issue_tile(1);
    bool ring_issued = issue_ring(0);
    for (int nn = 0; nn <= nlast; ++nn) {
      const int zp = zA - 2 + nn;
      make_phi(zp, nn, ring_issued);
      gr_named_sync(2, kGS);  // ring and (phi-only) tile consumed, phi ring written
      ring_issued = nn + 1 <= nlast ? issue_ring(nn + 1) : false;
      if (!is_coll(nn) && a == 0) gr_arrive(&sm.gt_empty[nn & 3]);  // a phi-only tile: its slot is free
      if (nn >= 2) {
        compute_P(zp - 1);  // needs phi(zp-2 .. zp)
        gr_named_sync(2, kGS);
        if (nn == 2) {
          double unused[3];
          own_P(Pz_prev, unused);
        } else if (nn == 3) {
          own_P(Pz_cur, Fxy_cur);
        } else {
          double Pz_next[3], Fxy_next[3];
          own_P(Pz_next, Fxy_next);
          // hand mu, F of plane j = zp - 2 to the collision warps
          const int j = zp - 2;
          const int q = seq & 1, u = seq >> 1;
          if (u >= 1) mbar_wait(&sm.q_empty[q], (u - 1) & 1);
          const double* r0 = sm.sPhi[wslot<kGNPHI>(j)];
          const double* rm = sm.sPhi[wslot<kGNPHI>(j - 1)];
          const double* rp = sm.sPhi[wslot<kGNPHI>(j + 1)];
          const int cbox = (a / TX + 2) * BX + (a % TX + 2);
          const double ph = r0[cbox];
          const double lap = (r0[cbox + 1] + r0[cbox - 1]) + (r0[cbox + BX] + r0[cbox - BX]) + (rp[cbox] + rm[cbox]) -
                             6.0 * ph;
          sm.sQ[q][0][a] = chem_pot(p, ph, lap);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            sm.sQ[q][1 + c][a] = Fxy_cur[c] - 0.5 * (Pz_next[c] - Pz_prev[c]);
            Pz_prev[c] = Pz_cur[c];
            Pz_cur[c] = Pz_next[c];
            Fxy_cur[c] = Fxy_next[c];
          }
          gr_arrive(&sm.q_full[q]);
          ++seq;
        }
      }
      // the g tile of box nn + 2 into the slot of box nn - 2, once that box's tile
      // has been read (by the collision of its plane, just handed over above, or
      // by the phi of a phi-only box)
      if (nn + 2 <= nlast) {
        if (nn - 2 >= 0 && a == 0) mbar_wait(&sm.gt_empty[(nn - 2) & 3], (unsigned)(((nn - 2) >> 2) & 1));
        issue_tile(nn + 2);
      }
    }
    cp_wait<0>();
  } else {
    // ============================== collision warps ==============================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 176;");
    const unsigned long long pol_f = policy_rt(l2.ftile);
    const int lx = tid % TX, ly = tid / TX;
    const int x = x0 + lx, y = y0 + ly;
    const bool active = (x < G.nx) && (y < G.ny);
    const int xm1 = wrapx(x - 1), xp1 = wrapx(x + 1), ym1 = wrapy(y - 1), yp1 = wrapy(y + 1);
    const long long site_xy = (long long)(active ? y : 0) * G.nx + (active ? x : 0);
    unsigned seq = 0;
    for (int k = zA; k < zB; ++k) {
      const int n = k - zA + 2;  // this plane's box
      double f[Q], g[Q];
      const double* fp = A + (long long)(k + GZ) * G.plane + site_xy;
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = ldg_hint(fp + (long long)slot(0, i) * nxy, pol_f);
      const int q = seq & 1, u = seq >> 1;
      mbar_wait(&sm.q_full[q], u & 1);
      const double mu = sm.sQ[q][0][tid];
      double F[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) F[c] = sm.sQ[q][1 + c][tid];
      gr_arrive(&sm.q_empty[q]);
      ++seq;
      mbar_wait(&sm.gt_full[n & 3], (unsigned)((n >> 2) & 1));
#pragma unroll
      for (int i = 0; i < Q; ++i) g[i] = sm.sGt[n & 3][grank(i)][tid];
      gr_named_sync(1, NT);  // the slot is read
      if (tid == 0) gr_arrive(&sm.gt_empty[n & 3]);
      double ph = g[0];  // A.3, canonical order: the stencil's bits
#pragma unroll
      for (int i = 1; i < Q; ++i) ph += g[i];
      if (active) {
        double* const zb[3] = {push_plane(G, B, pr, k - 1), push_plane(G, B, pr, k), push_plane(G, B, pr, k + 1)};
        auto push = [&](int i, double fs, double gs) {
          const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
          const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
          LB_CHECK(hl, xd >= 0 && xd < G.nx && yd >= 0 && yd < G.ny);
          double* d = zb[cz(i) + 1] + (long long)yd * G.nx + xd;  // A.8 push
          __stcs(d + (long long)slot(0, i) * nxy, fs);
          __stcs(d + (long long)slot(1, i) * nxy, gs);
        };
        const double rho = collide(p, f, g, ph, mu, F, push);
        if (!(rho > 0.0) || !isfinite(rho) || !isfinite(ph)) health_report(hl, G, x, y, k);  // R22
      }
    }
    gr_named_sync(1, NT);
    if (tid == 0) health_tick(hl);
  }
}

}  // namespace

bool step_gr_fits(const Geom& G, const StepMaps* maps) {
  return maps && maps->ok && maps->ty == kGY && G.nx % 2 == 0 && G.nx >= 4 && G.ny >= 4;
}

cudaError_t prepare_gr_kernels() {
  int r = 0;
  return prepare_kernel(reinterpret_cast<const void*>(k_step_gr), sizeof(GrSmem), kGT + kGS, &r);
}

cudaError_t launch_step_gr(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                           const Launch& ln, const Health& hl, const StepMaps* maps, cudaStream_t st, const Peers& pr) {
  if (!step_gr_fits(G, maps) || p.coll != 0) return cudaErrorInvalidValue;
  int resid = 0;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(k_step_gr), sizeof(GrSmem), kGT + kGS, &resid);
  if (e != cudaSuccess) return e;
  TileOrder ord = ln.order;
  if (ord.resid <= 0) ord.resid = resid;
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  const int zc = ln.zc;
  const int nblk = ((G.nx + kGX - 1) / kGX) * ((G.ny + kGY - 1) / kGY) * ((G.nzl + zc - 1) / zc);
  k_step_gr<<<(unsigned)nblk, kGT + kGS, sizeof(GrSmem), st>>>(G, p, A, B, phig, zc, ord, ln.l2, hl, pr, m[0], m[1],
                                                               m[4], m[5], m[6], m[7]);
  return cudaGetLastError();
}

}  // namespace lbk
