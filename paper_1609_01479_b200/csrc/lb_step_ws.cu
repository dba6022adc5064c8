// lb_step_ws.cu -- warp-specialised variant of the fused D3Q19 binary-fluid step.
//
// Same arithmetic, same HBM traffic and same results (bit for bit) as the tile
// kernel of lb_step.cu, but the two
// halves of an iteration run CONCURRENTLY on different warps of the CTA instead
// of one after the other between __syncthreads:
//
//   collision warps (TX*TY threads, one per column): wait for the TMA tile of
//       f, g at plane k, take phi, mu, F of plane k from the hand-off buffer sQ,
//       collide (A.6, A.7) and push f*, g* to x + c_i (A.8).  They are the only
//       warps that store, so the store stream never pauses for stencil work.
//   stencil warps (one thread per column for 32 x 8 tiles, with the register
//       file split between the roles by setmaxnreg; one warpgroup for 32 x 4
//       tiles): run one or two planes ahead -- wait for
//       the g box of plane j+2 (TMA), phi(j+2) = sum_i g_i on the box (A.3),
//       the chemical stress P(j+1) (A.4), the force F(j) = -div P (A.5) and
//       mu(j) (A.4) -- and hands phi, mu, F of plane j over through sQ (two
//       slots, mbarrier full/empty pairs).
//
// The tile kernel is one CTA per SM at 32 x 8 tiles; there, every __syncthreads
// between the phi/P phases and the collision phase stalled the store stream
// (DESIGN.md "Tuning").  Needs 16-byte rows (nx even: TMA).
#include "lb_device.cuh"
#include "lb_tma.cuh"

namespace lbk {
namespace {

constexpr int kWTX = 32;
#ifndef LB_WS_NA
#define LB_WS_NA 256
#endif
// stencil threads: one or two warpgroups, at most one per site
__host__ __device__ constexpr int ws_na(int ty) { return LB_WS_NA < kWTX * ty ? LB_WS_NA : kWTX * ty; }
// register split between the roles for 32 x 8 tiles with 256 stencil threads
// (setmaxnreg: 512 threads launch at 128 registers; the collision needs ~170)
#ifndef LB_WS_REGS_STENCIL
#define LB_WS_REGS_STENCIL 80
#endif
#ifndef LB_WS_REGS_COLL
#define LB_WS_REGS_COLL 176
#endif
// the MRT collision (COLL 1) keeps more values live
#ifndef LB_WS_REGS_STENCIL_MRT
#define LB_WS_REGS_STENCIL_MRT 64
#endif
#ifndef LB_WS_REGS_COLL_MRT
#define LB_WS_REGS_COLL_MRT 192
#endif
__host__ __device__ constexpr bool ws_split_regs(int ty) {
  return LB_WS_REGS_STENCIL > 0 && kWTX * ty == 256 && ws_na(ty) == 256;
}
// pushes: st.global.cs (LB_WS_ST_POL < 0) or an L2 policy (policy_of kind)
#ifndef LB_WS_ST_POL
#define LB_WS_ST_POL (-1)
#endif

// XCH: planes the stencil's P / F / mu work trails its phi (the neighbours' slack)
constexpr int kXchLag = 4;

template <int R>
__device__ __forceinline__ int wslot(int z) {
  const int s = z % R;
  return s < 0 ? s + R : s;
}
__host__ __device__ constexpr int ws_threads(int ty, bool) { return kWTX * ty + ws_na(ty); }
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int TY, int COLL, bool XCH = false>
struct alignas(128) WsSmem {
  static constexpr int NPHI = XCH ? kXchLag + 4 : 5;  // phi ring planes (XCH: lag planes more)
  static constexpr int NQ = COLL == 1 ? 8 : 5;  // hand-off values per site
  static constexpr int TX = kWTX, NT = TX * TY;
  static constexpr int BX = TX + 4, BY = TY + 4, NB = BX * BY;  // phi box: tile + 2 halo
  static constexpr int PX = TX + 2, PY = TY + 2, NP = PX * PY;  // P box: tile + 1 halo
  alignas(128) double sTf[Q][NT];  // f of the tile, f-slot order (TMA boxes TX x TY x 5|9|5)
  alignas(128) double sTg[Q][NT];  // g of the tile, g-slot order
  // g on the box, g-slot order (TMA boxes BX x BY x 5|9|5); XCH: two g tiles [Q][NT]
  alignas(128) double sG[Q][XCH ? 2 * NT : NB];
  double sPhi[NPHI][NB];           // ring of phi planes on the box
  double sP[6][NP];                // chemical stress of one plane on the P box
  double sQ[2][NQ][NT];            // hand-off: phi, mu, then Fx, Fy, Fz (COLL 0) or P (COLL 1)
  // box of a tile at a periodic edge: the TMA copy fills what lies inside the
  // lattice (zeros outside); the wrapped column pair (all BY rows) and row pairs
  // (all BX columns) come here by per-thread copies
  alignas(16) double sWc[Q][XCH ? 1 : BY][2];
  alignas(16) double sWr[Q][2][XCH ? 2 : BX];
  unsigned long long bar_f, bar_g, bar_box, bar_xb[2], q_full[2], q_empty[2];
};

// XCH (phi exchange; one periodic slab, whole 32 x 8 tiles): the stencil warps
// load only the g TILE of plane j+2, not the tile + 2-site halo box (-40% of the
// box bytes), store phi of their tile to an L2-resident array (xa.cur) and take
// the phi halo from the neighbouring tiles' stores there.  Empty sites hold the
// NaN kXchEmpty, so a value is its own flag (no fences, no flag words); each
// block resets its sites in last step's array (xa.old) for the next step.  A
// halo site still empty when needed (its tile runs behind or has not started --
// the next wave) is summed from g here: nobody waits, so no schedule can
// deadlock, and phi is the same sum in the same order either way -- the results
// are bit for bit those of the plain kernel.  Default where all blocks run in
// one wave (the tiles' CTAs start together and stay within the lag of each
// other: 128^3, 64^3); over several waves the neighbours drift apart and the
// fallback sums cost more than the box.
#ifdef LB_TRACE
// block schedule trace (measurement build only, scripts/trace_schedule.py): per
// block start / end globaltimer, SM, tile and first plane
__device__ unsigned long long lb_trace_buf[1 << 16][4];
#endif

template <int TY, int COLL, bool XCH = false>
__global__ void __launch_bounds__(ws_threads(TY, XCH), 1)
    k_step_ws(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B,
              const double* __restrict__ phig, int zc, TileOrder ord, L2Pol l2, Health hl, Peers pr, XchArgs xa,
              const __grid_constant__ CUtensorMap tm_t5, const __grid_constant__ CUtensorMap tm_t9,
              const __grid_constant__ CUtensorMap tm_g5, const __grid_constant__ CUtensorMap tm_g9) {
  using S = WsSmem<TY, COLL, XCH>;
  static_assert(!XCH || (TY == 8 && COLL == 0), "phi exchange: 32 x 8 tiles, BGK");
  constexpr int TX = kWTX, NT = S::NT;
  constexpr int BX = S::BX, BY = S::BY, NB = S::NB, PX = S::PX, NP = S::NP;
  constexpr unsigned TILE_BYTES = Q * NT * 8, BOX_BYTES = Q * NB * 8;
  constexpr int kNA = ws_na(TY);
  constexpr int SPT = NT / kNA;  // sites per stencil thread
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const int tid = threadIdx.x;
  const TileId tb = tile_of_block(blockIdx.x, (G.nx + TX - 1) / TX, (G.ny + TY - 1) / TY, (G.nzl + zc - 1) / zc, ord);
  const int x0 = tb.bx * TX, y0 = tb.by * TY;
  const int zA = tb.bz * zc, zB = min(zA + zc, G.nzl);
  const long long nxy = G.nxy;

  auto wrapx = [&](int v) { v %= G.nx; return v < 0 ? v + G.nx : v; };
  auto wrapy = [&](int v) { v %= G.ny; return v < 0 ? v + G.ny : v; };

  if (tid == 0) {
    mbar_init(&sm.bar_f, 1);
    mbar_init(&sm.bar_g, 1);
    mbar_init(&sm.bar_box, 1);
    mbar_init(&sm.bar_xb[0], 1);
    mbar_init(&sm.bar_xb[1], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.q_full[s], kNA);
      mbar_init(&sm.q_empty[s], NT);
    }
    fence_barrier_init();
  }
  __syncthreads();
#ifdef LB_TRACE
  if (tid == 0 && blockIdx.x < (1u << 16)) {
    unsigned sm_id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_id));
    lb_trace_buf[blockIdx.x][0] = globaltimer_ns();
    lb_trace_buf[blockIdx.x][2] = ((unsigned long long)zB << 32) | sm_id;
    lb_trace_buf[blockIdx.x][3] = ((unsigned long long)tb.bx << 40) | ((unsigned long long)tb.by << 20) | (unsigned)zA;
  }
#endif

  if (tid >= NT) {
    // ============================ stencil warps ============================
    if constexpr (ws_split_regs(TY))
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(COLL == 1 ? LB_WS_REGS_STENCIL_MRT : LB_WS_REGS_STENCIL));
    const int a = tid - NT;
    const unsigned long long pol_last = policy_rt(l2.box);
    if (pr.sync && !G.zwrap && (zA - 2 < 0 || zB + 1 >= G.nzl)) {  // peer transport: a slab-edge chunk
      if (a == 0) sync_wait_ghost_phi(G, pr, zA, zB);                 // waits for the neighbours' K_phi
      named_sync(2, kNA);
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
    constexpr int BROWU = BX / 2, BOXU = BY * BROWU, BOXR = (BOXU + kNA - 1) / kNA;
    unsigned ph_box = 0;
    unsigned ph_xb = 0;  // XCH: parity bits of the two g tile buffers
    unsigned seq = 0;  // planes handed off so far: slot seq & 1, use seq >> 1
    double Pz_prev[SPT][3], Pz_cur[SPT][3], Fxy_cur[SPT][3];
    double P6_cur[SPT][COLL == 1 ? 6 : 1];  // COLL 1: P at the site, plane j
    const bool box_interior = x0 >= 2 && x0 + TX + 2 <= G.nx && y0 >= 2 && y0 + TY + 2 <= G.ny;
    // a whole tile at an edge of a lattice of >= 2 x 2 tiles: every box column or
    // row wraps at most once, on one side (the side pieces); otherwise (narrow or
    // ragged lattices) the whole box by per-thread copies
    const bool box_side = !box_interior && x0 + TX <= G.nx && y0 + TY <= G.ny && G.nx >= 2 * TX && G.ny >= 2 * TY;
    const int wcol = x0 == 0 ? 0 : (x0 + TX + 2 > G.nx ? TX + 2 : -1);  // first wrapped box column (a pair)
    const int nrow_top = y0 < 2 ? 2 - y0 : 0;                           // wrapped box rows at the top ...
    const int nrow_bot = y0 + TY + 2 > G.ny ? y0 + TY + 2 - G.ny : 0;   // ... and at the bottom (<= 2)
    auto row_wrapped = [&](int r) { return r < nrow_top || r >= BY - nrow_bot; };
    auto row_side = [&](int r) { return r < 2 ? r : r - (BY - 2); };  // slot of a wrapped row in sWr
    constexpr bool use_box = !XCH;
    // per-thread copy plan of a wrapped halo box: 16-byte units
    long long box_src[BOXR];
    int box_dst[BOXR];
#pragma unroll
    for (int r = 0; r < BOXR; ++r) {
      const int u = a + r * kNA;
      const int row = u / BROWU, cu = u - row * BROWU;
      box_src[r] = (long long)wrapy(y0 - 2 + row) * G.nx + wrapx(x0 - 2 + cu * 2);
      box_dst[r] = u < BOXU ? row * BX + cu * 2 : -1;
      LB_CHECK(hl, box_dst[r] < 0 || (box_dst[r] + 1 < NB && box_src[r] >= 0 && box_src[r] + 1 < nxy));
    }
    // box n (n = 0 .. nlast) is the g box of plane zA - 2 + n
    const int nlast = zB - zA + 3;  // plane zB + 1
    auto issue_box = [&](int n) -> bool {
      const int zp = zA - 2 + n;
      bool ghost;
      const int zs = zsrc(zp, ghost);
      if (ghost) return false;
      if (XCH && !use_box) {
        if (a == 0) {  // the g tile only, in tile layout, into buffer n & 1
          const int cpl = (zs + GZ) * NSLOT;
          double* dst = &sm.sG[0][0] + (n & 1) * Q * NT;
          unsigned long long* bar = &sm.bar_xb[n & 1];
          fence_proxy_async();
          mbar_expect_tx(bar, TILE_BYTES);
          tma_load_3d(dst, &tm_t5, x0, y0, cpl + 5, bar, pol_last);
          tma_load_3d(dst + 5 * NT, &tm_t9, x0, y0, cpl + 19, bar, pol_last);
          tma_load_3d(dst + 14 * NT, &tm_t5, x0, y0, cpl + 33, bar, pol_last);
        }
      } else if (box_interior || box_side) {
        if (a == 0) {  // (at an edge the parts outside the lattice are zero-filled: the side pieces have them)
          const int cpl = (zs + GZ) * NSLOT;
          fence_proxy_async();
          mbar_expect_tx(&sm.bar_box, BOX_BYTES);
          tma_load_3d(&sm.sG[0][0], &tm_g5, x0 - 2, y0 - 2, cpl + 5, &sm.bar_box, pol_last);
          tma_load_3d(&sm.sG[5][0], &tm_g9, x0 - 2, y0 - 2, cpl + 19, &sm.bar_box, pol_last);
          tma_load_3d(&sm.sG[14][0], &tm_g5, x0 - 2, y0 - 2, cpl + 33, &sm.bar_box, pol_last);
        }
        if (box_side) {  // 16-byte copies: the wrapped column pair, then the wrapped rows
          const double* base = A + (long long)(zs + GZ) * G.plane;
          const int ncu = wcol >= 0 ? Q * BY : 0;
          const int nrows = nrow_top + nrow_bot, nru = Q * nrows * (BX / 2);
          for (int u = a; u < ncu + nru; u += kNA) {
            if (u < ncu) {
              const int j = u / BY, r = u - j * BY;
              const long long o = (long long)wrapy(y0 - 2 + r) * G.nx + wrapx(x0 - 2 + wcol);
              LB_CHECK(hl, j < Q && r < BY && o >= 0 && o + 1 < nxy);
              cp_async_v<2>(&sm.sWc[j][r][0], base + (long long)gslot_of_rank(j) * nxy + o);
            } else {
              const int v = u - ncu, j = v / (nrows * (BX / 2)), w = v - j * (nrows * (BX / 2));
              const int q = w / (BX / 2), c = 2 * (w - q * (BX / 2));
              const int r = q < nrow_top ? q : BY - nrow_bot + (q - nrow_top);
              const long long o = (long long)wrapy(y0 - 2 + r) * G.nx + wrapx(x0 - 2 + c);
              LB_CHECK(hl, j < Q && row_side(r) >= 0 && row_side(r) < 2 && c + 1 < BX && o >= 0 && o + 1 < nxy);
              cp_async_v<2>(&sm.sWr[j][row_side(r)][c], base + (long long)gslot_of_rank(j) * nxy + o);
            }
          }
          cp_commit();
        }
      } else {
        const double* base = A + (long long)(zs + GZ) * G.plane;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          const double* bj = base + (long long)gslot_of_rank(j) * nxy;
#pragma unroll
          for (int r = 0; r < BOXR; ++r)
            if (box_dst[r] >= 0) cp_async_v<2>(&sm.sG[j][box_dst[r]], bj + box_src[r]);
        }
        cp_commit();
      }
      return true;
    };
    // wait for the box, then make it visible to the whole role
    auto wait_box = [&](bool issued, int n) {
      if (XCH && !use_box) {  // g tile n (always issued: one periodic slab)
        mbar_wait(&sm.bar_xb[n & 1], (ph_xb >> (n & 1)) & 1);
        ph_xb ^= 1u << (n & 1);
      } else if (issued) {
        if (box_interior || box_side) {
          if (box_side) cp_wait<0>();
          mbar_wait(&sm.bar_box, ph_box);
          ph_box ^= 1;
        } else {
          cp_wait<0>();
        }
      }
      named_sync(2, kNA);
    };
    auto make_phi = [&](int zp, int n) {
      bool ghost;
      const int zs = zsrc(zp, ghost);
      double* ring = sm.sPhi[wslot<S::NPHI>(zp)];
      if (XCH && !ghost) {
        double* xp = xa.cur + (long long)zs * nxy;
        double* xo = xa.old + (long long)zs * nxy;
        if (!use_box) {  // phi of the tile from the g tile
          const double(*gt)[NT] = reinterpret_cast<const double(*)[NT]>(&sm.sG[0][0] + (n & 1) * Q * NT);
          for (int s = a; s < NT; s += kNA) {
            double v = gt[grank(0)][s];  // A.3, canonical order (same as phi_sum)
#pragma unroll
            for (int i = 1; i < Q; ++i) v += gt[grank(i)][s];
            ring[(s / TX + 2) * BX + s % TX + 2] = v;
            const long long o = (long long)(y0 + s / TX) * G.nx + x0 + s % TX;
            st_relaxed_f64(xp + o, v);  // published to the neighbouring tiles' CTAs
            st_relaxed_f64(xo + o, __longlong_as_double((long long)kXchEmpty));
          }
          return;
        }
      }
      if (ghost) {
        for (int b = a; b < NB; b += kNA) {
          const int gx = wrapx(x0 - 2 + b % BX), gy = wrapy(y0 - 2 + b / BX);
          LB_CHECK(hl, zs >= -GP && zs < G.nzl + GP && gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny);
          ring[b] = ldg(phig + phi_plane_index(G, zs) + (long long)gy * G.nx + gx);
        }
        return;
      }
      // two neighbouring sites per thread with 16-byte shared loads (BX even: a pair
      // never straddles a row): every thread of the role has at most one pair, so
      // phi of the box is ready after 19 loads instead of up to 38 -- and the next
      // box goes out sooner.  Each site's sum is in the canonical order (A.3, as
      // phi_sum): the same bits.
      static_assert(BX % 2 == 0 && NB % 2 == 0, "pairs of box sites");
      for (int pb = a; pb < NB / 2; pb += kNA) {
        const int b = 2 * pb;
        const double* src = &sm.sG[0][b];  // component rank j of the pair at src + j * stride
        int stride = NB;
        if (box_side) {
          const int r = b / BX, c = b - r * BX;
          if (wcol >= 0 && (c == wcol)) {
            src = &sm.sWc[0][r][0];
            stride = BY * 2;
          } else if (row_wrapped(r)) {
            src = &sm.sWr[0][row_side(r)][c];
            stride = 2 * BX;
          }
        }
        double2 v = *reinterpret_cast<const double2*>(src + grank(0) * stride);
#pragma unroll
        for (int i = 1; i < Q; ++i) {
          const double2 w = *reinterpret_cast<const double2*>(src + grank(i) * stride);
          v.x += w.x;
          v.y += w.y;
        }
        *reinterpret_cast<double2*>(&ring[b]) = v;
      }
    };
    auto compute_P = [&](int zp) {
      const double* f0 = sm.sPhi[wslot<S::NPHI>(zp - 1)];
      const double* f1 = sm.sPhi[wslot<S::NPHI>(zp)];
      const double* f2 = sm.sPhi[wslot<S::NPHI>(zp + 1)];
      for (int e = a; e < NP; e += kNA) {
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
    auto own_P6 = [&](int site, double* P6) {
      const int e = (site / TX + 1) * PX + (site % TX + 1);
#pragma unroll
      for (int q = 0; q < 6; ++q) P6[q] = sm.sP[q][e];
    };
    auto own_P = [&](int site, double Pz[3], double Fxy[3]) {
      const int e = (site / TX + 1) * PX + (site % TX + 1);
      const auto& P = sm.sP;
      Pz[0] = P[PXZ][e];
      Pz[1] = P[PYZ][e];
      Pz[2] = P[PZZ][e];
      Fxy[0] = -0.5 * (P[PXX][e + 1] - P[PXX][e - 1]) - 0.5 * (P[PXY][e + PX] - P[PXY][e - PX]);
      Fxy[1] = -0.5 * (P[PXY][e + 1] - P[PXY][e - 1]) - 0.5 * (P[PYY][e + PX] - P[PYY][e - PX]);
      Fxy[2] = -0.5 * (P[PXZ][e + 1] - P[PXZ][e - 1]) - 0.5 * (P[PYZ][e + PX] - P[PYZ][e - PX]);
    };

    // XCH lags kXchLag planes: iteration nn makes phi of the tile on box nn
    // (stored to xa.cur); each halo thread loads its site of box nn - lag + 1
    // from the owner's store in xa.cur (L2) and uses it an iteration later -- if
    // it still reads kXchEmpty the owner is behind (started later, runs slower)
    // and the site's phi is summed from g here.  The value is its own flag: no
    // fence, no flag word, no waiting.
    constexpr int lag = XCH ? kXchLag : 0;
    constexpr int NH = 4 * BX + 4 * TY;  // halo: top and bottom 2 rows, left and right 2 columns
    int h_ring = -1;
    long long h_off = 0;
    if (XCH && !use_box && a < NH) {
      int bx, by;
      if (a < 4 * BX) {
        const int r = a / BX;
        bx = a - r * BX;
        by = r < 2 ? r : TY + r;  // rows 0, 1, TY + 2, TY + 3
      } else {
        const int q = a - 4 * BX, c = q / TY;
        by = 2 + (q - c * TY);
        bx = c < 2 ? c : TX + c;  // columns 0, 1, TX + 2, TX + 3
      }
      h_ring = by * BX + bx;
      h_off = (long long)wrap_n(y0 - 2 + by, G.ny) * G.nx + wrap_n(x0 - 2 + bx, G.nx);
      LB_CHECK(hl, h_ring >= 0 && h_ring < NB && h_off >= 0 && h_off < nxy);
    }
    auto xsite = [&](int b) { return xa.cur + (long long)wrap_n(zA - 2 + b, G.nzl) * nxy + h_off; };
    // the owner has not stored it yet (a neighbouring tile that started later or
    // runs behind): phi from g here instead, the same sum in the same order
    auto phi_here = [&](int b) {
      return phi_sum(A + (long long)(wrap_n(zA - 2 + b, G.nzl) + GZ) * G.plane + h_off, nxy);
    };
    double pf = 0.0;  // the halo site of box hb + 1, loaded an iteration ahead
    bool issued = issue_box(0);
    if (XCH && xa.depth == 2 && 1 <= nlast) issue_box(1);  // two g tiles in flight
    for (int nn = 0; nn <= nlast + lag; ++nn) {
      double hv = 0.0;
      const int hb = nn - lag;  // the halo box completed in this iteration
      const bool hw = XCH && h_ring >= 0 && hb >= 0 && hb <= nlast;
      if (hw) {
        hv = pf;
        if (__double_as_longlong(hv) == (long long)kXchEmpty) hv = phi_here(hb);  // owner behind: sum it here
      }
      if (XCH && h_ring >= 0 && hb + 1 >= 0 && hb + 1 <= nlast) pf = ld_relaxed_f64(xsite(hb + 1));
      if (nn <= nlast) {
        wait_box(issued, nn);  // (also: everyone is past the previous hand-off)
        make_phi(zA - 2 + nn, nn);
      } else {
        named_sync(2, kNA);
      }
      if (hw) sm.sPhi[wslot<S::NPHI>(zA - 2 + hb)][h_ring] = hv;
      named_sync(2, kNA);  // sG consumed, ring written
      if (nn <= nlast) {
        if (XCH && xa.depth == 2)
          issued = nn + 2 <= nlast ? issue_box(nn + 2) : false;
        else
          issued = nn + 1 <= nlast ? issue_box(nn + 1) : false;
      }
      const int n = nn - lag, zp = zA - 2 + n;
      if (n < 2) continue;
      compute_P(zp - 1);  // needs phi(zp-2 .. zp)
      named_sync(2, kNA);
      if (n == 2) {
#pragma unroll
        for (int s = 0; s < SPT; ++s) {
          double unused[3];
          own_P(a + s * kNA, Pz_prev[s], unused);
        }
        continue;
      }
      if (n == 3) {
#pragma unroll
        for (int s = 0; s < SPT; ++s) {
          own_P(a + s * kNA, Pz_cur[s], Fxy_cur[s]);
          if constexpr (COLL == 1) own_P6(a + s * kNA, P6_cur[s]);
        }
        continue;
      }
      double Pz_next[SPT][3], Fxy_next[SPT][3];
      double P6_next[SPT][COLL == 1 ? 6 : 1];
#pragma unroll
      for (int s = 0; s < SPT; ++s) {
        own_P(a + s * kNA, Pz_next[s], Fxy_next[s]);
        if constexpr (COLL == 1) own_P6(a + s * kNA, P6_next[s]);
      }
      // hand phi, mu, F of plane j = zp - 2 to the collision warps
      const int j = zp - 2;
      const int q = seq & 1, u = seq >> 1;
      if (u >= 1) mbar_wait(&sm.q_empty[q], (u - 1) & 1);
      const double* r0 = sm.sPhi[wslot<S::NPHI>(j)];
      const double* rm = sm.sPhi[wslot<S::NPHI>(j - 1)];
      const double* rp = sm.sPhi[wslot<S::NPHI>(j + 1)];
#pragma unroll
      for (int s = 0; s < SPT; ++s) {
        const int site = a + s * kNA;
        const int cbox = (site / TX + 2) * BX + (site % TX + 2);
        const double ph = r0[cbox];
        const double lap = (r0[cbox + 1] + r0[cbox - 1]) + (r0[cbox + BX] + r0[cbox - BX]) + (rp[cbox] + rm[cbox]) -
                           6.0 * ph;
        sm.sQ[q][0][site] = ph;
        sm.sQ[q][1][site] = chem_pot(p, ph, lap);
        if constexpr (COLL == 1) {
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            sm.sQ[q][2 + c][site] = P6_cur[s][c];
            P6_cur[s][c] = P6_next[s][c];
          }
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            sm.sQ[q][2 + c][site] = Fxy_cur[s][c] - 0.5 * (Pz_next[s][c] - Pz_prev[s][c]);
            Pz_prev[s][c] = Pz_cur[s][c];
            Pz_cur[s][c] = Pz_next[s][c];
            Fxy_cur[s][c] = Fxy_next[s][c];
          }
        }
      }
      mbar_arrive(&sm.q_full[q]);
      ++seq;
    }
    cp_wait<0>();
    return;
  }

  // ============================== collision warps ==============================
  if constexpr (ws_split_regs(TY))
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(COLL == 1 ? LB_WS_REGS_COLL_MRT : LB_WS_REGS_COLL));
  const unsigned long long pol_f = policy_rt(l2.ftile), pol_g = policy_rt(l2.gtile);
  const unsigned long long pol_st = policy_of<(LB_WS_ST_POL < 0 ? 1 : LB_WS_ST_POL)>();
  unsigned ph_f = 0, ph_g = 0, seq = 0;
  auto issue_tile = [&](int zp, int dist) {
    if (tid == 0) {
      double(*dst)[NT] = dist == 0 ? sm.sTf : sm.sTg;
      unsigned long long* bar = dist == 0 ? &sm.bar_f : &sm.bar_g;
      const unsigned long long pol = dist == 0 ? pol_f : pol_g;
      const int cp0 = (zp + GZ) * NSLOT + (dist == 0 ? 0 : 5);
      fence_proxy_async();
      mbar_expect_tx(bar, TILE_BYTES);
      tma_load_3d(&dst[0][0], &tm_t5, x0, y0, cp0, bar, pol);
      tma_load_3d(&dst[5][0], &tm_t9, x0, y0, cp0 + (dist == 0 ? 10 : 14), bar, pol);
      tma_load_3d(&dst[14][0], &tm_t5, x0, y0, cp0 + 28, bar, pol);
    }
  };
  issue_tile(zA, 0);
  issue_tile(zA, 1);
  const int lx = tid % TX, ly = tid / TX;
  const int x = x0 + lx, y = y0 + ly;
  const bool active = (x < G.nx) && (y < G.ny);
  const int xm1 = wrapx(x - 1), xp1 = wrapx(x + 1), ym1 = wrapy(y - 1), yp1 = wrapy(y + 1);
  for (int k = zA; k < zB; ++k) {
    double f[Q], g[Q];
    mbar_wait(&sm.bar_f, ph_f);
    ph_f ^= 1;
#pragma unroll
    for (int i = 0; i < Q; ++i) f[i] = sm.sTf[frank(i)][tid];
    named_sync(1, NT);  // sTf consumed
    if (k + 1 < zB) issue_tile(k + 1, 0);
    const int q = seq & 1, u = seq >> 1;
    mbar_wait(&sm.q_full[q], u & 1);
    const double ph = sm.sQ[q][0][tid], mu = sm.sQ[q][1][tid];
    double V[S::NQ - 2];  // F (COLL 0) or P (COLL 1)
#pragma unroll
    for (int c = 0; c < S::NQ - 2; ++c) V[c] = sm.sQ[q][2 + c][tid];
    mbar_arrive(&sm.q_empty[q]);
    ++seq;
    mbar_wait(&sm.bar_g, ph_g);
    ph_g ^= 1;
#pragma unroll
    for (int i = 0; i < Q; ++i) g[i] = sm.sTg[grank(i)][tid];
    named_sync(1, NT);  // sTg consumed
    if (k + 1 < zB) issue_tile(k + 1, 1);
    if (active) {
      double* const zb[3] = {push_plane(G, B, pr, k - 1), push_plane(G, B, pr, k), push_plane(G, B, pr, k + 1)};
      auto push = [&](int i, double fs, double gs) {
        const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
        const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
        LB_CHECK(hl, xd >= 0 && xd < G.nx && yd >= 0 && yd < G.ny);
        double* d = zb[cz(i) + 1] + (long long)yd * G.nx + xd;  // A.8 push
        if (LB_WS_ST_POL < 0) {
          __stcs(d + (long long)slot(0, i) * nxy, fs);
          __stcs(d + (long long)slot(1, i) * nxy, gs);
        } else {
          st_hint(d + (long long)slot(0, i) * nxy, fs, pol_st);
          st_hint(d + (long long)slot(1, i) * nxy, gs, pol_st);
        }
      };
      double rho;
      if constexpr (COLL == 1) rho = collide_mrt(p, f, g, ph, mu, V, push);
      else rho = collide(p, f, g, ph, mu, V, push);
      if (!(rho > 0.0) || !isfinite(rho) || !isfinite(ph)) health_report(hl, G, x, y, k);  // R22
    }
  }
  named_sync(1, NT);  // every thread's pushes before the CTA's publication
  if (tid == 0) {
    health_tick(hl);
#ifdef LB_TRACE
    if (blockIdx.x < (1u << 16)) lb_trace_buf[blockIdx.x][1] = globaltimer_ns();
#endif
  }
}

template <int TY, int COLL, bool XCH = false>
cudaError_t launch_ws_t(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                        const Launch& ln, const Health& hl, const StepMaps* maps, cudaStream_t st, const Peers& pr,
                        const XchArgs* xch = nullptr) {
  constexpr size_t smem = sizeof(WsSmem<TY, COLL, XCH>);
  static_assert(smem <= 232448, "shared memory per CTA exceeds 227 KB");
  auto kern = k_step_ws<TY, COLL, XCH>;
  int resid = 0;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), smem, ws_threads(TY, XCH), &resid);
  if (e != cudaSuccess) return e;
  TileOrder ord = ln.order;
  if (ord.resid <= 0) ord.resid = resid;
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  const int zc = ln.zc;
  const int nitems = ((G.nx + kWTX - 1) / kWTX) * ((G.ny + TY - 1) / TY) * ((G.nzl + zc - 1) / zc);
  if (XCH && (!xch || !xch->cur || !xch->old)) return cudaErrorInvalidValue;
  const XchArgs xa = xch ? *xch : XchArgs{};
  kern<<<(unsigned)nitems, ws_threads(TY, XCH), smem, st>>>(G, p, A, B, phig, zc, ord, ln.l2, hl, pr, xa, m[0], m[1],
                                                            m[2], m[3]);
  return cudaGetLastError();
}

}  // namespace

bool step_ws_fits(const StepMaps* maps) { return maps && maps->ok && (maps->ty == 8 || maps->ty == 4); }

bool step_xch_fits(const Geom& G, const StepMaps* maps) {
  return step_ws_fits(maps) && maps->ty == 8 && G.zwrap && G.nx % kWTX == 0 && G.ny % 8 == 0;
}
int ws_xch_blocks(const Geom& G, int zc) { return (G.nx / kWTX) * ((G.ny + 7) / 8) * ((G.nzl + zc - 1) / zc); }
namespace {
__global__ void k_fill_u64(unsigned long long* p, long long n, unsigned long long v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
}  // namespace
cudaError_t fill_xch_empty(double* buf, long long n, cudaStream_t st) {
  k_fill_u64<<<592, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(buf), n, kXchEmpty);
  return cudaGetLastError();
}

cudaError_t prepare_ws_kernels() {
  int r = 0;
  cudaError_t e = cudaSuccess;
  auto prep = [&](const void* fn, size_t smem, int threads) {
    if (e == cudaSuccess) e = prepare_kernel(fn, smem, threads, &r);
  };
  prep(reinterpret_cast<const void*>(k_step_ws<8, 0, false>), sizeof(WsSmem<8, 0, false>), ws_threads(8, false));
  prep(reinterpret_cast<const void*>(k_step_ws<8, 1, false>), sizeof(WsSmem<8, 1, false>), ws_threads(8, false));
  prep(reinterpret_cast<const void*>(k_step_ws<8, 0, true>), sizeof(WsSmem<8, 0, true>), ws_threads(8, true));
  prep(reinterpret_cast<const void*>(k_step_ws<4, 0, false>), sizeof(WsSmem<4, 0, false>), ws_threads(4, false));
  prep(reinterpret_cast<const void*>(k_step_ws<4, 1, false>), sizeof(WsSmem<4, 1, false>), ws_threads(4, false));
  return e;
}

cudaError_t launch_step_ws(const Geom& G, const DevParams& p, const double* A, double* B, const double* phig,
                           const Launch& ln, const Health& hl, const StepMaps* maps, cudaStream_t st, const Peers& pr,
                           const XchArgs* xch) {
  if (!step_ws_fits(maps)) return cudaErrorInvalidValue;
  const bool t8 = maps->ty == 8;
  if (xch && p.coll == 0) {  // (MRT: the plain kernel -- same bits)
    if (!step_xch_fits(G, maps)) return cudaErrorInvalidValue;
    return launch_ws_t<8, 0, true>(G, p, A, B, phig, ln, hl, maps, st, pr, xch);
  }
  if (p.coll == 1)
    return t8 ? launch_ws_t<8, 1>(G, p, A, B, phig, ln, hl, maps, st, pr)
              : launch_ws_t<4, 1>(G, p, A, B, phig, ln, hl, maps, st, pr);
  return t8 ? launch_ws_t<8, 0>(G, p, A, B, phig, ln, hl, maps, st, pr)
            : launch_ws_t<4, 0>(G, p, A, B, phig, ln, hl, maps, st, pr);
}

}  // namespace lbk

#ifdef LB_TRACE
// copy the trace of the last launches out and clear it (measurement build only)
extern "C" int lb_debug_trace_get(unsigned long long* out, int nblocks) {
  if (nblocks < 0 || nblocks > (1 << 16)) return 1;
  static unsigned long long zero[1 << 16][4];
  return cudaMemcpyFromSymbol(out, lbk::lb_trace_buf, (size_t)nblocks * 32) != cudaSuccess ||
         cudaMemcpyToSymbol(lbk::lb_trace_buf, zero, sizeof(zero)) != cudaSuccess;
}
#endif
