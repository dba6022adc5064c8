// lb_step_ch.cu -- the NEXT-2 variant of the step (DESIGN.md readings
// R29-R33): phi is a field evolved by a finite-difference Cahn-Hilliard update
// with first-order upwind advective fluxes, instead of the g distribution
// ("Advection" and the finite-difference order-parameter update of Ludwig,
// PAPER.md P:176-183); f collides with the chemical stress in its
// equilibrium and a three-rate MRT (R23-R25, `collide_mrt`), so u = j / rho.
//
// One fused single pass per step, like the main step kernel: per site f is read
// and written once (304 B) and phi read and written once (16 B) -- 320 B/site
// instead of 608.  A CTA owns a TX x TY tile and marches in z:
//
//   sF  : f of planes k and k+1 on the tile + 1-site halo (TMA, one copy per
//         component into 128-byte-aligned slots; per-thread 16-byte cp.async
//         where the halo wraps), two buffers
//   sPhi: ring of 5 phi planes on the tile + 2-site halo (cp.async)
//   sU  : ring of 3 planes of u = j / rho on the tile + 1 halo (R32)
//   sMu : ring of 3 planes of mu on the tile + 1 halo (R3)
//
// Iteration k: wait f(k+1), phi(k+2) -> u(k+1), mu(k+1) on the halo box; f(k)
// to registers; issue f(k+2), phi(k+3); P(k) at the site (R4); collide f and
// push (A.8); phi(k+1 step) = phi - div J + M lap mu (R30, R31) -> next phi
// buffer.  A z-slab reads f's edge planes of its neighbours (for u at z +- 1) and
// phi on two planes from ghost planes, and pushes the leaving f components into
// the ghost planes of B, like the other step kernels.
#include "lb_device.cuh"
#include "lb_tma.cuh"

namespace lbk {
namespace {

constexpr int kCX = 32;

// z wrapped into [0, n) for z in [-n, 2n): one compare and add, no division (the
// kernel reaches planes zA - 2 .. zB + 1 of a periodic slab, nzl >= 3)
__device__ __forceinline__ int zwrap1(int z, int n) { return z < 0 ? z + n : (z >= n ? z - n : z); }
// ring slot of plane z >= -60: the floored z mod N (N divides 60), by an unsigned
// modulo by a constant (multiply-high, no sign fix-up)
template <int N>
__device__ __forceinline__ int rslot(int z) {
  static_assert(60 % N == 0, "ring size must divide 60");
  return (int)((unsigned)(z + 60) % (unsigned)N);
}

// f box buffers: 3 (the box of plane k+2 goes out while plane k is collided: two
// iterations of lead) where shared memory allows, else 2
template <int TY>
struct alignas(128) ChSmem {
  static constexpr int NBUF = TY == 8 ? 3 : 2;
  static constexpr int TX = kCX, NT = TX * TY;
  static constexpr int FX = TX + 4, FY = TY + 2;              // f box: x0-2 .. x0+TX+1 (16-byte start), y +- 1
  static constexpr int FS = ((FX * FY + 15) / 16) * 16;       // component slot, 128-byte multiple
  static constexpr int BX = TX + 4, BY = TY + 4, NB = BX * BY;  // phi box: +- 2
  static constexpr int UX = TX + 2, UY = TY + 2, NU = UX * UY;  // u, mu box: +- 1
  alignas(128) double sF[NBUF][Q][FS];
  alignas(128) double sPhi[5][NB];
  double sU[3][3][NU];
  double sMu[3][NU];
  unsigned long long bar[NBUF];
};

template <int TY>
__global__ void __launch_bounds__(kCX* TY, 1)
    k_step_ch(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B,
              const double* __restrict__ phiA, double* __restrict__ phiB, int zc, Health hl,
              const __grid_constant__ CUtensorMap tm_f1) {
  using S = ChSmem<TY>;
  constexpr int TX = kCX, NT = S::NT;
  constexpr int FX = S::FX, FY = S::FY, FS = S::FS, BX = S::BX, UX = S::UX, NU = S::NU, NBUF = S::NBUF;
  constexpr unsigned FBOX_BYTES = Q * FX * FY * 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const int tid = threadIdx.x;
  const int lx = tid % TX, ly = tid / TX;
  const int ntx = (G.nx + TX - 1) / TX, nty = (G.ny + TY - 1) / TY;
  const int tile = blockIdx.x % (ntx * nty);
  const int x0 = (tile % ntx) * TX, y0 = (tile / ntx) * TY;
  const int zA = (blockIdx.x / (ntx * nty)) * zc;
  const int zB = min(zA + zc, G.nzl);
  const int x = x0 + lx, y = y0 + ly;
  const bool active = x < G.nx && y < G.ny;
  const long long nxy = G.nxy;
  const bool fbox_tma = x0 >= 2 && x0 + TX + 2 <= G.nx && y0 >= 1 && y0 + TY + 1 <= G.ny;

  auto wrapx = [&](int v) { v %= G.nx; return v < 0 ? v + G.nx : v; };
  auto wrapy = [&](int v) { v %= G.ny; return v < 0 ? v + G.ny : v; };
  auto wz = [&](int z) { return zwrap1(z, G.nzl); };
  // plane read at z: periodic within a whole-lattice slab, else the ghost planes
  // (f: -1 and nzl, holding the neighbours' edge planes; phi: -2 .. nzl+1)
  auto zf = [&](int z) { return G.zwrap ? wz(z) : z; };

  if (tid == 0) {
    for (int b = 0; b < NBUF; ++b) mbar_init(&sm.bar[b], 1);
    fence_barrier_init();
  }
  __syncthreads();
  unsigned ph = 0;  // bit b: parity of bar[b]
  const unsigned long long pol_f = policy_evict_last();  // the halo rows are re-read by the neighbours

  // ---- f box of plane zp -> buffer zp % NBUF (TMA per component, or per-thread copies)
  constexpr int FROWU = FX / 2, FBU = FY * FROWU, FBR = (FBU + NT - 1) / NT;
  long long fb_src[FBR];
  int fb_dst[FBR];
#pragma unroll
  for (int r = 0; r < FBR; ++r) {
    const int u = tid + r * NT;
    const int row = u / FROWU, cu = u - row * FROWU;
    fb_src[r] = (long long)wrapy(y0 - 1 + row) * G.nx + wrapx(x0 - 2 + cu * 2);
    fb_dst[r] = u < FBU ? row * FX + cu * 2 : -1;
  }
  auto issue_f = [&](int zp) {
    const int b = rslot<NBUF>(zp);
    const int zs = zf(zp);
    if (fbox_tma) {
      if (tid == 0) {
        fence_proxy_async();
        mbar_expect_tx(&sm.bar[b], FBOX_BYTES);
        const int cpl = (zs + GZ) * NSLOT;
#pragma unroll 1
        for (int j = 0; j < Q; ++j)
          tma_load_3d(&sm.sF[b][j][0], &tm_f1, x0 - 2, y0 - 1, cpl + fslot_of_rank(j), &sm.bar[b], pol_f);
      }
    } else {
      const double* base = A + (long long)(zs + GZ) * G.plane;
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const double* bj = base + (long long)fslot_of_rank(j) * nxy;
#pragma unroll
        for (int r = 0; r < FBR; ++r)
          if (fb_dst[r] >= 0) cp_async_v<2>(&sm.sF[b][j][fb_dst[r]], bj + fb_src[r]);
      }
    }
  };
  auto wait_f = [&](int zp) {
    const int b = rslot<NBUF>(zp);
    if (fbox_tma) {
      mbar_wait(&sm.bar[b], (ph >> b) & 1);
      ph ^= 1u << b;
    }
  };
  // ---- phi box of plane zp -> ring slot zp % 5 (per-thread 16-byte copies)
  constexpr int PROWU = BX / 2, PBU = (TY + 4) * PROWU, PBR = (PBU + NT - 1) / NT;
  long long pb_src[PBR];
  int pb_dst[PBR];
#pragma unroll
  for (int r = 0; r < PBR; ++r) {
    const int u = tid + r * NT;
    const int row = u / PROWU, cu = u - row * PROWU;
    pb_src[r] = (long long)wrapy(y0 - 2 + row) * G.nx + wrapx(x0 - 2 + cu * 2);
    pb_dst[r] = u < PBU ? row * BX + cu * 2 : -1;
  }
  auto issue_phi = [&](int zp) {
    const double* base = phiA + phi_plane_index(G, zf(zp));
    double* ring = sm.sPhi[rslot<5>(zp)];
#pragma unroll
    for (int r = 0; r < PBR; ++r)
      if (pb_dst[r] >= 0) cp_async_v<2>(&ring[pb_dst[r]], base + pb_src[r]);
  };

  // ---- u and mu of plane zp on the +-1 box (needs f box zp, phi zp-1 .. zp+1)
  auto make_u_mu_at = [&](int zp, int e) {
    const double(*fb)[FS] = sm.sF[rslot<NBUF>(zp)];
    double(*u3)[NU] = sm.sU[rslot<3>(zp)];
    double* mu = sm.sMu[rslot<3>(zp)];
    const double* f0 = sm.sPhi[rslot<5>(zp - 1)];
    const double* f1 = sm.sPhi[rslot<5>(zp)];
    const double* f2 = sm.sPhi[rslot<5>(zp + 1)];
    {
      const int ex = e % UX, ey = e / UX;
      const int fi = ey * FX + ex + 1;  // f box: x offset 2, y offset 1; u box: offsets 1, 1
      double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
      for (int i = 0; i < Q; ++i) {  // A.3, canonical order
        const double v = fb[frank(i)][fi];
        rho += v;
        if (cx(i)) jx += cx(i) * v;
        if (cy(i)) jy += cy(i) * v;
        if (cz(i)) jz += cz(i) * v;
      }
      const double rinv = 1.0 / rho;
      u3[0][e] = jx * rinv;  // R32
      u3[1][e] = jy * rinv;
      u3[2][e] = jz * rinv;
      const int c = (ey + 1) * BX + (ex + 1);
      const double phc = f1[c];
      const double lap = (f1[c + 1] + f1[c - 1]) + (f1[c + BX] + f1[c - BX]) + (f2[c] + f0[c]) - 6.0 * phc;
      mu[e] = chem_pot(p, phc, lap);
    }
  };
  auto make_u_mu = [&](int zp) {
    for (int e = tid; e < NU; e += NT) make_u_mu_at(zp, e);
  };
  // the ring of the +-1 box around the tile: rows 0 and UY-1, then columns 0 and UX-1
  constexpr int NRING = NU - NT;
  auto ring_site = [&](int r) {
    if (r < UX) return r;
    if (r < 2 * UX) return (S::UY - 1) * UX + (r - UX);
    const int t = r - 2 * UX;
    return (1 + t / 2) * UX + ((t & 1) ? UX - 1 : 0);
  };

  // ---- prologue: phi zA-2 .. zA+1, f boxes zA-1, zA; u, mu of zA-1 and zA
  for (int zp = zA - 2; zp <= zA + 1; ++zp) issue_phi(zp);
  issue_f(zA - 1);
  issue_f(zA);
  if (NBUF == 3) issue_f(zA + 1);
  cp_commit();
  cp_wait<0>();
  wait_f(zA - 1);
  __syncthreads();
  make_u_mu(zA - 1);
  __syncthreads();
  if (NBUF == 2) issue_f(zA + 1);  // into the buffer of zA - 1
  issue_phi(zA + 2);
  cp_commit();
  wait_f(zA);
  __syncthreads();
  make_u_mu(zA);

  const int xm1 = wrapx(x - 1), xp1 = wrapx(x + 1), ym1 = wrapy(y - 1), yp1 = wrapy(y + 1);
  const int cb = (ly + 2) * BX + (lx + 2);  // own site in the phi box
  const int cu = (ly + 1) * UX + (lx + 1);  // own site in the u / mu box
  const int cf = (ly + 1) * FX + (lx + 2);  // own site in the f box

  for (int k = zA; k < zB; ++k) {
    cp_wait<0>();  // phi(k+2)
    wait_f(k + 1);
    __syncthreads();  // (also: everyone is past iteration k-1)
    double f[Q];
    if constexpr (NBUF == 3) {
      // one barrier per plane: the buffer of plane k-1 and the ring slots of k-2 are
      // free; u, mu (k+1) at this thread's own site are computed by this thread (all
      // the update of plane k reads of plane k+1), the ring of the box by the first
      // NRING threads (read only after the next barrier)
      if (k + 2 <= zB) issue_f(k + 2);
      if (k + 3 <= zB + 1) issue_phi(k + 3);
      cp_commit();
      make_u_mu_at(k + 1, cu);
      if (tid < NRING) make_u_mu_at(k + 1, ring_site(tid));
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = sm.sF[rslot<NBUF>(k)][frank(i)][cf];
    } else {
      make_u_mu(k + 1);
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = sm.sF[rslot<NBUF>(k)][frank(i)][cf];
      __syncthreads();  // f(k) consumed, u / mu (k+1) written
      if (k + 2 <= zB) issue_f(k + 2);
      if (k + 3 <= zB + 1) issue_phi(k + 3);
      cp_commit();
    }
    if (!active) continue;
    // ring slots of planes k - 1, k, k + 1 (one modulo each per plane)
    const int p0 = rslot<5>(k), pm = p0 == 0 ? 4 : p0 - 1, pp = p0 == 4 ? 0 : p0 + 1;
    const int u0 = rslot<3>(k), um = u0 == 0 ? 2 : u0 - 1, up = u0 == 2 ? 0 : u0 + 1;
    // P(k) at the site (R4, A.2)
    const double* r0 = sm.sPhi[p0];
    const double* rm = sm.sPhi[pm];
    const double* rp = sm.sPhi[pp];
    const double ph = r0[cb];
    const double xp = r0[cb + 1], xm = r0[cb - 1], yp = r0[cb + BX], ym = r0[cb - BX], zp = rp[cb], zm = rm[cb];
    const double lap = (xp + xm) + (yp + ym) + (zp + zm) - 6.0 * ph;
    double P6[6];
    stress6(p, ph, 0.5 * (xp - xm), 0.5 * (yp - ym), 0.5 * (zp - zm), lap, P6);
    // collide f (R23-R25) and push (A.8); g is not used in this variant
    double* const zb[3] = {push_plane(G, B, Peers{}, k - 1), push_plane(G, B, Peers{}, k),
                           push_plane(G, B, Peers{}, k + 1)};  // A.8; ghost planes for slabs
    const double g0[Q] = {};
    const double rho = collide_mrt(p, f, g0, 0.0, 0.0, P6, [&](int i, double fs, double) {
      const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
      const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
      LB_CHECK(hl, xd >= 0 && xd < G.nx && yd >= 0 && yd < G.ny);
      double* d = zb[cz(i) + 1] + (long long)yd * G.nx + xd;
      __stcs(d + (long long)slot(0, i) * nxy, fs);
    });
    // phi update (R30, R31): upwind fluxes through the six faces, M lap mu
    const double* uk = &sm.sU[u0][0][0];
    const double* ukm = &sm.sU[um][0][0];
    const double* ukp = &sm.sU[up][0][0];
    auto flux = [](double ua, double ub, double pa, double pb) {  // face between a and b = a + e
      const double uf = 0.5 * (ua + ub);
      return uf * (uf > 0.0 ? pa : pb);
    };
    double div = 0.0;
    div = div + (flux(uk[cu], uk[cu + 1], ph, xp) - flux(uk[cu - 1], uk[cu], xm, ph));
    div = div + (flux(uk[NU + cu], uk[NU + cu + UX], ph, yp) - flux(uk[NU + cu - UX], uk[NU + cu], ym, ph));
    div = div + (flux(uk[2 * NU + cu], ukp[2 * NU + cu], ph, zp) - flux(ukm[2 * NU + cu], uk[2 * NU + cu], zm, ph));
    const double* mk = sm.sMu[u0];
    const double lapmu = (mk[cu + 1] + mk[cu - 1]) + (mk[cu + UX] + mk[cu - UX]) +
                         (sm.sMu[up][cu] + sm.sMu[um][cu]) - 6.0 * mk[cu];
    const double phn = (ph - div) + p.mob * lapmu;
    phiB[phi_plane_index(G, k) + (long long)y * G.nx + x] = phn;
    if (!(rho > 0.0) || !isfinite(rho) || !isfinite(phn)) health_report(hl, G, x, y, k);  // R22
  }
  cp_wait<0>();
  __syncthreads();
  if (tid == 0) health_tick(hl);
}

// ============================================================================
// Warp-specialised variant (32 x 8 tiles; the default): the same arithmetic in
// the same order as k_step_ch -- so the same bits -- split between two roles
// that never wait for each other inside a plane:
//
//   collision warps (256 threads, one per column): f of plane k from the f box,
//       P(k) from the phi ring (R4), the MRT collision and the push (A.8); they
//       also issue every copy (f boxes by TMA -- per-thread cp.async where the box
//       wraps -- and the phi boxes by cp.async, completing on mbarriers);
//   stencil warps (256 threads): u, mu of plane k+1 on the +-1 box from the f box
//       of plane k+1 (R32, R3) and the phi update of plane k (R30, R31), which
//       needs only their own rings.
//
// Iteration k of the collision waits for the f box of plane k and for the stencil
// to be done with plane k-1 (then the slots of box k and phi k-2 are free: it
// issues box k+3 and phi k+4 into them), then phi(k+1) for P(k).  Iteration j of
// the stencil waits for box j+1 and phi j+2.  No cycle: the stencil's inputs of
// iteration j were issued by the collision's iterations j-2 and j-2 or earlier.
// Measured at 512 x 512 x 64 (B200): 15,240 MLUPS against 13,300 for k_step_ch.
template <int TY, int NPR_ = 6>
struct alignas(128) ChWsSmem {
  static constexpr int NBUF = 3;
  static constexpr int TX = kCX, NT = TX * TY;
  static constexpr int FX = TX + 4, FY = TY + 2;
  static constexpr int FB = FX * FY;  // one component of the f box
  // the box as the three f slot runs (5, 9, 5 components, each one TMA copy), each
  // run starting 128-byte aligned
  static constexpr int al16(int v) { return (v + 15) / 16 * 16; }
  static constexpr int RUN1 = al16(5 * FB), RUN2 = al16(RUN1 + 9 * FB), BOXD = al16(RUN2 + 5 * FB);
  static constexpr int BX = TX + 4, BY = TY + 4, NB = BX * BY;
  static constexpr int UX = TX + 2, UY = TY + 2, NU = UX * UY;
  // component of rank j (f slot order) in a box
  __device__ static constexpr int fofs(int j) { return j < 5 ? j * FB : (j < 14 ? RUN1 + (j - 5) * FB : RUN2 + (j - 14) * FB); }
  static constexpr int NPR = NPR_;  // phi ring: planes k-1 .. k+NPR-2 (phi of plane k+NPR-2 goes out at iteration k)
  alignas(128) double sF[NBUF][BOXD];
  alignas(128) double sPhi[NPR][NB];
  double sU[3][3][NU];
  double sMu[3][NU];
  unsigned long long box_full[NBUF], phi_full[NPR], sdone[2];
};

__device__ __forceinline__ void ch_named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void ch_mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on `bar` once every cp.async this thread issued so far has completed
__device__ __forceinline__ void cp_async_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int TY, int NPR_ = 6>
__global__ void __launch_bounds__(2 * kCX * TY, 1)
    k_step_ch_ws(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B,
                 const double* __restrict__ phiA, double* __restrict__ phiB, int zc, Health hl,
                 const __grid_constant__ CUtensorMap tm_f5, const __grid_constant__ CUtensorMap tm_f9,
                 const __grid_constant__ CUtensorMap tm_phi) {
  using S = ChWsSmem<TY, NPR_>;
  constexpr int TX = kCX, NT = S::NT;
  constexpr int FX = S::FX, FY = S::FY, BX = S::BX, UX = S::UX, NU = S::NU;
  constexpr unsigned FBOX_BYTES = Q * S::FB * 8, PBOX_BYTES = S::NB * 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const int tid = threadIdx.x;
  const int ntx = (G.nx + TX - 1) / TX, nty = (G.ny + TY - 1) / TY;
  const int tile = blockIdx.x % (ntx * nty);
  const int x0 = (tile % ntx) * TX, y0 = (tile / ntx) * TY;
  const int zA = (blockIdx.x / (ntx * nty)) * zc;
  const int zB = min(zA + zc, G.nzl);
  const long long nxy = G.nxy;
  const bool fbox_tma = x0 >= 2 && x0 + TX + 2 <= G.nx && y0 >= 1 && y0 + TY + 1 <= G.ny;
  const bool pbox_tma = x0 >= 2 && x0 + TX + 2 <= G.nx && y0 >= 2 && y0 + TY + 2 <= G.ny;
  auto wrapx = [&](int v) { v %= G.nx; return v < 0 ? v + G.nx : v; };
  auto wrapy = [&](int v) { v %= G.ny; return v < 0 ? v + G.ny : v; };
  auto zf = [&](int z) { return G.zwrap ? zwrap1(z, G.nzl) : z; };
  // ring slots and mbarrier parities relative to the first box (zA - 1) / phi (zA - 2)
  auto bslot = [&](int b) { return (b - (zA - 1)) % 3; };
  auto bpar = [&](int b) { return (unsigned)(((b - (zA - 1)) / 3) & 1); };
  constexpr int NPR = S::NPR;
  auto pslot = [&](int q) { return (q - (zA - 2)) % NPR; };
  auto ppar = [&](int q) { return (unsigned)(((q - (zA - 2)) / NPR) & 1); };

  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&sm.box_full[b], fbox_tma ? 1 : NT);
    for (int q = 0; q < NPR; ++q) mbar_init(&sm.phi_full[q], pbox_tma ? 1 : NT);
    for (int d = 0; d < 2; ++d) mbar_init(&sm.sdone[d], NT);
    fence_barrier_init();
  }
  __syncthreads();

  if (tid < NT) {
    // ============================ collision warps ============================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
    const int lx = tid % TX, ly = tid / TX;
    const int x = x0 + lx, y = y0 + ly;
    const bool active = x < G.nx && y < G.ny;
    const unsigned long long pol_f = policy_evict_last();  // the halo rows are re-read by the neighbours
    constexpr int FROWU = FX / 2, FBU = FY * FROWU, FBR = (FBU + NT - 1) / NT;
    long long fb_src[FBR];
    int fb_dst[FBR];
#pragma unroll
    for (int r = 0; r < FBR; ++r) {
      const int u = tid + r * NT;
      const int row = u / FROWU, cu = u - row * FROWU;
      fb_src[r] = (long long)wrapy(y0 - 1 + row) * G.nx + wrapx(x0 - 2 + cu * 2);
      fb_dst[r] = u < FBU ? row * FX + cu * 2 : -1;
      LB_CHECK(hl, fb_dst[r] < 0 || (fb_dst[r] + 1 < S::FB && fb_src[r] >= 0 && fb_src[r] + 1 < nxy));
    }
    auto issue_box = [&](int b) {  // f box of plane b into its slot (b <= zB)
      const int sl = bslot(b);
      const int zs = zf(b);
      double* box = sm.sF[sl];
      if (fbox_tma) {
        if (tid == 0) {  // three copies: the f slot runs 0..4, 10..18, 28..32
          fence_proxy_async();
          mbar_expect_tx(&sm.box_full[sl], FBOX_BYTES);
          const int cpl = (zs + GZ) * NSLOT;
          tma_load_3d(box, &tm_f5, x0 - 2, y0 - 1, cpl, &sm.box_full[sl], pol_f);
          tma_load_3d(box + S::RUN1, &tm_f9, x0 - 2, y0 - 1, cpl + 10, &sm.box_full[sl], pol_f);
          tma_load_3d(box + S::RUN2, &tm_f5, x0 - 2, y0 - 1, cpl + 28, &sm.box_full[sl], pol_f);
        }
      } else {
        const double* base = A + (long long)(zs + GZ) * G.plane;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          const double* bj = base + (long long)fslot_of_rank(j) * nxy;
#pragma unroll
          for (int r = 0; r < FBR; ++r)
            if (fb_dst[r] >= 0) cp_async_v<2>(box + S::fofs(j) + fb_dst[r], bj + fb_src[r]);
        }
        cp_async_arrive_noinc(&sm.box_full[sl]);
      }
    };
    constexpr int PROWU = BX / 2, PBU = (TY + 4) * PROWU, PBR = (PBU + NT - 1) / NT;
    long long pb_src[PBR];
    int pb_dst[PBR];
#pragma unroll
    for (int r = 0; r < PBR; ++r) {
      const int u = tid + r * NT;
      const int row = u / PROWU, cu = u - row * PROWU;
      pb_src[r] = (long long)wrapy(y0 - 2 + row) * G.nx + wrapx(x0 - 2 + cu * 2);
      pb_dst[r] = u < PBU ? row * BX + cu * 2 : -1;
      LB_CHECK(hl, pb_dst[r] < 0 || (pb_dst[r] + 1 < S::NB && pb_src[r] >= 0 && pb_src[r] + 1 < nxy));
    }
    auto issue_phi = [&](int q) {  // phi box of plane q into its ring slot (q <= zB + 1)
      double* ring = sm.sPhi[pslot(q)];
      if (pbox_tma) {
        if (tid == 0) {
          fence_proxy_async();
          mbar_expect_tx(&sm.phi_full[pslot(q)], PBOX_BYTES);
          tma_load_3d(ring, &tm_phi, x0 - 2, y0 - 2, zf(q) + GP, &sm.phi_full[pslot(q)], pol_f);
        }
        return;
      }
      const double* base = phiA + phi_plane_index(G, zf(q));
#pragma unroll
      for (int r = 0; r < PBR; ++r)
        if (pb_dst[r] >= 0) cp_async_v<2>(&ring[pb_dst[r]], base + pb_src[r]);
      cp_async_arrive_noinc(&sm.phi_full[pslot(q)]);
    };

    for (int b = zA - 1; b <= min(zA + 1, zB); ++b) issue_box(b);
    for (int q = zA - 2; q <= min(zA + NPR - 3, zB + 1); ++q) issue_phi(q);
    mbar_wait(&sm.phi_full[pslot(zA - 1)], ppar(zA - 1));
    mbar_wait(&sm.phi_full[pslot(zA)], ppar(zA));

    const int xm1 = wrapx(x - 1), xp1 = wrapx(x + 1), ym1 = wrapy(y - 1), yp1 = wrapy(y + 1);
    const int cb = (ly + 2) * BX + (lx + 2);  // own site in the phi box
    const int cf = (ly + 1) * FX + (lx + 2);  // own site in the f box
    for (int k = zA; k < zB; ++k) {
      double f[Q];
      mbar_wait(&sm.box_full[bslot(k)], bpar(k));
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = sm.sF[bslot(k)][S::fofs(frank(i)) + cf];
      // the stencil is past plane k-1: box k (u, mu(k)) and phi k-2 are free once
      // every collision thread has read f(k) too (and is past P(k-1))
      const int jd = k - 1 - (zA - 2);
      mbar_wait(&sm.sdone[jd & 1], (unsigned)((jd >> 1) & 1));
      ch_named_sync(1, NT);
      if (k == zA && zA + 2 <= zB) issue_box(zA + 2);  // (slot of box zA - 1)
      if (k + 3 <= zB) issue_box(k + 3);
      if (k + NPR - 2 <= zB + 1) issue_phi(k + NPR - 2);  // (into the slot of plane k-2)
      mbar_wait(&sm.phi_full[pslot(k + 1)], ppar(k + 1));
      if (!active) continue;
      const double* r0 = sm.sPhi[pslot(k)];
      const double* rm = sm.sPhi[pslot(k - 1)];
      const double* rp = sm.sPhi[pslot(k + 1)];
      const double ph = r0[cb];
      const double xp = r0[cb + 1], xm = r0[cb - 1], yp = r0[cb + BX], ym = r0[cb - BX], zp = rp[cb], zm = rm[cb];
      const double lap = (xp + xm) + (yp + ym) + (zp + zm) - 6.0 * ph;
      double P6[6];
      stress6(p, ph, 0.5 * (xp - xm), 0.5 * (yp - ym), 0.5 * (zp - zm), lap, P6);  // P(k) (R4, A.2)
      double* const zb[3] = {push_plane(G, B, Peers{}, k - 1), push_plane(G, B, Peers{}, k),
                             push_plane(G, B, Peers{}, k + 1)};
      const double g0[Q] = {};
      const double rho = collide_mrt(p, f, g0, 0.0, 0.0, P6, [&](int i, double fs, double) {
        const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
        const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
        LB_CHECK(hl, xd >= 0 && xd < G.nx && yd >= 0 && yd < G.ny);
        double* d = zb[cz(i) + 1] + (long long)yd * G.nx + xd;
        __stcs(d + (long long)slot(0, i) * nxy, fs);
      });
      if (!(rho > 0.0) || !isfinite(rho)) health_report(hl, G, x, y, k);  // R22
    }
    cp_wait<0>();
  } else {
    // ============================== stencil warps ==============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    const int a = tid - NT;
    const int lx = a % TX, ly = a / TX;
    const int x = x0 + lx, y = y0 + ly;
    const bool active = x < G.nx && y < G.ny;
    auto make_u_mu_at = [&](int zp, int e) {  // u, mu of plane zp at box site e (k_step_ch's arithmetic)
      const double* fb = sm.sF[bslot(zp)];
      double(*u3)[NU] = sm.sU[rslot<3>(zp)];
      double* mu = sm.sMu[rslot<3>(zp)];
      const double* f0 = sm.sPhi[pslot(zp - 1)];
      const double* f1 = sm.sPhi[pslot(zp)];
      const double* f2 = sm.sPhi[pslot(zp + 1)];
      const int ex = e % UX, ey = e / UX;
      const int fi = ey * FX + ex + 1;
      double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
      for (int i = 0; i < Q; ++i) {  // A.3, canonical order
        const double v = fb[S::fofs(frank(i)) + fi];
        rho += v;
        if (cx(i)) jx += cx(i) * v;
        if (cy(i)) jy += cy(i) * v;
        if (cz(i)) jz += cz(i) * v;
      }
      const double rinv = 1.0 / rho;
      u3[0][e] = jx * rinv;  // R32
      u3[1][e] = jy * rinv;
      u3[2][e] = jz * rinv;
      const int c = (ey + 1) * BX + (ex + 1);
      const double phc = f1[c];
      const double lap = (f1[c + 1] + f1[c - 1]) + (f1[c + BX] + f1[c - BX]) + (f2[c] + f0[c]) - 6.0 * phc;
      mu[e] = chem_pot(p, phc, lap);
    };
    const int cb = (ly + 2) * BX + (lx + 2);
    const int cu = (ly + 1) * UX + (lx + 1);
    mbar_wait(&sm.phi_full[pslot(zA - 2)], ppar(zA - 2));
    mbar_wait(&sm.phi_full[pslot(zA - 1)], ppar(zA - 1));
    for (int j = zA - 2; j < zB; ++j) {
      // s(j): u, mu (j+1) on the box; the phi update of plane j (j >= zA)
      mbar_wait(&sm.box_full[bslot(j + 1)], bpar(j + 1));
      mbar_wait(&sm.phi_full[pslot(j + 2)], ppar(j + 2));
      ch_named_sync(2, NT);  // every stencil thread is past s(j-1): the u, mu slot of j-2 is free
      for (int e = a; e < NU; e += NT) make_u_mu_at(j + 1, e);
      ch_named_sync(2, NT);  // u, mu (j+1) on the whole box
      if (j >= zA && active) {
        const int u0 = rslot<3>(j), um = rslot<3>(j - 1), up = rslot<3>(j + 1);
        const double* r0 = sm.sPhi[pslot(j)];
        const double* rm = sm.sPhi[pslot(j - 1)];
        const double* rp = sm.sPhi[pslot(j + 1)];
        const double ph = r0[cb];
        const double xp = r0[cb + 1], xm = r0[cb - 1], yp = r0[cb + BX], ym = r0[cb - BX], zp = rp[cb], zm = rm[cb];
        const double* uk = &sm.sU[u0][0][0];
        const double* ukm = &sm.sU[um][0][0];
        const double* ukp = &sm.sU[up][0][0];
        auto flux = [](double ua, double ub, double pa, double pb) {  // face between a and b = a + e
          const double uf = 0.5 * (ua + ub);
          return uf * (uf > 0.0 ? pa : pb);
        };
        double div = 0.0;
        div = div + (flux(uk[cu], uk[cu + 1], ph, xp) - flux(uk[cu - 1], uk[cu], xm, ph));
        div = div + (flux(uk[NU + cu], uk[NU + cu + UX], ph, yp) - flux(uk[NU + cu - UX], uk[NU + cu], ym, ph));
        div = div + (flux(uk[2 * NU + cu], ukp[2 * NU + cu], ph, zp) - flux(ukm[2 * NU + cu], uk[2 * NU + cu], zm, ph));
        const double* mk = sm.sMu[u0];
        const double lapmu = (mk[cu + 1] + mk[cu - 1]) + (mk[cu + UX] + mk[cu - UX]) +
                             (sm.sMu[up][cu] + sm.sMu[um][cu]) - 6.0 * mk[cu];
        const double phn = (ph - div) + p.mob * lapmu;  // R30
        phiB[phi_plane_index(G, j) + (long long)y * G.nx + x] = phn;
        if (!isfinite(phn)) health_report(hl, G, x, y, j);  // R22
      }
      ch_mbar_arrive(&sm.sdone[(j - (zA - 2)) & 1]);
    }
  }
  __syncthreads();
  if (tid == 0) health_tick(hl);
}

template <int TY>
cudaError_t launch_ch_t(const Geom& G, const DevParams& p, const double* A, double* B, const double* phiA,
                        double* phiB, int zc, const Health& hl, const ChMaps* maps, cudaStream_t st) {
  constexpr size_t smem = sizeof(ChSmem<TY>);
  static_assert(smem <= 232448, "shared memory per CTA exceeds 227 KB");
  auto kern = k_step_ch<TY>;
  int resid = 0;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), smem, kCX * TY, &resid);
  if (e != cudaSuccess) return e;
  const int tiles = ((G.nx + kCX - 1) / kCX) * ((G.ny + TY - 1) / TY);
  const int nblk = tiles * ((G.nzl + zc - 1) / zc);
  kern<<<nblk, kCX * TY, smem, st>>>(G, p, A, B, phiA, phiB, zc, hl, reinterpret_cast<const CUtensorMap*>(maps->m)[0]);
  return cudaGetLastError();
}

template <int TY, int NPR>
cudaError_t launch_ch_ws_t(const Geom& G, const DevParams& p, const double* A, double* B, const double* phiA,
                           double* phiB, int zc, const Health& hl, const ChMaps* maps, cudaStream_t st) {
  constexpr size_t smem = sizeof(ChWsSmem<TY, NPR>);
  static_assert(smem <= 232448, "shared memory per CTA exceeds 227 KB");
  auto kern = k_step_ch_ws<TY, NPR>;
  int resid = 0;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), smem, 2 * kCX * TY, &resid);
  if (e != cudaSuccess) return e;
  const int tiles = ((G.nx + kCX - 1) / kCX) * ((G.ny + TY - 1) / TY);
  const int nblk = tiles * ((G.nzl + zc - 1) / zc);
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  kern<<<nblk, 2 * kCX * TY, smem, st>>>(G, p, A, B, phiA, phiB, zc, hl, m[1], m[2], m[3]);
  return cudaGetLastError();
}

}  // namespace

cudaError_t prepare_ch_kernels() {
  int r = 0;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(k_step_ch<8>), sizeof(ChSmem<8>), kCX * 8, &r);
  if (e == cudaSuccess)
    e = prepare_kernel(reinterpret_cast<const void*>(k_step_ch_ws<8, 6>), sizeof(ChWsSmem<8, 6>), 2 * kCX * 8, &r);
  if (e == cudaSuccess)
    e = prepare_kernel(reinterpret_cast<const void*>(k_step_ch_ws<8, 5>), sizeof(ChWsSmem<8, 5>), 2 * kCX * 8, &r);
  if (e == cudaSuccess) e = prepare_kernel(reinterpret_cast<const void*>(k_step_ch<4>), sizeof(ChSmem<4>), kCX * 4, &r);
  return e;
}

bool make_ch_maps(const Geom& G, const double* buf, const double* phibuf, int ty, ChMaps* out) {
  out->ok = false;
  out->ty = ty;
  if (G.nx % 2 != 0) return false;
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(out->m);
  if (!encode_dist_map(&m[0], G, buf, kCX + 4, ty + 2, 1) || !encode_dist_map(&m[1], G, buf, kCX + 4, ty + 2, 5) ||
      !encode_dist_map(&m[2], G, buf, kCX + 4, ty + 2, 9) || !encode_phi_map(&m[3], G, phibuf, kCX + 4, ty + 4))
    return false;
  out->ok = true;
  return true;
}

cudaError_t launch_step_ch(const Geom& G, const DevParams& p, const double* A, double* B, const double* phiA,
                           double* phiB, int zc, const Health& hl, const ChMaps* maps, cudaStream_t st, bool ws,
                           int variant) {
  if (!maps || !maps->ok) return cudaErrorInvalidValue;
  if (maps->ty == 8 && ws) {
    // phi ring of 6 planes over several waves (512 x 512 x 64: +2% over 5), of 5 where
    // every block runs in the first wave (128^3: +2% over 6); variant 1 forces 5
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long nblk = (long long)((G.nx + kCX - 1) / kCX) * ((G.ny + 7) / 8) * ((G.nzl + zc - 1) / zc);
    return variant == 1 || nblk <= sms ? launch_ch_ws_t<8, 5>(G, p, A, B, phiA, phiB, zc, hl, maps, st)
                                       : launch_ch_ws_t<8, 6>(G, p, A, B, phiA, phiB, zc, hl, maps, st);
  }
  if (maps->ty == 8) return launch_ch_t<8>(G, p, A, B, phiA, phiB, zc, hl, maps, st);
  return launch_ch_t<4>(G, p, A, B, phiA, phiB, zc, hl, maps, st);
}

}  // namespace lbk
