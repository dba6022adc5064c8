// lb_step_lc.cu -- the NEXT-4 workload (readings R34-R45): the
// paper's liquid-crystal test case.  A Q tensor (symmetric, traceless: five stored
// components) evolves by the finite-difference Beris-Edwards "LC Update" with the
// Landau-de Gennes free energy and the "Advection" flux; the LB fluid f feels the
// divergence of the "Chemical stress" (stencils P:185-190).
//
// One fused single pass per step: per site f is read and written once (304 B),
// Q (80 B) and the stored velocity u (48 B) likewise -- 432 B/site.  A CTA owns a
// 32 x 8 tile (one thread per column) and marches in z:
//
//   sF  : f of planes k (being collided) and k+1 (in flight), TMA, tile only
//   sQ  : ring of 4 Q planes (k .. k+3) on the tile + 2-site halo (cp.async)
//   sU  : ring of 3 planes of the stored u (k .. k+2) on the tile + 1-site halo
//   sSig: the in-plane columns of the stress sigma_ax, sigma_ay of planes k, k+1
//         on the tile + 1-site halo
//
// Iteration k (one CTA barrier): gradients, H, fed and sigma of plane k+1 on the
// +-1 box (each thread its own site, the first 84 threads the ring: R35-R38);
// F(k) = div sigma at the site (in-plane columns from sSig, the z column from the
// sigma_az the thread kept for planes k-1 and k+1: R39); collide f(k) (Guo BGK,
// R40) and push (A.8); store u' = (j + F/2)/rho; LC update of Q(k) with the stored
// u (co-rotation R41, upwind advection and Gamma H, R42) -> next Q buffer.
// A whole periodic lattice wraps in z; a z-slab reads Q on two ghost planes and u
// on one at each end (filled by the exchange before the step) and pushes the f
// components that leave it into the ghost planes of B (sent after the step), as
// the binary-fluid step does.
#include "lb_device.cuh"
#include "lb_tma.cuh"

namespace lbk {
namespace {

constexpr int kLX = 32, kLY = 8, kLT = kLX * kLY;

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

struct alignas(128) LcSmem {
  static constexpr int BX = kLX + 4, BY = kLY + 4, NB = BX * BY;  // Q box: +-2
  static constexpr int UX = kLX + 4, UY = kLY + 2, NU = UX * UY;  // u box: x -2..+1 (16-byte rows), y +-1
  static constexpr int SX = kLX + 2, SY = kLY + 2, NS = SX * SY;  // sigma box: +-1
  alignas(128) double sF[2][Q][kLT];
  alignas(16) double sQ[4][5][NB];
  alignas(16) double sU[3][3][NU];
  double sSig[2][6][NS];  // [0..2]: sigma_ax (a = x, y, z), [3..5]: sigma_ay
  unsigned long long bar[2];
};

// ---- R34: five stored components -> the full symmetric traceless tensor
__device__ __forceinline__ void full3(const double (&v)[5], double (&M)[3][3]) {
  M[0][0] = v[0];
  M[0][1] = v[1];
  M[0][2] = v[2];
  M[1][0] = v[1];
  M[1][1] = v[3];
  M[1][2] = v[4];
  M[2][0] = v[2];
  M[2][1] = v[4];
  M[2][2] = -v[0] - v[3];
}

// ---- R35-R38 at one site: molecular field H (five components) and the stress
// sigma (full, not symmetric) from Q, dq[c] = d_c Q and the 7-point lap Q.
//   H     = -A0 (1 - gamma/3) Q + A0 gamma (Q Q - I Q:Q/3) - A0 gamma (Q:Q) Q + kappa lap Q
//   fed   = A0/2 (1 - gamma/3) Q:Q - A0 gamma/3 tr Q^3 + A0 gamma/4 (Q:Q)^2 + kappa/2 |d Q|^2
//   sigma = fed I + 2 xi Qt (Q:H) - xi (M + M^T) - kappa G + (M^T - M),
// with Qt = Q + I/3, M = H Qt (so Qt H = M^T, Q H - H Q = M^T - M) and
// G_ab = d_a Q_cd d_b Q_cd.
__device__ __forceinline__ void lc_fields(const DevParams& p, const double (&q)[5], const double (&dq)[3][5],
                                          const double (&lap)[5], double (&H)[5], double (&sg)[3][3]) {
  double Qm[3][3], L[3][3], QQ[3][3], Hf[3][3];
  full3(q, Qm);
  full3(lap, L);
  double q2 = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      q2 += Qm[a][b] * Qm[a][b];
      QQ[a][b] = Qm[a][0] * Qm[0][b] + Qm[a][1] * Qm[1][b] + Qm[a][2] * Qm[2][b];
    }
  const double c1 = -p.lc_a0 * (1.0 - p.lc_gamma * (1.0 / 3.0)), c2 = p.lc_a0 * p.lc_gamma;
  double tr3 = 0.0, qh = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double qq = a == b ? QQ[a][b] - q2 * (1.0 / 3.0) : QQ[a][b];
      Hf[a][b] = (c1 * Qm[a][b] + c2 * qq - c2 * q2 * Qm[a][b]) + p.kappa * L[a][b];
      tr3 += QQ[a][b] * Qm[a][b];
      qh += Qm[a][b] * Hf[a][b];
    }
  H[0] = Hf[0][0];
  H[1] = Hf[0][1];
  H[2] = Hf[0][2];
  H[3] = Hf[1][1];
  H[4] = Hf[1][2];
  // G_ab = d_a Q_cd d_b Q_cd over the symmetric pairs (cd): the diagonal and twice the
  // three off-diagonal entries (Q_zz = -Q_xx - Q_yy); |grad Q|^2 = tr G
  double dzz[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) dzz[c] = -dq[c][0] - dq[c][3];
  auto gab = [&](int a, int b) {
    return (dq[a][0] * dq[b][0] + dq[a][3] * dq[b][3] + dzz[a] * dzz[b]) +
           2.0 * (dq[a][1] * dq[b][1] + dq[a][2] * dq[b][2] + dq[a][4] * dq[b][4]);
  };
  const double Gxx = gab(0, 0), Gyy = gab(1, 1), Gzz = gab(2, 2), Gxy = gab(0, 1), Gxz = gab(0, 2), Gyz = gab(1, 2);
  const double Gm[3][3] = {{Gxx, Gxy, Gxz}, {Gxy, Gyy, Gyz}, {Gxz, Gyz, Gzz}};
  const double g2 = Gxx + Gyy + Gzz;
  const double bulk = 0.5 * p.lc_a0 * (1.0 - p.lc_gamma * (1.0 / 3.0)) * q2 - p.lc_a0 * p.lc_gamma * (1.0 / 3.0) * tr3 +
                      0.25 * p.lc_a0 * p.lc_gamma * q2 * q2;
  const double fed = bulk + 0.5 * p.kappa * g2;
  double M[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      M[a][b] = Hf[a][0] * (Qm[0][b] + (b == 0 ? 1.0 / 3.0 : 0.0)) + Hf[a][1] * (Qm[1][b] + (b == 1 ? 1.0 / 3.0 : 0.0)) +
                Hf[a][2] * (Qm[2][b] + (b == 2 ? 1.0 / 3.0 : 0.0));
  const double xi = p.lc_xi;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double G = Gm[a][b];
      const double qt = Qm[a][b] + (a == b ? 1.0 / 3.0 : 0.0);
      sg[a][b] = ((a == b ? fed : 0.0) + 2.0 * xi * qt * qh) - xi * (M[a][b] + M[b][a]) - p.kappa * G +
                 (M[b][a] - M[a][b]);
    }
}

// ---- R41: co-rotation S(W, Q) with its trace removed; A = xi D + Omega, so
// xi D - Omega = A^T and S = A Qt + (A Qt)^T - 2 xi Qt tr(Q W).  Five components.
__device__ __forceinline__ void corotation(double xi, const double (&W)[3][3], const double (&q)[5], double (&S5)[5]) {
  double Qm[3][3];
  full3(q, Qm);
  double Am[3][3], N[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) Am[a][b] = xi * (0.5 * (W[a][b] + W[b][a])) + 0.5 * (W[a][b] - W[b][a]);
  double trQW = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      N[a][b] = Am[a][0] * (Qm[0][b] + (b == 0 ? 1.0 / 3.0 : 0.0)) + Am[a][1] * (Qm[1][b] + (b == 1 ? 1.0 / 3.0 : 0.0)) +
                Am[a][2] * (Qm[2][b] + (b == 2 ? 1.0 / 3.0 : 0.0));
      trQW += Qm[a][b] * W[b][a];
    }
  double S[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      S[a][b] = (N[a][b] + N[b][a]) - 2.0 * xi * (Qm[a][b] + (a == b ? 1.0 / 3.0 : 0.0)) * trQW;
  const double t3 = (S[0][0] + S[1][1] + S[2][2]) * (1.0 / 3.0);
  S5[0] = S[0][0] - t3;
  S5[1] = S[0][1];
  S5[2] = S[0][2];
  S5[3] = S[1][1] - t3;
  S5[4] = S[1][2];
}

__global__ void __launch_bounds__(kLT, 1)
    k_step_lc(Geom G, DevParams p, const double* __restrict__ A, double* __restrict__ B, const double* __restrict__ qA,
              double* __restrict__ qB, const double* __restrict__ uA, double* __restrict__ uB, int zc,
              Health hl, const __grid_constant__ CUtensorMap tm5, const __grid_constant__ CUtensorMap tm9) {
  using S = LcSmem;
  constexpr int BX = S::BX, NB = S::NB, UX = S::UX, NU = S::NU, SX = S::SX, NS = S::NS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const int tid = threadIdx.x;
  const int lx = tid % kLX, ly = tid / kLX;
  const int ntx = (G.nx + kLX - 1) / kLX, nty = (G.ny + kLY - 1) / kLY;
  const int tile = blockIdx.x % (ntx * nty);
  const int x0 = (tile % ntx) * kLX, y0 = (tile / ntx) * kLY;
  const int zA = (blockIdx.x / (ntx * nty)) * zc;
  const int zB = min(zA + zc, G.nzl);
  const int x = x0 + lx, y = y0 + ly;
  const bool active = x < G.nx && y < G.ny;
  const long long nxy = G.nxy;

  auto wrapx = [&](int v) { v %= G.nx; return v < 0 ? v + G.nx : v; };
  auto wrapy = [&](int v) { v %= G.ny; return v < 0 ? v + G.ny : v; };
  auto wz = [&](int z) { return zwrap1(z, G.nzl); };
  // plane of the Q and u fields: periodic within a whole-lattice slab, else the
  // ghost planes (Q: -2 .. nzl+1, u: -1 .. nzl; qA, uA point at plane 0)
  auto zf = [&](int z) { return G.zwrap ? zwrap1(z, G.nzl) : z; };

  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  unsigned ph = 0;
  const unsigned long long pol_f = policy_evict_first();

  // ---- f tile of plane zp -> buffer zp % 2 (three TMA boxes: the f slot runs)
  auto issue_f = [&](int zp) {
    if (tid == 0) {
      const int b = ((zp) & 1);
      fence_proxy_async();
      mbar_expect_tx(&sm.bar[b], Q * kLT * 8);
      const int cpl = (wz(zp) + GZ) * NSLOT;
      tma_load_3d(&sm.sF[b][0][0], &tm5, x0, y0, cpl + 0, &sm.bar[b], pol_f);
      tma_load_3d(&sm.sF[b][5][0], &tm9, x0, y0, cpl + 10, &sm.bar[b], pol_f);
      tma_load_3d(&sm.sF[b][14][0], &tm5, x0, y0, cpl + 28, &sm.bar[b], pol_f);
    }
  };
  auto wait_f = [&](int zp) {
    const int b = ((zp) & 1);
    mbar_wait(&sm.bar[b], (ph >> b) & 1);
    ph ^= 1u << b;
  };
  // ---- Q box (+-2) of plane zp -> ring slot zp % 4; u box -> ring slot zp % 3.
  // 16-byte copies of (even, odd) x pairs: nx is even, so a pair never straddles the wrap.
  constexpr int ROWU = BX / 2;  // 18 pairs per row (both boxes are 36 wide)
  const int qrow = tid / ROWU, qcu = tid - qrow * ROWU;
  const bool has_q = tid < S::BY * ROWU, has_u = tid < S::UY * ROWU;
  const long long qsrc = (long long)wrapy(y0 - 2 + qrow) * G.nx + wrapx(x0 - 2 + 2 * qcu);
  const long long usrc = (long long)wrapy(y0 - 1 + qrow) * G.nx + wrapx(x0 - 2 + 2 * qcu);
  const int bdst = qrow * BX + 2 * qcu;  // same row pitch (36) in both boxes
  auto issue_q = [&](int zp) {
    if (!has_q) return;
    const double* base = qA + (long long)zf(zp) * 5 * nxy + qsrc;
    double(*ring)[NB] = sm.sQ[((zp) & 3)];
#pragma unroll
    for (int c = 0; c < 5; ++c) cp_async_v<2>(&ring[c][bdst], base + c * nxy);
  };
  auto issue_u = [&](int zp) {
    if (!has_u) return;
    const double* base = uA + (long long)zf(zp) * 3 * nxy + usrc;
    double(*ring)[NU] = sm.sU[rslot<3>(zp)];
#pragma unroll
    for (int a = 0; a < 3; ++a) cp_async_v<2>(&ring[a][bdst], base + a * nxy);
  };

  // ---- H, sigma of plane zp at sigma-box site e; the in-plane stress columns go to sSig
  // (ring slots: & 3 and & 1 are the non-negative residues also for zp < 0)
  auto fields_at = [&](int zp, int e, double (&q)[5], double (&H)[5], double (&sg)[3][3]) {
    const int ex = e % SX, ey = e / SX;
    const int c = (ey + 1) * BX + (ex + 1);
    const double(*Q0)[NB] = sm.sQ[((zp) & 3)];
    const double(*Qm)[NB] = sm.sQ[((zp - 1) & 3)];
    const double(*Qp)[NB] = sm.sQ[((zp + 1) & 3)];
    double dq[3][5], lap[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {  // R37: central gradient, 7-point Laplacian
      const double v = Q0[k][c];
      const double xp = Q0[k][c + 1], xm = Q0[k][c - 1], yp = Q0[k][c + BX], ym = Q0[k][c - BX];
      const double zp_ = Qp[k][c], zm = Qm[k][c];
      q[k] = v;
      dq[0][k] = 0.5 * (xp - xm);
      dq[1][k] = 0.5 * (yp - ym);
      dq[2][k] = 0.5 * (zp_ - zm);
      lap[k] = (xp + xm) + (yp + ym) + (zp_ + zm) - 6.0 * v;
    }
    lc_fields(p, q, dq, lap, H, sg);
    double(*s)[NS] = sm.sSig[((zp) & 1)];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      s[a][e] = sg[a][0];
      s[3 + a][e] = sg[a][1];
    }
  };
  // the ring of the +-1 box around the tile: rows 0 and SY-1, then columns 0 and SX-1
  constexpr int NRING = NS - kLT;
  auto ring_site = [&](int r) {
    if (r < SX) return r;
    if (r < 2 * SX) return (S::SY - 1) * SX + (r - SX);
    const int t = r - 2 * SX;
    return (1 + t / 2) * SX + ((t & 1) ? SX - 1 : 0);
  };
  const int cs = (ly + 1) * SX + (lx + 1);  // own site in the sigma box
  const int cq = (ly + 2) * BX + (lx + 2);  // own site in the Q box
  const int cu = (ly + 1) * UX + (lx + 2);  // own site in the u box
  // plane zp on the whole box; returns the own site's Q, H and sigma_az.  One call
  // site of fields_at for the own site and the ring site (a loop that is not
  // unrolled): the same instructions, so the same bits wherever a site falls in its
  // tile -- shifted lattices give shifted results bitwise, as in the oracle.
  auto box_plane = [&](int zp, double (&q)[5], double (&H)[5], double (&sz)[3]) {
    const int nsite = tid < NRING ? 2 : 1;
#pragma unroll 1
    for (int r = 0; r < nsite; ++r) {
      double q_[5], H_[5], sg[3][3];
      fields_at(zp, r == 0 ? cs : ring_site(tid), q_, H_, sg);
      if (r == 0) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          q[c] = q_[c];
          H[c] = H_[c];
        }
        sz[0] = sg[0][2];
        sz[1] = sg[1][2];
        sz[2] = sg[2][2];
      }
    }
  };

  // ---- prologue: Q zA-2 .. zA+1, u zA-1 .. zA+1, f(zA); planes zA-1, zA
  for (int zp = zA - 2; zp <= zA + 1; ++zp) issue_q(zp);
  for (int zp = zA - 1; zp <= zA + 1; ++zp) issue_u(zp);
  issue_f(zA);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  double qm1[5], q0[5], H0[5], szm[3], sz0[3], um[3];
  {
    double Hd[5];
    box_plane(zA - 1, qm1, Hd, szm);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) um[a] = sm.sU[rslot<3>(zA - 1)][a][cu];
  __syncthreads();  // the slot of Q(zA-2) is free
  issue_q(zA + 2);
  cp_commit();
  box_plane(zA, q0, H0, sz0);

  const int xm1 = wrapx(x - 1), xp1 = wrapx(x + 1), ym1 = wrapy(y - 1), yp1 = wrapy(y + 1);
  for (int k = zA; k < zB; ++k) {
    cp_wait<0>();  // Q(k+2), u(k+1)
    wait_f(k);
    __syncthreads();  // also: everyone is past iteration k-1 (its ring slots and f buffer are free)
    if (k + 3 <= zB + 1) issue_q(k + 3);
    if (k + 2 <= zB) issue_u(k + 2);
    if (k + 1 < zB) issue_f(k + 1);
    cp_commit();
    double q1[5], H1[5], sz1[3];
    box_plane(k + 1, q1, H1, sz1);
    const double(*uk)[NU] = sm.sU[rslot<3>(k)];
    double up[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) up[a] = sm.sU[rslot<3>(k + 1)][a][cu];
    if (active) {
      // R39: F = div sigma (= -div P^th), the in-plane columns from sSig(k)
      const double(*s)[NS] = sm.sSig[((k) & 1)];
      double F[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        F[a] = (0.5 * (s[a][cs + 1] - s[a][cs - 1]) + 0.5 * (s[3 + a][cs + SX] - s[3 + a][cs - SX])) +
               0.5 * (sz1[a] - szm[a]);
      // R40: Guo BGK of f (A.7) and push (A.8); u' = (j + F/2) / rho
      double f[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = sm.sF[((k) & 1)][frank(i)][tid];
      // A.8 push targets (push_plane of lb_kernels.cuh without peers, spelled out
      // for the three planes): periodic in z for a whole lattice, else planes -1 /
      // nzl are the ghost planes the exchange sends to the neighbouring slabs
      const long long pl = G.plane;
      double* const zk = B + (long long)(k + GZ) * pl;
      double* const zb[3] = {G.zwrap && k == 0 ? B + (long long)(G.nzl - 1 + GZ) * pl : zk - pl, zk,
                             G.zwrap && k == G.nzl - 1 ? B + (long long)GZ * pl : zk + pl};
      const double g0[Q] = {};
      double un[3];
      const double rho = collide(
          p, f, g0, 0.0, 0.0, F,
          [&](int i, double fs, double) {
            const int xd = cx(i) > 0 ? xp1 : (cx(i) < 0 ? xm1 : x);
            const int yd = cy(i) > 0 ? yp1 : (cy(i) < 0 ? ym1 : y);
            LB_CHECK(hl, xd >= 0 && xd < G.nx && yd >= 0 && yd < G.ny);
            double* d = zb[cz(i) + 1] + (yd * G.nx + xd);  // in-plane offset < nx ny < 2^31
            __stcs(d + (long long)slot(0, i) * nxy, fs);
          },
          un);
      // R41: velocity gradient of the stored u, co-rotation
      double W[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        W[a][0] = 0.5 * (uk[a][cu + 1] - uk[a][cu - 1]);
        W[a][1] = 0.5 * (uk[a][cu + UX] - uk[a][cu - UX]);
        W[a][2] = 0.5 * (up[a] - um[a]);
      }
      double S5[5];
      corotation(p.lc_xi, W, q0, S5);
      // R42 (R31 per component): upwind fluxes through the six faces, then the update
      const double(*Qk)[NB] = sm.sQ[((k) & 3)];
      const double ufx_p = 0.5 * (uk[0][cu] + uk[0][cu + 1]), ufx_m = 0.5 * (uk[0][cu - 1] + uk[0][cu]);
      const double ufy_p = 0.5 * (uk[1][cu] + uk[1][cu + UX]), ufy_m = 0.5 * (uk[1][cu - UX] + uk[1][cu]);
      const double ufz_p = 0.5 * (uk[2][cu] + up[2]), ufz_m = 0.5 * (um[2] + uk[2][cu]);
      auto J = [](double uf, double qa, double qb) { return uf * (uf > 0.0 ? qa : qb); };
      // in-plane faces: the upwind site is chosen once per face for all five
      // components (an offset into the Q box: Qk[c][cq] is q0[c]), so each flux is
      // one load and one product, the same values as J
      const int oxp = ufx_p > 0.0 ? cq : cq + 1, oxm = ufx_m > 0.0 ? cq - 1 : cq;
      const int oyp = ufy_p > 0.0 ? cq : cq + BX, oym = ufy_m > 0.0 ? cq - BX : cq;
      const long long zq = (long long)k * 5 * nxy + (long long)y * G.nx + x;
      double chk = rho;
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double v = q0[c];
        double div = 0.0;
        div = div + (ufx_p * Qk[c][oxp] - ufx_m * Qk[c][oxm]);
        div = div + (ufy_p * Qk[c][oyp] - ufy_m * Qk[c][oym]);
        div = div + (J(ufz_p, v, q1[c]) - J(ufz_m, qm1[c], v));
        const double qn = ((v - div) + S5[c]) + p.lc_Gamma * H0[c];
        __stcs(qB + zq + c * nxy, qn);
        chk += qn;
      }
      const long long zu = (long long)k * 3 * nxy + (long long)y * G.nx + x;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        __stcs(uB + zu + a * nxy, un[a]);
        chk += un[a];
      }
      if (!(rho > 0.0) || !isfinite(chk)) health_report(hl, G, x, y, k);  // R22
    }
    // rotate the per-thread planes
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      um[a] = uk[a][cu];
      szm[a] = sz0[a];
      sz0[a] = sz1[a];
    }
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      qm1[c] = q0[c];
      q0[c] = q1[c];
      H0[c] = H1[c];
    }
  }
  cp_wait<0>();
  __syncthreads();
  if (threadIdx.x == 0) health_tick(hl);
}

}  // namespace

cudaError_t prepare_lc_kernels() {
  int r = 0;
  return prepare_kernel(reinterpret_cast<const void*>(k_step_lc), sizeof(LcSmem), kLT, &r);
}

int lc_zchunk(const Geom& G, int num_sms) {
  const long long tiles = (long long)((G.nx + kLX - 1) / kLX) * ((G.ny + kLY - 1) / kLY);
  // fewer tiles than SMs: one wave, as many chunks as fit beside each other (128^3:
  // 2 x 64 planes, +11% over 3 waves of 19-plane chunks); otherwise >= 3 waves of one
  // CTA per SM; chunks of >= 16 planes (the prologue costs two planes)
  long long nchunks = tiles < num_sms ? num_sms / tiles : (3LL * num_sms + tiles - 1) / tiles;
  const long long maxchunks = G.nzl >= 32 ? G.nzl / 16 : 1;
  if (nchunks > maxchunks) nchunks = maxchunks;
  if (nchunks < 1) nchunks = 1;
  return (int)((G.nzl + nchunks - 1) / nchunks);
}

cudaError_t launch_step_lc(const Geom& G, const DevParams& p, const double* A, double* B, const double* qA,
                           double* qB, const double* uA, double* uB, int zc, const Health& hl, const StepMaps* maps,
                           cudaStream_t st) {
  if (!maps || !maps->ok || maps->ty != kLY || G.nx % 2 != 0) return cudaErrorInvalidValue;
  constexpr size_t smem = sizeof(LcSmem);
  static_assert(smem <= 232448, "shared memory per CTA exceeds 227 KB");
  int resid = 0;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(k_step_lc), smem, kLT, &resid);
  if (e != cudaSuccess) return e;
  const int tiles = ((G.nx + kLX - 1) / kLX) * ((G.ny + kLY - 1) / kLY);
  const int nblk = tiles * ((G.nzl + zc - 1) / zc);
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  k_step_lc<<<nblk, kLT, smem, st>>>(G, p, A, B, qA, qB, uA, uB, zc, hl, m[0], m[1]);
  return cudaGetLastError();
}

}  // namespace lbk
