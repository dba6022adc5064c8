// lb_kernels.cu -- sm_100a kernels of the D3Q19 binary-fluid step (first,
// site-parallel version: K_phi + K_step).
//
// Equations: DESIGN.md readings R1-R14 (PAPER.md P:163-190 names the pieces:
// "Collision", "Propagation", "Chemical stress", "Order Parameter Gradients").
// Everything is fp64.  The device code is an independent
// transcription; it shares nothing with oracle/.
#include <cuda_runtime.h>

#include "lb_kernels.cuh"

namespace lbk {
namespace {

constexpr int TPB = 128;

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// phi at (x, y, z) of the local slab; x, y periodic; z wraps only when G.zwrap,
// otherwise z in [-GP, nzl + GP) reads the ghost planes filled by the halo exchange.
__device__ __forceinline__ double phi_at(const Geom& G, const double* __restrict__ phi, int x, int y, int z) {
  x = wrap_n(x, G.nx);
  y = wrap_n(y, G.ny);
  if (G.zwrap) z = wrap_n(wrap_n(z, G.nzl), G.nzl);
  return ldg(phi + phi_plane_index(G, z) + (long long)y * G.nx + x);
}

// A.2: central gradient and 7-point Laplacian at (x, y, z) (R6).
__device__ __forceinline__ void grad_lap(const Geom& G, const double* __restrict__ phi, int x, int y, int z,
                                         double& ph, double gr[3], double& lap) {
  ph = phi_at(G, phi, x, y, z);
  const double xp = phi_at(G, phi, x + 1, y, z), xm = phi_at(G, phi, x - 1, y, z);
  const double yp = phi_at(G, phi, x, y + 1, z), ym = phi_at(G, phi, x, y - 1, z);
  const double zp = phi_at(G, phi, x, y, z + 1), zm = phi_at(G, phi, x, y, z - 1);
  gr[0] = 0.5 * (xp - xm);
  gr[1] = 0.5 * (yp - ym);
  gr[2] = 0.5 * (zp - zm);
  lap = (xp + xm) + (yp + ym) + (zp + zm) - 6.0 * ph;
}

// A.4 (R4): "Chemical Stress" P_ab; only row/column b is needed by the caller,
// returned as P[a] = P_ab.
__device__ __forceinline__ void stress_col(const DevParams& p, double ph, const double gr[3], double lap, int b,
                                           double P[3]) {
  const double p0 = 0.5 * p.A * ph * ph + 0.75 * p.B * (ph * ph * ph * ph);
  const double g2 = gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2];
  const double iso = p0 - p.kappa * ph * lap - 0.5 * p.kappa * g2;
#pragma unroll
  for (int a = 0; a < 3; ++a) P[a] = (a == b ? iso : 0.0) + p.kappa * gr[a] * gr[b];
}

// A.5 (R5): F_a = -sum_b (P_ab(x+e_b) - P_ab(x-e_b)) / 2.
__device__ __forceinline__ void force_at(const Geom& G, const DevParams& p, const double* __restrict__ phi, int x,
                                         int y, int z, double F[3]) {
  F[0] = F[1] = F[2] = 0.0;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const int dx = (b == 0), dy = (b == 1), dz = (b == 2);
    double ph, gr[3], lap, Pu[3], Pd[3];
    grad_lap(G, phi, x + dx, y + dy, z + dz, ph, gr, lap);
    stress_col(p, ph, gr, lap, b, Pu);
    grad_lap(G, phi, x - dx, y - dy, z - dz, ph, gr, lap);
    stress_col(p, ph, gr, lap, b, Pd);
#pragma unroll
    for (int a = 0; a < 3; ++a) F[a] -= 0.5 * (Pu[a] - Pd[a]);
  }
}

// A.3, A.6, A.7: moments, velocity, BGK of f with Guo source, BGK of g.
// f, g are overwritten by f*, g*.  Returns rho (for the R22 check).
__device__ __forceinline__ double collide(const DevParams& p, double (&f)[Q], double (&g)[Q], double phi, double mu,
                                          const double F[3]) {
  double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    rho += f[i];
    if (cx(i)) jx += cx(i) * f[i];
    if (cy(i)) jy += cy(i) * f[i];
    if (cz(i)) jz += cz(i) * f[i];
  }
  const double ux = (jx + 0.5 * F[0]) / rho;  // R7: u = (j + F/2) / rho
  const double uy = (jy + 0.5 * F[1]) / rho;
  const double uz = (jz + 0.5 * F[2]) / rho;
  const double uu = ux * ux + uy * uy + uz * uz;
  const double uF = ux * F[0] + uy * F[1] + uz * F[2];
  const double gmu = p.gamma * mu;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const double cu = cx(i) * ux + cy(i) * uy + cz(i) * uz;
    const double cF = cx(i) * F[0] + cy(i) * F[1] + cz(i) * F[2];
    const double w = wgt(i);
    const double feq = w * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * uu);   // R8
    const double S = w * (3.0 * (cF - uF) + 9.0 * cu * cF);                       // R7
    f[i] = f[i] - (f[i] - feq) * p.inv_tau_f + p.guo_pref * S;
    double geq = w * (3.0 * phi * cu + 4.5 * gmu * (double)(csq(i) - 1) + 4.5 * phi * (cu * cu - uu / 3.0));  // R9
    if (i == 0) geq += phi;
    g[i] = g[i] - (g[i] - geq) * p.inv_tau_g;
  }
  return rho;
}

// K_phi: phi = sum_i g_i over local planes [z0, z1) (A.3).  Summation in
// canonical order i = 0..18 (the same order every kernel uses).
__global__ void __launch_bounds__(TPB) k_phi(Geom G, const double* __restrict__ A, double* __restrict__ phi, int z0,
                                             int z1) {
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= G.nxy * (z1 - z0)) return;
  const int z = z0 + (int)(t / G.nxy);
  const long long xy = t - (long long)(z - z0) * G.nxy;
  const double* a = A + dist_index(G, z, 0, xy);
  double s = ldg(a + (long long)slot(1, 0) * G.nxy);
#pragma unroll
  for (int i = 1; i < Q; ++i) s += ldg(a + (long long)slot(1, i) * G.nxy);
  phi[phi_plane_index(G, z) + xy] = s;
}

// K_step: one site per thread.  Reads the pre-collision f, g at the site
// (coalesced, aligned), phi on the radius-2 stencil, collides, and PUSHES
// f_i*, g_i* to x + c_i (A.8).  With COLLIDE = false it only propagates (test
// support: the integer map alone).
template <bool COLLIDE>
__global__ void __launch_bounds__(TPB) k_step(Geom G, DevParams p, const double* __restrict__ A,
                                              double* __restrict__ B, const double* __restrict__ phi, int z0, int z1,
                                              int* __restrict__ flag) {
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= G.nxy * (z1 - z0)) return;
  const int z = z0 + (int)(t / G.nxy);
  const long long xy = t - (long long)(z - z0) * G.nxy;
  const int y = (int)(xy / G.nx);
  const int x = (int)(xy - (long long)y * G.nx);

  double f[Q], g[Q];
  const double* a = A + dist_index(G, z, 0, xy);
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    f[i] = ldg(a + (long long)slot(0, i) * G.nxy);
    g[i] = ldg(a + (long long)slot(1, i) * G.nxy);
  }
  if (COLLIDE) {
    double ph, gr[3], lap, F[3];
    grad_lap(G, phi, x, y, z, ph, gr, lap);
    const double mu = p.A * ph + p.B * (ph * ph * ph) - p.kappa * lap;  // R3
    force_at(G, p, phi, x, y, z, F);
    const double rho = collide(p, f, g, ph, mu, F);
    if (!(rho > 0.0) || !isfinite(rho) || !isfinite(ph)) *flag = 1;  // R22
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const long long d = push_target(G, i, x, y, z);
    __stcs(B + d + (long long)slot(0, i) * G.nxy, f[i]);
    __stcs(B + d + (long long)slot(1, i) * G.nxy, g[i]);
  }
}

// Initial state at local equilibrium (R15): f = f^eq(rho, u), g = g^eq(phi, u, Gamma mu),
// mu from the 7-point Laplacian of phi.  rho/u may be null (1 / 0).
__global__ void __launch_bounds__(TPB) k_init_eq(Geom G, DevParams p, const double* __restrict__ phi,
                                                 const double* __restrict__ rho_in, const double* __restrict__ u_in,
                                                 double* __restrict__ A) {
  const long long nloc = G.nxy * G.nzl;
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= nloc) return;
  const int z = (int)(t / G.nxy);
  const long long xy = t - (long long)z * G.nxy;
  const int y = (int)(xy / G.nx);
  const int x = (int)(xy - (long long)y * G.nx);
  double ph, gr[3], lap;
  grad_lap(G, phi, x, y, z, ph, gr, lap);
  const double mu = p.A * ph + p.B * (ph * ph * ph) - p.kappa * lap;
  const double rho = rho_in ? rho_in[t] : 1.0;
  const double ux = u_in ? u_in[t] : 0.0, uy = u_in ? u_in[nloc + t] : 0.0, uz = u_in ? u_in[2 * nloc + t] : 0.0;
  const double uu = ux * ux + uy * uy + uz * uz;
  const double gmu = p.gamma * mu;
  double* a = A + dist_index(G, z, 0, xy);
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const double cu = cx(i) * ux + cy(i) * uy + cz(i) * uz;
    const double w = wgt(i);
    a[(long long)slot(0, i) * G.nxy] = w * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * uu);
    double geq = w * (3.0 * ph * cu + 4.5 * gmu * (double)(csq(i) - 1) + 4.5 * ph * (cu * cu - uu / 3.0));
    if (i == 0) geq += ph;
    a[(long long)slot(1, i) * G.nxy] = geq;
  }
}

// canonical c[d*19*nloc + i*nloc + s]  <->  plane-major buffer (exact copies).
template <bool TO_PLANES>
__global__ void __launch_bounds__(TPB) k_permute(Geom G, const double* __restrict__ src, double* __restrict__ dst) {
  const long long nloc = G.nxy * G.nzl;
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= nloc * NSLOT) return;
  const int di = (int)(t / nloc);  // d * 19 + i
  const long long s = t - (long long)di * nloc;
  const int d = di / Q, i = di - d * Q;
  const int z = (int)(s / G.nxy);
  const long long xy = s - (long long)z * G.nxy;
  const long long b = dist_index(G, z, slot(d, i), xy);
  if (TO_PLANES)
    dst[b] = src[t];
  else
    dst[t] = src[b];
}

inline unsigned blocks_for(long long n) { return (unsigned)((n + TPB - 1) / TPB); }

}  // namespace

cudaError_t launch_phi(const Geom& G, const double* A, double* phi, int z0, int z1, cudaStream_t st) {
  const long long n = G.nxy * (z1 - z0);
  if (n <= 0) return cudaSuccess;
  k_phi<<<blocks_for(n), TPB, 0, st>>>(G, A, phi, z0, z1);
  return cudaGetLastError();
}

cudaError_t launch_step(const Geom& G, const DevParams& p, const double* A, double* B, const double* phi, int z0,
                        int z1, int* flag, bool collide, cudaStream_t st) {
  const long long n = G.nxy * (z1 - z0);
  if (n <= 0) return cudaSuccess;
  if (collide)
    k_step<true><<<blocks_for(n), TPB, 0, st>>>(G, p, A, B, phi, z0, z1, flag);
  else
    k_step<false><<<blocks_for(n), TPB, 0, st>>>(G, p, A, B, phi, z0, z1, flag);
  return cudaGetLastError();
}

cudaError_t launch_init_eq(const Geom& G, const DevParams& p, const double* phi, const double* rho, const double* u,
                           double* A, cudaStream_t st) {
  k_init_eq<<<blocks_for(G.nxy * G.nzl), TPB, 0, st>>>(G, p, phi, rho, u, A);
  return cudaGetLastError();
}

cudaError_t launch_canon_to_planes(const Geom& G, const double* canon, double* buf, cudaStream_t st) {
  k_permute<true><<<blocks_for(G.nxy * G.nzl * NSLOT), TPB, 0, st>>>(G, canon, buf);
  return cudaGetLastError();
}

cudaError_t launch_planes_to_canon(const Geom& G, const double* buf, double* canon, cudaStream_t st) {
  k_permute<false><<<blocks_for(G.nxy * G.nzl * NSLOT), TPB, 0, st>>>(G, buf, canon);
  return cudaGetLastError();
}

}  // namespace lbk
