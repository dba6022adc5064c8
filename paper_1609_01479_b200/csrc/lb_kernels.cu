// lb_kernels.cu -- auxiliary sm_100a kernels: phi = sum_i g_i (slab edge planes,
// lb_get_phi), equilibrium initialisation, propagation only (tests), and the
// canonical <-> plane-major layout permutations.  The step kernel itself is in
// lb_step.cu.
//
// Equations: DESIGN.md readings R1-R15 (PAPER.md P:163-190 names the pieces).
// fp64 throughout.  Independent of oracle/.
#include <cuda_runtime.h>

#include "lb_device.cuh"

namespace lbk {
namespace {

constexpr int TPB = 128;

inline unsigned blocks_for(long long n) { return (unsigned)((n + TPB - 1) / TPB); }

// phi at (x, y, z) of the local slab; x, y periodic; z wraps when G.zwrap,
// otherwise z in [-GP, nzl + GP) reads the ghost planes of the phi buffer.
__device__ __forceinline__ double phi_at(const Geom& G, const double* __restrict__ phi, int x, int y, int z) {
  x = wrap_n(x, G.nx);
  y = wrap_n(y, G.ny);
  if (G.zwrap) z = wrap_n(z, G.nzl);
  return ldg(phi + phi_plane_index(G, z) + (long long)y * G.nx + x);
}

// K_phi: phi = sum_i g_i over local planes [z0, z1) (A.3).
// With peers (fused halo), planes 0, 1 are also stored into ghost planes nzl, nzl+1
// of the slab below and planes nzl-2, nzl-1 into ghost planes -2, -1 of the slab
// above (P2P stores over NVLink between GPUs).
__global__ void __launch_bounds__(TPB) k_phi(Geom G, const double* __restrict__ A, double* __restrict__ phi, int z0,
                                             int z1, Peers pr) {
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= G.nxy * (z1 - z0)) return;
  const int z = z0 + (int)(t / G.nxy);
  const long long xy = t - (long long)(z - z0) * G.nxy;
  const double v = phi_sum(A + dist_index(G, z, 0, xy), G.nxy);
  phi[phi_plane_index(G, z) + xy] = v;
  if (pr.phi_dn && z < GP) pr.phi_dn[phi_plane_index(G, G.nzl + z) + xy] = v;
  if (pr.phi_up && z >= G.nzl - GP) pr.phi_up[phi_plane_index(G, z - G.nzl) + xy] = v;
  if (pr.phi_dn || pr.phi_up) __threadfence_system();
}

// K_phi of the peer transport (NEXT-1): phi of planes 0, 1, nzl-2, nzl-1 (A.3),
// stored here and into the neighbours' ghost planes; one site per thread.  The
// ordering is done by the one-thread kernels around it on the same stream
// (k_sync_wait before it: the neighbours' step of the previous timestep has
// stored into planes 0 / nzl-1 of this slab and stopped reading its ghost
// planes; k_sync_publish after it: this slab's phi epoch) -- kernel boundaries
// order the rest, so no CTA of this kernel waits or fences (in-kernel, one
// acquire and one system fence per CTA cost 60 us per launch at 512 x 512).
__global__ void __launch_bounds__(TPB) k_phi_edges(Geom G, const double* __restrict__ A, double* __restrict__ phi,
                                                   Peers pr) {
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= 4 * G.nxy) return;
  const int k = (int)(t / G.nxy);
  const int z = k < 2 ? k : G.nzl - 4 + k;
  const long long xy = t - (long long)k * G.nxy;
  const double v = phi_sum(A + dist_index(G, z, 0, xy), G.nxy);
  phi[phi_plane_index(G, z) + xy] = v;
  if (z < GP) pr.phi_dn[phi_plane_index(G, G.nzl + z) + xy] = v;
  if (z >= G.nzl - GP) pr.phi_up[phi_plane_index(G, z - G.nzl) + xy] = v;
}

// One thread: wait until both neighbours' epoch words w_dn, w_up of this slab
// reach this slab's own epoch `ew` (bounded wait, lb_device.cuh).
__global__ void k_sync_wait(Peers pr, int w_dn, int w_up, int ew) {
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(pr.sync + ew);
  sync_wait_ge(pr.sync, w_dn, e);
  sync_wait_ge(pr.sync, w_up, e);
}

// One thread, after the kernel whose stores it publishes (stream order: that
// kernel has completed): a system-scope fence, then this slab's epoch `ew` + 1
// released into the neighbours' words (to_dn in the slab below, to_up above).
__global__ void k_sync_publish(Peers pr, int ew, int to_dn, int to_up) {
  __threadfence_system();
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(pr.sync + ew) + 1;
  pr.sync[ew] = e;
  st_release_sys_u64(pr.sync_dn + to_dn, e);
  st_release_sys_u64(pr.sync_up + to_up, e);
}

// Propagation only (test support, lb_debug_stream): the push of A.8 with the
// same addressing (push_target) and slot map as the step kernel.
__global__ void __launch_bounds__(TPB) k_stream(Geom G, const double* __restrict__ A, double* __restrict__ B, Peers pr) {
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= G.nxy * G.nzl) return;
  const int z = (int)(t / G.nxy);
  const long long xy = t - (long long)z * G.nxy;
  const int y = (int)(xy / G.nx);
  const int x = (int)(xy - (long long)y * G.nx);
  const double* a = A + dist_index(G, z, 0, xy);
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const long long d = push_in_plane(G, i, x, y);
    double* b = push_plane(G, B, pr, z + cz(i));
    b[d + (long long)slot(0, i) * G.nxy] = a[(long long)slot(0, i) * G.nxy];
    b[d + (long long)slot(1, i) * G.nxy] = a[(long long)slot(1, i) * G.nxy];
  }
  if (pr.dn || pr.up) __threadfence_system();
}

// Initial state at local equilibrium (R15): f = f^eq(rho, u), g = g^eq(phi, u, Gamma mu),
// mu from the 7-point Laplacian of phi (A.2, A.4).  rho/u may be null (1 / 0).
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
  const double ph = phi_at(G, phi, x, y, z);
  const double lap = (phi_at(G, phi, x + 1, y, z) + phi_at(G, phi, x - 1, y, z)) +
                     (phi_at(G, phi, x, y + 1, z) + phi_at(G, phi, x, y - 1, z)) +
                     (phi_at(G, phi, x, y, z + 1) + phi_at(G, phi, x, y, z - 1)) - 6.0 * ph;
  const double mu = chem_pot(p, ph, lap);
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
    double geq = w * (3.0 * ph * cu + 4.5 * gmu * (double)(csq(i) - 1) + 4.5 * ph * (cu * cu - uu * (1.0 / 3.0)));
    if (i == 0) geq += ph;
    a[(long long)slot(1, i) * G.nxy] = geq;
  }
}

// slot of (d, i) for runtime d, i (no local-memory table): the cz group and
// the rank within it, from the compile-time map via a small switch-free search.
__device__ __forceinline__ int slot_rt(int d, int i) {
  int s = 0;
#pragma unroll
  for (int k = 0; k < Q; ++k)
    if (k == i) s = slot(d, k);
  return s;
}

// canonical c[(d*19 + i)*nloc + s]  <->  plane-major buffer (exact copies).
template <bool TO_PLANES>
__global__ void __launch_bounds__(TPB) k_permute(Geom G, const double* __restrict__ src, double* __restrict__ dst) {
  const long long nloc = G.nxy * G.nzl;
  const long long t = (long long)blockIdx.x * TPB + threadIdx.x;
  if (t >= nloc * NSLOT) return;
  const int di = (int)(t / nloc);
  const long long s = t - (long long)di * nloc;
  const int d = di / Q, i = di - d * Q;
  const int z = (int)(s / G.nxy);
  const long long xy = s - (long long)z * G.nxy;
  const long long b = dist_index(G, z, d ? slot_rt(1, i) : slot_rt(0, i), xy);
  if (TO_PLANES)
    dst[b] = src[t];
  else
    dst[t] = src[b];
}

}  // namespace

cudaError_t launch_phi(const Geom& G, const double* A, double* phi, int z0, int z1, cudaStream_t st, const Peers& pr) {
  const long long n = G.nxy * (z1 - z0);
  if (n <= 0) return cudaSuccess;
  k_phi<<<blocks_for(n), TPB, 0, st>>>(G, A, phi, z0, z1, pr);
  return cudaGetLastError();
}

cudaError_t launch_phi_edges(const Geom& G, const double* A, double* phi, cudaStream_t st, const Peers& pr) {
  if (!pr.sync || !pr.sync_dn || !pr.sync_up || !pr.phi_dn || !pr.phi_up || G.zwrap || G.nzl < 2)
    return cudaErrorInvalidValue;
  // wait for the neighbours' pushes of the previous step; the edges; publish phi
  // (nzl = 2 or 3: the edge pairs overlap; a plane is summed once per occurrence, same bits)
  k_sync_wait<<<1, 1, 0, st>>>(pr, SW_PUSH_FROM_DN, SW_PUSH_FROM_UP, SW_PUSH_EPOCH);
  k_phi_edges<<<blocks_for(4 * G.nxy), TPB, 0, st>>>(G, A, phi, pr);
  k_sync_publish<<<1, 1, 0, st>>>(pr, SW_PHI_EPOCH, SW_PHI_FROM_UP, SW_PHI_FROM_DN);
  return cudaGetLastError();
}

cudaError_t launch_publish_push(const Peers& pr, cudaStream_t st) {
  if (!pr.sync) return cudaSuccess;
  k_sync_publish<<<1, 1, 0, st>>>(pr, SW_PUSH_EPOCH, SW_PUSH_FROM_UP, SW_PUSH_FROM_DN);
  return cudaGetLastError();
}

cudaError_t launch_wait_inbound(const Peers& pr, cudaStream_t st) {
  if (!pr.sync) return cudaSuccess;
  k_sync_wait<<<1, 1, 0, st>>>(pr, SW_PUSH_FROM_DN, SW_PUSH_FROM_UP, SW_PUSH_EPOCH);
  return cudaGetLastError();
}

cudaError_t launch_stream(const Geom& G, const double* A, double* B, cudaStream_t st, const Peers& pr) {
  k_stream<<<blocks_for(G.nxy * G.nzl), TPB, 0, st>>>(G, A, B, pr);
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
