// lb_device.cuh -- device-side building blocks of the step, shared by every kernel
// so the arithmetic (and its rounding) is the same everywhere: a site updated by
// the fused kernel, by a slab-boundary launch or on another slab decomposition
// gives the same bits.
//
// Equations: DESIGN.md readings R3-R9 / SURVEY Appendix A.  fp64.
#pragma once

#include "lb_kernels.cuh"

namespace lbk {

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// phi = sum_i g_i (A.3): canonical order i = 0..18, starting from g_0.
// `a` points at (plane, slot 0, site); stride = nxy between slots.
__device__ __forceinline__ double phi_sum(const double* __restrict__ a, long long nxy) {
  double s = ldg(a + (long long)slot(1, 0) * nxy);
#pragma unroll
  for (int i = 1; i < Q; ++i) s += ldg(a + (long long)slot(1, i) * nxy);
  return s;
}

// R22: record site (x, y, local z) of this launch's slab as offending,
// tagged with the step in progress; the smallest (step, site) of a call wins.
__device__ __forceinline__ void health_report(const Health& h, const Geom& G, int x, int y, int z) {
  const unsigned long long site =
      (unsigned long long)(h.site0 + (long long)z * G.nxy + (long long)y * G.nx + x);
  const unsigned long long step = *reinterpret_cast<volatile unsigned long long*>(h.step);
  atomicMin(h.flag, (step << 40) | site);
}
// One thread per CTA, after the CTA's reports (a CTA barrier before): the last
// CTA of the launch to finish advances the step counter -- every report of this
// launch has read the step number by then (its value, not its visibility, is
// what matters: the reports are atomics the host reads after a stream sync, so
// no fence -- a gpu-scope fence here held every CTA until its pushes drained).
__device__ __forceinline__ void health_tick(const Health& h) {
  if (!h.done) return;
  if (atomicAdd(h.done, 1u) == gridDim.x - 1) {
    *h.done = 0;
    atomicAdd(h.step, 1ULL);
  }
}

// ---- device-side ordering of the peer transport (lb_kernels.cuh "SyncWord") ----
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait (one thread) until local sync word w >= target; bounded: after
// kSyncTimeoutNs, or once any wait of this slab has timed out, give up and leave
// SW_ERR set (lb_step reports it) -- a broken peer never hangs the GPU.
__device__ __forceinline__ void sync_wait_ge(unsigned long long* sync, int w, unsigned long long target) {
  if (ld_acquire_sys_u64(sync + w) >= target) return;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys_u64(sync + w) < target) {
    if (*reinterpret_cast<volatile unsigned long long*>(sync + SW_ERR)) return;
    if (globaltimer_ns() - t0 > kSyncTimeoutNs) {
      atomicExch(sync + SW_ERR, 1ULL);
      return;
    }
    __nanosleep(200);
  }
}
// Step kernels: a CTA whose planes need the ghost phi planes of the slab below
// (zA - 2 < 0) or above (zB + 1 >= nzl) waits for that neighbour's K_phi of this
// step (this slab's own K_phi ran just before, so its phi epoch is the target).
__device__ __forceinline__ void sync_wait_ghost_phi(const Geom& G, const Peers& pr, int zA, int zB) {
  if (!pr.sync || G.zwrap) return;
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(pr.sync + SW_PHI_EPOCH);
  if (zA - 2 < 0) sync_wait_ge(pr.sync, SW_PHI_FROM_DN, e);
  if (zB + 1 >= G.nzl) sync_wait_ge(pr.sync, SW_PHI_FROM_UP, e);
}

// A.4 (R3): mu = A phi + B phi^3 - kappa lap phi
__device__ __forceinline__ double chem_pot(const DevParams& p, double ph, double lap) {
  return p.A * ph + p.B * (ph * ph * ph) - p.kappa * lap;
}

// A.4 (R4): "Chemical Stress" P_ab from phi, grad phi, lap phi.
// Component order: xx, yy, zz, xy, xz, yz.
enum { PXX = 0, PYY, PZZ, PXY, PXZ, PYZ };
__device__ __forceinline__ void stress6(const DevParams& p, double ph, double gx, double gy, double gz, double lap,
                                        double P[6]) {
  const double p0 = 0.5 * p.A * ph * ph + 0.75 * p.B * (ph * ph * ph * ph);
  const double g2 = gx * gx + gy * gy + gz * gz;
  const double iso = p0 - p.kappa * ph * lap - 0.5 * p.kappa * g2;
  P[PXX] = iso + p.kappa * gx * gx;
  P[PYY] = iso + p.kappa * gy * gy;
  P[PZZ] = iso + p.kappa * gz * gz;
  P[PXY] = p.kappa * gx * gy;
  P[PXZ] = p.kappa * gx * gz;
  P[PYZ] = p.kappa * gy * gz;
}

// A.3, A.6, A.7: moments, velocity u = (j + F/2)/rho, BGK of f with the Guo
// source, BGK of g towards g^eq(phi, u, Gamma mu):
//   f_i* = f_i (1 - 1/tau_f) + f_i^eq / tau_f + (1 - 1/(2 tau_f)) S_i
//   g_i* = g_i (1 - 1/tau_g) + g_i^eq / tau_g
// Evaluated per antipodal pair (i, 19 - i): c_{19-i} = -c_i and w equal, so each
// of f^eq, S, g^eq splits into a part even in c (shared by the pair) and a part
// odd in c (sign-flipped), which roughly halves the fp64 work.  emit(i, f_i*, g_i*)
// is called once per component.  Returns rho (for the R22 numerical-domain check).
// uo (optional): receives u = (j + F/2)/rho (the liquid-crystal workload stores it, R40).
template <class GetF, class GetG, class Emit>
__device__ __forceinline__ double collide_acc(const DevParams& p, GetF&& getf, GetG&& getg, double phi, double mu,
                                              const double F[3], Emit&& emit, double* uo = nullptr) {
  double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const double fi = getf(i);
    rho += fi;
    if (cx(i)) jx += cx(i) * fi;
    if (cy(i)) jy += cy(i) * fi;
    if (cz(i)) jz += cz(i) * fi;
  }
  const double rinv = 1.0 / rho;
  const double ux = (jx + 0.5 * F[0]) * rinv;  // R7
  const double uy = (jy + 0.5 * F[1]) * rinv;
  const double uz = (jz + 0.5 * F[2]) * rinv;
  if (uo) {
    uo[0] = ux;
    uo[1] = uy;
    uo[2] = uz;
  }
  const double uu = ux * ux + uy * uy + uz * uz;
  const double uF = ux * F[0] + uy * F[1] + uz * F[2];
  const double gmu = p.gamma * mu;
  const double omf = p.inv_tau_f, omg = p.inv_tau_g, keepf = 1.0 - p.inv_tau_f, keepg = 1.0 - p.inv_tau_g;
  // parts of f^eq (R8), S (R7), g^eq (R9) that depend only on |c|^2 (weight class)
  const double rho_even = rho * (1.0 - 1.5 * uu);   // f^eq/w without the c.u terms
  const double s_even = -3.0 * uF;                  // S/w without the c terms
  const double phi_even = -1.5 * phi * uu;          // g^eq/w: -4.5 phi uu/3
  {  // rest particle: c = 0, |c|^2 - 1 = -1.  g is written with explicit roundings:
     // left to the compiler, its FMA contraction differed between kernels (1 ulp)
    const double w = wgt(0);
    const double feq = w * rho_even, S = w * s_even;
    const double geq = __fma_rn(w, __fma_rn(-4.5, gmu, phi_even), phi);
    emit(0, keepf * getf(0) + (omf * feq + p.guo_pref * S), __fma_rn(keepg, getg(0), __dmul_rn(omg, geq)));
  }
#pragma unroll
  for (int i = 1; i <= 9; ++i) {
    const int ia = Q - i;  // antipode (Appendix B)
    const double w = wgt(i);
    const double cu = cx(i) * ux + cy(i) * uy + cz(i) * uz;
    const double cF = cx(i) * F[0] + cy(i) * F[1] + cz(i) * F[2];
    const double cu2 = cu * cu;
    // even / odd parts, each already times w
    const double feq_e = w * (rho_even + 4.5 * rho * cu2), feq_o = (3.0 * w * rho) * cu;
    const double S_e = w * (s_even + 9.0 * cu * cF), S_o = (3.0 * w) * cF;
    const double geq_e = w * (4.5 * gmu * (double)(csq(i) - 1) + phi_even + 4.5 * phi * cu2);
    const double geq_o = (3.0 * w * phi) * cu;
    const double sym = omf * feq_e + p.guo_pref * S_e;
    const double anti = omf * feq_o + p.guo_pref * S_o;
    const double gsym = omg * geq_e, ganti = omg * geq_o;
    emit(i, keepf * getf(i) + sym + anti, keepg * getg(i) + gsym + ganti);
    emit(ia, keepf * getf(ia) + sym - anti, keepg * getg(ia) + gsym - ganti);
  }
  return rho;
}

// NEXT-3 variant (readings R23-R26): the chemical stress P in the second moment of
// f's equilibrium, no force, u = j / rho, and a three-rate MRT of f in projection
// form.  With X = P + rho u u and f^neq = f - f^eq, Pi = sum c c f^neq,
// t = tr Pi, S = Pi - t/3 I, h_i = 4.5 w_i (S:c c + t/3 (|c|^2 - 1)):
//   f_i^eq = w_i [rho + 3 rho c.u + 4.5 (X:c c - tr X/3)]
//   f_i*   = f_i^eq + 4.5 w_i [k_s S:c c + k_b t/3 (|c|^2 - 1)] + k_g (f_i^neq - h_i)
//          = f_i^eq + k_g f_i^neq + 4.5 w_i [(k_s - k_g) S:c c + (k_b - k_g) t/3 (|c|^2 - 1)]
// with k_s = 1 - 1/tau_s, k_b = 1 - 1/tau_b, k_g = 1 - 1/tau_ghost; g as in collide_acc
// with the force-free u.  Evaluated per antipodal pair: X:c c, S:c c and |c|^2 are
// even in c, c.u is odd.  P6 = (xx, yy, zz, xy, xz, yz).  Returns rho.
template <class Emit>
__device__ __forceinline__ double collide_mrt(const DevParams& p, double (&f)[Q], const double (&g)[Q], double phi,
                                              double mu, const double P6[6], Emit&& emit) {
  double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    rho += f[i];
    if (cx(i)) jx += cx(i) * f[i];
    if (cy(i)) jy += cy(i) * f[i];
    if (cz(i)) jz += cz(i) * f[i];
  }
  const double rinv = 1.0 / rho;
  const double ux = jx * rinv, uy = jy * rinv, uz = jz * rinv;  // R23
  const double X[6] = {P6[PXX] + rho * ux * ux, P6[PYY] + rho * uy * uy, P6[PZZ] + rho * uz * uz,
                       P6[PXY] + rho * ux * uy, P6[PXZ] + rho * ux * uz, P6[PYZ] + rho * uy * uz};
  const double trX3 = (X[0] + X[1] + X[2]) * (1.0 / 3.0);
  auto cMc = [](int i, const double M[6]) {  // c_i . M . c_i (even in c)
    double v = 0.0;
    if (cx(i)) v += M[0];
    if (cy(i)) v += M[1];
    if (cz(i)) v += M[2];
    if (cx(i) && cy(i)) v += 2.0 * cx(i) * cy(i) * M[3];
    if (cx(i) && cz(i)) v += 2.0 * cx(i) * cz(i) * M[4];
    if (cy(i) && cz(i)) v += 2.0 * cy(i) * cz(i) * M[5];
    return v;
  };
  // pass 1: f^neq in place, and its second moment Pi
  double Pi[6] = {0, 0, 0, 0, 0, 0};
  f[0] -= wgt(0) * (rho - 4.5 * trX3);  // rest: X:cc = 0
#pragma unroll
  for (int i = 1; i <= 9; ++i) {
    const int ia = Q - i;
    const double w = wgt(i);
    const double e = w * (rho + 4.5 * (cMc(i, X) - trX3));
    const double o = (3.0 * w * rho) * (cx(i) * ux + cy(i) * uy + cz(i) * uz);
    f[i] -= e + o;
    f[ia] -= e - o;
    const double s = f[i] + f[ia];  // c c is even: the pair contributes c c (f_i + f_ia)
    if (cx(i)) Pi[0] += s;
    if (cy(i)) Pi[1] += s;
    if (cz(i)) Pi[2] += s;
    if (cx(i) && cy(i)) Pi[3] += cx(i) * cy(i) * s;
    if (cx(i) && cz(i)) Pi[4] += cx(i) * cz(i) * s;
    if (cy(i) && cz(i)) Pi[5] += cy(i) * cz(i) * s;
  }
  const double t3 = (Pi[0] + Pi[1] + Pi[2]) * (1.0 / 3.0);
  const double S[6] = {Pi[0] - t3, Pi[1] - t3, Pi[2] - t3, Pi[3], Pi[4], Pi[5]};
  const double kg = 1.0 - p.inv_tau_ghost;
  const double dks = (1.0 - p.inv_tau_s) - kg, dkb = (1.0 - p.inv_tau_b) - kg;
  // g (R26): as collide_acc with F = 0
  const double uu = ux * ux + uy * uy + uz * uz;
  const double gmu = p.gamma * mu;
  const double omg = p.inv_tau_g, keepg = 1.0 - p.inv_tau_g;
  const double phi_even = -1.5 * phi * uu;
  {  // rest particle
    const double w = wgt(0);
    const double feq = w * (rho - 4.5 * trX3);
    const double fs = feq + kg * f[0] + 4.5 * w * (dkb * t3 * -1.0);
    const double geq = __fma_rn(w, __fma_rn(-4.5, gmu, phi_even), phi);
    emit(0, fs, __fma_rn(keepg, g[0], __dmul_rn(omg, geq)));
  }
#pragma unroll
  for (int i = 1; i <= 9; ++i) {
    const int ia = Q - i;
    const double w = wgt(i);
    const double e = w * (rho + 4.5 * (cMc(i, X) - trX3));
    const double cu = cx(i) * ux + cy(i) * uy + cz(i) * uz;
    const double o = (3.0 * w * rho) * cu;
    const double even = 4.5 * w * (dks * cMc(i, S) + dkb * t3 * (double)(csq(i) - 1));
    const double geq_e = w * (4.5 * gmu * (double)(csq(i) - 1) + phi_even + 4.5 * phi * cu * cu);
    const double geq_o = (3.0 * w * phi) * cu;
    const double gsym = omg * geq_e, ganti = omg * geq_o;
    emit(i, (e + o) + kg * f[i] + even, keepg * g[i] + gsym + ganti);
    emit(ia, (e - o) + kg * f[ia] + even, keepg * g[ia] + gsym - ganti);
  }
  return rho;
}

template <class Emit>
__device__ __forceinline__ double collide(const DevParams& p, const double (&f)[Q], const double (&g)[Q], double phi,
                                          double mu, const double F[3], Emit&& emit, double* uo = nullptr) {
  return collide_acc(
      p, [&](int i) { return f[i]; }, [&](int i) { return g[i]; }, phi, mu, F, emit, uo);
}

}  // namespace lbk
