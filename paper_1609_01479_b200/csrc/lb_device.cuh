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

// A.3, A.6, A.7: moments, velocity u = (j + F/2)/rho, BGK of f with Guo source,
// BGK of g towards g^eq(phi, u, Gamma mu).  emit(i, f_i*, g_i*) is called once
// per component, in canonical order, as soon as it is known (so stores can
// retire registers early).  Returns rho (for the R22 numerical-domain check).
// Same, reading f_i / g_i through accessors (e.g. from shared memory) and
// emitting only components I0 <= i < I1; the moments always use all 19 f_i in
// canonical order, so every caller computes identical rho, u.
template <int I0, int I1, class GetF, class GetG, class Emit>
__device__ __forceinline__ double collide_range(const DevParams& p, GetF&& getf, GetG&& getg, double phi, double mu,
                                                const double F[3], Emit&& emit) {
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
  const double uu = ux * ux + uy * uy + uz * uz;
  const double uF = ux * F[0] + uy * F[1] + uz * F[2];
  const double gmu = p.gamma * mu;
#pragma unroll
  for (int i = I0; i < I1; ++i) {
    const double cu = cx(i) * ux + cy(i) * uy + cz(i) * uz;
    const double cF = cx(i) * F[0] + cy(i) * F[1] + cz(i) * F[2];
    const double w = wgt(i);
    const double feq = w * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * uu);  // R8
    const double S = w * (3.0 * (cF - uF) + 9.0 * cu * cF);                      // R7
    const double fi = getf(i), gi = getg(i);
    const double fs = fi - (fi - feq) * p.inv_tau_f + p.guo_pref * S;
    double geq = w * (3.0 * phi * cu + 4.5 * gmu * (double)(csq(i) - 1) + 4.5 * phi * (cu * cu - uu * (1.0 / 3.0)));  // R9
    if (i == 0) geq += phi;
    emit(i, fs, gi - (gi - geq) * p.inv_tau_g);
  }
  return rho;
}

template <class Emit>
__device__ __forceinline__ double collide(const DevParams& p, const double (&f)[Q], const double (&g)[Q], double phi,
                                          double mu, const double F[3], Emit&& emit) {
  return collide_range<0, Q>(
      p, [&](int i) { return f[i]; }, [&](int i) { return g[i]; }, phi, mu, F, emit);
}


}  // namespace lbk
