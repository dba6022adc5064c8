"""Oracle of the NEXT-2 variant: the order parameter phi
evolved as a field by a finite-difference Cahn-Hilliard update with an advective
flux, replacing the g distribution.  Plain NumPy fp64.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Nothing in the product
path imports this module.

What it follows
---------------
The paper's Ludwig step has, besides the LB kernels, an "Advection" kernel
computing "the order parameter flux due to the bulk flow" and finite-difference
updates of the order parameter (stencils P:187-188).  For the binary
fluid that is the Cahn-Hilliard equation d_t phi + div(phi u) = M lap mu.  The
paper gives neither the scheme nor the coupling, so:

* R29  State = (f, phi) at integer t: f pre-collision as in R12, phi a field.
* R30  phi(t+1) = phi - sum_a [J_a(x + e_a/2) - J_a(x - e_a/2)] + M lap mu
       (explicit Euler, dt = 1, 7-point Laplacian of mu (R6), mu of R3).
* R31  Face flux, first-order upwind: u_f = (u(x) + u(x + e_a))/2,
       J_a(x + e_a/2) = u_f * (phi(x) if u_f > 0 else phi(x + e_a)).
* R32  The fluid: f collides as in the NEXT-3 variant (chemical stress in f^eq,
       three-rate MRT, R23-R25), so u = j / rho exactly and the advection
       velocity needs only f's moments -- no force on the halo.
* R33  Step order: moments -> gradients -> mu, P -> u -> collide f -> phi update
       -> propagate f.  Every term of the phi update uses fields at time t.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import lb_mrt as M
from . import lb_ref as R


@dataclass(frozen=True)
class ChParams:
    """Thermodynamics and mobility from ``base`` (M enters R30 directly; tau_f and
    tau_g are unused) and the MRT times of f (R32)."""

    base: R.Params = R.Params()
    tau_s: float = 0.8
    tau_b: float = 1.1
    tau_ghost: float = 1.0

    @property
    def mrt(self) -> M.MrtParams:
        return M.MrtParams(base=self.base, tau_s=self.tau_s, tau_b=self.tau_b, tau_ghost=self.tau_ghost)


def advective_divergence(phi: np.ndarray, u: np.ndarray) -> np.ndarray:
    """R31: sum_a [J_a(x + e_a/2) - J_a(x - e_a/2)], first-order upwind fluxes."""
    div = np.zeros_like(phi)
    for a in range(3):
        uf = 0.5 * (u[a] + R.shifted(u[a], a, +1))
        J = uf * np.where(uf > 0.0, phi, R.shifted(phi, a, +1))
        div = div + (J - R.shifted(J, a, -1))
    return div


def phi_update(phi: np.ndarray, u: np.ndarray, mu: np.ndarray, p: ChParams) -> np.ndarray:
    """R30: phi - div J + M lap mu."""
    return (phi - advective_divergence(phi, u)) + p.base.mobility * R.laplacian(mu)


@dataclass
class Fields:
    rho: np.ndarray
    j: np.ndarray
    grad: np.ndarray
    lap: np.ndarray
    mu: np.ndarray
    P: np.ndarray
    u: np.ndarray
    fstar: np.ndarray
    phi_next: np.ndarray


def check_domain(f: np.ndarray, phi: np.ndarray, rho: np.ndarray) -> None:
    """R22 for this variant."""
    bad = ~np.isfinite(f).all(axis=0) | ~np.isfinite(phi) | ~(rho > 0.0)
    if bad.any():
        z, y, x = (int(v) for v in np.argwhere(bad)[0])
        raise R.NumericalDomainError(f"rho <= 0 or non-finite value at site (x={x}, y={y}, z={z})")


def step_fields(f: np.ndarray, phi: np.ndarray, p: ChParams) -> Fields:
    """R33: everything but the propagation of f."""
    b = p.base
    rho = R.density(f)
    j = R.momentum(f)
    check_domain(f, phi, rho)
    grad = R.gradient(phi)
    lap = R.laplacian(phi)
    mu = R.chemical_potential(phi, lap, b)
    P = R.chemical_stress(phi, grad, lap, b)
    u = M.velocity(rho, j)
    fstar = M.collide_f(f, rho, u, P, p.mrt)
    phi_next = phi_update(phi, u, mu, p)
    return Fields(rho, j, grad, lap, mu, P, u, fstar, phi_next)


def step(f: np.ndarray, phi: np.ndarray, p: ChParams) -> tuple[np.ndarray, np.ndarray]:
    fl = step_fields(f, phi, p)
    return R.propagate(fl.fstar), fl.phi_next


def run(f: np.ndarray, phi: np.ndarray, p: ChParams, nsteps: int) -> tuple[np.ndarray, np.ndarray]:
    for _ in range(nsteps):
        f, phi = step(f, phi, p)
    return f, phi
