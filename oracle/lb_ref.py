"""Plain NumPy fp64 oracle of the D3Q19 binary-fluid LB timestep.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Nothing in the product
path imports this module.

What it follows
---------------
The paper (PAPER.md, Gray & Stratford) names the pieces of a Ludwig timestep but
gives none of the binary-fluid equations:

* P:144-152 (sec. 2.1.1): 3-D lattice, a set of double-precision values per
  site; LB evolves the hydrodynamics, coupled with finite differences.
* P:163-176 (sec. 2.1.1): a "distribution" field for the flow; "Collision";
  "Propagation" = "displacing the fluid data one lattice spacing in the
  appropriate direction"; the coupling force "is calculated as the divergence
  of the 'Chemical stress'", itself "a function of the order parameter field
  and its 'Order Parameter Gradients' derivatives".
* Propagation and the gradients are stencils; Collision and
  Chemical Stress are site-local.
* BGK collision and propagation (D2Q9 forms of SPEC's CPU program).

Every equation below is therefore a *reading*, numbered R1-R22 in DESIGN.md
(section "Readings of the paper"), and written in the paper's order of
components.  Arrays are shaped ``(19, nz, ny, nx)``: component-major, then z,
y, x with x fastest, so ``a.reshape(19, -1)`` is the canonical flat layout
``a[p*N + x + nx*(y + ny*z)]`` used at the C ABI.

Plain means: no blocking, no fusion, no FMA; every shift is ``np.roll``; each
field is materialised; the step runs in the order moments -> gradients ->
mu, P -> F -> u -> collide f -> collide g -> propagate (R14).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# --------------------------------------------------------------------------
# R1 / Appendix B: canonical D3Q19 velocity set.  Rest first, then the 18
# moving velocities in descending lexicographic (cx, cy, cz).  Antipode of
# p >= 1 is 18 - p + 1 = 19 - p.
# --------------------------------------------------------------------------
C = np.array(
    [
        [0, 0, 0],
        [1, 1, 0], [1, 0, 1], [1, 0, 0], [1, 0, -1], [1, -1, 0],
        [0, 1, 1], [0, 1, 0], [0, 1, -1], [0, 0, 1], [0, 0, -1],
        [0, -1, 1], [0, -1, 0], [0, -1, -1],
        [-1, 1, 0], [-1, 0, 1], [-1, 0, 0], [-1, 0, -1], [-1, -1, 0],
    ],
    dtype=np.int64,
)
NVEL = 19
_W_REST, _W_FACE, _W_EDGE = 1.0 / 3.0, 1.0 / 18.0, 1.0 / 36.0
W = np.array(
    [_W_REST if (c * c).sum() == 0 else (_W_FACE if (c * c).sum() == 1 else _W_EDGE) for c in C],
    dtype=np.float64,
)
CS2 = 1.0 / 3.0  # R1: lattice speed of sound squared

# array axis of each Cartesian direction a in (x, y, z) for (z, y, x) arrays
_AXIS = (2, 1, 0)


@dataclass(frozen=True)
class Params:
    """Parameters of the problem statement (BASELINE north_star; R2, R10, R16).

    tau_f, tau_g : BGK relaxation times of f and g (each > 1/2)
    A, B, kappa  : free energy  A/2 phi^2 + B/4 phi^4 + kappa/2 |grad phi|^2  (R2)
    mobility     : M; the g relaxation uses Gamma = M / (tau_g - 1/2)         (R10)
    """

    tau_f: float = 0.8
    tau_g: float = 1.3
    A: float = -0.0625
    B: float = 0.0625
    kappa: float = 0.04
    mobility: float = 0.05

    @property
    def gamma(self) -> float:
        """R10: Gamma = M / (tau_g - 1/2) (Chapman-Enskog of BGK g)."""
        return self.mobility / (self.tau_g - 0.5)


class NumericalDomainError(ArithmeticError):
    """R22 / S:335: density <= 0 or a non-finite value at some site."""


# --------------------------------------------------------------------------
# shifts
# --------------------------------------------------------------------------
def shifted(a: np.ndarray, axis_dir: int, s: int) -> np.ndarray:
    """Value at x + s*e_a of a periodic (z, y, x) field (R13: fully periodic)."""
    return np.roll(a, -s, axis=_AXIS[axis_dir])


# --------------------------------------------------------------------------
# A.3 moments (R12: state = pre-collision f, g at integer t)
# --------------------------------------------------------------------------
def density(f: np.ndarray) -> np.ndarray:
    """rho = sum_i f_i."""
    out = np.zeros(f.shape[1:])
    for i in range(NVEL):
        out = out + f[i]
    return out


def momentum(f: np.ndarray) -> np.ndarray:
    """j_a = sum_i c_ia f_i, returned as (3, nz, ny, nx)."""
    j = np.zeros((3,) + f.shape[1:])
    for i in range(NVEL):
        for a in range(3):
            if C[i, a] != 0:
                j[a] = j[a] + C[i, a] * f[i]
    return j


def order_parameter(g: np.ndarray) -> np.ndarray:
    """phi = sum_i g_i (zeroth moment of the second distribution, R9)."""
    return density(g)


# --------------------------------------------------------------------------
# A.2 "Order Parameter Gradients" (stencil; R6)
# --------------------------------------------------------------------------
def gradient(phi: np.ndarray) -> np.ndarray:
    """d_a phi = (phi(x+e_a) - phi(x-e_a)) / 2, returned as (3, nz, ny, nx)."""
    return np.stack([0.5 * (shifted(phi, a, +1) - shifted(phi, a, -1)) for a in range(3)])


def laplacian(phi: np.ndarray) -> np.ndarray:
    """7-point: sum_a (phi(x+e_a) + phi(x-e_a)) - 6 phi."""
    s = np.zeros_like(phi)
    for a in range(3):
        s = s + (shifted(phi, a, +1) + shifted(phi, a, -1))
    return s - 6.0 * phi


# --------------------------------------------------------------------------
# A.4 thermodynamics: chemical potential and "Chemical Stress" (R3, R4)
# --------------------------------------------------------------------------
def free_energy_density(phi: np.ndarray, p: Params) -> np.ndarray:
    """Bulk part of R2: psi(phi) = A/2 phi^2 + B/4 phi^4 (test helper)."""
    return 0.5 * p.A * phi * phi + 0.25 * p.B * phi * phi * phi * phi


def chemical_potential(phi: np.ndarray, lap: np.ndarray, p: Params) -> np.ndarray:
    """R3: mu = A phi + B phi^3 - kappa lap(phi)  (phi^3 as phi*phi*phi)."""
    return p.A * phi + p.B * (phi * phi * phi) - p.kappa * lap


def chemical_stress(phi: np.ndarray, grad: np.ndarray, lap: np.ndarray, p: Params) -> np.ndarray:
    """R4: P_ab = [p0 - kappa phi lap - kappa/2 |grad|^2] delta_ab + kappa d_a phi d_b phi,
    p0 = A/2 phi^2 + 3B/4 phi^4.  Returned as (3, 3, nz, ny, nx)."""
    p0 = 0.5 * p.A * phi * phi + 0.75 * p.B * (phi * phi * phi * phi)
    g2 = grad[0] * grad[0] + grad[1] * grad[1] + grad[2] * grad[2]
    iso = p0 - p.kappa * phi * lap - 0.5 * p.kappa * g2
    P = np.empty((3, 3) + phi.shape)
    for a in range(3):
        for b in range(3):
            P[a, b] = p.kappa * grad[a] * grad[b]
            if a == b:
                P[a, b] = iso + P[a, b]
    return P


# --------------------------------------------------------------------------
# A.5 force = -divergence of the chemical stress (R5)
# --------------------------------------------------------------------------
def force(P: np.ndarray) -> np.ndarray:
    """F_a = - sum_b (P_ab(x+e_b) - P_ab(x-e_b)) / 2, returned as (3, nz, ny, nx)."""
    F = np.zeros((3,) + P.shape[2:])
    for a in range(3):
        for b in range(3):
            F[a] = F[a] - 0.5 * (shifted(P[a, b], b, +1) - shifted(P[a, b], b, -1))
    return F


def velocity(rho: np.ndarray, j: np.ndarray, F: np.ndarray) -> np.ndarray:
    """R7 (Guo): u = (j + F/2) / rho."""
    return (j + 0.5 * F) / rho


# --------------------------------------------------------------------------
# A.6 equilibria (R8, R9) and A.7 Guo source (R7)
# --------------------------------------------------------------------------
def _cdot(i: int, v: np.ndarray) -> np.ndarray:
    """c_i . v for a (3, ...) field v."""
    return C[i, 0] * v[0] + C[i, 1] * v[1] + C[i, 2] * v[2]


def f_equilibrium(rho: np.ndarray, u: np.ndarray) -> np.ndarray:
    """R8: f_i^eq = w_i rho [1 + 3 c.u + 4.5 (c.u)^2 - 1.5 u.u]."""
    uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2]
    out = np.empty((NVEL,) + rho.shape)
    for i in range(NVEL):
        cu = _cdot(i, u)
        out[i] = W[i] * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * uu)
    return out


def g_equilibrium(phi: np.ndarray, u: np.ndarray, mu: np.ndarray, gamma: float) -> np.ndarray:
    """R9 (Hermite projection, phi in the rest particle):
    g_i^eq = w_i [3 phi c.u + 4.5 Gamma mu (|c|^2 - 1) + 4.5 phi ((c.u)^2 - u.u/3)] + phi delta_i0."""
    uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2]
    gmu = gamma * mu
    out = np.empty((NVEL,) + phi.shape)
    for i in range(NVEL):
        cu = _cdot(i, u)
        c2 = float((C[i] * C[i]).sum())
        out[i] = W[i] * (3.0 * phi * cu + 4.5 * gmu * (c2 - 1.0) + 4.5 * phi * (cu * cu - uu / 3.0))
        if i == 0:
            out[i] = out[i] + phi
    return out


def guo_source(u: np.ndarray, F: np.ndarray) -> np.ndarray:
    """R7: S_i = w_i [3 (c_i - u).F + 9 (c_i.u)(c_i.F)]."""
    uF = u[0] * F[0] + u[1] * F[1] + u[2] * F[2]
    out = np.empty((NVEL,) + F.shape[1:])
    for i in range(NVEL):
        out[i] = W[i] * (3.0 * (_cdot(i, F) - uF) + 9.0 * _cdot(i, u) * _cdot(i, F))
    return out


# --------------------------------------------------------------------------
# A.7 collision ("Collision", local P:189-190; BGK form S:331-339)
# --------------------------------------------------------------------------
def collide_f(f: np.ndarray, rho: np.ndarray, u: np.ndarray, F: np.ndarray, p: Params) -> np.ndarray:
    """f_i* = f_i - (f_i - f_i^eq)/tau_f + (1 - 1/(2 tau_f)) S_i."""
    feq = f_equilibrium(rho, u)
    S = guo_source(u, F)
    return f - (f - feq) / p.tau_f + (1.0 - 1.0 / (2.0 * p.tau_f)) * S


def collide_g(g: np.ndarray, phi: np.ndarray, u: np.ndarray, mu: np.ndarray, p: Params) -> np.ndarray:
    """g_i* = g_i - (g_i - g_i^eq)/tau_g."""
    geq = g_equilibrium(phi, u, mu, p.gamma)
    return g - (g - geq) / p.tau_g


# --------------------------------------------------------------------------
# A.8 propagation ("Propagation": "displacing the fluid data one
# lattice spacing in the appropriate direction")
# --------------------------------------------------------------------------
def propagate(a: np.ndarray) -> np.ndarray:
    """out_i(x + c_i) = a_i(x), periodic (R13)."""
    out = np.empty_like(a)
    for i in range(NVEL):
        out[i] = np.roll(a[i], shift=(int(C[i, 2]), int(C[i, 1]), int(C[i, 0])), axis=(0, 1, 2))
    return out


# --------------------------------------------------------------------------
# R22: numerical-domain check
# --------------------------------------------------------------------------
def check_domain(f: np.ndarray, g: np.ndarray, rho: np.ndarray) -> None:
    bad = ~np.isfinite(f).all(axis=0) | ~np.isfinite(g).all(axis=0) | ~(rho > 0.0)
    if bad.any():
        z, y, x = (int(v) for v in np.argwhere(bad)[0])
        raise NumericalDomainError(f"rho <= 0 or non-finite value at site (x={x}, y={y}, z={z})")


# --------------------------------------------------------------------------
# the step (R14 order) and helpers
# --------------------------------------------------------------------------
@dataclass
class Fields:
    """Every intermediate of one step (for unit pins)."""

    rho: np.ndarray
    j: np.ndarray
    phi: np.ndarray
    grad: np.ndarray
    lap: np.ndarray
    mu: np.ndarray
    P: np.ndarray
    F: np.ndarray
    u: np.ndarray
    fstar: np.ndarray
    gstar: np.ndarray


def step_fields(f: np.ndarray, g: np.ndarray, p: Params) -> Fields:
    """Steps 1-8 of the oracle step (everything but propagation)."""
    rho = density(f)  # 1. moments
    j = momentum(f)
    phi = order_parameter(g)
    check_domain(f, g, rho)
    grad = gradient(phi)  # 2. gradients
    lap = laplacian(phi)
    mu = chemical_potential(phi, lap, p)  # 3. mu
    P = chemical_stress(phi, grad, lap, p)  # 4. P
    F = force(P)  # 5. F
    u = velocity(rho, j, F)  # 6. u
    fstar = collide_f(f, rho, u, F, p)  # 7. collide f
    gstar = collide_g(g, phi, u, mu, p)  # 8. collide g
    return Fields(rho, j, phi, grad, lap, mu, P, F, u, fstar, gstar)


def step(f: np.ndarray, g: np.ndarray, p: Params) -> tuple[np.ndarray, np.ndarray]:
    """One timestep t -> t+1 of the pre-collision state (f, g)."""
    fl = step_fields(f, g, p)
    return propagate(fl.fstar), propagate(fl.gstar)  # 9. propagate


def run(f: np.ndarray, g: np.ndarray, p: Params, nsteps: int) -> tuple[np.ndarray, np.ndarray]:
    for _ in range(nsteps):
        f, g = step(f, g, p)
    return f, g


def equilibrium_state(rho: np.ndarray, u: np.ndarray, phi: np.ndarray, p: Params) -> tuple[np.ndarray, np.ndarray]:
    """R15 initial state: f = f^eq(rho, u), g = g^eq(phi, u, Gamma mu[phi]), with mu from
    the 7-point stencil of phi (R3, R6)."""
    mu = chemical_potential(phi, laplacian(phi), p)
    return f_equilibrium(rho, u), g_equilibrium(phi, u, mu, p.gamma)


def macroscopic(f: np.ndarray, g: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(rho, j, phi) of a state (diagnostics)."""
    return density(f), momentum(f), order_parameter(g)
