"""Oracle of the NEXT-4 workload: the paper's liquid-crystal
test case -- a Q-tensor order parameter evolved by a finite-difference
Beris-Edwards update with the Landau-de Gennes free energy, coupled to the D3Q19
LB fluid through the divergence of the "Chemical stress".  Plain NumPy fp64.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Nothing in the product
path imports this module.

What it follows
---------------
P:158-183 (sec. 2.1.1): the LC simulation "couples an 'order parameter' field (a
3x3 tensor, which is symmetric and traceless) ... and a 'distribution' field
representing the flow".  The order parameter "is evolved via an
advection-diffusion equation appropriate for rod-like molecules", the
distribution "via LB"; "they interact through a local force, derived from the
former".  The kernels: "Collision", "Propagation", the force "calculated as the
divergence of the 'Chemical stress'", itself "a function of the order parameter
field and its 'Order Parameter Gradients' derivatives", the "LC Update" ("a
finite difference implementation of the Beris-Edwards model with the Landau-de
Gennes free energy functional", citing Beris & Edwards 1994 and de Gennes &
Prost 1995) and the "Advection" ("the flux in the order parameter due to the
advective bulk flow").  P:185-190: gradients and advection are stencils;
collision, chemical stress and LC update are site-local.

The paper prints none of the equations, so each is a reading (R34-R45):

* R34  State = (f, Q, u) at integer t: f pre-collision (R12); Q by its five
       independent components (xx, xy, xz, yy, yz), Q_zz = -Q_xx - Q_yy; u the
       fluid velocity of the previous step's collision (Ludwig's hydrodynamic
       velocity, used by the next LC update).
* R35  Landau-de Gennes free energy density (one elastic constant, nematic):
       f_Q = A0/2 (1 - gamma/3) Q:Q - A0 gamma/3 tr(Q^3) + A0 gamma/4 (Q:Q)^2
             + kappa/2 (d_c Q_ab)(d_c Q_ab).
* R36  Molecular field H = -dF/dQ projected on symmetric traceless tensors:
       H = -A0 (1 - gamma/3) Q + A0 gamma (Q Q - I Q:Q/3) - A0 gamma (Q:Q) Q
           + kappa lap Q.
* R37  "Order Parameter Gradients": central d_c Q_ab and the 7-point lap Q_ab
       component by component (the stencils of R6).
* R38  Chemical stress (Beris-Edwards), sigma_ab =
         -p0 delta_ab + 2 xi (Q_ab + delta_ab/3) Q:H
         - xi H_ac (Q_cb + delta_cb/3) - xi (Q_ac + delta_ac/3) H_cb
         - kappa d_a Q_cd d_b Q_cd + Q_ac H_cb - H_ac Q_cb,
       p0 = -f_Q (the ideal-gas pressure rho/3 is carried by the LB); returned as
       P^th = -sigma, as in R4.
* R39  Force F_a = -sum_b (P^th_ab(x + e_b) - P^th_ab(x - e_b))/2 (R5: divergence
       on the second index, so sum_x F = 0).
* R40  Fluid: BGK of f with the Guo source (R7, R8) and this F; the new velocity
       u' = (j + F/2)/rho is the next state's u.
* R41  Velocity gradient W_ab = d_b u_a (central, of the stored u), D = (W + W^T)/2,
       Omega = (W - W^T)/2; co-rotation
         S = (xi D + Omega)(Q + I/3) + (Q + I/3)(xi D - Omega) - 2 xi (Q + I/3) tr(Q W),
       then its trace (2 xi div u / 3, non-zero only where the flow is
       compressible) removed: S <- S - I tr(S)/3.
* R42  "LC Update": Q(t+1) = Q - sum_a [J_a(x + e_a/2) - J_a(x - e_a/2)] + S + Gamma H,
       explicit Euler, dt = 1, with the first-order upwind flux of R31 per
       component ("Advection") and the stored u.
* R43  Step order: moments -> gradients of Q -> H -> P^th -> F -> u', collide f ->
       LC update (stored u) -> propagate f; the state becomes (f', Q', u').
* R44  Defaults: A0 = 0.01, gamma = 3.2, kappa = 0.01, xi = 0.7, Gamma = 0.3,
       tau_f = 0.8.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import lb_ch as CH
from . import lb_ref as R

# the five stored components (R34) as (a, b) index pairs
QCOMP = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2))


@dataclass(frozen=True)
class LcParams:
    """R35-R44.  tau_f: BGK time of f (> 1/2); A0, gamma: bulk LdG coefficients;
    kappa: elastic constant (>= 0); xi: flow-aligning parameter; Gamma: rotational
    diffusion constant (>= 0) of the LC update."""

    tau_f: float = 0.8
    A0: float = 0.01
    gamma: float = 3.2
    kappa: float = 0.01
    xi: float = 0.7
    Gamma: float = 0.3

    @property
    def fluid(self) -> R.Params:
        return R.Params(tau_f=self.tau_f)


def uniaxial_order(gamma: float) -> float:
    """Scalar order S0 of the bulk minimum of R35 for gamma > 8/3 (H = 0 for
    Q = S (n n - I/3)):  S0 = 1/4 + 3/4 sqrt(1 - 8/(3 gamma))."""
    return 0.25 + 0.75 * np.sqrt(1.0 - 8.0 / (3.0 * gamma))


# --------------------------------------------------------------------------
# R34: five components <-> the full symmetric traceless tensor
# --------------------------------------------------------------------------
def q_full(q5: np.ndarray) -> np.ndarray:
    """(5, ...) -> (3, 3, ...), symmetric, Q_zz = -Q_xx - Q_yy."""
    Q = np.empty((3, 3) + q5.shape[1:])
    for k, (a, b) in enumerate(QCOMP):
        Q[a, b] = q5[k]
        Q[b, a] = q5[k]
    Q[2, 2] = -q5[0] - q5[3]
    return Q


def q_five(Q: np.ndarray) -> np.ndarray:
    """(3, 3, ...) -> (5, ...)."""
    return np.stack([Q[a, b] for (a, b) in QCOMP])


def _matmul(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """(X Y)_ab = sum_c X_ac Y_cb, site by site."""
    Z = np.zeros(np.broadcast_shapes(X.shape, Y.shape))
    for a in range(3):
        for b in range(3):
            for c in range(3):
                Z[a, b] = Z[a, b] + X[a, c] * Y[c, b]
    return Z


def _contract(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """X:Y = sum_ab X_ab Y_ab."""
    s = np.zeros(np.broadcast_shapes(X.shape, Y.shape)[2:])
    for a in range(3):
        for b in range(3):
            s = s + X[a, b] * Y[a, b]
    return s


def _trace(X: np.ndarray) -> np.ndarray:
    return X[0, 0] + X[1, 1] + X[2, 2]


def _eye(shape) -> np.ndarray:
    I = np.zeros((3, 3) + tuple(shape))
    for a in range(3):
        I[a, a] = 1.0
    return I


# --------------------------------------------------------------------------
# R37 "Order Parameter Gradients"
# --------------------------------------------------------------------------
def q_gradient(Q: np.ndarray) -> np.ndarray:
    """dQ[c, a, b] = d_c Q_ab, central differences (R6)."""
    return np.stack([np.stack([np.stack([0.5 * (R.shifted(Q[a, b], c, +1) - R.shifted(Q[a, b], c, -1))
                                         for b in range(3)]) for a in range(3)]) for c in range(3)])


def q_laplacian(Q: np.ndarray) -> np.ndarray:
    """7-point Laplacian of every component (R6)."""
    return np.stack([np.stack([R.laplacian(Q[a, b]) for b in range(3)]) for a in range(3)])


# --------------------------------------------------------------------------
# R35 free energy, R36 molecular field
# --------------------------------------------------------------------------
def bulk_free_energy(Q: np.ndarray, p: LcParams) -> np.ndarray:
    """A0/2 (1 - gamma/3) Q:Q - A0 gamma/3 tr(Q^3) + A0 gamma/4 (Q:Q)^2."""
    q2 = _contract(Q, Q)
    q3 = _trace(_matmul(_matmul(Q, Q), Q))
    return 0.5 * p.A0 * (1.0 - p.gamma / 3.0) * q2 - p.A0 * p.gamma / 3.0 * q3 + 0.25 * p.A0 * p.gamma * q2 * q2


def free_energy_density(Q: np.ndarray, dQ: np.ndarray, p: LcParams) -> np.ndarray:
    """R35: bulk + kappa/2 (d_c Q_ab)^2."""
    g2 = np.zeros(Q.shape[2:])
    for c in range(3):
        for a in range(3):
            for b in range(3):
                g2 = g2 + dQ[c, a, b] * dQ[c, a, b]
    return bulk_free_energy(Q, p) + 0.5 * p.kappa * g2


def molecular_field(Q: np.ndarray, lapQ: np.ndarray, p: LcParams) -> np.ndarray:
    """R36: H = -A0 (1 - gamma/3) Q + A0 gamma (Q Q - I Q:Q/3) - A0 gamma (Q:Q) Q + kappa lap Q."""
    q2 = _contract(Q, Q)
    QQ = _matmul(Q, Q)
    H = np.empty_like(Q)
    for a in range(3):
        for b in range(3):
            qq = QQ[a, b] - q2 / 3.0 if a == b else QQ[a, b]
            H[a, b] = (-p.A0 * (1.0 - p.gamma / 3.0) * Q[a, b] + p.A0 * p.gamma * qq
                       - p.A0 * p.gamma * q2 * Q[a, b]) + p.kappa * lapQ[a, b]
    return H


# --------------------------------------------------------------------------
# R38 chemical stress, R39 force
# --------------------------------------------------------------------------
def chemical_stress(Q: np.ndarray, dQ: np.ndarray, H: np.ndarray, fed: np.ndarray, p: LcParams) -> np.ndarray:
    """R38: P^th = -sigma, with sigma the Beris-Edwards stress and p0 = -fed
    (fed = the free energy density of R35 at the site).  Shape (3, 3, ...)."""
    I = _eye(Q.shape[2:])
    Qt = Q + I / 3.0
    qh = _contract(Q, H)
    HQt = _matmul(H, Qt)
    QtH = _matmul(Qt, H)
    QH = _matmul(Q, H)
    HQ = _matmul(H, Q)
    P = np.empty_like(Q)
    for a in range(3):
        for b in range(3):
            grad_term = np.zeros(Q.shape[2:])
            for c in range(3):
                for d in range(3):
                    grad_term = grad_term + dQ[a, c, d] * dQ[b, c, d]
            sigma = (fed * I[a, b] + 2.0 * p.xi * Qt[a, b] * qh) - p.xi * HQt[a, b] - p.xi * QtH[a, b] \
                - p.kappa * grad_term + (QH[a, b] - HQ[a, b])
            P[a, b] = -sigma
    return P


def force(P: np.ndarray) -> np.ndarray:
    """R39 = R5: F_a = -sum_b (P_ab(x+e_b) - P_ab(x-e_b))/2."""
    return R.force(P)


# --------------------------------------------------------------------------
# R41 co-rotation, R42 LC update
# --------------------------------------------------------------------------
def velocity_gradient(u: np.ndarray) -> np.ndarray:
    """W[a, b] = d_b u_a, central differences."""
    return np.stack([np.stack([0.5 * (R.shifted(u[a], b, +1) - R.shifted(u[a], b, -1)) for b in range(3)])
                     for a in range(3)])


def corotation(W: np.ndarray, Q: np.ndarray, xi: float) -> np.ndarray:
    """R41: S(W, Q) with its trace removed."""
    I = _eye(Q.shape[2:])
    Qt = Q + I / 3.0
    D = 0.5 * (W + W.transpose(1, 0, *range(2, W.ndim)))
    Om = 0.5 * (W - W.transpose(1, 0, *range(2, W.ndim)))
    trQW = _trace(_matmul(Q, W))
    S = (_matmul(xi * D + Om, Qt) + _matmul(Qt, xi * D - Om)) - 2.0 * xi * Qt * trQW
    return S - I * (_trace(S) / 3.0)


def lc_update(Q: np.ndarray, u: np.ndarray, H: np.ndarray, p: LcParams) -> np.ndarray:
    """R42: the five components of Q - div J + S + Gamma H."""
    S = corotation(velocity_gradient(u), Q, p.xi)
    out = np.empty((5,) + Q.shape[2:])
    for k, (a, b) in enumerate(QCOMP):
        out[k] = ((Q[a, b] - CH.advective_divergence(Q[a, b], u)) + S[a, b]) + p.Gamma * H[a, b]
    return out


# --------------------------------------------------------------------------
# the step (R43)
# --------------------------------------------------------------------------
def check_domain(f: np.ndarray, q5: np.ndarray, u: np.ndarray, rho: np.ndarray) -> None:
    """R22 for this workload."""
    bad = (~np.isfinite(f).all(axis=0) | ~np.isfinite(q5).all(axis=0) | ~np.isfinite(u).all(axis=0)
           | ~(rho > 0.0))
    if bad.any():
        z, y, x = (int(v) for v in np.argwhere(bad)[0])
        raise R.NumericalDomainError(f"rho <= 0 or non-finite value at site (x={x}, y={y}, z={z})")


@dataclass
class Fields:
    rho: np.ndarray
    j: np.ndarray
    Q: np.ndarray
    dQ: np.ndarray
    lapQ: np.ndarray
    H: np.ndarray
    fed: np.ndarray
    P: np.ndarray
    F: np.ndarray
    u_new: np.ndarray
    fstar: np.ndarray
    q_next: np.ndarray


def step_fields(f: np.ndarray, q5: np.ndarray, u: np.ndarray, p: LcParams) -> Fields:
    """R43: everything but the propagation of f."""
    rho = R.density(f)
    j = R.momentum(f)
    check_domain(f, q5, u, rho)
    Q = q_full(q5)
    dQ = q_gradient(Q)
    lapQ = q_laplacian(Q)
    H = molecular_field(Q, lapQ, p)
    fed = free_energy_density(Q, dQ, p)
    P = chemical_stress(Q, dQ, H, fed, p)
    F = force(P)
    u_new = R.velocity(rho, j, F)
    fstar = R.collide_f(f, rho, u_new, F, p.fluid)
    q_next = lc_update(Q, u, H, p)
    return Fields(rho, j, Q, dQ, lapQ, H, fed, P, F, u_new, fstar, q_next)


def step(f: np.ndarray, q5: np.ndarray, u: np.ndarray, p: LcParams):
    """One timestep: (f, Q, u) at t -> at t + 1."""
    fl = step_fields(f, q5, u, p)
    return R.propagate(fl.fstar), fl.q_next, fl.u_new


def run(f: np.ndarray, q5: np.ndarray, u: np.ndarray, p: LcParams, nsteps: int):
    for _ in range(nsteps):
        f, q5, u = step(f, q5, u, p)
    return f, q5, u


def nematic_q(n: np.ndarray, S: float) -> np.ndarray:
    """Five components of S (n n - I/3) for a (3, ...) director field n (R45)."""
    Q = np.empty((3, 3) + n.shape[1:])
    for a in range(3):
        for b in range(3):
            Q[a, b] = S * (n[a] * n[b] - (1.0 / 3.0 if a == b else 0.0))
    return q_five(Q)


def initial_state(rho: np.ndarray, u: np.ndarray, n: np.ndarray, p: LcParams):
    """R45: f = f^eq(rho, u) (R8), Q = S0 (n n - I/3) with S0 of R35's bulk minimum,
    the stored velocity = u."""
    return R.f_equilibrium(rho, u), nematic_q(n, uniaxial_order(p.gamma)), u.copy()


def _window(a: np.ndarray, x: int, y: int, z: int, r: int) -> np.ndarray:
    """Periodic window of radius r around (x, y, z) of a (..., nz, ny, nx) array."""
    nz, ny, nx = a.shape[-3:]
    zi = np.arange(z - r, z + r + 1) % nz
    yi = np.arange(y - r, y + r + 1) % ny
    xi = np.arange(x - r, x + r + 1) % nx
    return a[..., zi[:, None, None], yi[None, :, None], xi[None, None, :]]


def step_at_sites(f: np.ndarray, q5: np.ndarray, u: np.ndarray, p: LcParams, sites):
    """One step evaluated only at the given sites: the whole-lattice ``step`` on a
    periodic window of radius 4 around each site (a new f at x depends on F at
    x - c_i, hence on P^th within radius 2 and Q within radius 3), centre kept.
    Returns (f (19, n), q (5, n), u (3, n))."""
    r = 4
    fo, qo, uo = [], [], []
    for (x, y, z) in sites:
        f1, q1, u1 = step(_window(f, x, y, z, r), _window(q5, x, y, z, r), _window(u, x, y, z, r), p)
        fo.append(f1[:, r, r, r])
        qo.append(q1[:, r, r, r])
        uo.append(u1[:, r, r, r])
    return np.stack(fo, axis=1), np.stack(qo, axis=1), np.stack(uo, axis=1)
