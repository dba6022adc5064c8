"""Oracle of the NEXT-3 collision variant: the thermodynamic
stress in the second moment of f's equilibrium instead of a body force, relaxed
by a three-rate multiple-relaxation-time (MRT) operator.  Plain NumPy fp64.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Nothing in the product
path imports this module.

What it follows
---------------
The paper names a "Collision" kernel and says the coupling to the order
parameter goes through the "Chemical Stress"; it gives no
collision operator.  The main path reads that as a force F = -div P with Guo
forcing (R5, R7).  This variant is the other standard reading of the same
sentence, used by Ludwig's original binary-fluid method (Swift et al. 1996):
the chemical stress enters f's equilibrium itself, and the fluid sees
-div P through the divergence of the second moment.  Readings:

* R23  u = j / rho (no force); f_i^eq = w_i [rho + 3 rho c_i.u
       + 4.5 (P_ab + rho u_a u_b)(c_ia c_ib - delta_ab/3)], so that
       sum f^eq = rho, sum c f^eq = rho u, sum c c f^eq = rho/3 I + P + rho u u.
       With P = 0 it is R8's f^eq.
* R24  Three-rate MRT in projection form.  f^neq = f - f^eq; its second moment
       Pi = sum_i c_i c_i f_i^neq splits into the traceless S = Pi - (tr Pi/3) I
       and the trace; the "stress" part h_i = 4.5 w_i Pi:(c_i c_i - I/3)
       carries all of Pi, and the remainder (ghost part) gamma_i = f_i^neq - h_i
       carries no mass, momentum or stress.  Post-collision:
           f_i* = f_i^eq + 4.5 w_i [(1 - 1/tau_s) S:(c_i c_i)
                  + (1 - 1/tau_b) (tr Pi/3)(|c_i|^2 - 1)] + (1 - 1/tau_ghost) gamma_i.
       All three times equal reduce it to BGK exactly (up to rounding).
* R25  Shear viscosity nu = (tau_s - 1/2)/3; tau_b sets the bulk viscosity,
       tau_ghost the ghost-mode damping (1 projects the ghosts out).
* R26  g: BGK towards g^eq(phi, u, Gamma mu) (R9, R10) with the same u = j/rho.
* R27  Step order: moments -> gradients -> mu, P -> u -> collide f (MRT) ->
       collide g -> propagate.  No force is formed.

Plain means the same as in ``lb_ref``: no blocking, no fusion, no FMA, np.roll
for shifts, every field materialised.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import lb_ref as R

C, W, NVEL = R.C, R.W, R.NVEL


@dataclass(frozen=True)
class MrtParams:
    """R23-R26: the thermodynamic parameters and tau_g of the main path (``base``;
    its tau_f is not used), and the three MRT relaxation times of f."""

    base: R.Params = R.Params()
    tau_s: float = 0.8      # shear (traceless stress) -- nu = (tau_s - 1/2)/3
    tau_b: float = 1.0      # bulk (trace of the stress)
    tau_ghost: float = 1.0  # ghost modes (1: projected out each step)


def velocity(rho: np.ndarray, j: np.ndarray) -> np.ndarray:
    """R23: u = j / rho (no force shift)."""
    return j / rho


def f_equilibrium_stress(rho: np.ndarray, u: np.ndarray, P: np.ndarray) -> np.ndarray:
    """R23: f_i^eq = w_i [rho + 3 rho c.u + 4.5 (X:(c c) - tr X / 3)], X = P + rho u u."""
    X = np.empty_like(P)
    for a in range(3):
        for b in range(3):
            X[a, b] = P[a, b] + rho * u[a] * u[b]
    trX = X[0, 0] + X[1, 1] + X[2, 2]
    out = np.empty((NVEL,) + rho.shape)
    for i in range(NVEL):
        cXc = np.zeros(rho.shape)
        for a in range(3):
            for b in range(3):
                if C[i, a] != 0 and C[i, b] != 0:
                    cXc = cXc + C[i, a] * C[i, b] * X[a, b]
        out[i] = W[i] * (rho + 3.0 * rho * R._cdot(i, u) + 4.5 * (cXc - trX / 3.0))
    return out


def second_moment(a: np.ndarray) -> np.ndarray:
    """Pi_ab = sum_i c_ia c_ib a_i, returned as (3, 3, ...)."""
    Pi = np.zeros((3, 3) + a.shape[1:])
    for i in range(NVEL):
        for x in range(3):
            for y in range(3):
                if C[i, x] != 0 and C[i, y] != 0:
                    Pi[x, y] = Pi[x, y] + C[i, x] * C[i, y] * a[i]
    return Pi


def stress_part(Pi: np.ndarray) -> np.ndarray:
    """R24: h_i = 4.5 w_i (Pi:(c_i c_i) - tr Pi / 3)."""
    tr = Pi[0, 0] + Pi[1, 1] + Pi[2, 2]
    out = np.empty((NVEL,) + Pi.shape[2:])
    for i in range(NVEL):
        cPc = np.zeros(Pi.shape[2:])
        for a in range(3):
            for b in range(3):
                if C[i, a] != 0 and C[i, b] != 0:
                    cPc = cPc + C[i, a] * C[i, b] * Pi[a, b]
        out[i] = 4.5 * W[i] * (cPc - tr / 3.0)
    return out


def collide_f(f: np.ndarray, rho: np.ndarray, u: np.ndarray, P: np.ndarray, p: MrtParams) -> np.ndarray:
    """R24 in the order written there."""
    feq = f_equilibrium_stress(rho, u, P)
    fneq = f - feq
    Pi = second_moment(fneq)
    tr = Pi[0, 0] + Pi[1, 1] + Pi[2, 2]
    S = Pi.copy()
    for a in range(3):
        S[a, a] = Pi[a, a] - tr / 3.0
    gamma = fneq - stress_part(Pi)
    ks, kb, kg = 1.0 - 1.0 / p.tau_s, 1.0 - 1.0 / p.tau_b, 1.0 - 1.0 / p.tau_ghost
    out = np.empty_like(f)
    for i in range(NVEL):
        cSc = np.zeros(rho.shape)
        for a in range(3):
            for b in range(3):
                if C[i, a] != 0 and C[i, b] != 0:
                    cSc = cSc + C[i, a] * C[i, b] * S[a, b]
        c2 = float((C[i] * C[i]).sum())
        out[i] = feq[i] + 4.5 * W[i] * (ks * cSc + kb * (tr / 3.0) * (c2 - 1.0)) + kg * gamma[i]
    return out


def collide_g(g: np.ndarray, phi: np.ndarray, u: np.ndarray, mu: np.ndarray, p: MrtParams) -> np.ndarray:
    """R26: BGK of g with the force-free u."""
    return R.collide_g(g, phi, u, mu, p.base)


@dataclass
class Fields:
    rho: np.ndarray
    j: np.ndarray
    phi: np.ndarray
    grad: np.ndarray
    lap: np.ndarray
    mu: np.ndarray
    P: np.ndarray
    u: np.ndarray
    fstar: np.ndarray
    gstar: np.ndarray


def step_fields(f: np.ndarray, g: np.ndarray, p: MrtParams) -> Fields:
    """R27: everything but propagation."""
    b = p.base
    rho = R.density(f)
    j = R.momentum(f)
    phi = R.order_parameter(g)
    R.check_domain(f, g, rho)
    grad = R.gradient(phi)
    lap = R.laplacian(phi)
    mu = R.chemical_potential(phi, lap, b)
    P = R.chemical_stress(phi, grad, lap, b)
    u = velocity(rho, j)
    fstar = collide_f(f, rho, u, P, p)
    gstar = collide_g(g, phi, u, mu, p)
    return Fields(rho, j, phi, grad, lap, mu, P, u, fstar, gstar)


def step(f: np.ndarray, g: np.ndarray, p: MrtParams) -> tuple[np.ndarray, np.ndarray]:
    fl = step_fields(f, g, p)
    return R.propagate(fl.fstar), R.propagate(fl.gstar)


def run(f: np.ndarray, g: np.ndarray, p: MrtParams, nsteps: int) -> tuple[np.ndarray, np.ndarray]:
    for _ in range(nsteps):
        f, g = step(f, g, p)
    return f, g
