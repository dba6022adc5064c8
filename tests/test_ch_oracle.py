"""Pins of the NEXT-2 oracle (``oracle/lb_ch.py``: finite-difference Cahn-Hilliard
update of phi with first-order upwind advective fluxes, readings R29-R33).

Closed forms of the discrete scheme: with u = 0 a Fourier mode of phi grows or
decays by exactly 1 - M khat^2 (A + kappa khat^2) per step (B = 0); in a uniform
flow U a passive mode is multiplied by 1 - U (1 - e^{-ik}) (U > 0) or
1 - U (e^{ik} - 1) (U < 0) -- which fixes the upwind direction on every axis.
Plus conservation, the fixed point, bitwise symmetries and the flat interface.
"""
import math

import numpy as np
import pytest

from oracle import lb_ch as CH
from oracle import lb_ref as R
from paper_1609_01479_b200 import synth
from symmetry import CUBIC, cube_transform


def _mode(field, axis, k_index):
    """Complex amplitude of Fourier mode k_index along `axis` (0=x, 1=y, 2=z) of a (z, y, x) field."""
    ax = (2, 1, 0)[axis]
    prof = field.mean(axis=tuple(a for a in range(3) if a != ax))
    return np.fft.fft(prof)[k_index]


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("A,kappa", [(0.1, 0.0), (-0.0625, 0.04), (0.05, 0.02)])
def test_linear_cahn_hilliard_factor_per_step(axis, A, kappa):
    """u = 0 in the first step (f at rest, the collision conserves j): a mode eps cos(k x_a)
    is multiplied by exactly 1 - M khat^2 (A + kappa khat^2), khat^2 = 2 (1 - cos k)."""
    n = (16, 12, 10)[axis]
    sh = [6, 5, 4]
    sh[axis] = n
    nx, ny, nz = sh
    base = R.Params(A=A, B=0.0, kappa=kappa, mobility=0.3)
    p = CH.ChParams(base=base)
    k = 2 * np.pi * 2 / n
    coord = np.indices((nz, ny, nx))[(2, 1, 0)[axis]]
    phi = 1e-3 * np.cos(k * coord)
    f = R.f_equilibrium(np.ones((nz, ny, nx)), np.zeros((3, nz, ny, nx)))
    f1, phi1 = CH.step(f, phi, p)
    kh2 = 2 * (1 - math.cos(k))
    lam = 1 - base.mobility * kh2 * (A + kappa * kh2)
    assert abs(_mode(phi1, axis, 2) / _mode(phi, axis, 2) - lam) < 1e-13


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("U", [0.07, -0.05])
def test_upwind_advection_factor(axis, U):
    """A = B = kappa = M = 0, rho = 1, uniform u = U e_a (f = f^eq, a fixed point): the
    mode is multiplied by 1 - U (1 - e^{-ik}) for U > 0 and 1 - U (e^{ik} - 1) for U < 0."""
    n = (16, 12, 10)[axis]
    sh = [5, 4, 3]
    sh[axis] = n
    nx, ny, nz = sh
    base = R.Params(A=0.0, B=0.0, kappa=0.0, mobility=0.0)
    p = CH.ChParams(base=base)
    u = np.zeros((3, nz, ny, nx))
    u[axis] = U
    f = R.f_equilibrium(np.ones((nz, ny, nx)), u)
    k = 2 * np.pi / n
    coord = np.indices((nz, ny, nx))[(2, 1, 0)[axis]]
    phi = 0.3 + 0.1 * np.cos(k * coord)
    f1, phi1 = CH.step(f, phi, p)
    lam = 1 - U * (1 - np.exp(-1j * k)) if U > 0 else 1 - U * (np.exp(1j * k) - 1)
    assert abs(_mode(phi1, axis, 1) / _mode(phi, axis, 1) - lam) < 1e-13
    assert np.abs(f1 - f).max() < 1e-16 * 4  # the uniform flow is a fixed point of f


def test_multi_step_spinodal_growth():
    """20 steps of a small mode (B = 0, eps = 1e-7): u stays O(eps^2), so the growth is the
    linear factor to the 20th power (1e-9)."""
    base = R.Params(A=-0.0625, B=0.0, kappa=0.04, mobility=0.4)
    p = CH.ChParams(base=base)
    n = 32
    k = 2 * np.pi / n
    x = np.arange(n)
    phi = np.broadcast_to(1e-7 * np.cos(k * x), (4, 4, n)).copy()
    f = R.f_equilibrium(np.ones((4, 4, n)), np.zeros((3, 4, 4, n)))
    f1, phi1 = CH.run(f, phi, p, 20)
    kh2 = 2 * (1 - math.cos(k))
    lam = 1 - base.mobility * kh2 * (base.A + base.kappa * kh2)
    assert lam > 1  # the mode grows (spinodal)
    assert abs(_mode(phi1, 0, 1) / _mode(phi, 0, 1) / lam**20 - 1) < 1e-9


def _rough(nx, ny, nz, seed):
    rho, u, phi, nf, _ = synth.rough_fields(nx, ny, nz, seed)
    return R.f_equilibrium(rho, u) + nf, phi


def test_conservation_of_phi_mass_and_momentum():
    p = CH.ChParams()
    f, phi = _rough(8, 6, 5, 41)
    f1, phi1 = CH.run(f, phi, p, 3)
    assert abs(phi1.sum() - phi.sum()) < 1e-13 * np.abs(phi).sum()
    assert abs(f1.sum() - f.sum()) < 1e-13 * f.sum()
    j0, j1 = R.momentum(f).sum(axis=(1, 2, 3)), R.momentum(f1).sum(axis=(1, 2, 3))
    assert np.abs(j1 - j0).max() < 1e-13


@pytest.mark.parametrize("u0", [(0.0, 0.0, 0.0), (0.03, -0.02, 0.01)])
def test_uniform_state_is_fixed_point(u0):
    sh = (4, 5, 6)
    p = CH.ChParams()
    u = np.broadcast_to(np.array(u0)[:, None, None, None], (3,) + sh).copy()
    phi = np.full(sh, -0.4)
    fl = CH.step_fields(R.f_equilibrium(np.full(sh, 0.9), u), phi, p)
    from oracle import lb_mrt as M

    feq = M.f_equilibrium_stress(fl.rho, fl.u, fl.P)
    f1, phi1 = CH.run(feq, phi, p, 3)
    assert np.abs(f1 - feq).max() < 1e-15
    assert np.abs(phi1 - phi).max() < 1e-15


def test_phi_sign_symmetry_and_shift_invariance_bitwise():
    p = CH.ChParams()
    f, phi = _rough(6, 5, 4, 42)
    f1, p1 = CH.run(f, phi, p, 2)
    f2, p2 = CH.run(f, -phi, p, 2)
    assert np.array_equal(f1, f2) and np.array_equal(p1, -p2)
    sh = lambda a: np.roll(a, (1, -2, 3), axis=(-3, -2, -1))  # noqa: E731
    f3, p3 = CH.run(sh(f), sh(phi), p, 2)
    assert np.array_equal(f3, sh(f1)) and np.array_equal(p3, sh(p1))


@pytest.mark.slow
def test_flat_interface_is_steady():
    base = R.Params(mobility=0.45)
    p = CH.ChParams(base=base)
    nx, ny, nz = 4, 4, 64
    xi = math.sqrt(-2 * base.kappa / base.A)
    z = np.arange(nz)
    prof = np.where(z < 32, np.tanh((z - 16) / xi), -np.tanh((z - 48) / xi))
    sh = (nz, ny, nx)
    phi = np.broadcast_to(prof[:, None, None], sh).copy()
    f = R.f_equilibrium(np.ones(sh), np.zeros((3,) + sh))
    f, phi = CH.run(f, phi, p, 2000)
    fl = CH.step_fields(f, phi, p)
    ph, mu = phi[:, 0, 0], fl.mu[:, 0, 0]
    assert np.abs(ph - prof).max() < 3e-2
    assert mu.max() - mu.min() < 1e-4
    assert np.abs(fl.u).max() < 1e-6
    phi_b = math.sqrt(-base.A / base.B)
    assert abs(ph[32 - 8] - phi_b) < 1e-3 and abs(ph[64 - 8] + phi_b) < 1e-3


@pytest.mark.parametrize("Mc", CUBIC)
def test_step_commutes_with_cubic_symmetry(Mc):
    """The finite-difference Cahn-Hilliard + upwind advection step
    uses the same stencil on every axis, with the upwind side chosen by the
    sign of u along that axis, so it commutes with reflections and axis
    permutations of the lattice (up to rounding)."""
    p = CH.ChParams()
    n = 5
    f, phi = _rough(n, n, n, 14)
    f1, p1 = CH.run(f, phi, p, 2)
    T = lambda a: cube_transform(a, Mc, n)  # noqa: E731
    f2, p2 = CH.run(T(f), T(phi), p, 2)
    assert np.abs(f2 - T(f1)).max() <= 1e-13 * np.abs(f1).max()
    assert np.abs(p2 - T(p1)).max() <= 1e-13 * np.abs(p1).max()
