"""Pins of the NEXT-3 oracle (``oracle/lb_mrt.py``: thermodynamic stress in f's
equilibrium, three-rate MRT; readings R23-R27 of DESIGN.md).

As for the main oracle, none of these compares the oracle with itself: moments
come from ``lb_brute``'s independently enumerated velocity set, the reductions
are to the BGK form of S:331-339 and to R8's f^eq, and the hydrodynamic pins
are closed forms.
"""
import math

import numpy as np
import pytest

from oracle import lb_brute as BR
from oracle import lb_mrt as M
from oracle import lb_ref as R
from paper_1609_01479_b200 import synth
from symmetry import CUBIC, cube_transform

P0 = R.Params()
MP0 = M.MrtParams(base=P0, tau_s=0.8, tau_b=1.1, tau_ghost=1.0)


def _brute_moments(dist):
    m0 = sum(dist[i] for i in range(19))
    m1 = [sum(BR.CV[i][a] * dist[i] for i in range(19)) for a in range(3)]
    m2 = [[sum(BR.CV[i][a] * BR.CV[i][b] * dist[i] for i in range(19)) for b in range(3)] for a in range(3)]
    return m0, m1, m2


def _random_fields(seed=21, sh=(4, 4, 4)):
    r = np.random.default_rng(seed)
    rho = r.uniform(0.5, 1.5, sh)
    u = r.uniform(-0.1, 0.1, (3,) + sh) / math.sqrt(3)
    A = r.uniform(-1e-2, 1e-2, (3, 3) + sh)
    P = 0.5 * (A + A.transpose(1, 0, 2, 3, 4))  # symmetric, like the chemical stress
    return rho, u, P


def test_stress_equilibrium_moments_bruteforce():
    """R23: sum f^eq = rho, sum c f^eq = rho u, sum c c f^eq = rho/3 I + P + rho u u."""
    rho, u, P = _random_fields()
    m0, m1, m2 = _brute_moments(M.f_equilibrium_stress(rho, u, P))
    tol = 2e-15
    assert np.abs(m0 - rho).max() < tol
    for a in range(3):
        assert np.abs(m1[a] - rho * u[a]).max() < tol
        for b in range(3):
            want = P[a, b] + rho * u[a] * u[b] + (rho / 3.0 if a == b else 0.0)
            assert np.abs(m2[a][b] - want).max() < tol


def test_stress_equilibrium_without_stress_is_r8():
    rho, u, P = _random_fields(22)
    a = M.f_equilibrium_stress(rho, u, np.zeros_like(P))
    b = R.f_equilibrium(rho, u)
    assert np.abs(a - b).max() < 1e-16 * 4


def _random_f(seed=23, sh=(4, 4, 4)):
    r = np.random.default_rng(seed)
    rho, u, P = _random_fields(seed, sh)
    f = R.f_equilibrium(rho, u) + r.uniform(-2e-3, 2e-3, (19,) + sh)
    rho_f, j = R.density(f), R.momentum(f)
    return f, rho_f, M.velocity(rho_f, j), P


def test_projection_parts_carry_stress_and_ghosts_carry_nothing():
    """R24: the stress part h reproduces Pi; the ghost part has no mass, momentum or stress."""
    f, rho, u, P = _random_f()
    fneq = f - M.f_equilibrium_stress(rho, u, P)
    Pi = M.second_moment(fneq)
    h = M.stress_part(Pi)
    gam = fneq - h
    tol = 4e-15  # ~20 eps x the O(1) sums; a structural error is O(1e-3)
    m0, m1, m2 = _brute_moments(h)
    assert np.abs(m0).max() < tol
    for a in range(3):
        assert np.abs(m1[a]).max() < tol
        for b in range(3):
            assert np.abs(m2[a][b] - Pi[a, b]).max() < tol
    m0, m1, m2 = _brute_moments(gam)
    assert np.abs(m0).max() < tol
    for a in range(3):
        assert np.abs(m1[a]).max() < tol
        for b in range(3):
            assert np.abs(m2[a][b]).max() < tol
    assert np.abs(gam).max() > 1e-5  # the random f does have ghost content


@pytest.mark.parametrize("tau", [0.7, 1.0, 1.7])
def test_equal_relaxation_times_reduce_to_bgk(tau):
    """R24 with tau_s = tau_b = tau_ghost = tau is BGK."""
    f, rho, u, P = _random_f(24)
    p = M.MrtParams(base=P0, tau_s=tau, tau_b=tau, tau_ghost=tau)
    feq = M.f_equilibrium_stress(rho, u, P)
    want = f - (f - feq) / tau
    got = M.collide_f(f, rho, u, P, p)
    assert np.abs(got - want).max() < 4e-15


def test_each_part_relaxes_at_its_own_rate():
    """R24: Pi(f* - f^eq) = (1-1/tau_s) S + (1-1/tau_b) tr/3 I; ghosts scale by (1-1/tau_ghost);
    mass and momentum of f* are those of f."""
    f, rho, u, P = _random_f(25)
    p = M.MrtParams(base=P0, tau_s=0.65, tau_b=1.4, tau_ghost=0.9)
    feq = M.f_equilibrium_stress(rho, u, P)
    fs = M.collide_f(f, rho, u, P, p)
    Pi = M.second_moment(f - feq)
    tr = Pi[0, 0] + Pi[1, 1] + Pi[2, 2]
    m0, m1, m2 = _brute_moments(fs - feq)
    tol = 4e-15
    assert np.abs(m0).max() < tol
    for a in range(3):
        assert np.abs(m1[a]).max() < tol
        for b in range(3):
            S = Pi[a, b] - (tr / 3.0 if a == b else 0.0)
            want = (1 - 1 / p.tau_s) * S + ((1 - 1 / p.tau_b) * tr / 3.0 if a == b else 0.0)
            assert np.abs(m2[a][b] - want).max() < tol
    gam_before = (f - feq) - M.stress_part(Pi)
    gam_after = (fs - feq) - M.stress_part(M.second_moment(fs - feq))
    assert np.abs(gam_after - (1 - 1 / p.tau_ghost) * gam_before).max() < tol


def test_step_conserves_mass_phi_and_momentum_exactly_locally():
    """No force: the collision conserves j site by site, so the step conserves the totals."""
    rho, u, phi, nf, ng = synth.rough_fields(8, 6, 5, 3)
    f, g = R.equilibrium_state(rho, u, phi, P0)
    f, g = f + nf, g + ng
    fl = M.step_fields(f, g, MP0)
    assert np.abs(R.momentum(fl.fstar) - R.momentum(f)).max() < 1e-16 * 20
    f1, g1 = M.step(f, g, MP0)
    assert abs(f1.sum() - f.sum()) < 1e-12 * f.sum()
    assert abs(g1.sum() - g.sum()) < 1e-12 * np.abs(g).sum()
    assert np.abs(R.momentum(f1).sum(axis=(1, 2, 3)) - R.momentum(f).sum(axis=(1, 2, 3))).max() < 1e-13


@pytest.mark.parametrize("u0", [(0.0, 0.0, 0.0), (0.03, -0.02, 0.01)])
def test_uniform_equilibrium_is_fixed_point(u0):
    sh = (4, 5, 6)
    u = np.broadcast_to(np.array(u0)[:, None, None, None], (3,) + sh).copy()
    phi = np.full(sh, 0.3)
    f, g = R.equilibrium_state(np.full(sh, 1.1), u, phi, P0)
    # the uniform state has P = p0(phi) I: the stress equilibrium adds it to f
    fl = M.step_fields(f, g, MP0)
    feq = M.f_equilibrium_stress(fl.rho, fl.u, fl.P)
    f1, g1 = M.run(feq, g, MP0, 3)
    assert np.abs(f1 - feq).max() < 1e-15
    assert np.abs(g1 - g).max() < 1e-15


def test_phi_sign_symmetry_and_shift_invariance_bitwise():
    rho, u, phi, nf, ng = synth.rough_fields(6, 5, 4, 4)
    f, g = R.equilibrium_state(rho, u, phi, P0)
    f, g = f + nf, g + ng
    f1, g1 = M.step(f, g, MP0)
    f2, g2 = M.step(f, -g, MP0)
    assert np.array_equal(f1, f2) and np.array_equal(g1, -g2)
    sh = lambda a: np.roll(a, (1, -2, 3), axis=(1, 2, 3))  # noqa: E731
    f3, g3 = M.step(sh(f), sh(g), MP0)
    assert np.array_equal(f3, sh(f1)) and np.array_equal(g3, sh(g1))


def _mode_amplitude(field, k_index, n):
    prof = field.mean(axis=(0, 1))
    return abs(np.fft.rfft(prof)[k_index]) * 2 / n


@pytest.mark.parametrize("tb,tg", [(1.0, 1.0), (0.7, 1.6)])
def test_shear_wave_viscosity_is_set_by_tau_s_alone(tb, tg):
    """R25: u_y = U sin(kx) decays as exp(-nu k^2 t), nu = (tau_s - 1/2)/3 (2%), whatever the
    bulk and ghost times (a shear wave has no trace and, at this k, negligible ghost content)."""
    base = R.Params(A=0.0, B=0.0, kappa=0.0, mobility=0.0)
    p = M.MrtParams(base=base, tau_s=0.9, tau_b=tb, tau_ghost=tg)
    nx, ny, nz, T = 64, 4, 4, 200
    k = 2 * np.pi / nx
    x = np.arange(nx)
    sh = (nz, ny, nx)
    u = np.zeros((3,) + sh)
    u[1] = 1e-3 * np.sin(k * x)
    f, g = R.equilibrium_state(np.ones(sh), u, np.zeros(sh), base)
    a0 = _mode_amplitude(u[1], 1, nx)
    f, g = M.run(f, g, p, T)
    a1 = _mode_amplitude(R.momentum(f)[1] / R.density(f), 1, nx)
    nu_meas = -math.log(a1 / a0) / (k * k * T)
    assert abs(nu_meas / ((p.tau_s - 0.5) / 3) - 1) < 0.02


@pytest.mark.slow
def test_flat_interface_is_steady_with_stress_in_equilibrium():
    """The flat interface (A.9 profile) relaxes to a steady state: mu uniform, bulk at
    +-sqrt(-A/B), and the transient flow set off by the discrete stress dies out (|u| is
    3.8e-5 after 1000 steps, 2.4e-7 after 2000)."""
    base = R.Params(mobility=0.45)
    p = M.MrtParams(base=base, tau_s=0.8, tau_b=1.0, tau_ghost=1.0)
    nx, ny, nz = 4, 4, 64
    xi = math.sqrt(-2 * base.kappa / base.A)
    z = np.arange(nz)
    prof = np.where(z < 32, np.tanh((z - 16) / xi), -np.tanh((z - 48) / xi))
    sh = (nz, ny, nx)
    phi = np.broadcast_to(prof[:, None, None], sh).copy()
    f, g = R.equilibrium_state(np.ones(sh), np.zeros((3,) + sh), phi, base)
    f, g = M.run(f, g, p, 2000)
    fl = M.step_fields(f, g, p)
    ph, mu = fl.phi[:, 0, 0], fl.mu[:, 0, 0]
    assert np.abs(ph - prof).max() < 3e-2
    assert mu.max() - mu.min() < 1e-4
    assert np.abs(fl.u).max() < 1e-6
    phi_b = math.sqrt(-base.A / base.B)
    assert abs(ph[32 - 8] - phi_b) < 1e-3 and abs(ph[64 - 8] + phi_b) < 1e-3


@pytest.mark.parametrize("Mc", CUBIC)
def test_step_commutes_with_cubic_symmetry(Mc):
    """Stress-in-equilibrium MRT keeps the cubic isotropy of the
    BGK step: its moment projections split the second moment into trace and
    traceless parts, both invariant under reflections and axis permutations.
    A wrongly indexed stress component or projection row breaks this."""
    n = 5
    rho, u, phi, nf, ng = synth.rough_fields(n, n, n, 13)
    f, g = R.equilibrium_state(rho, u, phi, P0)
    f, g = f + nf, g + ng
    f1, g1 = M.step(f, g, MP0)
    T = lambda a: cube_transform(a, Mc, n)  # noqa: E731
    f2, g2 = M.step(T(f), T(g), MP0)
    assert np.abs(f2 - T(f1)).max() <= 1e-13 * np.abs(f1).max()
    assert np.abs(g2 - T(g1)).max() <= 1e-13 * np.abs(g1).max()
