"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these compares the oracle with itself: each checks a closed form, an
exact rational identity, a conservation law, a bitwise symmetry, a second
independent transcription (``lb_brute``), or a hydrodynamic limit.  A dropped
term, a wrong sign or index, or a transposed operand in ``oracle/lb_ref.py``
fails at least one of them.
"""
from fractions import Fraction
import math
import os

import numpy as np
import pytest

from oracle import lb_brute as BR
from oracle import lb_ref as R
from paper_1609_01479_b200 import synth
from symmetry import CUBIC, cube_transform

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "d3q19_appendix_b.txt")
P0 = R.Params()  # R16 defaults


def _golden_table():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        p, cx, cy, cz, w = line.split()
        rows.append((int(p), (int(cx), int(cy), int(cz)), Fraction(w)))
    return rows


def _rough_state(nx, ny, nz, seed=1, p=P0):
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, seed)
    f, g = R.equilibrium_state(rho, u, phi, p)
    return f + nf, g + ng


def _spinodal_state(nx, ny, nz, seed=0, p=P0):
    rho, u, phi = synth.spinodal_fields(nx, ny, nz, seed)
    return R.equilibrium_state(rho, u, phi, p)


# ---------------------------------------------------------------- D3Q19 table
def test_table_matches_golden_and_enumeration():
    """R1: typed table (lb_ref) == Appendix B golden == enumerated set (lb_brute), bitwise."""
    rows = _golden_table()
    assert len(rows) == 19
    for p, c, w in rows:
        assert tuple(int(v) for v in R.C[p]) == c
        assert R.W[p] == float(w)
        assert BR.CV[p] == c
        assert BR.WV[p] == float(w)


def test_table_exact_moments():
    """Sum w = 1, sum w c = 0, sum w cc = I/3, odd 3rd moments 0, 4th = (dd+dd+dd)/9 (exact rationals)."""
    rows = _golden_table()
    d = lambda a, b: 1 if a == b else 0
    assert sum(w for _, _, w in rows) == 1
    for a in range(3):
        assert sum(w * c[a] for _, c, w in rows) == 0
        for b in range(3):
            assert sum(w * c[a] * c[b] for _, c, w in rows) == Fraction(d(a, b), 3)
            for e in range(3):
                assert sum(w * c[a] * c[b] * c[e] for _, c, w in rows) == 0
                for h in range(3):
                    m4 = sum(w * c[a] * c[b] * c[e] * c[h] for _, c, w in rows)
                    assert m4 == Fraction(d(a, b) * d(e, h) + d(a, e) * d(b, h) + d(a, h) * d(b, e), 9)


def test_antipodes_and_component_sets():
    """Antipode of p >= 1 is 19 - p; the c_z = +-1 sets of Appendix B."""
    for p in range(1, 19):
        assert (R.C[19 - p] == -R.C[p]).all()
    assert [p for p in range(19) if R.C[p, 2] == 1] == [2, 6, 9, 11, 15]
    assert [p for p in range(19) if R.C[p, 2] == -1] == [4, 8, 10, 13, 17]


# ---------------------------------------------------------------- equilibria
def _brute_moments(dist):
    """Explicit-loop zeroth, first and second moments of (19, ...) arrays."""
    m0 = sum(dist[i] for i in range(19))
    m1 = [sum(BR.CV[i][a] * dist[i] for i in range(19)) for a in range(3)]
    m2 = [[sum(BR.CV[i][a] * BR.CV[i][b] * dist[i] for i in range(19)) for b in range(3)] for a in range(3)]
    return m0, m1, m2


def test_equilibrium_and_source_moments_bruteforce():
    """R7-R9 moments on a 4^3 lattice with random rho, u, phi, mu, F (north_star pin)."""
    r = np.random.default_rng(11)
    sh = (4, 4, 4)
    rho = r.uniform(0.5, 1.5, sh)
    u = r.uniform(-0.1, 0.1, (3,) + sh) / math.sqrt(3)
    phi = r.uniform(-1, 1, sh)
    mu = r.uniform(-0.1, 0.1, sh)
    F = r.uniform(-1e-2, 1e-2, (3,) + sh)
    gam = P0.gamma
    tol = 2e-15
    m0, m1, m2 = _brute_moments(R.f_equilibrium(rho, u))
    assert np.abs(m0 - rho).max() < tol
    for a in range(3):
        assert np.abs(m1[a] - rho * u[a]).max() < tol
        for b in range(3):
            want = rho * (u[a] * u[b] + (1.0 / 3.0 if a == b else 0.0))
            assert np.abs(m2[a][b] - want).max() < tol
    m0, m1, m2 = _brute_moments(R.g_equilibrium(phi, u, mu, gam))
    assert np.abs(m0 - phi).max() < tol
    for a in range(3):
        assert np.abs(m1[a] - phi * u[a]).max() < tol
        for b in range(3):
            want = phi * u[a] * u[b] + (gam * mu if a == b else 0.0)
            assert np.abs(m2[a][b] - want).max() < tol
    m0, m1, m2 = _brute_moments(R.guo_source(u, F))
    assert np.abs(m0).max() < tol
    for a in range(3):
        assert np.abs(m1[a] - F[a]).max() < tol
        for b in range(3):
            assert np.abs(m2[a][b] - (u[a] * F[b] + F[a] * u[b])).max() < tol


def test_g_equilibrium_rest_particle_closed_form():
    """R9 at rest: g0 = phi - 1.5 Gamma mu - phi u^2/2; faces carry no mu term; edges Gamma mu / 8."""
    phi, mu, gam = np.array(0.3), np.array(0.02), 0.7
    u = np.zeros((3,))
    geq = R.g_equilibrium(phi, u, mu, gam)
    assert abs(geq[0] - (0.3 - 1.5 * 0.7 * 0.02)) < 1e-16
    assert abs(geq[3]) < 1e-18 and abs(geq[9]) < 1e-18
    assert abs(geq[1] - 0.7 * 0.02 / 8) < 1e-17


# ---------------------------------------------------------------- stencils
@pytest.mark.parametrize("m", [(1, 0, 0), (2, 3, 1), (5, 1, 3)])
def test_stencils_fourier_mode(m):
    """Central gradient of eps cos(k.x+t) is -eps sin(k.x+t) sin k_a; 7-point Laplacian
    eigenvalue is -sum 2(1 - cos k_a), exactly (up to rounding)."""
    nx, ny, nz = 12, 10, 8
    k = np.array([2 * np.pi * m[0] / nx, 2 * np.pi * m[1] / ny, 2 * np.pi * m[2] / nz])
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    th = k[0] * x + k[1] * y + k[2] * z + 0.3
    eps = 0.01
    phi = eps * np.cos(th)
    grad = R.gradient(phi)
    for a in range(3):
        assert np.abs(grad[a] + eps * np.sin(th) * np.sin(k[a])).max() < 1e-16
    lam = -sum(2 * (1 - np.cos(k[a])) for a in range(3))
    assert np.abs(R.laplacian(phi) - lam * phi).max() < 1e-15


# ---------------------------------------------------------------- thermodynamics
def test_chemical_potential_is_free_energy_derivative():
    """R3 vs R2: uniform phi, mu = d psi / d phi (central difference of psi)."""
    phi = np.linspace(-1.3, 1.3, 27)
    h = 1e-5
    dpsi = (R.free_energy_density(phi + h, P0) - R.free_energy_density(phi - h, P0)) / (2 * h)
    mu = R.chemical_potential(phi, np.zeros_like(phi), P0)
    assert np.abs(mu - dpsi).max() < 1e-10


def test_bulk_pressure_is_legendre_transform():
    """R4 vs R2/R3: uniform phi, P = (phi mu - psi) I."""
    phi = np.linspace(-1.3, 1.3, 27).reshape(3, 3, 3)
    z = np.zeros((3,) + phi.shape)
    P = R.chemical_stress(phi, z, np.zeros_like(phi), P0)
    mu = R.chemical_potential(phi, np.zeros_like(phi), P0)
    p_thermo = phi * mu - R.free_energy_density(phi, P0)
    for a in range(3):
        for b in range(3):
            want = p_thermo if a == b else 0.0
            assert np.abs(P[a, b] - want).max() < 1e-16


def test_force_converges_to_phi_grad_mu():
    """R4/R5: div P = phi grad mu in the continuum (Gibbs-Duhem), so the discrete
    F = -div P -> -phi grad mu at second order.  Halving k shrinks the error ~4x."""
    errs = []
    for L in (32, 64):
        x = np.arange(L)
        k = 2 * np.pi / L
        prof = 0.5 * np.cos(k * x) + 0.2 * np.sin(2 * k * x)  # varies along x only
        phi = np.broadcast_to(prof, (3, 3, L)).copy()
        lap = R.laplacian(phi)
        F = R.force(R.chemical_stress(phi, R.gradient(phi), lap, P0))
        mu = R.chemical_potential(phi, lap, P0)
        want = -phi * R.gradient(mu)[0]
        errs.append(np.abs(F[0] - want).max() / np.abs(want).max())
        assert np.abs(F[1]).max() < 1e-18 and np.abs(F[2]).max() < 1e-18
    assert errs[0] < 0.15
    assert 3.5 < errs[0] / errs[1] < 4.5


def _mode3d(L, k_int, amp, th0):
    """amp cos(2 pi (k_int . x) / L + th0) on an L^3 lattice, (z, y, x) array."""
    z, y, x = np.meshgrid(np.arange(L), np.arange(L), np.arange(L), indexing="ij")
    k = 2 * np.pi * np.asarray(k_int, dtype=np.float64) / L
    th = k[0] * x + k[1] * y + k[2] * z + th0
    return amp * np.cos(th), th, k


def test_stress_single_mode_closed_form():
    """R4 (A.4) on phi = eps cos(k.x + t): the discrete gradient is exactly
    -eps sin(k.x + t) sin k_a (A.2), so every off-diagonal component is
    P_ab = kappa eps^2 sin^2(k.x + t) sin k_a sin k_b (a != b), and the diagonal ones
    add the isotropic part p0 - kappa phi lap phi - kappa/2 |grad phi|^2 with the
    Laplacian eigenvalue -sum 2(1 - cos k_a).  A mode with k_x, k_y, k_z all non-zero
    exercises every off-diagonal term."""
    L, eps = 12, 0.3
    phi, th, k = _mode3d(L, (1, 2, 3), eps, 0.4)
    lam = -sum(2 * (1 - np.cos(k[a])) for a in range(3))
    grad = R.gradient(phi)
    lap = R.laplacian(phi)
    P = R.chemical_stress(phi, grad, lap, P0)
    s2 = np.sin(th) ** 2
    g2 = eps * eps * s2 * sum(np.sin(k[a]) ** 2 for a in range(3))
    iso = 0.5 * P0.A * phi ** 2 + 0.75 * P0.B * phi ** 4 - P0.kappa * lam * phi ** 2 - 0.5 * P0.kappa * g2
    for a in range(3):
        for b in range(3):
            want = P0.kappa * eps * eps * s2 * np.sin(k[a]) * np.sin(k[b])
            if a == b:
                want = want + iso
            assert np.abs(P[a, b] - want).max() < 2e-16, (a, b)
            assert np.abs(P[a, b] - P[b, a]).max() < 1e-18  # symmetric


@pytest.mark.parametrize("modes,sizes", [
    # (k vector, amplitude, phase) triples summed into phi; every pair of axes coupled
    ((((1, 1, 0), 0.5, 0.3), ((0, 1, 1), 0.3, 1.1), ((1, 0, 2), 0.2, 2.0)), (16, 32)),
    ((((1, 2, 1), 0.6, 0.0), ((2, -1, 1), 0.25, 0.7)), (32, 64)),
])
def test_force_converges_to_phi_grad_mu_3d(modes, sizes):
    """Gibbs-Duhem in 3-D: div P = phi grad mu holds identically in the continuum
    for P_ab of R4 (A.4) -- the off-diagonal kappa d_a phi d_b phi and the
    cross-derivatives d_b P_ab (a != b) of F (A.5) are what cancel the
    kappa d_a(|grad phi|^2)/2 and kappa phi d_a lap phi terms.  So for a smooth
    field varying along all three axes the discrete F = -div P approaches
    -phi grad mu in EVERY component at second order: the error falls ~4x when
    the lattice (and every wavelength) doubles.  A wrong factor or sign on the
    off-diagonal stress, or a dropped cross-derivative, leaves an O(1) error."""
    errs = []
    for L in sizes:
        phi = np.zeros((L, L, L))
        for kv, amp, th0 in modes:
            phi = phi + _mode3d(L, kv, amp, th0)[0]
        lap = R.laplacian(phi)
        F = R.force(R.chemical_stress(phi, R.gradient(phi), lap, P0))
        mu = R.chemical_potential(phi, lap, P0)
        gmu = R.gradient(mu)
        e = []
        for a in range(3):
            want = -phi * gmu[a]
            assert np.abs(want).max() > 1e-5  # every component is driven
            e.append(np.abs(F[a] - want).max() / np.abs(want).max())
        errs.append(e)
    for a in range(3):
        assert errs[0][a] < 0.3, errs
        assert 3.5 < errs[0][a] / errs[1][a] < 4.5, errs


def test_force_sums_to_zero():
    """R5: sum_x F = 0 (telescoping), so total momentum is conserved."""
    f, g = _rough_state(7, 6, 5)
    fl = R.step_fields(f, g, P0)
    scale = np.abs(fl.F).max() * fl.F[0].size
    for a in range(3):
        assert abs(fl.F[a].sum()) < 1e-14 * scale


# ---------------------------------------------------------------- collision
def test_collision_invariants():
    """Per site: sum f* = rho; sum c f* = j + F; sum g* = phi (A.9)."""
    f, g = _rough_state(5, 4, 3)
    fl = R.step_fields(f, g, P0)
    m0, m1, _ = _brute_moments(fl.fstar)
    assert np.abs(m0 - fl.rho).max() < 1e-15
    for a in range(3):
        assert np.abs(m1[a] - (fl.j[a] + fl.F[a])).max() < 1e-15
    assert np.abs(sum(fl.gstar[i] for i in range(19)) - fl.phi).max() < 1e-15


def test_collision_tau_one_special_case():
    """S:339 analogue: tau = 1 relaxes fully; f* = f^eq + S/2 and g* = g^eq."""
    p = R.Params(tau_f=1.0, tau_g=1.0)
    f, g = _rough_state(4, 4, 4, p=p)
    fl = R.step_fields(f, g, p)
    feq = R.f_equilibrium(fl.rho, fl.u)
    S = R.guo_source(fl.u, fl.F)
    geq = R.g_equilibrium(fl.phi, fl.u, fl.mu, p.gamma)
    assert np.abs(fl.fstar - (feq + 0.5 * S)).max() < 1e-16
    assert np.abs(fl.gstar - geq).max() < 1e-16


# ---------------------------------------------------------------- propagation
def test_propagation_matches_integer_map_and_is_permutation():
    """A.8 / S:343-348: out_i(x) = a_i(x - c_i) bitwise; each component's multiset preserved."""
    nx, ny, nz = 5, 4, 3
    a = np.random.default_rng(3).random((19, nz, ny, nx))
    out = R.propagate(a)
    for i in range(19):
        assert np.array_equal(np.sort(out[i].ravel()), np.sort(a[i].ravel()))
        for z in range(nz):
            for y in range(ny):
                for x in range(nx):
                    sx, sy, sz = BR.propagation_source(nx, ny, nz, x, y, z, i)
                    assert out[i, z, y, x] == a[i, sz, sy, sx]


def test_propagation_returns_after_lcm_steps():
    """stream-only for L = lcm(nx, ny, nz) steps returns the start, bitwise."""
    nx, ny, nz = 4, 6, 3
    a = np.random.default_rng(4).random((19, nz, ny, nx))
    b = a
    for _ in range(math.lcm(nx, ny, nz)):
        b = R.propagate(b)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- full step
def test_vectorised_equals_bruteforce():
    """Two independent transcriptions agree: lb_ref (np.roll) vs lb_brute (scalar loops)."""
    f, g = _rough_state(5, 4, 3, seed=2)
    fa, ga = f, g
    fb, gb = f, g
    for _ in range(2):
        fa, ga = R.step(fa, ga, P0)
        fb, gb = BR.step(fb, gb, P0)
    assert np.abs(fa - fb).max() < 1e-14
    assert np.abs(ga - gb).max() < 1e-14


def test_site_sampler_matches_full_step():
    f, g = _rough_state(6, 5, 4, seed=5)
    fa, ga = R.step(f, g, P0)
    smp = BR.SiteSampler(f, g, P0)
    for (x, y, z) in synth.sample_sites(6, 5, 4, 20):
        fo, go = smp.after_step(x, y, z)
        assert np.abs(np.array(fo) - fa[:, z, y, x]).max() < 1e-14
        assert np.abs(np.array(go) - ga[:, z, y, x]).max() < 1e-14


def test_step_conserves_mass_phi_momentum():
    """north_star pin: sum f, sum g and sum c f unchanged by a step (to rounding)."""
    f, g = _rough_state(8, 7, 6, seed=6)
    m0, j0, p0 = (v.sum(axis=(-1, -2, -3)) for v in R.macroscopic(f, g))
    for _ in range(3):
        f, g = R.step(f, g, P0)
    m1, j1, p1 = (v.sum(axis=(-1, -2, -3)) for v in R.macroscopic(f, g))
    assert abs(m1 - m0) < 1e-12 * abs(m0)
    assert np.abs(j1 - j0).max() < 1e-13 * np.abs(f).sum()
    assert abs(p1 - p0) < 1e-12 * np.abs(g).sum()


@pytest.mark.parametrize("u0", [(0.0, 0.0, 0.0), (0.03, -0.02, 0.01)])
def test_uniform_equilibrium_is_fixed_point(u0):
    """north_star / S:337: uniform rho0, u0 (Galilean), phi0 at equilibrium is unchanged."""
    sh = (4, 5, 6)
    rho = np.full(sh, 1.1)
    u = np.stack([np.full(sh, v) for v in u0])
    phi = np.full(sh, 0.4)
    f, g = R.equilibrium_state(rho, u, phi, P0)
    f1, g1 = R.step(f, g, P0)
    assert np.abs(f1 - f).max() <= 1e-15 * np.abs(f).max()
    assert np.abs(g1 - g).max() <= 1e-15 * np.abs(g).max()


def test_shift_invariance_bitwise():
    """step(shift_v(s)) == shift_v(step(s)) bitwise for lattice vectors v."""
    f, g = _rough_state(6, 5, 4, seed=8)
    f1, g1 = R.step(f, g, P0)
    for v in [(1, 0, 0), (0, 2, 0), (0, 0, 3), (2, 1, 1)]:
        sh = lambda a: np.roll(a, shift=(v[2], v[1], v[0]), axis=(1, 2, 3))
        f2, g2 = R.step(sh(f), sh(g), P0)
        assert np.array_equal(f2, sh(f1)) and np.array_equal(g2, sh(g1))


def test_phi_sign_symmetry_bitwise():
    """step(f, -g) == (f', -g') bitwise: mu and g^eq are odd in phi; P, F even."""
    f, g = _rough_state(5, 5, 4, seed=9)
    f1, g1 = R.step(f, g, P0)
    f2, g2 = R.step(f, -g, P0)
    assert np.array_equal(f1, f2) and np.array_equal(-g1, g2)


def test_numerical_domain_error_names_site():
    """R22 / S:335: rho <= 0 raises."""
    f, g = _rough_state(4, 4, 4)
    f[:, 2, 1, 3] = 0.0
    with pytest.raises(R.NumericalDomainError, match=r"x=3, y=1, z=2"):
        R.step(f, g, P0)


# ---------------------------------------------------------------- hydrodynamic limits
def _mode_amplitude(field, k_index, axis_len):
    """|Fourier coefficient| of a field varying along x."""
    prof = field.mean(axis=(0, 1))
    return abs(np.fft.rfft(prof)[k_index]) * 2 / axis_len


def test_shear_wave_viscosity():
    """S:362 analogue: u_y = U sin(kx) decays as exp(-nu k^2 t), nu = (tau_f - 1/2)/3, within 2%."""
    p = R.Params(A=0.0, B=0.0, kappa=0.0, mobility=0.0)
    nx, ny, nz, T = 64, 4, 4, 200
    k = 2 * np.pi / nx
    x = np.arange(nx)
    sh = (nz, ny, nx)
    u = np.zeros((3,) + sh)
    u[1] = 1e-3 * np.sin(k * x)
    f, g = R.equilibrium_state(np.ones(sh), u, np.zeros(sh), p)
    a0 = _mode_amplitude(u[1], 1, nx)
    f, g = R.run(f, g, p, T)
    a1 = _mode_amplitude(R.momentum(f)[1] / R.density(f), 1, nx)
    nu_meas = -math.log(a1 / a0) / (k * k * T)
    nu = (p.tau_f - 0.5) / 3
    assert abs(nu_meas / nu - 1) < 0.02


def test_phi_diffusion_rate():
    """R10: A > 0, B = kappa = 0: d_t phi = M A lap(phi); a cos mode decays at M A k^2 (3%)."""
    p = R.Params(A=0.1, B=0.0, kappa=0.0, mobility=0.2)
    nx, ny, nz, T = 32, 4, 4, 300
    k = 2 * np.pi / nx
    x = np.arange(nx)
    sh = (nz, ny, nx)
    phi = np.broadcast_to(1e-4 * np.cos(k * x), sh).copy()
    f, g = R.equilibrium_state(np.ones(sh), np.zeros((3,) + sh), phi, p)
    a0 = _mode_amplitude(R.order_parameter(g), 1, nx)
    f, g = R.run(f, g, p, T)
    a1 = _mode_amplitude(R.order_parameter(g), 1, nx)
    rate = -math.log(a1 / a0) / T
    assert abs(rate / (p.mobility * p.A * k * k) - 1) < 0.03


def test_spinodal_linear_growth_rate():
    """A.9: linear Cahn-Hilliard growth omega = M khat^2 (-A - kappa khat^2),
    khat^2 = 2(1 - cos k) (7-point mu), within 5% at early times."""
    p = R.Params(mobility=0.45)
    nx, ny, nz, T = 32, 4, 4, 300
    k = 2 * np.pi / nx
    x = np.arange(nx)
    sh = (nz, ny, nx)
    phi = np.broadcast_to(1e-6 * np.cos(k * x), sh).copy()
    f, g = R.equilibrium_state(np.ones(sh), np.zeros((3,) + sh), phi, p)
    f, g = R.run(f, g, p, 20)  # let the initial transient pass
    a0 = _mode_amplitude(R.order_parameter(g), 1, nx)
    f, g = R.run(f, g, p, T)
    a1 = _mode_amplitude(R.order_parameter(g), 1, nx)
    kh2 = 2 * (1 - math.cos(k))
    omega = p.mobility * kh2 * (-p.A - p.kappa * kh2)
    rate = math.log(a1 / a0) / T
    assert abs(rate / omega - 1) < 0.05


@pytest.mark.slow
def test_flat_interface_profile():
    """A.9: phi = tanh(z/xi), xi = sqrt(-2 kappa/A), solves mu = 0; bulk +-sqrt(-A/B).
    After 1000 steps the profile is steady (mu uniform, the stationarity condition of
    d_t phi = M lap mu), the bulk sits at +-1, and the discrete profile stays within 3%
    of the continuum tanh (xi = 1.13 lattice spacings, so the 7-point stencil's O(h^2/xi^2)
    error is a few percent)."""
    p = R.Params(mobility=0.45)
    nx, ny, nz = 4, 4, 64
    xi = math.sqrt(-2 * p.kappa / p.A)
    z = np.arange(nz)
    prof = np.where(z < 32, np.tanh((z - 16) / xi), -np.tanh((z - 48) / xi))
    sh = (nz, ny, nx)
    phi = np.broadcast_to(prof[:, None, None], sh).copy()
    f, g = R.equilibrium_state(np.ones(sh), np.zeros((3,) + sh), phi, p)
    f, g = R.run(f, g, p, 1000)
    fl = R.step_fields(f, g, p)
    ph, mu = fl.phi[:, 0, 0], fl.mu[:, 0, 0]
    assert np.abs(ph - prof).max() < 3e-2
    assert mu.max() - mu.min() < 1e-4
    phi_b = math.sqrt(-p.A / p.B)
    assert abs(ph[32 - 8] - phi_b) < 1e-3 and abs(ph[64 - 8] + phi_b) < 1e-3


@pytest.mark.parametrize("M", CUBIC)
def test_step_commutes_with_cubic_symmetry(M):
    """The model is isotropic under the cubic group (D3Q19, the
    free energy and P_ab are built from rotation-invariant terms), so
    step(T s) == T step(s) up to rounding for reflections and axis
    permutations.  A transposed P_ab index, a z-only sign slip in the force or
    a velocity component paired with the wrong axis breaks this, which the
    translation and phi-sign symmetries above cannot see."""
    n = 5
    f, g = _rough_state(n, n, n, seed=12)
    f1, g1 = R.step(f, g, P0)
    T = lambda a: cube_transform(a, M, n)  # noqa: E731
    f2, g2 = R.step(T(f), T(g), P0)
    assert np.abs(f2 - T(f1)).max() <= 1e-13 * np.abs(f1).max()
    assert np.abs(g2 - T(g1)).max() <= 1e-13 * np.abs(g1).max()
