"""Pins of the NEXT-4 oracle (``oracle/lb_lc.py``: Landau-de Gennes Q tensor,
Beris-Edwards LC update, chemical stress -> force on the LB fluid; readings
R34-R45 of DESIGN.md).  The paper prints no LC equation or number, so each part
is pinned by what the mathematics fixes:

* H = -dF/dQ: the molecular field is the (negative) derivative of the free
  energy, by finite differences of the bulk density and of the discrete total
  free energy (whose exact variational derivative has the 7-point Laplacian);
  the uniaxial bulk minimum S0 = 1/4 + 3/4 sqrt(1 - 8 / (3 gamma)) and the
  closed-form H of a uniaxial Q;
* the force: a Gibbs-Duhem-type identity (div sigma -> -dQ:H, second order),
  sum_x F = 0, and summation by parts sum_x u.F = sum_x P:W(u) (fixes the
  divergence index against the velocity-gradient convention);
* the co-rotation: the reversible coupling exchanges no energy, H:S + sigma:W = 0
  pointwise; a rigid rotation of the fluid rotates the director with it; the
  isotropic limit S = 2 xi D / 3;
* the LC update: the exact per-step factor of a small mode (relaxation
  1 + Gamma (-A0 (1 - gamma/3) - kappa khat^2)) and of passive upwind advection;
  the free energy decreases at rate Gamma sum H:H;
* the step: uniform nematic (also Galilean) fixed point, mass and momentum
  conservation, shift invariance (bitwise), lattice rotation and reflection
  covariance, the site sampler equal to the full step (bitwise).
"""
import math

import numpy as np
import pytest

from oracle import lb_lc as LC
from oracle import lb_ref as R
from paper_1609_01479_b200 import synth


def _rand_sym_traceless(r, shape=()):
    q5 = r.uniform(-0.4, 0.4, size=(5,) + shape)
    return LC.q_full(q5)


def _frob(X, Y):
    return float((X * Y).sum())


def test_five_components_roundtrip():
    r = np.random.default_rng(0)
    q5 = r.uniform(-1, 1, size=(5, 3, 4, 2))
    Q = LC.q_full(q5)
    assert np.array_equal(LC.q_five(Q), q5)
    assert np.array_equal(Q, Q.transpose(1, 0, 2, 3, 4))
    assert np.abs(Q[0, 0] + Q[1, 1] + Q[2, 2]).max() == 0.0


@pytest.mark.parametrize("gamma", [2.0, 2.9, 3.2, 4.0])
def test_bulk_molecular_field_is_minus_derivative(gamma):
    """For any symmetric traceless direction D: d/de f_bulk(Q + e D) = -H_bulk : D."""
    p = LC.LcParams(gamma=gamma, A0=0.7)
    r = np.random.default_rng(int(gamma * 10))
    for _ in range(5):
        Q = _rand_sym_traceless(r)
        D = _rand_sym_traceless(r)
        H = LC.molecular_field(Q, np.zeros_like(Q), p)
        e = 1e-5
        d = (LC.bulk_free_energy(Q + e * D, p) - LC.bulk_free_energy(Q - e * D, p)) / (2 * e)
        assert abs(d + _frob(H, D)) < 1e-9 * (1 + abs(d))


def _discrete_energy(q5, p):
    """sum_x f_bulk + kappa/2 sum_x sum_a |Q(x + e_a) - Q(x)|^2: the discrete energy whose
    exact variational derivative carries the 7-point Laplacian (summation by parts)."""
    Q = LC.q_full(q5)
    E = LC.bulk_free_energy(Q, p).sum()
    for a in range(3):
        d = np.stack([np.stack([R.shifted(Q[i, j], a, +1) - Q[i, j] for j in range(3)]) for i in range(3)])
        E += 0.5 * p.kappa * (d * d).sum()
    return E


def test_molecular_field_is_minus_gradient_of_discrete_energy():
    p = LC.LcParams(kappa=0.3, A0=0.5)
    r = np.random.default_rng(5)
    q5 = r.uniform(-0.4, 0.4, size=(5, 4, 5, 6))
    Q = LC.q_full(q5)
    H = LC.molecular_field(Q, LC.q_laplacian(Q), p)
    for (z, y, x) in [(0, 0, 0), (3, 4, 5), (1, 2, 3)]:
        Dq = r.uniform(-1, 1, size=5)
        D = LC.q_full(Dq.reshape(5, 1))[:, :, 0]
        e = 1e-5
        qp, qm = q5.copy(), q5.copy()
        qp[:, z, y, x] += e * Dq
        qm[:, z, y, x] -= e * Dq
        d = (_discrete_energy(qp, p) - _discrete_energy(qm, p)) / (2 * e)
        assert abs(d + _frob(H[:, :, z, y, x], D)) < 1e-8 * (1 + abs(d))


@pytest.mark.parametrize("gamma", [2.8, 3.0, 3.2, 4.5])
def test_uniaxial_bulk_minimum_and_closed_form_field(gamma):
    """Q = S (n n - I/3): H = A0 [-(1 - gamma/3) S + gamma S^2/3 - 2 gamma S^3/3] (n n - I/3),
    zero at S0 = 1/4 + 3/4 sqrt(1 - 8/(3 gamma)), which is a local minimum of f_bulk."""
    p = LC.LcParams(gamma=gamma, A0=0.3)
    n = np.array([0.36, -0.48, 0.8])
    N = np.outer(n, n) - np.eye(3) / 3
    S0 = LC.uniaxial_order(gamma)
    for S in (0.1, S0, 0.7):
        Q = S * N
        H = LC.molecular_field(Q, np.zeros_like(Q), p)
        coef = p.A0 * (-(1 - gamma / 3) * S + gamma * S * S / 3 - 2 * gamma * S ** 3 / 3)
        assert np.abs(H - coef * N).max() < 1e-15
    H0 = LC.molecular_field(S0 * N, np.zeros((3, 3)), p)
    assert np.abs(H0).max() < 1e-15
    f = lambda S: float(LC.bulk_free_energy(S * N, p))  # noqa: E731
    assert f(S0) < f(S0 - 0.01) and f(S0) < f(S0 + 0.01)


def test_gradient_index_order():
    """dQ[c, a, b] = d_c Q_ab: a mode along x only has x derivatives, of the right sign."""
    n = 12
    x = np.arange(n)
    sh = (3, 4, n)
    q5 = np.zeros((5,) + sh)
    q5[1] = np.broadcast_to(np.sin(2 * np.pi * x / n), sh)  # Q_xy
    dQ = LC.q_gradient(LC.q_full(q5))
    assert np.abs(dQ[1]).max() == 0 and np.abs(dQ[2]).max() == 0
    k = 2 * np.pi / n
    expect = math.sin(k) * np.cos(k * x)  # central difference of sin
    assert np.abs(dQ[0, 0, 1][0, 0] - expect).max() < 1e-15
    assert np.abs(dQ[0, 1, 0][0, 0] - expect).max() < 1e-15


def _diag_mode_field(n, eps=0.05):
    """A smooth diagonal Q (Q and H commute, so the antisymmetric stress vanishes)."""
    k = 2 * np.pi / n
    z, y, x = np.indices((n, n, n))
    q1 = eps * np.cos(k * x + 0.3) * (1 + 0.5 * np.sin(k * y))
    q2 = eps * np.sin(k * z - 0.2) + 0.5 * eps * np.cos(k * (x + y))
    q5 = np.zeros((5, n, n, n))
    q5[0], q5[3] = q1, q2
    return q5


def test_force_converges_to_minus_dq_h():
    """xi = 0, diagonal Q: div sigma = -sum_cd d_a Q_cd H_cd in the continuum (the LC
    Gibbs-Duhem relation behind R38's p0 = -f); the lattice error falls as k^2."""
    p = LC.LcParams(xi=0.0, kappa=0.5, A0=0.2)
    errs = []
    for n in (16, 32):
        q5 = _diag_mode_field(n)
        Q = LC.q_full(q5)
        dQ = LC.q_gradient(Q)
        H = LC.molecular_field(Q, LC.q_laplacian(Q), p)
        F = LC.force(LC.chemical_stress(Q, dQ, H, LC.free_energy_density(Q, dQ, p), p))
        T = -np.einsum("acdzyx,cdzyx->azyx", dQ, H)
        errs.append(np.abs(F - T).max() / np.abs(T).max())
    assert errs[0] < 0.1
    assert 3.3 < errs[0] / errs[1] < 4.7


def test_force_sums_to_zero_and_summation_by_parts():
    """sum_x F = 0; sum_x u.F = sum_x P:W(u) for any P and u (F = -div P, W_ab = d_b u_a)."""
    r = np.random.default_rng(9)
    sh = (5, 6, 7)
    P = r.uniform(-1, 1, size=(3, 3) + sh)
    u = r.uniform(-1, 1, size=(3,) + sh)
    F = LC.force(P)
    assert np.abs(F.sum(axis=(1, 2, 3))).max() < 1e-12
    W = LC.velocity_gradient(u)
    lhs = (u * F).sum()
    rhs = (P * W).sum()
    assert abs(lhs - rhs) < 1e-12 * (np.abs(u * F).sum() + np.abs(P * W).sum())


def test_reversible_coupling_exchanges_no_energy():
    """H:S(W, Q) + sigma_rev:W = 0 pointwise for any symmetric traceless Q, H and any
    traceless W (an incompressible flow; sigma_rev = the xi and antisymmetric parts: R38
    with dQ = 0, fed = 0).  For a compressible W the sum is 2 xi (Q:H) tr(W)/3."""
    r = np.random.default_rng(11)
    for xi in (0.0, 0.7, -0.4):
        p = LC.LcParams(xi=xi)
        Q = _rand_sym_traceless(r, (6,))
        H = _rand_sym_traceless(r, (6,))
        W = r.uniform(-1, 1, size=(3, 3, 6))
        sigma = -LC.chemical_stress(Q, np.zeros((3, 3, 3, 6)), H, np.zeros(6), p)
        trW = W[0, 0] + W[1, 1] + W[2, 2]
        qh = (Q * H).sum(axis=(0, 1))
        e = (H * LC.corotation(W, Q, xi)).sum(axis=(0, 1)) + (sigma * W).sum(axis=(0, 1))
        assert np.abs(e - 2 * xi * qh * trW / 3).max() < 1e-14
        W0 = W - np.eye(3)[:, :, None] * trW / 3
        e0 = (H * LC.corotation(W0, Q, xi)).sum(axis=(0, 1)) + (sigma * W0).sum(axis=(0, 1))
        assert np.abs(e0).max() < 1e-14


def _rodrigues(n, w, t):
    th = np.linalg.norm(w) * t
    k = w / np.linalg.norm(w)
    return n * math.cos(th) + np.cross(k, n) * math.sin(th) + k * (k @ n) * (1 - math.cos(th))


def test_rigid_rotation_rotates_the_director():
    """u = omega x r (W_ac = eps_abc omega_b, no strain): dQ/dt = S(W, Q) for
    Q = S (n n - I/3) equals the time derivative of the rotated director, for any xi."""
    w = np.array([0.3, -0.2, 0.5])
    W = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            for c in range(3):
                W[a, c] += np.linalg.det(np.eye(3)[[a, b, c]]) * w[b]
    n = np.array([0.6, 0.0, 0.8])
    Sc = 0.45
    h = 1e-5
    Qt = lambda t: Sc * (np.outer(_rodrigues(n, w, t), _rodrigues(n, w, t)) - np.eye(3) / 3)  # noqa: E731
    dQdt = (Qt(h) - Qt(-h)) / (2 * h)
    for xi in (0.0, 0.7):
        S = LC.corotation(W[:, :, None], Qt(0)[:, :, None], xi)[:, :, 0]
        assert np.abs(S - dQdt).max() < 1e-9


def test_isotropic_flow_alignment():
    """Q = 0: S = 2 xi/3 (D - I tr D/3)."""
    r = np.random.default_rng(13)
    W = r.uniform(-1, 1, size=(3, 3, 4))
    D = 0.5 * (W + W.transpose(1, 0, 2))
    xi = 0.7
    S = LC.corotation(W, np.zeros((3, 3, 4)), xi)
    trD = D[0, 0] + D[1, 1] + D[2, 2]
    expect = 2 * xi / 3 * (D - np.eye(3)[:, :, None] * trD / 3)
    assert np.abs(S - expect).max() < 1e-15


def _rest_f(sh, u=None):
    u = np.zeros((3,) + sh) if u is None else u
    return R.f_equilibrium(np.ones(sh), u)


def _mode(field, axis, k_index):
    ax = (2, 1, 0)[axis]
    prof = field.mean(axis=tuple(a for a in range(3) if a != ax))
    return np.fft.fft(prof)[k_index]


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("comp", [0, 2, 4])
def test_linear_relaxation_factor(axis, comp):
    """Isotropic phase (gamma = 2), stored u = 0, small mode eps cos(k x_a) in one stored
    component: multiplied per step by 1 + Gamma (-A0 (1 - gamma/3) - kappa khat^2) up to
    O(eps) (the cubic and quartic terms); 20 steps with xi = 0 (no stress linear in Q, so
    the flow stays O(eps^2)): the factor to the 20th power."""
    p = LC.LcParams(gamma=2.0, A0=0.05, kappa=0.04, Gamma=0.8, xi=0.0)
    n = (16, 12, 10)[axis]
    sh = [4, 4, 4]
    sh[axis] = n
    nx, ny, nz = sh
    k = 2 * np.pi * 2 / n
    coord = np.indices((nz, ny, nx))[(2, 1, 0)[axis]]
    q5 = np.zeros((5, nz, ny, nx))
    q5[comp] = 1e-7 * np.cos(k * coord)
    f, u = _rest_f((nz, ny, nx)), np.zeros((3, nz, ny, nx))
    kh2 = 2 * (1 - math.cos(k))
    lam = 1 + p.Gamma * (-p.A0 * (1 - p.gamma / 3) - p.kappa * kh2)
    _, q1, _ = LC.step(f, q5, u, p)
    assert abs(_mode(q1[comp], axis, 2) / _mode(q5[comp], axis, 2) - lam) < 1e-8
    _, q20, _ = LC.run(f, q5, u, p, 20)
    assert abs(_mode(q20[comp], axis, 2) / _mode(q5[comp], axis, 2) / lam**20 - 1) < 1e-7
    others = [c for c in range(5) if c != comp]
    assert np.abs(q20[others]).max() < 1e-12


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("U", [0.07, -0.05])
def test_upwind_advection_factor(axis, U):
    """A0 = kappa = 0 (H = 0), uniform stored u = U e_a (W = 0, S = 0; f = f^eq(1, u) with
    F = 0 is a fixed point): every component's mode is multiplied by 1 - U (1 - e^{-ik})
    for U > 0 and 1 - U (e^{ik} - 1) for U < 0."""
    p = LC.LcParams(A0=0.0, kappa=0.0)
    n = (16, 12, 10)[axis]
    sh = [5, 4, 3]
    sh[axis] = n
    nx, ny, nz = sh
    u = np.zeros((3, nz, ny, nx))
    u[axis] = U
    f = _rest_f((nz, ny, nx), u)
    k = 2 * np.pi / n
    coord = np.indices((nz, ny, nx))[(2, 1, 0)[axis]]
    q5 = np.stack([0.1 * (c + 1) * np.cos(k * coord + c) for c in range(5)])
    f1, q1, u1 = LC.step(f, q5, u, p)
    lam = 1 - U * (1 - np.exp(-1j * k)) if U > 0 else 1 - U * (np.exp(1j * k) - 1)
    for c in range(5):
        assert abs(_mode(q1[c], axis, 1) / _mode(q5[c], axis, 1) - lam) < 1e-13
    assert np.abs(f1 - f).max() < 4e-16 and np.abs(u1 - u).max() < 1e-16


def test_free_energy_decreases_at_rate_gamma_h2():
    """Stored u = 0: one LC update is Q + Gamma H, so the discrete free energy changes by
    -Gamma sum H:H + O(Gamma^2)."""
    p = LC.LcParams(Gamma=1e-4, kappa=0.05, A0=0.1)
    r = np.random.default_rng(17)
    q5 = r.uniform(-0.3, 0.3, size=(5, 5, 4, 6))
    sh = q5.shape[1:]
    fl = LC.step_fields(_rest_f(sh), q5, np.zeros((3,) + sh), p)
    dE = _discrete_energy(fl.q_next, p) - _discrete_energy(q5, p)
    rate = -p.Gamma * (fl.H * fl.H).sum()
    assert dE < 0 and abs(dE / rate - 1) < 1e-3


@pytest.mark.parametrize("u0", [(0.0, 0.0, 0.0), (0.03, -0.02, 0.01)])
def test_uniform_nematic_is_fixed_point(u0):
    sh = (4, 5, 6)
    p = LC.LcParams()
    u = np.broadcast_to(np.array(u0)[:, None, None, None], (3,) + sh).copy()
    n = np.broadcast_to(np.array([0.36, -0.48, 0.8])[:, None, None, None], (3,) + sh)
    f, q5, uu = LC.initial_state(np.full(sh, 0.9), u, n, p)
    f1, q1, u1 = LC.run(f, q5, uu, p, 3)
    assert np.abs(f1 - f).max() < 1e-15
    assert np.abs(q1 - q5).max() < 1e-15
    assert np.abs(u1 - u).max() < 1e-15


def _rough(nx, ny, nz, seed):
    rho, u, q5, nf = synth.rough_lc_fields(nx, ny, nz, seed)
    return R.f_equilibrium(rho, u) + nf, q5, u


def test_conservation_of_mass_and_momentum():
    p = LC.LcParams()
    f, q5, u = _rough(8, 6, 5, 21)
    f1, _, _ = LC.run(f, q5, u, p, 3)
    assert abs(f1.sum() - f.sum()) < 1e-13 * f.sum()
    j0, j1 = R.momentum(f).sum(axis=(1, 2, 3)), R.momentum(f1).sum(axis=(1, 2, 3))
    assert np.abs(j1 - j0).max() < 1e-13


def test_shift_invariance_bitwise():
    p = LC.LcParams()
    f, q5, u = _rough(6, 5, 4, 22)
    out = LC.run(f, q5, u, p, 2)
    sh = lambda a: np.roll(a, (1, -2, 3), axis=(-3, -2, -1))  # noqa: E731
    out2 = LC.run(sh(f), sh(q5), sh(u), p, 2)
    for a, b in zip(out, out2):
        assert np.array_equal(sh(a), b)


def _transform(f, q5, u, M):
    """Apply the lattice map x -> M x (M a signed permutation) to a state on a cubic lattice."""
    n = f.shape[-1]
    z, y, x = np.indices((n, n, n))
    pos = np.stack([x, y, z])  # destination coordinates of each source site
    dst = np.einsum("ab,bzyx->azyx", M, pos) % n

    def scalar(a):
        out = np.empty_like(a)
        out[..., dst[2], dst[1], dst[0]] = a
        return out

    fo = np.empty_like(f)
    for i in range(19):
        ci = M @ R.C[i]
        j = int(np.where((R.C == ci).all(axis=1))[0][0])
        fo[j] = scalar(f[i])
    Q = LC.q_full(q5)
    Qr = np.einsum("ac,cdzyx,bd->abzyx", M, Q, M)
    qo = scalar(LC.q_five(Qr))
    uo = scalar(np.einsum("ab,bzyx->azyx", M, u))
    return fo, qo, uo


@pytest.mark.parametrize("name,M", [
    ("cyclic", np.array([[0, 0, 1], [1, 0, 0], [0, 1, 0]])),
    ("reflect_x", np.diag([-1, 1, 1])),
    ("swap_xy", np.array([[0, 1, 0], [1, 0, 0], [0, 0, 1]])),
])
def test_lattice_symmetry_covariance(name, M):
    """step(M s) = M step(s) for the cubic lattice symmetries (to rounding): catches
    transposed operands and wrong signs that a rotation-covariant formula cannot have."""
    p = LC.LcParams()
    f, q5, u = _rough(6, 6, 6, 23)
    a = _transform(*LC.run(f, q5, u, p, 2), M)
    b = LC.run(*_transform(f, q5, u, M), p, 2)
    for x, y in zip(a, b):
        assert np.abs(x - y).max() < 1e-14 * max(1.0, np.abs(x).max())


def test_site_sampler_equals_full_step():
    p = LC.LcParams()
    f, q5, u = _rough(10, 9, 11, 24)
    sites = synth.sample_sites(10, 9, 11, 12)
    f1, q1, u1 = LC.step(f, q5, u, p)
    fs, qs, us = LC.step_at_sites(f, q5, u, p, sites)
    for k, (x, y, z) in enumerate(sites):
        assert np.array_equal(fs[:, k], f1[:, z, y, x])
        assert np.array_equal(qs[:, k], q1[:, z, y, x])
        assert np.array_equal(us[:, k], u1[:, z, y, x])


def test_domain_error_names_the_site():
    p = LC.LcParams()
    f, q5, u = _rough(4, 4, 4, 25)
    q5[2, 3, 1, 2] = np.nan
    with pytest.raises(R.NumericalDomainError, match=r"x=2, y=1, z=3"):
        LC.step(f, q5, u, p)
