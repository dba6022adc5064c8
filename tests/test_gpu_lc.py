"""GPU parity of the NEXT-4 liquid-crystal workload (lb_create_lc: Landau-de Gennes
Q tensor, Beris-Edwards LC update with upwind advection, chemical stress driving the
Guo-forced LB fluid; readings R34-R45) against ``oracle/lb_lc.py`` at the
tolerance of R18 (norm-wise 1e-12 per field)."""
import numpy as np
import pytest

from oracle import lb_lc as LC
from oracle import lb_ref as R
from paper_1609_01479_b200 import lb, synth

pytestmark = pytest.mark.gpu

TOL = 1e-12
LP = LC.LcParams()
# a second parameter set with every term large: isotropic-side gamma, strong elasticity
LP2 = LC.LcParams(tau_f=0.9, A0=0.2, gamma=2.6, kappa=0.05, xi=-0.4, Gamma=0.5)


def cparams(p: LC.LcParams):
    return lb.make_lc_params(p.tau_f, p.A0, p.gamma, p.kappa, p.xi, p.Gamma)


def rough(nx, ny, nz, seed=61):
    rho, u, q5, nf = synth.rough_lc_fields(nx, ny, nz, seed)
    return R.f_equilibrium(rho, u) + nf, q5, u


def quench(nx, ny, nz, seed=0, p=LP):
    """R45: rest fluid, Q = S0 (n n - I/3) from random directors."""
    n = synth.random_directors(nx, ny, nz, seed)
    return LC.initial_state(np.ones((nz, ny, nx)), np.zeros((3, nz, ny, nx)), n, p)


def gpu_run(state, p, nsteps):
    f = state[0]
    nz, ny, nx = f.shape[1:]
    with lb.LcLattice(nx, ny, nz, cparams(p)) as L:
        L.set_state(*state)
        L.step(nsteps)
        return L.get_state()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def assert_parity(got, ref, tol=TOL):
    (f1, q1, u1), (f0, q0, u0) = got, ref
    r0 = R.density(f0)
    cabs = np.sqrt((R.C * R.C).sum(axis=1)).reshape(19, 1, 1, 1)
    uscale = max(float(np.abs(u0).max()), float(((np.abs(f0) * cabs).sum(axis=0) / r0).max()))
    errs = {"f": rel(f1, f0), "Q": rel(q1, q0), "rho": rel(R.density(f1), r0),
            "u": float(np.abs(u1 - u0).max() / uscale)}
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"parity errors above {tol}: {bad} (all: {errs})"


def test_lc_set_get_roundtrip_bitwise():
    st = rough(16, 6, 5)
    with lb.LcLattice(16, 6, 5) as L:
        L.set_state(*st)
        got = L.get_state()
    for a, b in zip(got, st):
        assert np.array_equal(a, b)


def test_lc_init_matches_the_oracle_recipe():
    nx, ny, nz = 16, 8, 6
    r = np.random.default_rng(4)
    rho = 1.0 + 0.05 * r.random((nz, ny, nx))
    u = r.uniform(-0.02, 0.02, size=(3, nz, ny, nx))
    n = synth.random_directors(nx, ny, nz, 7)
    ref = LC.initial_state(rho, u, n, LP)
    with lb.LcLattice(nx, ny, nz, cparams(LP)) as L:
        L.init(n, rho, u)
        got = L.get_state()
    for a, b in zip(got, ref):
        assert rel(a, b) <= 1e-15


def test_lc_parity_16cubed_10_steps_quench():
    st = quench(16, 16, 16)
    assert_parity(gpu_run(st, LP, 10), LC.run(*st, LP, 10))


@pytest.mark.parametrize("shape", [(16, 16, 16), (34, 10, 7), (64, 20, 9), (4, 31, 6), (96, 40, 5)])
@pytest.mark.parametrize("p", [LP, LP2], ids=["default", "strong"])
def test_lc_parity_rough_ragged(shape, p):
    """Partial and wrapped tiles (nx < 32, ragged x and y), several tiles, short z."""
    st = rough(*shape)
    assert_parity(gpu_run(st, p, 4), LC.run(*st, p, 4))


def test_lc_parity_64cubed_10_steps():
    st = quench(64, 64, 64, seed=2)
    assert_parity(gpu_run(st, LP, 10), LC.run(*st, LP, 10))


def test_lc_z_chunks_parity():
    """128 x 64 x 40: 32 tiles, two z-chunks of 20 planes (lc_zchunk)."""
    st = quench(128, 64, 40, seed=3)
    assert_parity(gpu_run(st, LP, 2), LC.run(*st, LP, 2))


def test_lc_parity_bench_size_sampled():
    """The bench launch (512 x 512 x 64, lb_init_lc, one step) against the oracle on
    radius-4 windows around sampled sites (corners included)."""
    nx, ny, nz = 512, 512, 64
    n = synth.random_directors(nx, ny, nz, 0)
    with lb.LcLattice(nx, ny, nz, cparams(LP)) as L:
        L.init(n)
        L.step(1)
        f1, q1, u1 = L.get_state()
    sites = synth.sample_sites(nx, ny, nz, 40, seed=11)
    S0 = LC.uniaxial_order(LP.gamma)
    for (x, y, z) in sites:
        nw = LC._window(n, x, y, z, 4)
        sh = nw.shape[1:]
        f0, q0, u0 = LC.step(R.f_equilibrium(np.ones(sh), np.zeros((3,) + sh)), LC.nematic_q(nw, S0),
                             np.zeros((3,) + sh), LP)
        c = (slice(None), 4, 4, 4)
        assert rel(f1[:, z, y, x], f0[c]) <= TOL
        assert rel(q1[:, z, y, x], q0[c]) <= TOL
        assert np.abs(u1[:, z, y, x] - u0[c]).max() <= TOL


@pytest.mark.parametrize("u0", [(0.0, 0.0, 0.0), (0.03, -0.02, 0.01)])
def test_lc_uniform_nematic_fixed_point(u0):
    sh = (6, 5, 8)
    u = np.broadcast_to(np.array(u0)[:, None, None, None], (3,) + sh).copy()
    n = np.broadcast_to(np.array([0.36, -0.48, 0.8])[:, None, None, None], (3,) + sh)
    st = LC.initial_state(np.full(sh, 0.9), u, n, LP)
    got = gpu_run(st, LP, 5)
    for a, b in zip(got, st):
        assert np.abs(a - b).max() <= 5e-15


def test_lc_shift_invariance_bitwise():
    st = rough(32, 12, 10, seed=62)
    a = gpu_run(st, LP, 3)
    sh = lambda v: np.roll(v, (2, -3, 6), axis=(-3, -2, -1))  # noqa: E731
    b = gpu_run(tuple(sh(v) for v in st), LP, 3)
    for x, y in zip(a, b):
        assert np.array_equal(sh(x), y)


def test_lc_conservation_64cubed_200_steps():
    st = quench(64, 64, 64, seed=4)
    f = st[0]
    f1, _, _ = gpu_run(st, LP, 200)
    assert abs(f1.sum() - f.sum()) <= 1e-12 * f.sum()
    j0, j1 = R.momentum(f).sum(axis=(1, 2, 3)), R.momentum(f1).sum(axis=(1, 2, 3))
    assert np.abs(j1 - j0).max() <= 1e-13 * np.abs(f).sum()


def test_lc_errors():
    with lb.LcLattice(16, 8, 8) as L:
        for call in (lambda: lb.lb_step(L.h, 1),  # no state yet
                     ):
            with pytest.raises(lb.LBError) as e:
                call()
            assert e.value.code == lb.LB_ESTATE
        L.set_state(*rough(16, 8, 8))
        for call in (lambda: lb.lb_get_state(L.h), lambda: lb.lb_get_phi(L.h), lambda: lb.lb_set_collision(L.h, 1),
                     lambda: lb.lb_debug_step_kernel(L.h, 2),
                     lambda: lb.lb_init_equilibrium(L.h, None, None, np.zeros(16 * 8 * 8))):
            with pytest.raises(lb.LBError) as e:
                call()
            assert e.value.code == lb.LB_EINVAL
    with lb.LcLattice(16, 8, 8, lb.make_lc_params(gamma=2.5)) as L:
        with pytest.raises(lb.LBError) as e:
            L.init(synth.random_directors(16, 8, 8))
        assert e.value.code == lb.LB_EINVAL
    st = rough(16, 8, 8)
    st[1][0, 3, 2, 1] = np.nan
    with lb.LcLattice(16, 8, 8) as L:
        L.set_state(*st)
        with pytest.raises(lb.LBError) as e:
            L.step(2)
        assert e.value.code == lb.LB_ENUMERIC


def gpu_run_slabs(state, p, nsteps, nslabs):
    f = state[0]
    nz, ny, nx = f.shape[1:]
    with lb.LcLattice(nx, ny, nz, cparams(p), nslabs=nslabs) as L:
        L.set_state(*state)
        got = L.get_state()
        for a, b in zip(got, state):  # set/get through the slabs: bitwise
            assert np.array_equal(a, b)
        L.step(nsteps)
        return L.get_state()


@pytest.mark.parametrize("nslabs", [2, 4, 8])
@pytest.mark.parametrize("p", [LP, LP2], ids=["default", "strong"])
def test_lc_slabs_bitwise_equal_whole_lattice(nslabs, p):
    """z-slabs on one GPU (loopback: the ghost-plane exchanges of Q, u and f that the
    ranks do with NCCL) give the bits of the whole periodic lattice; 8 slabs = 2 planes
    each, so the Q halo is a whole slab."""
    st = rough(32, 12, 16, seed=63)
    a = gpu_run(st, p, 3)
    b = gpu_run_slabs(st, p, 3, nslabs)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_lc_slabs_parity_64cubed():
    st = quench(64, 64, 64, seed=5)
    assert_parity(gpu_run_slabs(st, LP, 10, 2), LC.run(*st, LP, 10))


def test_lc_quench_long_run_stable_and_conserving():
    """2000 steps of the R45 random-director quench at 64^3: the state stays finite,
    Q stays in the physical range (|Q_ab| < 2/3), mass and momentum are conserved to
    rounding, and the order relaxes (the mean Q:Q falls from 2 S0^2/3 as the random
    texture anneals)."""
    n = 64
    st = quench(n, n, n, seed=8)
    f0, q0 = st[0], st[1]
    f1, q1, u1 = gpu_run(st, LP, 2000)
    assert np.isfinite(f1).all() and np.isfinite(q1).all() and np.isfinite(u1).all()
    assert np.abs(q1).max() < 2.0 / 3.0
    assert abs(f1.sum() - f0.sum()) <= 1e-12 * f0.sum()
    j0, j1 = R.momentum(f0).sum(axis=(1, 2, 3)), R.momentum(f1).sum(axis=(1, 2, 3))
    assert np.abs(j1 - j0).max() <= 1e-12 * f0.sum()
    Q0, Q1 = LC.q_full(q0), LC.q_full(q1)
    assert (Q1 * Q1).sum(axis=(0, 1)).mean() < (Q0 * Q0).sum(axis=(0, 1)).mean()
