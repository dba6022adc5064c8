"""GPU parity of the NEXT-3 collision variant (lb_set_collision model 1: chemical
stress in f's equilibrium, three-rate MRT; readings R23-R27) against
``oracle/lb_mrt.py``, with the tolerance of R18, plus the bitwise properties the
main path has (kernels, slab decompositions, symmetries)."""
import numpy as np
import pytest

from oracle import lb_mrt as M
from oracle import lb_ref as R
from paper_1609_01479_b200 import lb, synth

pytestmark = pytest.mark.gpu

TOL = 1e-12
P0 = R.Params()
MP = M.MrtParams(base=P0, tau_s=0.8, tau_b=1.1, tau_ghost=1.0)


def cparams(p: R.Params):
    return lb.make_params(p.tau_f, p.tau_g, p.A, p.B, p.kappa, p.mobility)


def rough(nx, ny, nz, seed=31, p=P0):
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, seed)
    f, g = R.equilibrium_state(rho, u, phi, p)
    return f + nf, g + ng


def spinodal(nx, ny, nz, seed=0, p=P0):
    rho, u, phi = synth.spinodal_fields(nx, ny, nz, seed)
    return R.equilibrium_state(rho, u, phi, p)


def gpu_run(f, g, mp, nsteps, nslabs=1, kernel=0, halo=None):
    nz, ny, nx = f.shape[1:]
    with lb.Lattice(nx, ny, nz, cparams(mp.base), nslabs=nslabs) as L:
        lb.lb_debug_step_kernel(L.h, kernel)
        lb.lb_set_collision(L.h, 1, mp.tau_s, mp.tau_b, mp.tau_ghost)
        if halo is not None:
            lb.lb_debug_halo_mode(L.h, halo)
        L.set_state(f, g)
        L.step(nsteps)
        return L.get_state()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def assert_parity(got, ref, tol=TOL):
    (f1, g1), (f0, g0) = got, ref
    r1, j1, p1 = R.macroscopic(f1, g1)
    r0, j0, p0 = R.macroscopic(f0, g0)
    cabs = np.sqrt((R.C * R.C).sum(axis=1)).reshape(19, 1, 1, 1)
    uscale = max(float(np.abs(j0 / r0).max()), float(((np.abs(f0) * cabs).sum(axis=0) / r0).max()))
    errs = {"f": rel(f1, f0), "g": rel(g1, g0), "phi": rel(p1, p0), "rho": rel(r1, r0),
            "u": float(np.abs(j1 / r1 - j0 / r0).max() / uscale)}
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"parity errors above {tol}: {bad} (all: {errs})"


def test_mrt_parity_16cubed_10_steps_spinodal():
    f, g = spinodal(16, 16, 16)
    assert_parity(gpu_run(f, g, MP, 10), M.run(f, g, MP, 10))


@pytest.mark.parametrize("shape", [(16, 16, 16), (17, 19, 13), (24, 20, 18), (33, 5, 4), (4, 31, 6), (3, 3, 3)])
def test_mrt_parity_rough_ragged(shape):
    f, g = rough(*shape)
    assert_parity(gpu_run(f, g, MP, 5), M.run(f, g, MP, 5))


@pytest.mark.parametrize("taus", [(0.6, 0.6, 0.6), (0.7, 1.8, 1.3), (1.5, 0.9, 0.55)])
def test_mrt_parity_relaxation_times(taus):
    mp = M.MrtParams(base=R.Params(mobility=0.2), tau_s=taus[0], tau_b=taus[1], tau_ghost=taus[2])
    f, g = rough(12, 10, 9, seed=32, p=mp.base)
    assert_parity(gpu_run(f, g, mp, 4), M.run(f, g, mp, 4))


def test_mrt_parity_64cubed_10_steps():
    f, g = spinodal(64, 64, 64, seed=2)
    assert_parity(gpu_run(f, g, MP, 10), M.run(f, g, MP, 10))


@pytest.mark.parametrize("shape", [(16, 16, 16), (34, 10, 7), (64, 64, 16)])
def test_mrt_kernels_bitwise_equal(shape):
    """Tile and warp-specialised kernels share collide_mrt: same bits."""
    f, g = rough(*shape, seed=33)
    a = gpu_run(f, g, MP, 3, kernel=1)
    for k in (2,):
        b = gpu_run(f, g, MP, 3, kernel=k)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_mrt_32x8_tiles_bitwise_and_parity():
    """The bench's 32 x 8 tile shape (plane with >= 4 x 148 tiles), two z-chunks."""
    f, g = spinodal(512, 304, 16, seed=34)
    a = gpu_run(f, g, MP, 1, kernel=2)
    b = gpu_run(f, g, MP, 1, kernel=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("nslabs,halo", [(2, 1), (2, 0), (4, 1), (4, 0)])
def test_mrt_slabs_bitwise(nslabs, halo):
    f, g = rough(32, 16, 16, seed=35)
    a = gpu_run(f, g, MP, 4, nslabs=1, kernel=1)
    b = gpu_run(f, g, MP, 4, nslabs=nslabs, kernel=2, halo=halo)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_mrt_phi_sign_symmetry_and_shift_invariance_bitwise():
    f, g = rough(16, 12, 10, seed=36)
    f1, g1 = gpu_run(f, g, MP, 3)
    f2, g2 = gpu_run(f, -g, MP, 3)
    assert np.array_equal(f1, f2) and np.array_equal(g1, -g2)
    sh = lambda a: np.roll(a, (2, -3, 5), axis=(1, 2, 3))  # noqa: E731
    f3, g3 = gpu_run(sh(f), sh(g), MP, 3)
    assert np.array_equal(f3, sh(f1)) and np.array_equal(g3, sh(g1))


def test_mrt_conservation_64cubed_500_steps():
    """No force: mass, phi and momentum are conserved to rounding over 500 steps."""
    f, g = spinodal(64, 64, 64, seed=37)
    f1, g1 = gpu_run(f, g, MP, 500)
    assert abs(f1.sum() - f.sum()) <= 1e-12 * f.sum()
    assert abs(g1.sum() - g.sum()) <= 1e-12 * np.abs(g).sum()
    j0, j1 = R.momentum(f).sum(axis=(1, 2, 3)), R.momentum(f1).sum(axis=(1, 2, 3))
    assert np.abs(j1 - j0).max() <= 1e-13 * np.abs(f).sum()


def test_mrt_set_collision_errors_and_model_switch():
    with lb.Lattice(16, 8, 8) as L:
        for bad in ((1, 0.5, 1.0, 1.0), (1, 0.8, float("nan"), 1.0), (2, 0.8, 1.0, 1.0)):
            with pytest.raises(lb.LBError) as e:
                lb.lb_set_collision(L.h, *bad)
            assert e.value.code == lb.LB_EINVAL
    f, g = rough(16, 8, 8, seed=38)
    with lb.Lattice(16, 8, 8, cparams(P0)) as L:  # model 1, then back to model 0 = the main path
        L.set_state(f, g)
        lb.lb_set_collision(L.h, 1, 0.8, 1.1, 1.0)
        lb.lb_set_collision(L.h, 0)
        L.step(2)
        f1, g1 = L.get_state()
    f0, g0 = R.run(f, g, P0, 2)
    assert rel(f1, f0) <= TOL and rel(g1, g0) <= TOL


def test_mrt_parity_bench_launch_sampled():
    """bench.py --collision mrt: 512 x 512 x 64, lb_init_equilibrium on the spinodal
    phi, one step, sampled sites against the oracle on windows."""
    from sitewin import centre, crop, window

    nx, ny, nz = 512, 512, 64
    phi = synth.spinodal_phi(nx, ny, nz, seed=0)
    with lb.Lattice(nx, ny, nz, cparams(P0)) as L:
        lb.lb_set_collision(L.h, 1, MP.tau_s, MP.tau_b, MP.tau_ghost)
        L.init_equilibrium(phi)
        L.step(1)
        f1, g1 = L.get_state()
    fs, gs, fr, gr = [], [], [], []
    for (x, y, z) in synth.sample_sites(nx, ny, nz, 40, seed=13):
        pw = window(phi, x, y, z, 5)
        sh = pw.shape
        f0, g0 = R.equilibrium_state(np.ones(sh), np.zeros((3,) + sh), pw, P0)
        fo, go = M.step(crop(f0), crop(g0), MP)
        fr.append(centre(fo)), gr.append(centre(go))
        fs.append(f1[:, z, y, x]), gs.append(g1[:, z, y, x])
    assert rel(np.array(fs), np.array(fr)) <= TOL
    assert rel(np.array(gs), np.array(gr)) <= TOL
