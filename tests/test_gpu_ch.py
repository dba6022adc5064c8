"""GPU parity of the NEXT-2 variant (lb_create_ch: finite-difference Cahn-Hilliard
phi with upwind advection, f with the stress-in-equilibrium MRT collision;
readings R29-R33) against ``oracle/lb_ch.py`` at the tolerance of R18."""
import numpy as np
import pytest

from oracle import lb_ch as CH
from oracle import lb_ref as R
from paper_1609_01479_b200 import lb, synth

pytestmark = pytest.mark.gpu

TOL = 1e-12
CP = CH.ChParams(base=R.Params(mobility=0.2), tau_s=0.8, tau_b=1.1, tau_ghost=1.0)


def cparams(p: R.Params):
    return lb.make_params(p.tau_f, p.tau_g, p.A, p.B, p.kappa, p.mobility)


def rough(nx, ny, nz, seed=51):
    rho, u, phi, nf, _ = synth.rough_fields(nx, ny, nz, seed)
    return R.f_equilibrium(rho, u) + nf, phi


def spinodal(nx, ny, nz, seed=0):
    rho, u, phi = synth.spinodal_fields(nx, ny, nz, seed)
    return R.f_equilibrium(rho, u), phi


def gpu_run(f, phi, cp, nsteps):
    nz, ny, nx = f.shape[1:]
    with lb.ChLattice(nx, ny, nz, cparams(cp.base), cp.tau_s, cp.tau_b, cp.tau_ghost) as L:
        L.set_state(f, phi)
        L.step(nsteps)
        return L.get_state()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def assert_parity(got, ref, tol=TOL):
    (f1, p1), (f0, p0) = got, ref
    r1, j1 = R.density(f1), R.momentum(f1)
    r0, j0 = R.density(f0), R.momentum(f0)
    cabs = np.sqrt((R.C * R.C).sum(axis=1)).reshape(19, 1, 1, 1)
    uscale = max(float(np.abs(j0 / r0).max()), float(((np.abs(f0) * cabs).sum(axis=0) / r0).max()))
    errs = {"f": rel(f1, f0), "phi": rel(p1, p0), "rho": rel(r1, r0),
            "u": float(np.abs(j1 / r1 - j0 / r0).max() / uscale)}
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"parity errors above {tol}: {bad} (all: {errs})"


def test_ch_set_get_roundtrip_bitwise():
    f, phi = rough(16, 6, 5)
    with lb.ChLattice(16, 6, 5) as L:
        L.set_state(f, phi)
        f1, p1 = L.get_state()
        assert np.array_equal(L.get_phi(), phi)
    assert np.array_equal(f1, f) and np.array_equal(p1, phi)


def test_ch_parity_16cubed_10_steps_spinodal():
    f, phi = spinodal(16, 16, 16)
    assert_parity(gpu_run(f, phi, CP, 10), CH.run(f, phi, CP, 10))


@pytest.mark.parametrize("shape", [(16, 16, 16), (34, 10, 7), (64, 20, 9), (4, 31, 6), (96, 40, 5)])
def test_ch_parity_rough_ragged(shape):
    """Wrapped and partial tiles (per-thread copies), interior tiles (TMA), 32 x 4 tiles."""
    f, phi = rough(*shape)
    assert_parity(gpu_run(f, phi, CP, 5), CH.run(f, phi, CP, 5))


def test_ch_parity_64cubed_10_steps():
    f, phi = spinodal(64, 64, 64, seed=2)
    assert_parity(gpu_run(f, phi, CP, 10), CH.run(f, phi, CP, 10))


def test_ch_32x8_tiles_and_z_chunks_parity():
    """A plane with >= 4 x 148 tiles of 32 x 8 and two z-chunks (the bench's tile shape)."""
    f, phi = spinodal(512, 304, 16, seed=3)
    assert_parity(gpu_run(f, phi, CP, 1), CH.run(f, phi, CP, 1))


def test_ch_phi_sign_symmetry_and_shift_invariance_bitwise():
    f, phi = rough(32, 12, 10, seed=52)
    f1, p1 = gpu_run(f, phi, CP, 3)
    f2, p2 = gpu_run(f, -phi, CP, 3)
    assert np.array_equal(f1, f2) and np.array_equal(p1, -p2)
    sh = lambda a: np.roll(a, (2, -3, 6), axis=(-3, -2, -1))  # noqa: E731
    f3, p3 = gpu_run(sh(f), sh(phi), CP, 3)
    assert np.array_equal(f3, sh(f1)) and np.array_equal(p3, sh(p1))


def test_ch_conservation_64cubed_500_steps():
    f, phi = spinodal(64, 64, 64, seed=4)
    f1, p1 = gpu_run(f, phi, CP, 500)
    assert abs(p1.sum() - phi.sum()) <= 1e-12 * np.abs(phi).sum()
    assert abs(f1.sum() - f.sum()) <= 1e-12 * f.sum()
    j0, j1 = R.momentum(f).sum(axis=(1, 2, 3)), R.momentum(f1).sum(axis=(1, 2, 3))
    assert np.abs(j1 - j0).max() <= 1e-13 * np.abs(f).sum()


def test_ch_init_equilibrium_and_errors():
    rho, u, phi = synth.spinodal_fields(16, 8, 8, 5)
    with lb.ChLattice(16, 8, 8) as L:
        L.init_equilibrium(phi)
        f1, p1 = L.get_state()
        assert np.array_equal(p1, phi)
        assert rel(f1, R.f_equilibrium(np.ones_like(phi), np.zeros((3,) + phi.shape))) <= 1e-15
        for call in (lambda: lb.lb_get_state(L.h), lambda: lb.lb_set_collision(L.h, 1),
                     lambda: lb.lb_debug_step_kernel(L.h, 3)):
            with pytest.raises(lb.LBError) as e:
                call()
            assert e.value.code == lb.LB_EINVAL
    with pytest.raises(lb.LBError) as e:
        lb.ChLattice(15, 8, 8)  # nx odd
    assert e.value.code == lb.LB_EINVAL


def gpu_run_slabs(f, phi, cp, nsteps, nslabs):
    nz, ny, nx = f.shape[1:]
    with lb.ChLattice(nx, ny, nz, cparams(cp.base), cp.tau_s, cp.tau_b, cp.tau_ghost, nslabs=nslabs) as L:
        L.set_state(f, phi)
        f0, p0 = L.get_state()
        assert np.array_equal(f0, f) and np.array_equal(p0, phi)  # set/get through the slabs: bitwise
        L.step(nsteps)
        return L.get_state()


@pytest.mark.parametrize("nslabs", [2, 4, 8])
def test_ch_slabs_bitwise_equal_whole_lattice(nslabs):
    """z-slabs on one GPU (loopback: f edge planes and phi halos before the step, the
    leaving f components after it -- the exchanges the ranks do with NCCL) give the
    bits of the whole periodic lattice; 8 slabs = 2 planes each."""
    f, phi = rough(32, 12, 16, seed=53)
    f1, p1 = gpu_run(f, phi, CP, 3)
    f2, p2 = gpu_run_slabs(f, phi, CP, 3, nslabs)
    assert np.array_equal(f1, f2) and np.array_equal(p1, p2)


def test_ch_slabs_parity_64cubed():
    f, phi = spinodal(64, 64, 64, seed=6)
    assert_parity(gpu_run_slabs(f, phi, CP, 10, 2), CH.run(f, phi, CP, 10))


def test_ch_parity_bench_launch_sampled():
    """bench.py --collision ch: 512 x 512 x 64, lb_init_equilibrium (f = f^eq(1, 0),
    phi as given), one step, sampled sites against the oracle on radius-4 windows."""
    from sitewin import centre, window

    nx, ny, nz = 512, 512, 64
    phi = synth.spinodal_phi(nx, ny, nz, seed=0)
    with lb.ChLattice(nx, ny, nz, cparams(R.Params()), 0.8, 1.1, 1.0) as L:
        L.init_equilibrium(phi)
        L.step(1)
        f1, p1 = L.get_state()
    cp = CH.ChParams(base=R.Params(), tau_s=0.8, tau_b=1.1, tau_ghost=1.0)
    fs, ps, fr, pr = [], [], [], []
    for (x, y, z) in synth.sample_sites(nx, ny, nz, 40, seed=14):
        pw = window(phi, x, y, z, 4)
        sh = pw.shape
        fo, po = CH.step(R.f_equilibrium(np.ones(sh), np.zeros((3,) + sh)), pw, cp)
        fr.append(centre(fo)), pr.append(centre(po))
        fs.append(f1[:, z, y, x]), ps.append(p1[z, y, x])
    assert rel(np.array(fs), np.array(fr)) <= TOL
    assert rel(np.array(ps), np.array(pr)) <= TOL


@pytest.mark.parametrize("shape", [(64, 24, 12), (96, 40, 9)])
def test_ch_tile_rows_bitwise(shape):
    """32 x 4 tiles (two CTAs per SM) and 32 x 8 tiles (LB_TUNE_TILE_ROWS) give the
    same bits, and both meet the oracle."""
    nx, ny, nz = shape
    f, phi = rough(nx, ny, nz, seed=57)
    out = []
    for ty in (4, 8):
        with lb.ChLattice(nx, ny, nz, cparams(CP.base), CP.tau_s, CP.tau_b, CP.tau_ghost) as L:
            lb.lb_debug_tune(L.h, lb.LB_TUNE_TILE_ROWS, ty)
            L.set_state(f, phi)
            L.step(4)
            out.append(L.get_state())
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert_parity(out[0], CH.run(f, phi, CP, 4))


def _run_kernel(f, phi, nsteps, kernel, nslabs=1, zchunk=None, variant=0):
    nz, ny, nx = f.shape[1:]
    with lb.ChLattice(nx, ny, nz, cparams(CP.base), CP.tau_s, CP.tau_b, CP.tau_ghost, nslabs=nslabs) as L:
        lb.lb_debug_step_kernel(L.h, kernel)
        lb.lb_debug_tune(L.h, lb.LB_TUNE_VARIANT, variant)
        if zchunk:
            lb.lb_debug_tune(L.h, lb.LB_TUNE_ZCHUNK, zchunk)
        L.set_state(f, phi)
        L.step(nsteps)
        return L.get_state()


@pytest.mark.parametrize("shape,nslabs,zchunk", [((16, 16, 16), 1, None), ((34, 10, 7), 1, None),
                                                 ((64, 24, 12), 1, 1), ((64, 24, 12), 1, 2), ((96, 40, 9), 1, 4),
                                                 ((64, 16, 16), 2, None), ((32, 16, 12), 3, None),
                                                 ((512, 304, 8), 1, None)])
def test_ch_ws_kernel_bitwise_equal_tile_kernel(shape, nslabs, zchunk):
    """The warp-specialised Cahn-Hilliard kernel (collision warps: f box, P, MRT,
    push and every copy; stencil warps: u, mu and the phi update) gives the bits of
    the tile kernel k_step_ch: one tile, ragged and wrapped tiles, z-chunks of 1, 2
    and 4 planes, loopback slabs, several waves; and meets the oracle."""
    nx, ny, nz = shape
    f, phi = rough(nx, ny, nz, seed=58)
    steps = 3 if nx * ny * nz > 100_000 else 5
    a = _run_kernel(f, phi, steps, 2, nslabs, zchunk)
    b = _run_kernel(f, phi, steps, 1, nslabs, zchunk)
    c = _run_kernel(f, phi, steps, 2, nslabs, zchunk, variant=1)  # 5-plane phi ring
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(c[0], b[0]) and np.array_equal(c[1], b[1])
    if nx * ny * nz <= 40_000:
        assert_parity(a, CH.run(f, phi, CP, steps))
