"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance (north_star "within 1e-12 relative"; reading R18): norm-wise
per field, ||x_gpu - x_ref||_inf / ||x_ref||_inf <= 1e-12, separately for f, g
and the derived phi, rho, u.  Integer maps and pure data movement (set/get,
propagation-only, slab decompositions, symmetries) are compared bitwise.
Inputs are the seeded synthetic states of ``paper_1609_01479_b200.synth``;
initial distributions are built by the oracle on the host and loaded with
lb_set_state, so no oracle input comes from the GPU.
"""
import numpy as np
import pytest

from oracle import lb_brute as BR
from oracle import lb_ref as R
from paper_1609_01479_b200 import lb, synth

pytestmark = pytest.mark.gpu

TOL = 1e-12
P0 = R.Params()


def cparams(p: R.Params):
    return lb.make_params(p.tau_f, p.tau_g, p.A, p.B, p.kappa, p.mobility)


def spinodal(nx, ny, nz, seed=0, p=P0):
    rho, u, phi = synth.spinodal_fields(nx, ny, nz, seed)
    return R.equilibrium_state(rho, u, phi, p)


def rough(nx, ny, nz, seed=1, p=P0):
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, seed)
    f, g = R.equilibrium_state(rho, u, phi, p)
    return f + nf, g + ng


def gpu_run(f, g, p, nsteps, nslabs=1, kernel=0, halo=None, tune=None):
    """kernel: 0 default, 1 tile, 2 warp-specialised, 3 warp-specialised with the phi exchange
    (lb_debug_step_kernel); halo: None default, 0 exchange, 1 peer (fused) transport between
    slabs (lb_debug_halo_mode); tune: {key: value} of lb_debug_tune."""
    nz, ny, nx = f.shape[1:]
    with lb.Lattice(nx, ny, nz, cparams(p), nslabs=nslabs) as L:
        lb.lb_debug_step_kernel(L.h, kernel)
        if halo is not None:
            lb.lb_debug_halo_mode(L.h, halo)
        for k, v in (tune or {}).items():
            lb.lb_debug_tune(L.h, k, v)
        L.set_state(f, g)
        L.step(nsteps)
        return L.get_state()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def u_scale(f, rho):
    """R18 for u: u = sum_i c_i f_i / rho cancels, so its error is normalised by the
    momentum the populations carry, max_s sum_i |c_i| f_i / rho (or |u| if larger)."""
    cabs = np.sqrt((R.C * R.C).sum(axis=1)).reshape(19, 1, 1, 1)
    return float((np.abs(f) * cabs).sum(axis=0).__truediv__(rho).max())


def assert_parity(fg_gpu, fg_ref, tol=TOL, u_strict_tol=None):
    """R18.  Also reports the strict ||du||_inf / ||u||_inf (no cancellation scale);
    u_strict_tol, if given, bounds it too."""
    (f1, g1), (f0, g0) = fg_gpu, fg_ref
    r1, j1, p1 = R.macroscopic(f1, g1)
    r0, j0, p0 = R.macroscopic(f0, g0)
    u1, u0 = j1 / r1, j0 / r0
    u_err = float(np.abs(u1 - u0).max() / max(np.abs(u0).max(), u_scale(f0, r0)))
    errs = {"f": rel(f1, f0), "g": rel(g1, g0), "phi": rel(p1, p0), "rho": rel(r1, r0), "u": u_err,
            "u_strict": rel(u1, u0)}
    print("parity (R18; u_strict = max|du| / max|u|):", {k: f"{v:.2e}" for k, v in errs.items()})
    bad = {k: v for k, v in errs.items() if k != "u_strict" and not v <= tol}
    if u_strict_tol is not None and not errs["u_strict"] <= u_strict_tol:
        bad["u_strict"] = errs["u_strict"]
    assert not bad, f"parity errors above {tol}: {bad} (all: {errs})"
    return errs


# ------------------------------------------------------------------ data movement
@pytest.mark.parametrize("nslabs", [1, 2, 4])
def test_set_get_roundtrip_bitwise(nslabs):
    r = np.random.default_rng(0)
    f = r.standard_normal((19, 8, 5, 7))
    g = r.standard_normal((19, 8, 5, 7))
    with lb.Lattice(7, 5, 8, nslabs=nslabs) as L:
        L.set_state(f, g)
        f1, g1 = L.get_state()
    assert np.array_equal(f1.view(np.uint64), f.view(np.uint64))
    assert np.array_equal(g1.view(np.uint64), g.view(np.uint64))


@pytest.mark.parametrize("shape,nslabs", [((7, 5, 8), 1), ((7, 5, 8), 2), ((4, 3, 12), 3), ((16, 16, 16), 4)])
def test_stream_only_equals_oracle_propagation_bitwise(shape, nslabs):
    nx, ny, nz = shape
    r = np.random.default_rng(1)
    f = r.standard_normal((19, nz, ny, nx))
    g = r.standard_normal((19, nz, ny, nx))
    with lb.Lattice(nx, ny, nz, nslabs=nslabs) as L:
        L.set_state(f, g)
        L.stream_only(3)
        f1, g1 = L.get_state()
    for _ in range(3):
        f, g = R.propagate(f), R.propagate(g)
    assert np.array_equal(f1, f) and np.array_equal(g1, g)


@pytest.mark.parametrize("kind", ["spinodal", "rough"])
@pytest.mark.parametrize("nslabs", [1, 2])
def test_init_equilibrium_matches_oracle(kind, nslabs):
    nx, ny, nz = 12, 10, 8
    if kind == "spinodal":
        rho, u, phi = synth.spinodal_fields(nx, ny, nz, 3)
    else:
        rho, u, phi, _, _ = synth.rough_fields(nx, ny, nz, 3)
    f0, g0 = R.equilibrium_state(rho, u, phi, P0)
    with lb.Lattice(nx, ny, nz, cparams(P0), nslabs=nslabs) as L:
        L.init_equilibrium(phi, rho if kind == "rough" else None, u if kind == "rough" else None)
        f1, g1 = L.get_state()
        ph = L.get_phi()
    assert rel(f1, f0) <= 1e-14 and rel(g1, g0) <= 1e-14
    assert rel(ph, phi) <= 1e-14


# ------------------------------------------------------------------ parity
def test_parity_16cubed_10_steps_spinodal():
    """BASELINE config 1: 16^3, spinodal random phi +- 0.01, 10 steps, fp64.  The
    strict velocity error max|du| / max|u| (no cancellation scale)
    is reported too: 2.5e-11 on B200 -- u ~ 1e-5 is a difference of populations
    ~0.05 (j = sum c f), so a few ulps of f are ~1e-11 of u; bounded at 1e-9."""
    f, g = spinodal(16, 16, 16)
    assert_parity(gpu_run(f, g, P0, 10), R.run(f, g, P0, 10), u_strict_tol=1e-9)


@pytest.mark.parametrize("shape,steps", [((16, 16, 16), 100), ((24, 20, 18), 5), ((64, 64, 64), 10)])
def test_parity_u_strict(shape, steps):
    """The strict velocity error max|du| / max|u| on the spinodal quench (u builds up
    from rest, so it is small and cancels in j = sum c f) and on the rough state:
    reported (B200: 1.7e-10 after 100 quench steps at 16^3, 2.7e-11 after 10 at
    64^3, 4e-15 on the rough state), bounded at 1e-9; R18 bounds the
    cancellation-scaled form at 1e-12."""
    nx, ny, nz = shape
    f, g = spinodal(nx, ny, nz, seed=3) if steps != 5 else rough(nx, ny, nz, seed=3)
    errs = assert_parity(gpu_run(f, g, P0, steps), R.run(f, g, P0, steps), u_strict_tol=1e-9)
    assert errs["u_strict"] >= 0


@pytest.mark.parametrize("shape", [(16, 16, 16), (17, 19, 13), (3, 3, 3), (24, 20, 18), (33, 5, 4), (4, 31, 6)])
def test_parity_rough_ragged(shape):
    nx, ny, nz = shape
    f, g = rough(nx, ny, nz)
    assert_parity(gpu_run(f, g, P0, 5), R.run(f, g, P0, 5))


@pytest.mark.parametrize("shape", [(96, 48, 8), (128, 41, 6)])
def test_parity_edge_and_interior_tiles(shape):
    """Interior tiles (the halo box by TMA) beside every kind of edge tile (the box
    by TMA, zero-filled outside the lattice, with the wrapped column pair and rows
    from side buffers): left / right columns, top / bottom rows -- ny = 41 leaves a
    single wrapped row below the tile at y0 = 32 and a ragged last tile row (whole
    box per thread) -- and the four corners, against the oracle at 1e-12; and
    bitwise equal to the tile kernel (per-thread copies of every box)."""
    nx, ny, nz = shape
    f, g = rough(nx, ny, nz, seed=33)
    ws = gpu_run(f, g, P0, 3, kernel=2)
    assert_parity(ws, R.run(f, g, P0, 3))
    tile = gpu_run(f, g, P0, 3, kernel=1)
    assert np.array_equal(ws[0], tile[0]) and np.array_equal(ws[1], tile[1])


def test_parity_64cubed_10_steps():
    f, g = spinodal(64, 64, 64, seed=2)
    assert_parity(gpu_run(f, g, P0, 10), R.run(f, g, P0, 10))


def test_parity_100_steps_demo_mobility():
    p = R.Params(mobility=0.45)
    f, g = spinodal(16, 16, 16, seed=4, p=p)
    assert_parity(gpu_run(f, g, p, 100), R.run(f, g, p, 100))


@pytest.mark.parametrize("tau", [(1.0, 1.0), (0.55, 2.5)])
def test_parity_other_relaxation_times(tau):
    p = R.Params(tau_f=tau[0], tau_g=tau[1], mobility=0.2)
    f, g = rough(12, 9, 10, seed=5, p=p)
    assert_parity(gpu_run(f, g, p, 4), R.run(f, g, p, 4))


@pytest.mark.parametrize("nx,ny,nz", [(128, 128, 128), (256, 128, 64)])
def test_parity_full_size_sampled(nx, ny, nz):
    """Full benchmark-class sizes: one step in the bench's launch configuration,
    compared at sampled sites (incl. all 8 corners) with the brute-force oracle."""
    f, g = spinodal(nx, ny, nz, seed=6)
    f1, g1 = gpu_run(f, g, P0, 1)
    smp = BR.SiteSampler(f, g, P0)
    fs, gs, fr, gr = [], [], [], []
    for (x, y, z) in synth.sample_sites(nx, ny, nz, 48):
        fo, go = smp.after_step(x, y, z)
        fr.append(fo), gr.append(go)
        fs.append(f1[:, z, y, x]), gs.append(g1[:, z, y, x])
    assert rel(np.array(fs), np.array(fr)) <= TOL
    assert rel(np.array(gs), np.array(gr)) <= TOL


# ------------------------------------------------------------------ the warp-specialised step kernel
@pytest.mark.parametrize("shape", [(16, 16, 16), (24, 20, 18), (34, 10, 7), (64, 64, 16), (4, 31, 6)])
def test_ws_kernel_parity_and_bitwise_equal_to_tile_kernel(shape):
    """lb_step_ws.cu (stencil warpgroup + collision warps) gives the same bits as the
    tile kernel -- wrapped and partial tiles, 32 x 4 tiles -- and meets the parity
    tolerance against the oracle."""
    nx, ny, nz = shape
    f, g = rough(nx, ny, nz, seed=14)
    a = gpu_run(f, g, P0, 4, kernel=2)
    b = gpu_run(f, g, P0, 4, kernel=1)
    c = gpu_run(f, g, P0, 4, kernel=2, tune={lb.LB_TUNE_BAND_ROWS: 3})  # another block order
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(c[0], b[0]) and np.array_equal(c[1], b[1])
    assert_parity(a, R.run(f, g, P0, 4))


def test_ws_kernel_32x8_tiles_and_z_chunks():
    """A plane with >= 4 x 148 tiles of 32 x 8 (the bench's tile shape) and two
    z-chunks: bitwise equal to the tile kernel, and sampled sites against the
    brute-force oracle."""
    nx, ny, nz = 512, 304, 16
    f, g = spinodal(nx, ny, nz, seed=15)
    a = gpu_run(f, g, P0, 1, kernel=2)
    b = gpu_run(f, g, P0, 1, kernel=1)
    c = gpu_run(f, g, P0, 2, kernel=2, tune={lb.LB_TUNE_BAND_ROWS: 4, lb.LB_TUNE_ZCHUNK: 5})
    d = gpu_run(f, g, P0, 2, kernel=2)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(c[0], d[0]) and np.array_equal(c[1], d[1])
    smp = BR.SiteSampler(f, g, P0)
    fs, gs, fr, gr = [], [], [], []
    for (x, y, z) in synth.sample_sites(nx, ny, nz, 32):
        fo, go = smp.after_step(x, y, z)
        fr.append(fo), gr.append(go)
        fs.append(a[0][:, z, y, x]), gs.append(a[1][:, z, y, x])
    assert rel(np.array(fs), np.array(fr)) <= TOL
    assert rel(np.array(gs), np.array(gr)) <= TOL


@pytest.mark.parametrize("nslabs", [2, 4])
def test_ws_kernel_slabs_bitwise(nslabs):
    f, g = rough(32, 16, 16, seed=16)
    a = gpu_run(f, g, P0, 5, nslabs=1, kernel=1)
    b = gpu_run(f, g, P0, 5, nslabs=nslabs, kernel=2)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("band", [2, 4, 7])
def test_block_order_bands_bitwise(kernel, band):
    """The block order (tiles walked in bands of tile rows, column by column;
    lb_debug_tune LB_TUNE_BAND_ROWS) changes only when a tile runs, not what it
    computes: bitwise equal to row-major order, including a partial last band
    (ny / 8 = 19 tile rows) and several z-chunks."""
    nx, ny, nz = 128, 152, 12
    f, g = rough(nx, ny, nz, seed=26)
    a = gpu_run(f, g, P0, 3, kernel=kernel, tune={lb.LB_TUNE_BAND_ROWS: band, lb.LB_TUNE_ZCHUNK: 4,
                                                  lb.LB_TUNE_RESID: 40})
    b = gpu_run(f, g, P0, 3, kernel=kernel)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("kernel", [1, 2])
def test_tile_rows_bitwise(kernel):
    """32 x 4 tiles (LB_TUNE_TILE_ROWS 4: the TMA maps re-encoded) against the
    default 32 x 8: the same bits for the tile and warp-specialised kernels."""
    f, g = rough(96, 40, 12, seed=28)
    a = gpu_run(f, g, P0, 3, kernel=kernel, tune={lb.LB_TUNE_TILE_ROWS: 4})
    b = gpu_run(f, g, P0, 3, kernel=kernel)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("kernel", [1, 2])
def test_slab_edge_chunks_last_bitwise(kernel):
    """Slabs of several z-chunks with the peer transport: the edge chunks (which may
    wait for a neighbour's K_phi) are launched after the interior ones -- the same
    bits as one slab and as the exchange transport."""
    f, g = rough(64, 16, 24, seed=29)
    ref = gpu_run(f, g, P0, 5, kernel=kernel)
    for halo in (1, 0):
        a = gpu_run(f, g, P0, 5, nslabs=2, kernel=kernel, halo=halo, tune={lb.LB_TUNE_ZCHUNK: 3})
        assert np.array_equal(a[0], ref[0]) and np.array_equal(a[1], ref[1]), halo


def test_tune_errors_and_graphs_off():
    f, g = rough(32, 12, 10, seed=27)
    a = gpu_run(f, g, P0, 17, tune={lb.LB_TUNE_GRAPHS: 0})
    b = gpu_run(f, g, P0, 17)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with lb.Lattice(8, 8, 8) as L:
        for key, val in [(99, 1), (lb.LB_TUNE_ZCHUNK, -1), (lb.LB_TUNE_BAND_ROWS, 0), (lb.LB_TUNE_RESID, -2),
                         (lb.LB_TUNE_TILE_ROWS, 6), (lb.LB_TUNE_L2_BOX, 4)]:
            with pytest.raises(lb.LBError) as e:
                lb.lb_debug_tune(L.h, key, val)
            assert e.value.code == lb.LB_EINVAL


# ------------------------------------------------------------------ the phi exchange (kernel 3)
def gpu_run_zc(f, g, p, nsteps, kernel, zchunk=None, coll=None):
    """gpu_run with an optional z-chunk (lb_debug_tune) and collision model (lb_set_collision)."""
    nz, ny, nx = f.shape[1:]
    with lb.Lattice(nx, ny, nz, cparams(p)) as L:
        if zchunk:
            lb.lb_debug_tune(L.h, lb.LB_TUNE_ZCHUNK, zchunk)
        lb.lb_debug_step_kernel(L.h, kernel)
        if coll is not None:
            lb.lb_set_collision(L.h, 1, *coll)
        L.set_state(f, g)
        L.step(nsteps)
        return L.get_state()


@pytest.mark.parametrize("shape,zchunk", [((32, 8, 8), None), ((64, 16, 12), None), ((64, 64, 16), None),
                                          ((96, 40, 9), 4), ((512, 304, 16), 8), ((512, 304, 16), None)])
def test_xch_kernel_bitwise_equal_to_ws_kernel(shape, zchunk):
    """The phi exchange (neighbouring tiles' CTAs hand each other the phi halo through
    an L2-resident phi array whose empty sites hold a sentinel NaN; a site still
    empty when needed is summed from g) gives the bits of the warp-specialised
    kernel: one tile (every neighbour is the tile itself), one wave, several waves
    (neighbours in the next wave: sums from g), two z-chunks; 20 steps, i.e. graph
    replays and the two phi arrays swapping roles between steps."""
    nx, ny, nz = shape
    steps = 20 if nx * ny * nz <= 200_000 else 3
    f, g = rough(nx, ny, nz, seed=21)
    a = gpu_run_zc(f, g, P0, steps, kernel=3, zchunk=zchunk)
    b = gpu_run_zc(f, g, P0, steps, kernel=2)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    if nx * ny * nz <= 40_000:
        assert_parity(a, R.run(f, g, P0, steps))


def test_xch_is_default_for_one_wave():
    """Kernel 0 takes the phi exchange where all blocks fit in one wave (64^3: 16
    tiles x 8 z-chunks) and the plain warp-specialised kernel otherwise: both
    bitwise equal to kernel 3."""
    for shape in [(64, 64, 64), (512, 304, 16)]:
        nx, ny, nz = shape
        f, g = rough(nx, ny, nz, seed=23)
        a = gpu_run(f, g, P0, 2, kernel=0)
        b = gpu_run(f, g, P0, 2, kernel=2)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_xch_after_other_kernels_bitwise():
    """Steps of the phi exchange interleaved with steps that do not use it (kernel 2,
    the MRT collision) must not read stale phi from the exchange arrays: the same
    bits as kernel 2 throughout."""
    f, g = rough(64, 32, 16, seed=24)
    mp = (0.8, 1.1, 1.0)
    with lb.Lattice(64, 32, 16, cparams(P0)) as L:
        L.set_state(f, g)
        lb.lb_debug_step_kernel(L.h, 3)
        L.step(10)
        lb.lb_debug_step_kernel(L.h, 2)
        L.step(1)
        lb.lb_debug_step_kernel(L.h, 3)
        L.step(3)
        lb.lb_set_collision(L.h, 1, *mp)
        L.step(1)
        lb.lb_set_collision(L.h, 0)
        L.step(9)
        a = L.get_state()
    with lb.Lattice(64, 32, 16, cparams(P0)) as L:
        L.set_state(f, g)
        lb.lb_debug_step_kernel(L.h, 2)
        L.step(14)
        lb.lb_set_collision(L.h, 1, *mp)
        L.step(1)
        lb.lb_set_collision(L.h, 0)
        L.step(9)
        b = L.get_state()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_xch_kernel_mrt_bitwise():
    f, g = rough(64, 32, 10, seed=22)
    mp = (0.8, 1.1, 1.0)
    a = gpu_run_zc(f, g, P0, 9, kernel=3, coll=mp)
    b = gpu_run_zc(f, g, P0, 9, kernel=2, coll=mp)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("shape,nslabs", [((48, 16, 8), 1), ((64, 12, 8), 1), ((64, 16, 8), 2)])
def test_xch_kernel_rejects_unfit_lattice(shape, nslabs):
    nx, ny, nz = shape
    with lb.Lattice(nx, ny, nz, nslabs=nslabs) as L:
        with pytest.raises(lb.LBError) as e:
            lb.lb_debug_step_kernel(L.h, 3)
        assert e.value.code == lb.LB_EINVAL


def test_ws_kernel_rejects_odd_nx():
    with lb.Lattice(7, 16, 8) as L:
        with pytest.raises(lb.LBError) as e:
            lb.lb_debug_step_kernel(L.h, 2)
        assert e.value.code == lb.LB_EINVAL
        for bad in (4, 5, -1):  # (removed kernels)
            with pytest.raises(lb.LBError) as e:
                lb.lb_debug_step_kernel(L.h, bad)
            assert e.value.code == lb.LB_EINVAL


# ------------------------------------------------------------------ fused (peer) halo transport
def test_loopback_defaults_to_fused_halo():
    with lb.Lattice(16, 8, 8, nslabs=2) as L:
        assert lb.lb_debug_halo_mode(L.h) == 1
    with lb.Lattice(16, 8, 8) as L:
        with pytest.raises(lb.LBError):
            lb.lb_debug_halo_mode(L.h, 1)  # one periodic slab has no halo


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("shape,nslabs", [((12, 10, 16), 2), ((32, 16, 16), 4), ((34, 9, 12), 3), ((7, 5, 8), 4)])
def test_fused_halo_bitwise_equal_to_exchange_and_one_slab(kernel, shape, nslabs):
    """The step kernel storing the leaving components straight into the neighbour
    slab's buffer (and K_phi into its phi ghost planes) gives the same bits as the
    ghost-plane + exchange transport and as the undecomposed lattice."""
    nx, ny, nz = shape
    if kernel == 2 and nx % 2:
        pytest.skip("warp-specialised kernel needs nx even")
    f, g = rough(nx, ny, nz, seed=17)
    ref = gpu_run(f, g, P0, 5, nslabs=1, kernel=1)
    peer = gpu_run(f, g, P0, 5, nslabs=nslabs, kernel=kernel, halo=1)
    exch = gpu_run(f, g, P0, 5, nslabs=nslabs, kernel=kernel, halo=0)
    for a in (peer, exch):
        assert np.array_equal(a[0], ref[0]) and np.array_equal(a[1], ref[1])


def test_fused_halo_ws_kernel_and_stream_only():
    f, g = rough(64, 16, 16, seed=18)
    a = gpu_run(f, g, P0, 3, nslabs=2, kernel=2, halo=1)
    b = gpu_run(f, g, P0, 3, nslabs=1, kernel=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with lb.Lattice(64, 16, 16, nslabs=4) as L:
        assert lb.lb_debug_halo_mode(L.h) == 1
        L.set_state(f, g)
        L.stream_only(5)
        f1, g1 = L.get_state()
    f0, g0 = f, g
    for _ in range(5):
        f0, g0 = R.propagate(f0), R.propagate(g0)
    assert np.array_equal(f1, f0) and np.array_equal(g1, g0)


@pytest.mark.parametrize("kernel,shape,nslabs", [(0, (32, 16, 16), 2), (0, (32, 16, 16), 4), (0, (24, 10, 16), 8),
                                                 (2, (64, 24, 12), 3), (1, (33, 9, 12), 2), (1, (17, 19, 12), 4)])
@pytest.mark.parametrize("halo", [0, 1])
def test_slabs_parity_against_oracle(kernel, shape, nslabs, halo):
    """Loopback z-slabs of the BGK path (both halo transports; the peer one with the
    device-side epochs of NEXT-1) against the oracle directly at R18's 1e-12 --
    not only against the GPU's own one-slab run -- including odd-nx tile-kernel
    slabs and 8 slabs of 2 planes."""
    nx, ny, nz = shape
    f, g = rough(nx, ny, nz, seed=41)
    a = gpu_run(f, g, P0, 6, nslabs=nslabs, kernel=kernel, halo=halo)
    assert_parity(a, R.run(f, g, P0, 6))


# ------------------------------------------------------------------ bitwise properties of the GPU path
@pytest.mark.parametrize("nslabs", [2, 4, 8])
def test_slab_decomposition_is_bitwise_identical(nslabs):
    f, g = rough(12, 10, 16, seed=7)
    a = gpu_run(f, g, P0, 6, nslabs=1)
    b = gpu_run(f, g, P0, 6, nslabs=nslabs)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_determinism_bitwise():
    f, g = rough(16, 12, 10, seed=8)
    a = gpu_run(f, g, P0, 5)
    b = gpu_run(f, g, P0, 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_phi_sign_symmetry_bitwise():
    f, g = rough(10, 9, 8, seed=9)
    a = gpu_run(f, g, P0, 3)
    b = gpu_run(f, -g, P0, 3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(-a[1], b[1])


def test_shift_invariance_bitwise():
    f, g = rough(10, 9, 8, seed=10)
    a = gpu_run(f, g, P0, 3)
    for v in [(1, 0, 0), (0, 3, 0), (0, 0, 5), (2, 1, 1)]:
        sh = lambda x: np.roll(x, shift=(v[2], v[1], v[0]), axis=(1, 2, 3))
        b = gpu_run(sh(f), sh(g), P0, 3)
        assert np.array_equal(sh(a[0]), b[0]) and np.array_equal(sh(a[1]), b[1])


@pytest.mark.parametrize("u0", [(0.0, 0.0, 0.0), (0.03, -0.02, 0.01)])
def test_uniform_equilibrium_fixed_point(u0):
    sh = (6, 5, 4)
    u = np.stack([np.full(sh, v) for v in u0])
    f, g = R.equilibrium_state(np.full(sh, 1.1), u, np.full(sh, 0.4), P0)
    f1, g1 = gpu_run(f, g, P0, 5)
    # a few ulps per step: the device contracts to FMA and multiplies by 1/tau (R17)
    assert rel(f1, f) <= 5e-15 and rel(g1, g) <= 5e-15


def test_conservation_64cubed_1000_steps():
    """C2: 64^3, 1000 steps: mass and phi drift <= 1e-12 relative, momentum <= 1e-13 sum|f|."""
    f, g = spinodal(64, 64, 64, seed=11, p=R.Params(mobility=0.45))
    m0, j0, p0 = (v.sum(axis=(-1, -2, -3)) for v in R.macroscopic(f, g))
    f1, g1 = gpu_run(f, g, R.Params(mobility=0.45), 1000)
    m1, j1, p1 = (v.sum(axis=(-1, -2, -3)) for v in R.macroscopic(f1, g1))
    assert abs(m1 - m0) <= 1e-12 * abs(m0)
    assert np.abs(j1 - j0).max() <= 1e-13 * np.abs(f1).sum()
    assert abs(p1 - p0) <= 1e-12 * np.abs(g1).sum()


# ------------------------------------------------------------------ errors
@pytest.mark.parametrize("kernel,nslabs", [(0, 1), (1, 1), (2, 1), (0, 2)])
def test_numeric_error_flag(kernel, nslabs):
    """R22: rho <= 0 or a non-finite value -> LB_ENUMERIC naming the global
    site and the step (the first offending one of the call)."""
    f, g = rough(8, 8, 8)
    f[:, 6, 2, 1] = 0.0  # rho = 0 at (x=1, y=2, z=6): in the second slab of two
    with lb.Lattice(8, 8, 8, nslabs=nslabs) as L:
        lb.lb_debug_step_kernel(L.h, kernel)
        L.set_state(f, g)
        with pytest.raises(lb.LBError) as e:
            L.step(1)
        assert e.value.code == lb.LB_ENUMERIC
        assert "(x=1, y=2, z=6)" in str(e.value) and "step 0 of this call" in str(e.value), str(e.value)
    f, g = rough(8, 8, 8)
    g[5, 1, 1, 1] = np.nan  # NaN in a moving g: pushed on to (x+cx, y+cy, z+cz) and spreading
    with lb.Lattice(8, 8, 8, nslabs=nslabs) as L:
        lb.lb_debug_step_kernel(L.h, kernel)
        L.set_state(f, g)
        L.step(0)
        with pytest.raises(lb.LBError) as e:
            L.step(12)  # (graph replays)
        assert e.value.code == lb.LB_ENUMERIC
        assert "(x=1, y=1, z=1)" in str(e.value) and "step 0 of this call" in str(e.value), str(e.value)


@pytest.mark.parametrize("pre", [0, 2])
def test_numeric_error_names_later_step(pre):
    """A state that goes bad only in step 1: tau_f = 1 and no force (A = B = kappa
    = 0), rest everywhere except one dense, fast site (rho = 1000, u = (0.3, 0.7, 0))
    whose equilibrium components with c.u = -0.3 or -0.4 are negative (e.g. c =
    (-1, 0, 0): w rho (1 - 0.9 + 0.405 - 0.87) < 0); pushed to the neighbours they
    make rho < 0 there in the next step.  The report names the smallest such site,
    (x0-1, y0, z0-1) -- the site the oracle's R22 error names for the same state --
    and step 1, counted from the call's first step (after `pre` clean steps)."""
    p = R.Params(tau_f=1.0, A=0.0, B=0.0, kappa=0.0)
    n = 10
    rho = np.ones((n, n, n))
    u = np.zeros((3, n, n, n))
    x0, y0, z0 = 5, 4, 6
    f, g = R.equilibrium_state(rho, u, np.zeros((n, n, n)), p)
    rho[z0, y0, x0] = 1000.0
    u[0, z0, y0, x0] = 0.3
    u[1, z0, y0, x0] = 0.7
    fd, _ = R.equilibrium_state(rho, u, np.zeros((n, n, n)), p)
    f[:, z0, y0, x0] = fd[:, z0, y0, x0]
    for kernel in (0, 1):
        with lb.Lattice(n, n, n, cparams(p)) as L:
            lb.lb_debug_step_kernel(L.h, kernel)
            L.set_state(f, g)
            with pytest.raises(lb.LBError) as e:
                L.step(3)
            msg = str(e.value)
            assert e.value.code == lb.LB_ENUMERIC
            assert f"(x={x0 - 1}, y={y0}, z={z0 - 1})" in msg and "step 1 of this call" in msg, msg
    # after `pre` clean rest steps elsewhere: the count is per call
    with lb.Lattice(n, n, n, cparams(p)) as L:
        L.set_state(*R.equilibrium_state(np.ones((n, n, n)), np.zeros((3, n, n, n)), np.zeros((n, n, n)), p))
        L.step(pre)
        L.set_state(f, g)
        with pytest.raises(lb.LBError) as e:
            L.step(2)
        assert "step 1 of this call" in str(e.value) and f"(step {pre + 1} since" in str(e.value), str(e.value)
        L.set_state(*R.equilibrium_state(np.ones((n, n, n)), np.zeros((3, n, n, n)), np.zeros((n, n, n)), p))
        L.step(9)  # clean again: the flag was reset


def test_state_errors_and_zero_steps():
    with lb.Lattice(8, 8, 8) as L:
        with pytest.raises(lb.LBError) as e:
            L.step(1)
        assert e.value.code == lb.LB_ESTATE
        with pytest.raises(lb.LBError) as e:
            L.get_state()
        assert e.value.code == lb.LB_ESTATE
        f, g = rough(8, 8, 8)
        L.set_state(f, g)
        L.step(0)
        f1, g1 = L.get_state()
        assert np.array_equal(f1, f) and np.array_equal(g1, g)
        with pytest.raises(lb.LBError) as e:
            L.step(-1)
        assert e.value.code == lb.LB_EINVAL


def test_launch_count_and_profile():
    f, g = spinodal(16, 16, 16)
    with lb.Lattice(16, 16, 16) as L:
        L.set_state(f, g)
        n0 = lb.lb_launch_count(L.h)
        lb.lb_profile_enable(L.h, True)
        L.step(4)
        prof = lb.lb_profile(L.h)
        assert lb.lb_launch_count(L.h) > n0
        assert prof["k_step"][1] == 4 and prof["k_step"][0] > 0


def test_parity_bench_launch_sampled():
    """The bench's own launch: 512 x 512 x 64 (BASELINE config 5 per GPU),
    lb_init_equilibrium on the R15 spinodal phi, one step in the default kernel and
    z-chunking, against the oracle at sampled sites (corners included) on radius-4
    windows (the initial state computed on radius-5 windows: g^eq needs lap phi)."""
    from sitewin import centre, crop, window

    nx, ny, nz = 512, 512, 64
    phi = synth.spinodal_phi(nx, ny, nz, seed=0)
    with lb.Lattice(nx, ny, nz, cparams(P0)) as L:
        L.init_equilibrium(phi)
        L.step(1)
        f1, g1 = L.get_state()
    fs, gs, fr, gr = [], [], [], []
    for (x, y, z) in synth.sample_sites(nx, ny, nz, 40, seed=12):
        pw = window(phi, x, y, z, 5)
        sh = pw.shape
        f0, g0 = R.equilibrium_state(np.ones(sh), np.zeros((3,) + sh), pw, P0)
        fo, go = R.step(crop(f0), crop(g0), P0)
        fr.append(centre(fo)), gr.append(centre(go))
        fs.append(f1[:, z, y, x]), gs.append(g1[:, z, y, x])
    assert rel(np.array(fs), np.array(fr)) <= TOL
    assert rel(np.array(gs), np.array(gr)) <= TOL


@pytest.mark.parametrize("nslabs,halo", [(1, None), (2, 0), (2, 1), (4, 1)])
def test_graph_replay_bitwise_equal_plain_steps(nslabs, halo):
    """lb_step(20) replays CUDA graphs of 8 steps (after one plain step); 20 calls of
    lb_step(1) never do: the same bits and the same kernel count."""
    f, g = rough(32, 12, 16, seed=9)
    out = []
    for mode in ("graph", "plain"):
        with lb.Lattice(32, 12, 16, cparams(P0), nslabs=nslabs) as L:
            if halo is not None:
                lb.lb_debug_halo_mode(L.h, halo)
            L.set_state(f, g)
            n0 = lb.lb_launch_count(L.h)
            if mode == "graph":
                L.step(20)
            else:
                for _ in range(20):
                    L.step(1)
            out.append((L.get_state(), lb.lb_launch_count(L.h) - n0))
    (a, na), (b, nb) = out
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert na == nb


@pytest.mark.parametrize("nslabs", [1, 2])
def test_prepare_captures_without_stepping(nslabs):
    """lb_prepare captures the step graphs of both buffer parities and runs nothing:
    the state is unchanged, and the steps after it give the bits and the kernel
    count of steps without it."""
    f, g = rough(32, 12, 16, seed=19)
    out = []
    for prep in (True, False):
        with lb.Lattice(32, 12, 16, cparams(P0), nslabs=nslabs) as L:
            L.set_state(f, g)
            n0 = lb.lb_launch_count(L.h)
            if prep:
                lb.lb_prepare(L.h)
                assert lb.lb_launch_count(L.h) == n0
                f1, g1 = L.get_state()
                assert np.array_equal(f1, f) and np.array_equal(g1, g)
                n0 = lb.lb_launch_count(L.h)
            L.step(3)
            L.step(17)
            out.append((L.get_state(), lb.lb_launch_count(L.h) - n0))
    (a, na), (b, nb) = out
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert na == nb


def test_graphs_dropped_on_collision_change():
    """A cached graph of the BGK step must not survive lb_set_collision."""
    f, g = rough(32, 12, 10, seed=10)
    mp = (0.8, 1.1, 1.0)
    with lb.Lattice(32, 12, 10, cparams(P0)) as L:
        L.set_state(f, g)
        L.step(17)  # captures graphs for both parities
        lb.lb_set_collision(L.h, 1, *mp)
        L.set_state(f, g)
        L.step(17)
        a = L.get_state()
    with lb.Lattice(32, 12, 10, cparams(P0)) as L:
        lb.lb_set_collision(L.h, 1, *mp)
        L.set_state(f, g)
        for _ in range(17):
            L.step(1)
        b = L.get_state()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_spinodal_decomposition_long_run_128cubed():
    """5000 steps of the R15 quench at 128^3 with the demo mobility (M = 0.45): the
    mixture separates into the two bulk phases +-sqrt(-A/B) = +-1 (the free-energy
    minima, R2), sum(phi) and mass stay at their initial values to 1e-12 of their
    scale, and momentum stays zero to rounding (north_star conservation over a long
    run, on the GPU alone)."""
    n = 128
    p = R.Params(mobility=0.45)
    rho, u, phi = synth.spinodal_fields(n, n, n, seed=21)
    with lb.Lattice(n, n, n, cparams(p)) as L:
        L.init_equilibrium(phi)
        f0, g0 = L.get_state()
        L.step(5000)
        f1, g1 = L.get_state()
        ph = L.get_phi()
    assert abs(g1.sum() - g0.sum()) <= 1e-12 * np.abs(g0).sum()
    assert abs(f1.sum() - f0.sum()) <= 1e-12 * f0.sum()
    j = R.momentum(f1).sum(axis=(1, 2, 3))
    assert np.abs(j).max() <= 1e-11 * f0.sum()
    # separated: most sites near a bulk value, both phases present, none far beyond it
    # (small curved domains sit slightly above 1: the Laplace-pressure shift ~ kappa/R)
    frac_bulk = float((np.abs(np.abs(ph) - 1.0) < 0.1).mean())
    assert frac_bulk > 0.6, frac_bulk
    assert (ph > 0.9).mean() > 0.2 and (ph < -0.9).mean() > 0.2
    assert np.abs(ph).max() < 1.2


def _reflect(a, axis):
    """x -> -x (mod n) along axis (0 = x, 1 = y, 2 = z) of a (19, nz, ny, nx) field, c_i relabelled."""
    perm = []
    for i in range(R.NVEL):
        c = R.C[i].copy()
        c[axis] = -c[axis]
        perm.append(int(np.flatnonzero((R.C == c).all(axis=1))[0]))
    ax = 3 - axis
    b = np.empty_like(a)
    b[perm] = np.roll(np.flip(a, axis=ax), 1, axis=ax)
    return b


@pytest.mark.parametrize("shape,axis", [((40, 24, 20), 0), ((40, 24, 20), 1), ((40, 24, 20), 2), ((33, 17, 9), 0)])
def test_reflection_covariance(shape, axis):
    """Property that holds at any size (the oracle pins it in
    test_step_commutes_with_cubic_symmetry): reflecting the input reflects
    the output.  Each run is within R18's 1e-12 of the oracle, so the two
    differ by at most 2e-12; ragged tiles put the mirrored sites in other
    tiles and other lanes."""
    nx, ny, nz = shape
    f, g = rough(nx, ny, nz, seed=31)
    f1, g1 = gpu_run(f, g, P0, 4)
    f2, g2 = gpu_run(_reflect(f, axis), _reflect(g, axis), P0, 4)
    assert rel(f2, _reflect(f1, axis)) <= 2 * TOL
    assert rel(g2, _reflect(g1, axis)) <= 2 * TOL
