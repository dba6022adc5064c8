"""C-ABI tests that need no GPU: the library loads, exports every symbol
include/lb.h declares, validates arguments before touching CUDA, and its
integer propagation / halo maps equal the oracle's np.roll map bitwise."""
import os
import re

import numpy as np
import pytest

from oracle import lb_ref as R
from paper_1609_01479_b200 import lb

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "lb.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lb_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lb._lib, n), n
        assert n in lb.EXPORTS, n


def test_version_and_bytes_per_site():
    assert "sm_100a" in lb.lb_version()
    assert lb.lb_bytes_per_site() == 608.0


@pytest.mark.parametrize(
    "kw,msg",
    [
        (dict(nx=2, ny=8, nz=8), "extents"),
        (dict(tau_f=0.5), "tau_f"),
        (dict(tau_g=float("nan")), "tau_g"),
        (dict(kappa=-1.0), "kappa"),
        (dict(mobility=-0.1), "mobility"),
        (dict(A=float("inf")), "finite"),
    ],
)
def test_create_rejects_bad_arguments(kw, msg):
    dims = {k: kw.pop(k) for k in ("nx", "ny", "nz") if k in kw}
    nx, ny, nz = dims.get("nx", 8), dims.get("ny", 8), dims.get("nz", 8)
    with pytest.raises(lb.LBError) as e:
        lb.lb_create(nx, ny, nz, lb.make_params(**kw))
    assert e.value.code == lb.LB_EINVAL and msg in str(e.value)


@pytest.mark.parametrize(
    "nx,kw,msg",
    [
        (15, {}, "nx even"),
        (16, dict(tau_f=0.5), "tau_f"),
        (16, dict(kappa=-0.1), "kappa"),
        (16, dict(Gamma=-1.0), "Gamma"),
        (16, dict(xi=float("nan")), "finite"),
        (16, dict(A0=float("inf")), "finite"),
    ],
)
def test_create_lc_rejects_bad_arguments(nx, kw, msg):
    """The liquid-crystal handle validates before touching CUDA (no GPU here)."""
    with pytest.raises(lb.LBError) as e:
        lb.lb_create_lc(nx, 8, 8, lb.make_lc_params(**kw))
    assert e.value.code == lb.LB_EINVAL and msg in str(e.value)


def test_loopback_rejects_bad_slab_counts():
    with pytest.raises(lb.LBError) as e:
        lb.lb_create_loopback(8, 8, 9, lb.make_params(), 2)
    assert e.value.code == lb.LB_EINVAL
    with pytest.raises(lb.LBError) as e:
        lb.lb_create_loopback(8, 8, 8, lb.make_params(), 8)  # 1 plane per slab
    assert e.value.code == lb.LB_EINVAL


def _oracle_pull_map(nx, ny, nz):
    """np.roll of the global site-index field: out[i, s] = source site of s (A.8)."""
    idx = np.arange(nx * ny * nz, dtype=np.int64).reshape(nz, ny, nx)
    return R.propagate(np.broadcast_to(idx, (19, nz, ny, nx)).astype(np.float64)).astype(np.int64)


@pytest.mark.parametrize("shape,nslabs", [((4, 5, 6), 1), ((4, 5, 6), 2), ((4, 5, 6), 3), ((3, 3, 3), 1),
                                          ((7, 3, 8), 4), ((5, 6, 4), 2)])
def test_propagation_map_equals_oracle_bitwise(shape, nslabs):
    nx, ny, nz = shape
    got = lb.lb_debug_propagation_map(nx, ny, nz, nslabs)
    assert np.array_equal(got, _oracle_pull_map(nx, ny, nz))


@pytest.mark.parametrize("shape,nslabs", [((4, 5, 6), 1), ((4, 5, 6), 2), ((4, 5, 6), 3), ((3, 3, 3), 1),
                                          ((7, 3, 8), 4), ((5, 6, 4), 2), ((6, 4, 16), 8)])
def test_fused_halo_map_equals_oracle_bitwise(shape, nslabs):
    """The fused (peer) halo: destinations from the kernels' own push_plane address
    arithmetic into the neighbouring slabs' buffers, never a ghost plane -- the same
    permutation as np.roll (A.8)."""
    nx, ny, nz = shape
    got = lb.lb_debug_propagation_map_peers(nx, ny, nz, nslabs)
    assert np.array_equal(got, _oracle_pull_map(nx, ny, nz))


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
def test_halo_plan_ring(nranks):
    for r in range(nranks):
        p = lb.lb_halo_plan(16, 12, 32, nranks, r)
        assert p["up"] == (r + 1) % nranks and p["down"] == (r - 1) % nranks
        assert p["dist_doubles"] == 10 * 16 * 12 and p["phi_doubles"] == 2 * 16 * 12
    with pytest.raises(lb.LBError):
        lb.lb_halo_plan(16, 12, 33, 2, 0)


def _brute_xch_pre(nx, ny, band):
    """Sites some band takes as phi halo from a later band, by the definition: walk
    every tile (32 x 8, row-major, band = tile // band) and its 2-site ring."""
    ntx = nx // 32
    owner = lambda x, y: ((y % ny) // 8 * ntx + (x % nx) // 32) // band  # noqa: E731
    need = set()
    for t in range(ntx * (ny // 8)):
        x0, y0, b = (t % ntx) * 32, (t // ntx) * 8, t // band
        for y in range(y0 - 2, y0 + 10):
            for x in range(x0 - 2, x0 + 34):
                if owner(x, y) > b:
                    need.add((y % ny) * nx + x % nx)
    return sorted(need)


@pytest.mark.parametrize("nx,ny,band", [(128, 48, 5), (128, 48, 1), (128, 48, 4), (96, 40, 7), (512, 64, 16),
                                        (64, 32, 3), (32, 16, 1)])
def test_xch_prepass_sites_brute_force(nx, ny, band):
    """The pre-pass of the banded phi exchange (host-built site list, lb_step_ws.cu
    ws_xch_pre_sites: the 4 corners of the 5 x 5 window) covers exactly the halo
    sites a band takes from later bands -- brute force over every tile's 2-ring,
    including the periodic wrap in x and y and bands that split tile rows."""
    b, sites = lb.lb_debug_xch_bands(nx, ny, 8, 8, 148, band)
    assert b == band
    assert sites.tolist() == _brute_xch_pre(nx, ny, band)


def test_xch_automatic_bands():
    """Automatic bands: none where tiles x z-chunks fit one wave, else equal bands of
    whole tile rows that fit 148 CTAs (512 x 512 x 64: 8 bands of 8 rows = 128)."""
    assert lb.lb_debug_xch_bands(128, 128, 128, 64, 148)[0] == 0
    assert lb.lb_debug_xch_bands(512, 512, 64, 32, 148)[0] == 128
    assert lb.lb_debug_xch_bands(512, 304, 16, 16, 148)[0] == 128
    assert lb.lb_debug_xch_bands(256, 256, 32, 32, 148)[0] == 128
    b, sites = lb.lb_debug_xch_bands(512, 512, 64, 32, 148)
    assert len(sites) == 8 * 2 * 512  # two rows below each band boundary, and above band 0
    with pytest.raises(lb.LBError):
        lb.lb_debug_xch_bands(100, 64, 8, 8, 148)
