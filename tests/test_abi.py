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




@pytest.mark.parametrize("ntx,nty,nch,resid,band", [(16, 64, 2, 148, 1), (16, 64, 2, 148, 4), (16, 19, 3, 40, 4),
                                                    (5, 7, 1, 148, 3), (16, 64, 2, 148, 64), (3, 2, 4, 1, 2)])
def test_tile_order_is_a_permutation(ntx, nty, nch, resid, band):
    """lb_debug_tile_order (the kernels' tile_of_block): every (tile, z-chunk) once;
    chunk c of a tile after chunk c-1; with bands, consecutive blocks of a band
    walk its rows column by column (y neighbours adjacent in launch order)."""
    o = lb.lb_debug_tile_order(ntx, nty, nch, resid, band)
    keys = {tuple(r) for r in o.tolist()}
    assert len(keys) == ntx * nty * nch == len(o)
    assert all(0 <= bx < ntx and 0 <= by < nty and 0 <= bz < nch for bx, by, bz in keys)
    pos = {tuple(r): i for i, r in enumerate(o.tolist())}
    for (bx, by, bz), i in pos.items():
        if bz > 0:
            assert pos[(bx, by, bz - 1)] < i
    if band > 1 and nty % band == 0 and resid >= ntx * nty:
        # first group, chunk 0: rows of a band interleave
        assert o[0].tolist() == [0, 0, 0] and o[1].tolist() == [0, 1, 0]
        assert o[band].tolist() == [1, 0, 0]
    if band == 1 and resid >= ntx:
        assert o[1].tolist() == [1 % ntx, 1 // ntx, 0]


@pytest.mark.parametrize("ntx,nty,nch,resid", [(16, 64, 4, 148), (8, 8, 3, 64), (5, 7, 2, 148), (3, 2, 5, 4)])
def test_tile_order_edge_chunks_last(ntx, nty, nch, resid):
    """A z-slab with the peer transport (band < 0): the same permutation with the
    chunks that read a neighbour's phi planes (0 and nch-1) after the interior
    chunks of every group, so the CTAs that may wait come last."""
    o = lb.lb_debug_tile_order(ntx, nty, nch, resid, -1)
    ref = lb.lb_debug_tile_order(ntx, nty, nch, resid, 1)
    assert sorted(map(tuple, o.tolist())) == sorted(map(tuple, ref.tolist()))
    if nch >= 3:
        ntiles = ntx * nty
        grp = min(resid, ntiles)
        first = o[:grp * (nch - 2)]  # the interior chunks of the first group
        assert all(0 < c < nch - 1 for c in first[:, 2].tolist())
    else:
        assert np.array_equal(o, ref)
