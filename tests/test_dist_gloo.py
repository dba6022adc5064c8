"""Multi-rank host logic on CPU (gloo, world_size 2-4): no GPU needed.

* dist helpers used by bench.py / lb_create_slab bootstrap: broadcast of the
  128-byte NCCL unique id, max-over-ranks timing reduction, slab ranges.
* the z-slab halo plan of the C library (lb_halo_plan: peers and message
  sizes) driving a slab-decomposed run of the CPU oracle, with the same
  exchanges the CUDA path does (phi: 2 planes per direction before the step;
  distributions: the 10 components with c_z = +-1 of the boundary planes after
  it).  The decomposed result must equal the whole-lattice oracle bitwise
  (sub-domains surrounded by halos filled from neighbours).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lb_ref as R
from paper_1609_01479_b200 import dist as D
from paper_1609_01479_b200 import lb, synth

P0 = R.Params(mobility=0.2)
CZ_UP = [i for i in range(19) if R.C[i, 2] == 1]
CZ_DN = [i for i in range(19) if R.C[i, 2] == -1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(fn, world, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _sendrecv(send_arr, dst, recv_shape, src):
    """Paired exchange (isend + recv) of float64 arrays."""
    out = torch.empty(recv_shape, dtype=torch.float64)
    req = dist.isend(torch.from_numpy(np.ascontiguousarray(send_arr)), dst)
    dist.recv(out, src)
    req.wait()
    return out.numpy()


# ---------------------------------------------------------------- helpers
def _helpers_body(rank, world):
    uid = lb.lb_nccl_get_unique_id() if rank == 0 else None
    got = D.broadcast_bytes(uid)
    ref = [None]
    if rank == 0:
        ref = [got]
    dist.broadcast_object_list(ref, 0)
    assert len(got) == 128 and got == ref[0]
    assert D.max_over_ranks(float(rank) * 1.5) == 1.5 * (world - 1)
    assert D.sum_over_ranks(1.0) == float(world)
    z0, z1 = D.slab_range(8 * world, world, rank)
    assert (z0, z1) == (8 * rank, 8 * rank + 8)
    # the all-gather of lb_create_slab_ext's bootstrap (IPC handles, agreement flags)
    mine = bytes([rank, 255 - rank]) * 3
    assert D.allgather_bytes(mine) == b"".join(bytes([r, 255 - r]) * 3 for r in range(world))
    assert D.allgather_bytes(b"") == b""
    D.barrier()


@pytest.mark.parametrize("world", [2, 4])
def test_dist_helpers_gloo(world):
    _run(_helpers_body, world)


def test_slab_range_rejects_thin_slabs():
    with pytest.raises(ValueError):
        D.slab_range(6, 4, 0)
    with pytest.raises(ValueError):
        D.slab_range(3, 2, 0)


# ---------------------------------------------------------------- slab-decomposed oracle
def slab_step(f, g, p, plan, L):
    """One oracle step on a z-slab with the library's halo exchanges (A.8, R14)."""
    up, dn = plan["up"], plan["down"]
    nz_, ny, nx = f.shape[1:]
    assert nz_ == L
    # phi halo: planes [L-2, L) go up, [0, 2) go down (lb_api.cu exchange_phi)
    phi = R.order_parameter(g)
    assert plan["phi_doubles"] == 2 * nx * ny
    below = _sendrecv(phi[L - 2:], up, (2, ny, nx), dn)
    above = _sendrecv(phi[:2], dn, (2, ny, nx), up)
    ext = np.concatenate([below, phi, above])  # planes -2 .. L+1
    grad, lap = R.gradient(ext), R.laplacian(ext)
    F = R.force(R.chemical_stress(ext, grad, lap, p))[:, 2:L + 2]
    mu = R.chemical_potential(ext, lap, p)[2:L + 2]
    rho, j = R.density(f), R.momentum(f)
    R.check_domain(f, g, rho)
    u = R.velocity(rho, j, F)
    fs, gs = R.collide_f(f, rho, u, F, p), R.collide_g(g, phi, u, mu, p)
    # push with ghost planes -1 and L, then the distribution halo exchange
    outs = []
    for a in (fs, gs):
        o = np.zeros((19, L + 2, ny, nx))
        for i in range(19):
            shifted = np.roll(a[i], shift=(int(R.C[i, 1]), int(R.C[i, 0])), axis=(1, 2))
            o[i, 1 + int(R.C[i, 2]):L + 1 + int(R.C[i, 2])] += shifted
        outs.append(o)
    msg_up = np.stack([o[i, L + 1] for o in outs for i in CZ_UP])  # ghost plane L, c_z = +1
    msg_dn = np.stack([o[i, 0] for o in outs for i in CZ_DN])  # ghost plane -1, c_z = -1
    assert plan["dist_doubles"] == msg_up.size == msg_dn.size
    from_dn = _sendrecv(msg_up, up, msg_up.shape, dn)
    from_up = _sendrecv(msg_dn, dn, msg_dn.shape, up)
    k = 0
    for o in outs:
        for i in CZ_UP:
            o[i, 1] = from_dn[k]
            k += 1
    k = 0
    for o in outs:
        for i in CZ_DN:
            o[i, L] = from_up[k]
            k += 1
    return outs[0][:, 1:L + 1], outs[1][:, 1:L + 1]


def _slab_body(rank, world, shape, steps, out_dir):
    nx, ny, nz = shape
    plan = lb.lb_halo_plan(nx, ny, nz, world, rank)
    z0, z1 = D.slab_range(nz, world, rank)
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, seed=3)
    f, g = R.equilibrium_state(rho, u, phi, P0)
    f, g = (f + nf)[:, z0:z1].copy(), (g + ng)[:, z0:z1].copy()
    for _ in range(steps):
        f, g = slab_step(f, g, P0, plan, z1 - z0)
    np.save(os.path.join(out_dir, f"f{rank}.npy"), f)
    np.save(os.path.join(out_dir, f"g{rank}.npy"), g)


@pytest.mark.parametrize("world,shape", [(2, (6, 5, 8)), (3, (5, 4, 9)), (4, (4, 5, 8))])
def test_slab_decomposed_oracle_equals_whole_lattice(world, shape, tmp_path):
    steps = 3
    _run(_slab_body, world, shape, steps, str(tmp_path))
    nx, ny, nz = shape
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, seed=3)
    f, g = R.equilibrium_state(rho, u, phi, P0)
    f, g = R.run(f + nf, g + ng, P0, steps)
    fs = np.concatenate([np.load(tmp_path / f"f{r}.npy") for r in range(world)], axis=1)
    gs = np.concatenate([np.load(tmp_path / f"g{r}.npy") for r in range(world)], axis=1)
    assert np.array_equal(fs, f) and np.array_equal(gs, g)


# ---------------------------------------------------------------- liquid crystal (NEXT-4)
from oracle import lb_lc as LC  # noqa: E402

LP0 = LC.LcParams(A0=0.2, gamma=2.6, kappa=0.05, xi=-0.4, Gamma=0.5)


def slab_step_lc(f, q5, u, p, plan, L):
    """One LC oracle step on a z-slab with the exchanges of lb_api.cu (exchange_lc before
    the step: Q planes [L-2, L) up / [0, 2) down, u planes L-1 up / 0 down; after it
    the f components with c_z = +-1 that left the slab)."""
    up, dn = plan["up"], plan["down"]
    _, _, ny, nx = f.shape
    qb = _sendrecv(q5[:, L - 2:], up, (5, 2, ny, nx), dn)
    qa = _sendrecv(q5[:, :2], dn, (5, 2, ny, nx), up)
    ub = _sendrecv(u[:, L - 1:], up, (3, 1, ny, nx), dn)
    ua = _sendrecv(u[:, :1], dn, (3, 1, ny, nx), up)
    qe = np.concatenate([qb, q5, qa], axis=1)  # Q planes -2 .. L+1
    ue = np.concatenate([ub, u, ua], axis=1)  # u planes -1 .. L
    rho, j = R.density(f), R.momentum(f)
    LC.check_domain(f, q5, u, rho)
    Q = LC.q_full(qe)
    dQ, lapQ = LC.q_gradient(Q), LC.q_laplacian(Q)
    H = LC.molecular_field(Q, lapQ, p)
    P = LC.chemical_stress(Q, dQ, H, LC.free_energy_density(Q, dQ, p), p)
    F = LC.force(P)[:, 2:L + 2]
    u_new = R.velocity(rho, j, F)
    fs = R.collide_f(f, rho, u_new, F, p.fluid)
    q_next = LC.lc_update(Q[:, :, 1:L + 3], ue, H[:, :, 1:L + 3], p)[:, 1:L + 1]
    o = np.zeros((19, L + 2, ny, nx))
    for i in range(19):
        sh = np.roll(fs[i], shift=(int(R.C[i, 1]), int(R.C[i, 0])), axis=(1, 2))
        o[i, 1 + int(R.C[i, 2]):L + 1 + int(R.C[i, 2])] += sh
    msg_up = np.stack([o[i, L + 1] for i in CZ_UP])
    msg_dn = np.stack([o[i, 0] for i in CZ_DN])
    from_dn = _sendrecv(msg_up, up, msg_up.shape, dn)
    from_up = _sendrecv(msg_dn, dn, msg_dn.shape, up)
    for k, i in enumerate(CZ_UP):
        o[i, 1] = from_dn[k]
    for k, i in enumerate(CZ_DN):
        o[i, L] = from_up[k]
    return o[:, 1:L + 1], q_next, u_new


def _lc_rough(nx, ny, nz):
    rho, u, q5, nf = synth.rough_lc_fields(nx, ny, nz, seed=5)
    return R.f_equilibrium(rho, u) + nf, q5, u


def _slab_body_lc(rank, world, shape, steps, out_dir):
    nx, ny, nz = shape
    plan = lb.lb_halo_plan(nx, ny, nz, world, rank)
    z0, z1 = D.slab_range(nz, world, rank)
    f, q5, u = (a[:, z0:z1].copy() for a in _lc_rough(nx, ny, nz))
    for _ in range(steps):
        f, q5, u = slab_step_lc(f, q5, u, LP0, plan, z1 - z0)
    for name, a in (("f", f), ("q", q5), ("u", u)):
        np.save(os.path.join(out_dir, f"{name}{rank}.npy"), a)


@pytest.mark.parametrize("world,shape", [(2, (6, 5, 8)), (3, (4, 5, 9)), (4, (4, 4, 8))])
def test_lc_slab_decomposed_oracle_equals_whole_lattice(world, shape, tmp_path):
    """The liquid-crystal schedule of lb_create_lc_slab (Q on two halo planes, u on one,
    f's crossing components), run on the oracle over gloo ranks: bitwise the whole lattice."""
    steps = 3
    _run(_slab_body_lc, world, shape, steps, str(tmp_path))
    ref = LC.run(*_lc_rough(*shape), LP0, steps)
    for name, a in zip("fqu", ref):
        got = np.concatenate([np.load(tmp_path / f"{name}{r}.npy") for r in range(world)], axis=1)
        assert np.array_equal(got, a), name


# ---------------------------------------------------------------- Cahn-Hilliard (NEXT-2)
from oracle import lb_ch as CH  # noqa: E402
from oracle import lb_mrt as MRT  # noqa: E402

CP0 = CH.ChParams(base=R.Params(mobility=0.2))


def slab_step_ch(f, phi, p, plan, L):
    """One Cahn-Hilliard oracle step on a z-slab with the exchanges of lb_api.cu
    (exchange_fedge + exchange_phi before the step: f planes L-1 up / 0 down, all 19
    components; phi planes [L-2, L) up / [0, 2) down; after it the leaving f
    components)."""
    up, dn = plan["up"], plan["down"]
    _, _, ny, nx = f.shape
    fb = _sendrecv(f[:, L - 1:], up, (19, 1, ny, nx), dn)
    fa = _sendrecv(f[:, :1], dn, (19, 1, ny, nx), up)
    pb = _sendrecv(phi[L - 2:], up, (2, ny, nx), dn)
    pa = _sendrecv(phi[:2], dn, (2, ny, nx), up)
    fe = np.concatenate([fb, f, fa], axis=1)  # f planes -1 .. L
    pe = np.concatenate([pb, phi, pa])  # phi planes -2 .. L+1
    b = p.base
    rho_e, j_e = R.density(fe), R.momentum(fe)
    u_e = MRT.velocity(rho_e, j_e)  # planes -1 .. L
    grad_e, lap_e = R.gradient(pe), R.laplacian(pe)
    mu_e = R.chemical_potential(pe, lap_e, b)
    P = R.chemical_stress(pe, grad_e, lap_e, b)[:, :, 2:L + 2]
    rho, u = rho_e[1:L + 1], u_e[:, 1:L + 1]
    CH.check_domain(f, phi, rho)
    fs = MRT.collide_f(f, rho, u, P, p.mrt)
    phi_next = CH.phi_update(pe[1:L + 3], u_e, mu_e[1:L + 3], p)[1:L + 1]
    o = np.zeros((19, L + 2, ny, nx))
    for i in range(19):
        sh = np.roll(fs[i], shift=(int(R.C[i, 1]), int(R.C[i, 0])), axis=(1, 2))
        o[i, 1 + int(R.C[i, 2]):L + 1 + int(R.C[i, 2])] += sh
    msg_up = np.stack([o[i, L + 1] for i in CZ_UP])
    msg_dn = np.stack([o[i, 0] for i in CZ_DN])
    from_dn = _sendrecv(msg_up, up, msg_up.shape, dn)
    from_up = _sendrecv(msg_dn, dn, msg_dn.shape, up)
    for k, i in enumerate(CZ_UP):
        o[i, 1] = from_dn[k]
    for k, i in enumerate(CZ_DN):
        o[i, L] = from_up[k]
    return o[:, 1:L + 1], phi_next


def _ch_rough(nx, ny, nz):
    rho, u, phi, nf, _ = synth.rough_fields(nx, ny, nz, seed=6)
    return R.f_equilibrium(rho, u) + nf, phi


def _slab_body_ch(rank, world, shape, steps, out_dir):
    nx, ny, nz = shape
    plan = lb.lb_halo_plan(nx, ny, nz, world, rank)
    z0, z1 = D.slab_range(nz, world, rank)
    f, phi = _ch_rough(nx, ny, nz)
    f, phi = f[:, z0:z1].copy(), phi[z0:z1].copy()
    for _ in range(steps):
        f, phi = slab_step_ch(f, phi, CP0, plan, z1 - z0)
    np.save(os.path.join(out_dir, f"f{rank}.npy"), f)
    np.save(os.path.join(out_dir, f"p{rank}.npy"), phi)


@pytest.mark.parametrize("world,shape", [(2, (6, 5, 8)), (3, (4, 5, 9)), (4, (4, 4, 8))])
def test_ch_slab_decomposed_oracle_equals_whole_lattice(world, shape, tmp_path):
    """The Cahn-Hilliard schedule of lb_create_ch_slab on the oracle over gloo ranks:
    bitwise the whole lattice."""
    steps = 3
    _run(_slab_body_ch, world, shape, steps, str(tmp_path))
    f, phi = CH.run(*_ch_rough(*shape), CP0, steps)
    fs = np.concatenate([np.load(tmp_path / f"f{r}.npy") for r in range(world)], axis=1)
    ps = np.concatenate([np.load(tmp_path / f"p{r}.npy") for r in range(world)], axis=0)
    assert np.array_equal(fs, f) and np.array_equal(ps, phi)
