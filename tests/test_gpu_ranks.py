"""The inter-rank code of the peer transport, executed: two processes (ranks) of
a z-slab decomposition, bootstrapped by gloo through lb_create_slab_ext (CUDA IPC
mappings of the neighbour's A, B, phi and sync words; the end-to-end poke check),
stepping with the device-side ordering of NEXT-1 (K_phi edges into the
neighbour's ghost planes, step-kernel pushes into its next state, epochs
published with st.release.sys and polled with ld.acquire.sys).

Only one GPU is available, and two ranks' kernels must never wait on each other
on one GPU (B200_PROFILING.md): each step therefore runs in the three host-visible
phases of lb_debug_step_phase with a gloo barrier between them, so every
device-side wait is already satisfied when its kernel starts.  The ranks' results
are gathered and compared bitwise with one slab and with two loopback slabs, and
with the oracle at R18's 1e-12.  (With one GPU per rank -- the driver's scaling
run -- the same kernels overlap and the waits do the ordering.)"""
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

pytestmark = pytest.mark.gpu

P0 = R.Params()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _entry(rank, world, port, shape, nsteps, kernel, outdir, init=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        nx, ny, nz = shape
        rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, 3)
        f, g = R.equilibrium_state(rho, u, phi, P0)
        f, g = f + nf, g + ng
        z0, z1 = D.slab_range(nz, world, rank)
        params = lb.make_params(P0.tau_f, P0.tau_g, P0.A, P0.B, P0.kappa, P0.mobility)
        with lb.Lattice(nx, ny, nz, params, nranks=world, rank=rank, allgather=D.allgather_bytes) as L:
            assert lb.lb_debug_halo_mode(L.h) == 1  # peer transport mapped and checked end to end
            lb.lb_debug_step_kernel(L.h, kernel)
            if init:  # lb_init_equilibrium: phi ghost planes by P2P copies between the processes
                L.init_equilibrium(phi[z0:z1])
            else:
                L.set_state(f[:, z0:z1], g[:, z0:z1])
            for _ in range(nsteps):
                for phase in (0, 1):
                    lb.lb_debug_step_phase(L.h, phase)
                    dist.barrier()
            lb.lb_debug_step_phase(L.h, 2)
            fr, gr = L.get_state()
        np.save(os.path.join(outdir, f"f{rank}.npy"), fr)
        np.save(os.path.join(outdir, f"g{rank}.npy"), gr)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,kernel,init", [((32, 16, 16), 0, False), ((33, 9, 12), 1, False),
                                               ((64, 24, 8), 2, False), ((32, 16, 16), 0, True)])
def test_two_ranks_peer_transport_bitwise(shape, kernel, init, tmp_path):
    nx, ny, nz = shape
    nsteps = 5
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(r, 2, port, shape, nsteps, kernel, str(tmp_path), init))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    f = np.concatenate([np.load(tmp_path / f"f{r}.npy") for r in range(2)], axis=1)
    g = np.concatenate([np.load(tmp_path / f"g{r}.npy") for r in range(2)], axis=1)
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, 3)
    f0, g0 = R.equilibrium_state(rho, u, phi, P0)
    f0, g0 = f0 + nf, g0 + ng
    params = lb.make_params(P0.tau_f, P0.tau_g, P0.A, P0.B, P0.kappa, P0.mobility)
    if init:
        f0, g0 = R.equilibrium_state(np.ones_like(phi), np.zeros((3,) + phi.shape), phi, P0)
    for nslabs in (1, 2):
        with lb.Lattice(nx, ny, nz, params, nslabs=nslabs) as L:
            lb.lb_debug_step_kernel(L.h, kernel)
            if init:
                L.init_equilibrium(phi)
            else:
                L.set_state(f0, g0)
            L.step(nsteps)
            fl, gl = L.get_state()
        assert np.array_equal(f, fl) and np.array_equal(g, gl), nslabs
    fr, gr = R.run(f0, g0, P0, nsteps)
    assert np.abs(f - fr).max() / np.abs(fr).max() <= 1e-12
    assert np.abs(g - gr).max() / np.abs(gr).max() <= 1e-12


def _entry_nccl(rank, world, port, outdir):
    """lb_create_slab (NCCL bootstrap) with both ranks on one GPU: NCCL refuses two
    communicator ranks on one device, so creation must fail cleanly (LB_ENCCL, a
    message, no hang); if this NCCL accepts it, the ranks step in phases as above."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        uid = D.broadcast_bytes(lb.lb_nccl_get_unique_id() if rank == 0 else None)
        outcome = "created"
        try:
            L = lb.Lattice(16, 8, 8, nranks=world, rank=rank, uid=uid)
        except lb.LBError as e:
            outcome = f"error {e.code} {e}"
            L = None
        if L is not None:
            rho, u, phi, nf, ng = synth.rough_fields(16, 8, 8, 3)
            f, g = R.equilibrium_state(rho, u, phi, P0)
            z0, z1 = D.slab_range(8, world, rank)
            L.set_state(f[:, z0:z1] + nf[:, z0:z1], g[:, z0:z1] + ng[:, z0:z1])
            if lb.lb_debug_halo_mode(L.h) == 1:
                for _ in range(2):
                    for phase in (0, 1):
                        lb.lb_debug_step_phase(L.h, phase)
                        dist.barrier()
                lb.lb_debug_step_phase(L.h, 2)
            L.close()
        with open(os.path.join(outdir, f"nccl{rank}.txt"), "w") as fh:
            fh.write(outcome)
    finally:
        dist.destroy_process_group()


def test_nccl_bootstrap_two_ranks_one_gpu(tmp_path):
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_entry_nccl, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    assert not alive, "lb_create_slab hung with two ranks on one GPU"
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    outs = [open(tmp_path / f"nccl{r}.txt").read() for r in range(2)]
    print("lb_create_slab, two ranks on one GPU:", outs)
    for o in outs:
        assert o == "created" or o.startswith(f"error {lb.LB_ENCCL}"), o
