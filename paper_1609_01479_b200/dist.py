"""Process-group plumbing for the z-slab decomposition (PAPER.md P:185-193:
"domain decomposition and MPI in a standard way" -- here one process per GPU,
torch.distributed for bootstrap and timing reductions only).

torch.distributed never touches the data path: the library owns its NCCL
communicator (lb_create_slab) and torch only carries the 128-byte
ncclUniqueId from rank 0 to the others, barriers, and the max-over-ranks
reduction of timings.  Works with the "nccl" backend on GPUs and "gloo" on CPU
(tests).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1-process defaults)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str) -> None:
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)


def _device() -> torch.device:
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_bytes(payload: bytes | None, nbytes: int = 128, src: int = 0) -> bytes:
    """Rank src's `payload` (exactly nbytes) on every rank."""
    t = torch.zeros(nbytes, dtype=torch.uint8, device=_device())
    if dist.get_rank() == src:
        assert payload is not None and len(payload) == nbytes
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().numpy().tobytes())


def allgather_bytes(payload: bytes) -> bytes:
    """Every rank's `payload` (all the same length), concatenated in rank order: the
    bootstrap all-gather of lb_create_slab_ext (CUDA IPC handles, agreement flags,
    barriers) over whatever process group is initialised (gloo or NCCL)."""
    n = len(payload)
    t = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(_device()) if n else torch.zeros(0, dtype=torch.uint8, device=_device())
    out = [torch.zeros(n, dtype=torch.uint8, device=_device()) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return b"".join(bytes(o.cpu().numpy().tobytes()) for o in out)


def max_over_ranks(v: float) -> float:
    """Max of a float over all ranks (the timing rule: max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(v)
    t = torch.tensor([float(v)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(v)
    t = torch.tensor([float(v)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()


def slab_range(nz: int, nranks: int, rank: int) -> tuple[int, int]:
    """Global z range [z0, z1) owned by `rank` (include/lb.h lb_create_slab)."""
    if nz % nranks or nz // nranks < (2 if nranks > 1 else 3):
        raise ValueError(f"nz={nz} cannot be split into {nranks} slabs of >= 2 planes")
    L = nz // nranks
    return rank * L, (rank + 1) * L
