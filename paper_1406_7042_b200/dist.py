"""Multi-GPU plumbing: one process per GPU, torch.distributed
for rendezvous and the timing reductions.  The hot path has no data-path
collective: a reduced-hybrid run does not shard without a halo exchange, so
N GPUs run N independent replicas (weak scaling, "replicas only"); only the
timing (max over ranks) and the unit counts (sum over ranks) are reduced.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init(backend=None):
    """Initialise the process group from torchrun's environment (no-op for a
    single process).  Returns (rank, world, local_rank)."""
    world, rank, local = env_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def _device():
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def barrier():
    if dist.is_initialized():
        dist.barrier()


def reduce_max(x: float) -> float:
    """Max over ranks (the step time of the slowest rank)."""
    if not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float) -> float:
    if not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def replica_scale(rank: int) -> float:
    """Each replica runs an independent excitation: the source amplitude of
    replica r is scaled by (1 + r/8) (the work per rank is unchanged)."""
    return 1.0 + rank / 8.0


def finalize():
    if dist.is_initialized():
        dist.destroy_process_group()
