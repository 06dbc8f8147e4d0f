"""Multi-GPU plumbing for the replicas-only scaling mode.

The LTS path has no exchange step: every rank runs an independent replica of
the full pass on its own GPU.  The only collectives are the timing barrier and
the max-over-ranks reduction of the measured device time, done here so the
same code is exercised by the CPU (gloo) tests and by bench.py (nccl).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device=None):
    rank, world, local = env()
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    return rank, world, local


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) across the job."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank: int, world: int, ms_per_step_max: float) -> float:
    """Whole-job units/s: all ranks' units over the slowest rank's step time."""
    return world * units_per_rank / (ms_per_step_max / 1e3)


def shutdown():
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
