"""Replica plumbing for `bench.py --gpus N`: one process per
GPU, each solving its own seeded instance of the workload (no data-path
collective: the north-star solve runs on one GPU), timed as the maximum over
ranks. Backend-agnostic so the N > 1 logic is tested with `gloo` on CPU."""

from __future__ import annotations


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def replica_seed(rank: int) -> int:
    """Seed of the synthetic instance solved by `rank` (seed = rank)."""
    return int(rank)


def max_over_ranks(value: float) -> float:
    """Maximum of a per-rank scalar (elapsed seconds) over all ranks."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(value)
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    dist = _dist()
    if dist is not None and dist.get_world_size() > 1:
        dist.barrier()


def whole_job_rate(world: int, units_per_rank: float, elapsed_max: float) -> float:
    """Units all ranks processed / the slowest rank's time (weak scaling)."""
    return world * units_per_rank / elapsed_max
