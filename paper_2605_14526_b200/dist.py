"""Multi-GPU plumbing for bench.py: one process per GPU (torchrun), independent
replicas of the trajectory (a single trajectory does not shard, SURVEY.md
§8(e)); timing is the maximum over ranks and throughput counts every rank's
steps."""
from __future__ import annotations

import torch
import torch.distributed as dist


def max_over_ranks(ms: float) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return ms
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(steps: int, ms: float, world: int) -> float:
    """Whole-job steps/s: every rank ran `steps` steps within the slowest rank's time."""
    return world * steps / (ms / 1e3)
