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


# ---- batched system-ID (C5): samples shard across ranks --------------------

def shard(samples: int, rank: int, world: int) -> range:
    """Contiguous block of sample indices owned by `rank` (sizes differ by at
    most one; lower ranks take the remainder).  The global sample order is
    rank-major, so the all-reduced sum is a fixed function of (samples, world)."""
    base, rem = divmod(samples, world)
    lo = rank * base + min(rank, rem)
    return range(lo, lo + base + (1 if rank < rem else 0))


def allreduce_loss_grad(buf: torch.Tensor) -> torch.Tensor:
    """Sum [loss, dL/dtheta] over ranks in place — the only cross-GPU exchange of
    the batched path.  `buf` lives on this rank's GPU for
    NCCL (it is the device buffer hd_batch_evaluate filled) or on the CPU for
    gloo."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    return buf
