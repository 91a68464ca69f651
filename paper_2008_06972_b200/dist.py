"""Multi-GPU plumbing for batch encoding: one process per GPU, groups sharded
by rank, no data-path collective.

K+P groups are independent (no GOP chaining), so each rank
encodes its own contiguous block of groups.  The only collectives are the
final gather of per-group blob sizes and the max-over-ranks of the device
time.  Works with the NCCL backend on GPUs and gloo on CPU
(tests).
"""

from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def shard_range(n_groups: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of n_groups for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_groups, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _coll_device(device):
    """gloo collectives run on host tensors (also when the ranks use GPUs)."""
    return device if dist.get_backend() == "nccl" else torch.device("cpu")


def gather_sizes(local: torch.Tensor) -> torch.Tensor:
    """All ranks' per-group int64 sizes concatenated in rank order (every rank
    must pass the same length; pad with -1 and strip if shards are ragged)."""
    world = dist.get_world_size()
    if dist.get_backend() == "nccl":
        out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    src = local.detach().to("cpu").contiguous()
    out = torch.empty(world * src.numel(), dtype=src.dtype)
    dist.all_gather(list(out.chunk(world)), src)
    return out.to(local.device)


def max_over_ranks(value: float, device) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: int, device) -> int:
    t = torch.tensor([value], dtype=torch.int64, device=_coll_device(device))
    dist.all_reduce(t)
    return int(t.item())
