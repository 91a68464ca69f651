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


def gpu_numa_node(local: int) -> int:
    """NUMA node of CUDA device `local` (sysfs numa_node of its PCI address),
    or -1 when unknown."""
    import subprocess

    bus = None
    try:
        pr = torch.cuda.get_device_properties(local)
        bus = "%04x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
    except Exception:
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(local), "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                                 capture_output=True, text=True, timeout=20).stdout.strip()
            if out:
                bus = out.lower()[-12:]
        except Exception:
            return -1
    try:
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            return int(f.read().strip())
    except Exception:
        return -1


def _cpulist(spec: str):
    cpus = []
    for part in spec.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.extend(range(int(a), int(b) + 1))
        elif part:
            cpus.append(int(part))
    return cpus


def bind_to_gpu_numa(local: int) -> dict:
    """Pin this rank's threads to the CPUs of its GPU's NUMA node, so its
    pinned staging buffers (allocated afterwards, first touched by these
    threads) are node-local and its H2D copies do not cross the socket link.
    Returns {"numa_node", "cpus"}; a no-op where the topology is unknown."""
    import os

    node = gpu_numa_node(local)
    info = {"numa_node": node, "cpus": None}
    if node < 0:
        return info
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            cpus = set(_cpulist(f.read())) & set(os.sched_getaffinity(0))
        if cpus:
            os.sched_setaffinity(0, cpus)
            info["cpus"] = len(cpus)
    except Exception:
        pass
    return info


def gather_ragged(local: torch.Tensor, n_total: int, world: int) -> torch.Tensor:
    """Per-group int64 values of contiguous shards (shard_range) gathered in
    group order: each rank pads to the largest shard with -1, the padding is
    stripped after the gather."""
    width = -(-n_total // world)
    pad = torch.full((width,), -1, dtype=torch.int64, device=local.device)
    pad[: local.numel()] = local
    allv = gather_sizes(pad)
    parts = []
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        parts.append(allv[r * width: r * width + (hi - lo)])
    return torch.cat(parts)


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
