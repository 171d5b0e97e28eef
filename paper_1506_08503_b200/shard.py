"""Multi-GPU shard plan (north_star subsystem (4)).

The reference's data parallelism is a balanced contiguous row partition
(parallel.py:37-50, ``plan``) fanned out over threads (:66-75).  On an
8 x B200 box the same plan assigns contiguous block ranges to GPUs -- one
process (rank) per GPU, one stream each, no collective on the data path
because blocks are independent.  Only timing and the
optional verification reduce across ranks.

``plan`` is pure Python (CPU-testable); ``rank_slice`` / ``key_slice`` give a
rank its share; ``max_over_ranks`` is the one reduction the bench performs.
"""

from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class ParallelPlan:
    """Contiguous balanced partition of [0, N) into at most ``workers`` ranges
    (same contract as the reference's ParallelPlan, parallel.py:25-34)."""

    workers: int
    chunks: tuple

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("need at least one worker")


def plan(n_messages: int, workers: int) -> ParallelPlan:
    """Balanced contiguous ranges, sizes within one of each other, at most
    min(workers, n) of them (semantics of parallel.py:37-50).

    The first ``n % k`` ranges get the extra row; boundaries are
    ``i * q + min(i, r)`` with ``q, r = divmod(n, k)``.
    """
    if workers < 1:
        raise ValueError("need at least one worker")
    if n_messages < 0:
        raise ValueError("negative message count")
    k = min(workers, n_messages)
    if k == 0:
        return ParallelPlan(workers=workers, chunks=())
    q, r = divmod(n_messages, k)
    edges = [i * q + min(i, r) for i in range(k + 1)]
    return ParallelPlan(workers=workers, chunks=tuple(zip(edges[:-1], edges[1:])))


def rank_slice(n_messages: int, rank: int, world_size: int) -> tuple:
    """Rows [lo, hi) owned by `rank` (empty range if the plan has fewer chunks)."""
    if not 0 <= rank < world_size:
        raise ValueError("rank out of range")
    chunks = plan(n_messages, world_size).chunks
    return chunks[rank] if rank < len(chunks) else (n_messages, n_messages)


def key_slice(n_keys: int, rank: int, world_size: int) -> tuple:
    """Config 5 shards keys (and with them their blocks) contiguously."""
    return rank_slice(n_keys, rank, world_size)


def dist_env() -> tuple:
    """(rank, local_rank, world_size) from the torchrun environment (defaults 0, 0, 1)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (timing); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: int, device=None) -> int:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def gather_objects(obj) -> list:
    """Every rank's ``obj`` in rank order (``[obj]`` without a process group)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [obj]
    res = [None] * dist.get_world_size()
    dist.all_gather_object(res, obj)
    return res


def parse_cpulist(text: str) -> list:
    """CPU ids from a sysfs cpulist ("0-3,8,10-11")."""
    cpus = []
    for part in text.strip().split(","):
        if "-" in part:
            lo, hi = part.split("-")
            cpus.extend(range(int(lo), int(hi) + 1))
        elif part:
            cpus.append(int(part))
    return cpus


def host_threads_per_rank(n_cpus: int, ranks_sharing: int) -> int:
    """Copy threads for one rank when `ranks_sharing` ranks run on the same
    `n_cpus` CPUs: an even share, so N ranks' spinning host pools
    (csrc/host_pool.h) never oversubscribe a NUMA node."""
    return max(1, n_cpus // max(1, ranks_sharing))


def _gpu_cpulist(device_index: int) -> str:
    import torch
    props = torch.cuda.get_device_properties(device_index)
    bdf = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
    with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
        return f.read().strip()


def bind_to_gpu_numa_node(device_index: int) -> list | None:
    """Pin this process to the CPUs local to the GPU's PCIe root (one process
    per GPU): pinned staging buffers and host copies then stay on the GPU's
    NUMA node.  The host copy pool is sized to this rank's share of those
    CPUs (GAES_HOST_THREADS, unless the caller set it): the local ranks whose
    GPUs hang off the same node split its CPUs evenly.  Best effort; returns
    the CPU list used or None."""
    allowed = os.sched_getaffinity(0)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", 1))
    try:
        mine = _gpu_cpulist(device_index)
        sharing = 0
        for g in range(local_world):
            try:
                sharing += _gpu_cpulist(g) == mine
            except (OSError, RuntimeError, AssertionError):
                pass
        cpus = [c for c in parse_cpulist(mine) if c in allowed]
    except (OSError, ValueError, AttributeError, RuntimeError, AssertionError):
        cpus, sharing = [], local_world
    bound = bool(cpus) and len(cpus) != len(allowed)
    if bound:
        os.sched_setaffinity(0, cpus)
    if local_world > 1 and not os.environ.get("GAES_HOST_THREADS"):
        pool = cpus if bound else sorted(allowed)
        os.environ["GAES_HOST_THREADS"] = str(host_threads_per_rank(len(pool), max(1, sharing)))
    return cpus if bound else None
