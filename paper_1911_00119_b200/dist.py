"""Multi-GPU plumbing: streams shard, aggregates reduce once.

Streams / scenarios are independent, so rank r of W owns
the contiguous range ``shard(n, W, r)`` and runs it with no data-path
collective.  The only cross-GPU exchange is the final aggregate: each rank
reduces its per-stream blocks deterministically on its GPU (alert_reduce)
and ``reduce_aggregates`` all-gathers the 88-double vectors (NCCL over
NVLink on GPUs, gloo in the CPU tests) and sums them in rank order, so the
result is bit-reproducible for a given world size (an NCCL all-reduce's
summation order depends on the topology/algorithm).
"""

from __future__ import annotations


def shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of the items owned by ``rank`` (balanced, contiguous)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(n, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def reduce_aggregates(local, group=None):
    """Sum a 1-D aggregate tensor over all ranks in rank order (all_gather)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local.clone()
    src = local.contiguous()
    if dist.get_backend(group) == "gloo" and src.is_cuda:  # gloo gathers host tensors
        src = src.cpu()
    parts = [torch.empty_like(src) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, src, group=group)
    total = parts[0].clone()
    for p in parts[1:]:
        total += p
    return total.to(local.device)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    gloo = dist.get_backend(group) == "gloo"
    t = torch.tensor([value], dtype=torch.float64, device=None if gloo else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device=None, group=None) -> float:
    """Sum of a scalar over ranks (e.g. bytes copied by every rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    gloo = dist.get_backend(group) == "gloo"
    t = torch.tensor([float(value)], dtype=torch.float64, device=None if gloo else device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
