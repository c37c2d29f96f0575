"""Realization sharding across GPUs (one process per GPU, torch.distributed).

The reference parallelises only over realizations: contiguous chunks from
``_chunk_bounds`` (ensemble.py:596-606) run in worker processes, and the
host concatenates the chunk states to average them (ensemble.py:762-768).
Here each rank owns a contiguous realization shard for the whole run
(states never move between GPUs); the only cross-GPU traffic is, at each
post-processing point, an all-reduce of the per-rank diagonal partial sums
(NCCL over NVLink) plus a tiny all-gather of the per-rank norm statistics.
Purity, which needs overlaps between realizations on different ranks, is the
one exception and gathers the states (small problems only).

Everything here also runs on CPU tensors with the gloo backend, which is how
the multi-process logic is tested without GPUs.
"""

from __future__ import annotations


def _collective(group=None) -> bool:
    """Run the collectives?  Yes on more than one rank; also on one rank when
    CTQW_FORCE_COLLECTIVES=1 (exercises the NCCL path on a single-GPU box)."""
    import os

    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return False
    return dist.get_world_size(group) > 1 or os.environ.get("CTQW_FORCE_COLLECTIVES") == "1"


def world_info(group=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_bounds(realizations: int, world: int, rank: int):
    """Contiguous shard of ``rank`` (same split rule as ``_chunk_bounds``)."""
    base, extra = divmod(int(realizations), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def all_shards(realizations: int, world: int):
    return [shard_bounds(realizations, world, r) for r in range(world)]


def allreduce_sum_(tensor, group=None):
    """In-place sum over ranks (no-op on one rank)."""
    import torch.distributed as dist

    if _collective(group):
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def gather_objects(obj, group=None):
    """List of ``obj`` from every rank in rank order."""
    import torch.distributed as dist

    if _collective(group):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, obj, group=group)
        return out
    return [obj]


def merge_segment_stats(per_rank):
    """Combine per-rank segment statistics like the reference combines chunks.

    ``per_rank`` is a list (rank order) of dicts with keys event_count,
    corrections, max_deviation, events (list of tuples) and failure (None or
    (deviation, realization, step)).  Totals add, the maximum deviation is
    the max, events concatenate in shard order (ensemble.py:751-758), and the
    failure reported is the first shard's that failed -- the reference
    collects chunk futures in order (ensemble.py:727-730).
    """
    merged = {"event_count": 0, "corrections": 0, "max_deviation": 0.0, "events": [],
              "failure": None}
    for st in per_rank:
        merged["event_count"] += int(st["event_count"])
        merged["corrections"] += int(st["corrections"])
        merged["max_deviation"] = max(merged["max_deviation"], float(st["max_deviation"]))
        merged["events"].extend(st["events"])
        if merged["failure"] is None and st["failure"] is not None:
            merged["failure"] = st["failure"]
    return merged


def gather_states(local, group=None):
    """Concatenate every rank's state shard (used only for purity)."""
    import torch
    import torch.distributed as dist

    if not _collective(group):
        return local
    sizes = gather_objects(int(local.shape[0]), group)
    flat = torch.view_as_real(local) if local.is_complex() else local
    biggest = max(sizes)
    padded = torch.zeros((biggest,) + tuple(flat.shape[1:]), dtype=flat.dtype, device=flat.device)
    padded[: flat.shape[0]] = flat
    bufs = [torch.empty_like(padded) for _ in sizes]
    dist.all_gather(bufs, padded, group=group)
    out = torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0).contiguous()
    return torch.view_as_complex(out) if local.is_complex() else out


__all__ = ["world_info", "shard_bounds", "all_shards", "allreduce_sum_", "gather_objects",
           "merge_segment_stats", "gather_states"]
