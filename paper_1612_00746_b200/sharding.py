"""Realization sharding across GPUs (one process per GPU, torch.distributed).

The reference parallelises only over realizations: contiguous chunks from
``_chunk_bounds`` (ensemble.py:596-606) run in worker processes, and the
host concatenates the chunk states to average them (ensemble.py:762-768).
Here each rank owns a contiguous realization shard for the whole run
(states never move between GPUs); the only cross-GPU traffic is, at each
post-processing point, an all-reduce of the per-rank diagonal sums -- exact
int64 fixed-point limbs, so the result is bitwise the same for any number of
ranks -- (NCCL over NVLink) plus one all-gather of a fixed-size tensor of the
per-rank norm statistics.
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


def _comm_device(group=None):
    """Tensors for collectives live on the current CUDA device under NCCL, on
    the host under gloo (the CPU tests)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_objects(obj, group=None):
    """List of ``obj`` from every rank in rank order (small host-side objects,
    not on the per-collection-point path)."""
    import torch.distributed as dist

    if _collective(group):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, obj, group=group)
        return out
    return [obj]


def allreduce_int_(values, group=None):
    """Sum of a few host integers over ranks (one int64 tensor all-reduce)."""
    import torch
    import torch.distributed as dist

    if not _collective(group):
        return [int(v) for v in values]
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [int(v) for v in t.cpu().tolist()]


MAX_EVENTS = 100
_HEAD = 8  # event_count, corrections, max_deviation, failed, fail_dev, fail_real, fail_step, n_events


def pack_stats(st) -> list:
    """Fixed-size float64 record of one rank's segment statistics (counts and
    indices stay exact below 2^53)."""
    fail = st["failure"]
    events = list(st["events"])[:MAX_EVENTS]
    rec = [float(st["event_count"]), float(st["corrections"]), float(st["max_deviation"]),
           1.0 if fail is not None else 0.0,
           float(fail[0]) if fail else 0.0, float(fail[1]) if fail else 0.0, float(fail[2]) if fail else 0.0,
           float(len(events))]
    for dev, corrected, real, step in events:
        rec.extend((float(dev), 1.0 if corrected else 0.0, float(real), float(step)))
    rec.extend([0.0] * (4 * (MAX_EVENTS - len(events))))
    return rec


def unpack_stats(rec) -> dict:
    rec = [float(v) for v in rec]
    n_ev = int(rec[7])
    events = []
    for k in range(n_ev):
        dev, corr, real, step = rec[_HEAD + 4 * k: _HEAD + 4 * k + 4]
        events.append((dev, bool(corr), int(real), int(step)))
    failure = (rec[4], int(rec[5]), int(rec[6])) if rec[3] else None
    return {"event_count": int(rec[0]), "corrections": int(rec[1]), "max_deviation": rec[2],
            "events": events, "failure": failure}


def gather_stats(local, group=None):
    """Every rank's segment statistics, in rank order: ONE all-gather of a
    fixed-size float64 tensor (8 + 4*MAX_EVENTS entries per rank)."""
    import torch
    import torch.distributed as dist

    if not _collective(group):
        return [local]
    dev = _comm_device(group)
    mine = torch.tensor(pack_stats(local), dtype=torch.float64, device=dev)
    bufs = [torch.empty_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(bufs, mine, group=group)
    return [unpack_stats(b.cpu().tolist()) for b in bufs]


def gather_segment_events(per_segment, group=None):
    """Per-segment event lists of a group of collection points, merged over
    the ranks with ONE all-gather: ``per_segment`` is this rank's list (one
    entry per segment) of (deviation, corrected, realization, step) lists,
    each holding the rank's first MAX_EVENTS in (step, realization) order;
    the result keeps, per segment, the first MAX_EVENTS of the union in that
    order (merge_segment_stats' rule), so it does not depend on the split."""
    import torch
    import torch.distributed as dist

    if not _collective(group):
        return [sorted(evs, key=lambda e: (e[3], e[2]))[:MAX_EVENTS] for evs in per_segment]
    P = len(per_segment)
    rec = torch.zeros((P, 1 + 4 * MAX_EVENTS), dtype=torch.float64)
    for k, evs in enumerate(per_segment):
        evs = list(evs)[:MAX_EVENTS]
        rec[k, 0] = float(len(evs))
        for e, (dev, corrected, real, step) in enumerate(evs):
            rec[k, 1 + 4 * e: 5 + 4 * e] = torch.tensor([dev, 1.0 if corrected else 0.0, float(real), float(step)],
                                                        dtype=torch.float64)
    dev = _comm_device(group)
    mine = rec.to(dev)
    bufs = [torch.empty_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(bufs, mine, group=group)
    recs = [b.cpu().numpy() for b in bufs]
    out = []
    for k in range(P):
        evs = []
        for r in recs:
            for e in range(int(r[k, 0])):
                dv, corr, real, step = r[k, 1 + 4 * e: 5 + 4 * e]
                evs.append((float(dv), bool(corr), int(real), int(step)))
        evs.sort(key=lambda e: (e[3], e[2]))
        out.append(evs[:MAX_EVENTS])
    return out


def merge_segment_stats(per_rank):
    """Combine per-rank segment statistics independently of how the
    realizations were split.

    ``per_rank`` is a list (rank order) of dicts with keys event_count,
    corrections, max_deviation, events (list of (dev, corrected, realization,
    step)) and failure (None or (deviation, realization, step)).  Totals
    add, the maximum deviation is the max, the events kept are the first
    MAX_EVENTS in (step, realization) order -- each rank's list holds its own
    first MAX_EVENTS in that order, so the union contains the global first
    ones -- and the failure reported is the one a single process reports
    (the device reduction's rule): earliest step, then largest deviation,
    then lowest realization.  So 1, 2, 4 or 8 GPUs report the same events and
    the same culprit (the reference's single-chunk semantics,
    propagators.py:320-323, ensemble.py:503-516).
    """
    merged = {"event_count": 0, "corrections": 0, "max_deviation": 0.0, "events": [],
              "failure": None}
    events = []
    for st in per_rank:
        merged["event_count"] += int(st["event_count"])
        merged["corrections"] += int(st["corrections"])
        merged["max_deviation"] = max(merged["max_deviation"], float(st["max_deviation"]))
        events.extend(st["events"])
        f = st["failure"]
        if f is not None:
            cur = merged["failure"]
            if cur is None or (f[2], -f[0], f[1]) < (cur[2], -cur[0], cur[1]):
                merged["failure"] = (float(f[0]), int(f[1]), int(f[2]))
    events.sort(key=lambda e: (e[3], e[2]))
    merged["events"] = events[:MAX_EVENTS]
    return merged


def is_collective(group=None) -> bool:
    """Do collectives run for ``group`` (more than one rank, or forced)?"""
    return _collective(group)


def gather_states(local, group=None):
    """Concatenate every rank's state shard (used only for purity)."""
    import torch
    import torch.distributed as dist

    if not _collective(group):
        return local
    cnt = torch.tensor([int(local.shape[0])], dtype=torch.int64, device=_comm_device(group))
    cnts = [torch.empty_like(cnt) for _ in range(dist.get_world_size(group))]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    flat = torch.view_as_real(local) if local.is_complex() else local
    biggest = max(sizes)
    padded = torch.zeros((biggest,) + tuple(flat.shape[1:]), dtype=flat.dtype, device=flat.device)
    padded[: flat.shape[0]] = flat
    bufs = [torch.empty_like(padded) for _ in sizes]
    dist.all_gather(bufs, padded, group=group)
    out = torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0).contiguous()
    return torch.view_as_complex(out) if local.is_complex() else out


__all__ = ["world_info", "is_collective", "shard_bounds", "all_shards", "allreduce_sum_", "allreduce_int_", "gather_objects",
           "gather_stats", "pack_stats", "unpack_stats", "merge_segment_stats", "gather_states"]
