"""Multi-GPU plumbing for the checker.

CTA pairs are independent reference `check_equivalence` calls, so a grid
shards with no data-path exchange: rank r owns a contiguous range of CTA
pairs and checks it on its own GPU with its own term table. The one
exchange is the verdict combine — a sum all-reduce of small counters
(equal VCs, VCs, faults, missing outputs) plus a min all-reduce of the first
non-equal VC index — over NCCL on GPUs (gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Optional, Sequence, Tuple

COUNTERS = ("equal", "vcs", "faults", "missing")
NO_FAILURE = (1 << 62)


def shard_blocks(total_blocks: int, rank: int, world: int) -> Tuple[int, int]:
    """(first block, block count) of `rank`'s contiguous share of a grid of
    `total_blocks` CTA pairs; shares differ by at most one block."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    q, r = divmod(total_blocks, world)
    base = rank * q + min(rank, r)
    return base, q + (1 if rank < r else 0)


def combine_verdicts(counters: Sequence[int], first_failure: Optional[int], device=None, group=None):
    """All-reduce of the per-rank verdict counters (sum) and of the first
    failing global VC index (min). Returns (dict of totals, first failure or
    None). Uses the default process group when torch.distributed is
    initialised, else returns the local values."""
    import torch
    import torch.distributed as dist

    vals = [int(c) for c in counters] + [NO_FAILURE if first_failure is None else int(first_failure)]
    if not (dist.is_available() and dist.is_initialized()):
        tot, ff = vals[:-1], vals[-1]
    else:
        t = torch.tensor(vals[:-1], dtype=torch.int64, device=device)
        f = torch.tensor([vals[-1]], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(f, op=dist.ReduceOp.MIN, group=group)
        tot, ff = [int(x) for x in t.tolist()], int(f.item())
    return dict(zip(COUNTERS, tot)), (None if ff >= NO_FAILURE else ff)
