"""Multi-GPU plumbing for the checker.

CTA pairs are independent reference `check_equivalence` calls, so a grid
shards with no data-path exchange: rank r owns a contiguous range of CTA
pairs and checks it on its own GPU with its own term table. The one
exchange is the verdict combine: a sum all-reduce of small counters (equal
VCs, VCs, faults, missing outputs), a min all-reduce of the first non-equal
VC index, and an all-gather of per-VC verdict bytes and side-condition
(hash, discharged) pairs so one rank can aggregate the report
(pipeline.cpp:245-266). On GPUs this is the C-ABI's NCCL collective
(veq_comm_init / veq_comm_combine); `combine_verdicts` is the same exchange
over torch.distributed (gloo in the CPU tests) and `aggregate` the report
fold both feed.
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


def comm_init(sess, rank: int, world: int, group=None) -> bool:
    """NCCL communicator of the C-ABI for this rank's session: rank 0 makes
    the unique id, torch.distributed broadcasts it (plumbing only).
    Returns False when the library has no NCCL (the caller falls back to
    combine_verdicts)."""
    import ctypes as C
    import torch.distributed as dist
    from . import native as N

    L = N.lib()
    buf = C.create_string_buffer(128)
    ok = [True]
    if rank == 0:
        ok[0] = L.veq_comm_unique_id(buf) == 0
    obj = [bytes(buf.raw) if rank == 0 else None, ok[0]]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not obj[1]:
        return False
    st = L.veq_comm_init(sess.ctx, C.c_char_p(obj[0]), world, rank)
    return st == 0


def comm_combine(sess, first_failure: Optional[int]):
    """veq_comm_combine: (totals dict, first failure or None, per-VC verdict
    bytes of all ranks, side-condition (hash, discharged) pairs of all ranks,
    VC offsets per rank)."""
    import ctypes as C
    import numpy as np
    from . import native as N

    out = N.veq_combined()
    st = N.lib().veq_comm_combine(sess.ctx, NO_FAILURE if first_failure is None else int(first_failure),
                                  C.byref(out))
    if st != 0:
        raise N.VeqError(st, N.lib().veq_last_error(sess.ctx).decode())
    R = int(out.n_ranks)
    voff = np.ctypeslib.as_array(out.rank_vc_off, shape=(R + 1,)).copy()
    soff = np.ctypeslib.as_array(out.rank_sc_off, shape=(R + 1,)).copy()
    nv, ns = int(voff[R]), int(soff[R])
    verdict = np.ctypeslib.as_array(out.verdict, shape=(max(nv, 1),))[:nv].copy() if nv else np.zeros(0, np.uint8)
    sch = np.ctypeslib.as_array(out.sc_hash, shape=(max(ns, 1),))[:ns].copy() if ns else np.zeros(0, np.uint64)
    scd = np.ctypeslib.as_array(out.sc_discharged, shape=(max(ns, 1),))[:ns].copy() if ns else np.zeros(0, np.uint8)
    ff = int(out.first_fail)
    return (dict(zip(COUNTERS, [int(x) for x in out.totals])), None if ff >= NO_FAILURE else ff, verdict,
            list(zip(sch.tolist(), scd.tolist())), voff)


def aggregate(verdicts: Sequence[int], side_conditions: Sequence[Tuple[int, int]]) -> str:
    """The report fold of check_equivalence (pipeline.cpp:245-266) over VCs
    in order: side conditions de-duplicated by identity in first-occurrence
    order (structurally equal denominators share one Merkle hash); any
    residual (undischarged) one makes the verdict "unknown"; a VC that is
    not canonically equal is left to the host slow path ("undecided")."""
    seen, residual = set(), False
    for h, dis in side_conditions:
        if h not in seen:
            seen.add(h)
            residual |= not dis
    if not all(verdicts):
        return "undecided"
    return "unknown" if residual else "equivalent"
