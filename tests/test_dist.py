"""Multi-rank host path (CPU, gloo, world size 2): the grid of CTA pairs is
sharded with no data-path exchange (paper_2511_12638_b200.dist.shard_blocks)
and the verdicts are combined by one all-reduce (combine_verdicts), as
bench.py does over NCCL on GPUs. Each rank elaborates its
own shard with the product frontend; together the shards reproduce the
single-rank elaboration exactly. When the oracle is built, each rank also
checks its shard with the reference checker and the combined verdict
counts equal the single-process ones. A second 2-rank test all-gathers the
per-VC verdicts and side conditions of a sharded check (the exchange of
veq_comm_combine) and folds them into the reference's report verdict."""
import json
import os
import re
import socket
import subprocess
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
TOTAL, BLOCK = 5, 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_counts(w, blocks):
    """(pairs checked, equal VCs) of the reference checker on these CTA pairs."""
    d = tempfile.mkdtemp(prefix="veq_dist_")
    open(os.path.join(d, "a.mk"), "w").write(w.kernel_a)
    open(os.path.join(d, "b.mk"), "w").write(w.kernel_b)
    lst = []
    for b in blocks:
        p = os.path.join(d, f"cfg_{b}.cfg")
        open(p, "w").write(re.sub(r"params\.B = \d+", f"params.B = {b}", w.cfg))
        lst.append(p)
    open(os.path.join(d, "list.txt"), "w").write("\n".join(lst) + "\n")
    out = subprocess.run([HARNESS, "bench", os.path.join(d, "a.mk"), os.path.join(d, "b.mk"),
                          os.path.join(d, "list.txt"), "1", "60"], capture_output=True, text=True, timeout=300)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    return r["pairs"], r["equal"]


def _normal(bt):
    """Statement stream with batch-pool indices replaced by pool contents
    (sync sets, constants), so shards and the full grid compare directly."""
    out = []
    for st in bt.stmts.tolist():
        kind, op, arr, dst, a, b = st
        if kind == 6:  # SYNC: set contents
            q = bt.syncsets[a]
            words = tuple(int(x) for x in bt.set_words[int(q["word_off"]):int(q["word_off"]) + (int(q["n_bits"]) + 63) // 64])
            a = ("set", int(q["full"]), int(q["lo"]), int(q["n_bits"]), words)
        elif kind == 0 and op == 0:  # SETCONST: the constant
            a = ("const", int(bt.consts[a]["num"]), int(bt.consts[a]["den"]))
        out.append((kind, op, arr, dst, a, b))
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2511_12638_b200 import dist as D, frontend, workloads
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        w = workloads.c2_reduce(n_blocks=TOTAL, block=BLOCK)
        base, cnt = D.shard_blocks(TOTAL, rank, world)
        a, b, _ = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, "B", cnt, want_names=False, block_base=base)
        shards = [None] * world
        dist.all_gather_object(shards, (base, cnt, _normal(a), _normal(b)))
        pairs, equal = _oracle_counts(w, range(base, base + cnt))
        tot, ff = D.combine_verdicts([equal, pairs, 0, 0], None if equal == pairs else base)
        q.put((rank, shards, tot, ff))
    finally:
        dist.destroy_process_group()


def test_shard_blocks_partition():
    from paper_2511_12638_b200.dist import shard_blocks
    for total in (0, 1, 5, 1024, 1025):
        for world in (1, 2, 3, 8):
            got = [shard_blocks(total, r, world) for r in range(world)]
            assert sum(c for _, c in got) == total
            assert all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(world - 1))
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


@pytest.mark.skipif(not os.path.exists(HARNESS), reason="oracle not built (each rank checks its shard with it)")
def test_two_rank_gloo():
    from paper_2511_12638_b200 import frontend, workloads
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    w = workloads.c2_reduce(n_blocks=TOTAL, block=BLOCK)
    fa, fb, _ = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, "B", TOTAL, want_names=False)
    shards = res[0][1]
    assert [s[:2] for s in shards] == [(0, 3), (3, 2)]
    # the shards' statement streams concatenate to the full grid's
    assert sum((s[2] for s in shards), []) == _normal(fa)
    assert sum((s[3] for s in shards), []) == _normal(fb)
    for _, _, tot, ff in res:
        assert tot == {"equal": TOTAL, "vcs": TOTAL, "faults": 0, "missing": 0}
        assert ff is None


def _agg_worker(rank, world, port, q, gdir):
    import torch.distributed as dist
    from paper_2511_12638_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        g = json.load(open(os.path.join(gdir, "golden.json")))
        fp = g["fast_path"]
        base, cnt = D.shard_blocks(len(fp), rank, world)
        mine = [(1 if v["fast_equal"] else 0,
                 [(hash(c["denominator"]), int(c["discharged"])) for c in v["side_conditions"]])
                for v in fp[base:base + cnt]]
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        allv = [x for p in parts for x in p]  # rank order = VC order
        verdict = D.aggregate([v for v, _ in allv], [sc for _, scs in allv for sc in scs])
        q.put((rank, verdict, g["report"]["verdict"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["wl_c4_attn_l16_b2", "wl_c2_reduce_b2", "corpus_11_attn_ref__attn_opt__attn"])
def test_two_rank_report_aggregation(name):
    gdir = os.path.join(ROOT, "tests", "golden", name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agg_worker, args=(r, 2, port, q, gdir)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got, want in res:
        assert got == want
