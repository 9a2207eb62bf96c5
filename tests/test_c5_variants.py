"""Config 5: a batch of 1,000 generated kernel variants
against one reference kernel at N = 32 (workloads.c5_variants, seeded).

The generator yields 48 distinct (variant source, config) pairs; the
reference checker (oracle/_ref/ref_harness digest) ran each once and its
report is the golden (tests/golden/dg_c5_*, written by
make_digest_golden.py c5). Every one of the 1,000 variants is one of them,
so per-pair parity is parity on the whole batch.

CPU: the generator still yields exactly the goldens' sources, and the
product frontend's packed IR of every pair is byte-identical to the
reference's elaboration (CRC-32 + length).

GPU: each pair checked through the pipeline (check_batches: device run,
race scan, safety faults, compare, slow path) gives the reference's JSON
report byte for byte (report_to_json, timings omitted) — verdicts, race
pairs in Collector order, safety faults, counterexamples."""
import json
import os
import zlib
from collections import Counter

import pytest

from conftest import GOLDEN, golden_dirs, load_golden
from paper_2511_12638_b200 import frontend, workloads

DIRS = golden_dirs("dg_c5_")


def _case_name(kind, cfg):
    tk = cfg.split("params.TK = ")[1].split()[0]
    return f"dg_c5_{kind}_tk{tk}"


def _src(d, f):
    return open(os.path.join(d, f)).read()


def test_generator_matches_goldens():
    ref = workloads.c5_reference(32)
    seen = {}
    for kind, src, cfg in workloads.c5_variants(1000, 32):
        seen.setdefault((src, cfg), _case_name(kind, cfg))
    assert sorted(seen.values()) == sorted(os.path.basename(d) for d in DIRS)
    for (src, cfg), name in seen.items():
        d = os.path.join(GOLDEN, name)
        assert _src(d, "a.mk") == ref
        assert _src(d, "b.mk") == src
        assert _src(d, "cfg.cfg") == cfg


def test_verdict_tally():
    """The 1,000-variant verdict tally the reference reports (from the
    goldens): every racy, out-of-bounds and mis-indexed variant is caught."""
    verdict = {os.path.basename(d): load_golden(d)["report"]["verdict"] for d in DIRS}
    tally = Counter(verdict[_case_name(k, c)] for k, _, c in workloads.c5_variants(1000, 32))
    assert sum(tally.values()) == 1000
    kinds = Counter(k for k, _, _ in workloads.c5_variants(1000, 32))
    # semantics-preserving rewrites are equivalent; the rest are not
    assert tally["equivalent"] == sum(kinds[k] for k in ("tiled", "colmajor", "reverse_k", "unroll2"))
    assert tally["equivalent"] < 1000


def _dig(b: bytes):
    return {"crc32": "%08x" % zlib.crc32(b), "len": len(b)}


@pytest.mark.parametrize("d", DIRS, ids=os.path.basename)
def test_elaboration_matches_reference(d):
    g = load_golden(d)
    a, b, inputs = frontend.elaborate_pair(_src(d, "a.mk"), _src(d, "b.mk"), _src(d, "cfg.cfg"))
    assert inputs == [(x["name"], x["size"]) for x in g["inputs"]]
    assert _dig(a.image) == g["ir_a"]
    assert _dig(b.image) == g["ir_b"]


@pytest.mark.gpu
@pytest.mark.parametrize("d", DIRS, ids=os.path.basename)
def test_report_matches_reference(d):
    from paper_2511_12638_b200.engine import Session
    from paper_2511_12638_b200.pipeline import check_batches, report_to_json
    g = load_golden(d)
    want = dict(g["report"])
    want.pop("timings", None)
    a, b, inputs = frontend.elaborate_pair(_src(d, "a.mk"), _src(d, "b.mk"), _src(d, "cfg.cfg"))
    s = Session(0, max_nodes=1 << 22, max_kid_words=1 << 24, scratch_bytes=1 << 30, keep_regs=True)
    try:
        s.declare_inputs(inputs)
        (rep,) = check_batches(s, a, b)
        got = report_to_json(rep, want["kernels"]["a"], want["kernels"]["b"])
    finally:
        s.close()
    assert got["verdict"] == want["verdict"]
    for k in ("race", "safety", "deadlock", "vcs", "side_conditions", "error"):
        assert got.get(k) == want.get(k), k
    assert json.dumps(got) == json.dumps(want)


@pytest.mark.gpu
def test_fan_verdicts_match_reference():
    """bench.py's C5 path (reference kernel once + a batch of variants,
    veq_compare_fan, veq_decide_batch via pipeline.fan_verdicts) on the first
    160 variants of the batch: every verdict equals the reference's."""
    from paper_2511_12638_b200 import ir
    from paper_2511_12638_b200 import native as N
    from paper_2511_12638_b200.engine import Session
    from paper_2511_12638_b200.pipeline import fan_verdicts, out_array_pairs
    verdict = {os.path.basename(d): load_golden(d)["report"]["verdict"] for d in DIRS}
    variants = workloads.c5_variants(1000, 32)[:160]
    ref = workloads.c5_reference(32)
    cache, a0, inputs = {}, None, None
    for _, src, cfg in variants:
        if (src, cfg) not in cache:
            a, b, inputs = frontend.elaborate_pair(ref, src, cfg, want_names=False)
            a0 = a if a0 is None else a0
            assert bytes(a.image) == bytes(a0.image)
            cache[(src, cfg)] = b
    batch = ir.concat([a0] + [cache[(src, cfg)] for _, src, cfg in variants])
    S = len(batch.stmts)
    s = Session(0, max_nodes=max(1 << 22, S // 5), max_kid_words=(1 << 24) + 4 * S, scratch_bytes=4 << 30)
    try:
        s.declare_inputs(inputs)
        h = s.load(batch)
        oa, ob, names = out_array_pairs(a0, cache[(variants[0][1], variants[0][2])], 0)
        o0 = int(a0.progs[0]["array_off"])
        sizes = [int(a0.arrays[o0 + k]["size"]) for k in oa]
        for _ in range(2):  # the same batch re-run after clearing the term table
            assert N.lib().veq_clear_terms(s.ctx) == 0
            r = s.run_raw(h)
            got = fan_verdicts(s, h, 0, 1, len(variants), oa, ob, names, sizes, r)
            want = [verdict[_case_name(k, c)] for k, _, c in variants]
            assert got == want
    finally:
        s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dg_c5_index_bug_tk4", "dg_c5_wrong_guard_tk8"])
def test_decide_batch_matches_reference(name):
    """veq_decide_batch (one device launch for all differences, host
    decisions on a thread pool) gives every VC the reference's verdict."""
    import numpy as np
    from paper_2511_12638_b200 import native as N
    from paper_2511_12638_b200.engine import Session
    from paper_2511_12638_b200.pipeline import out_array_pairs, vc_seeds
    d = os.path.join(GOLDEN, name)
    g = load_golden(d)
    a, b, inputs = frontend.elaborate_pair(_src(d, "a.mk"), _src(d, "b.mk"), _src(d, "cfg.cfg"), want_names=False)
    s = Session(0, max_nodes=1 << 22, max_kid_words=1 << 24, scratch_bytes=1 << 30)
    try:
        s.declare_inputs(inputs)
        ba, bb = s.load(a), s.load(b)
        s.run_pair_raw(ba, bb)
        oa, ob, names = out_array_pairs(a, b, 0)
        vc = s.compare_raw(ba, bb, oa, ob)
        n = int(vc.n_vcs)
        f = np.array([vc.vcs[i].node_a for i in range(n)], dtype=np.uint32)
        gg = np.array([vc.vcs[i].node_b for i in range(n)], dtype=np.uint32)
        sizes = [int(a.arrays[int(a.progs[0]["array_off"]) + k]["size"]) for k in oa]
        kinds = s.decide_batch(f, gg, vc_seeds(names, sizes), 64)
        assert [N.VERDICT_KIND[k] for k in kinds] == [v["verdict"] for v in g["report"]["vcs"]]
        # single-VC API agrees on a sample
        for i in (0, n // 2, n - 1):
            assert s.decide(int(f[i]), int(gg[i]), int(vc_seeds(names, sizes)[i]))["verdict"] == N.VERDICT_KIND[kinds[i]]
    finally:
        s.close()
