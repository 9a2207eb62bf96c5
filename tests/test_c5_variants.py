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
