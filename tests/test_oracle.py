"""Oracle pinning (CPU). The oracle is the reference checker itself, compiled
from /root/reference/proj/src by oracle/Makefile into oracle/_ref/ (test
infrastructure only). These tests pin it and the committed golden fixtures
it produced (tests/golden/make_golden.sh, make_workload_golden.py):

* the fixtures carry the reference's own known answers — the 15 manifest
  verdicts (proj/kernels/manifest.txt:3-17), the softmax-nosync race census
  (proj/tests/test_symexec.cpp:360-384) and the warp-deadlock report;
* when oracle/_ref is built, re-running it reproduces every workload
  fixture byte for byte (the fixtures are the oracle's output, not edited);
* when the reference's unit-test executables are built (make -C oracle
  tests), they pass on this build (138 doctest cases + 9 acceptance
  criteria, proj/tests/*.cpp)."""
import json
import os
import subprocess
import tempfile

import pytest

from conftest import GOLDEN, golden_dirs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
HARNESS = os.path.join(REF, "ref_harness")


def _g(d):
    return json.load(open(os.path.join(d, "golden.json")))


@pytest.mark.parametrize("d", golden_dirs("corpus_"), ids=os.path.basename)
def test_manifest_verdicts(d):
    expected = open(os.path.join(d, "expected_verdict")).read().strip()
    assert _g(d)["report"]["verdict"] == expected


def test_softmax_nosync_race_census():
    g = _g(os.path.join(GOLDEN, "corpus_04_softmax_naive__softmax_naive_nosync__softmax4"))
    r = g["run_b"]
    assert r["outcome"] == "race"
    first = r["races"][0]
    assert (first["array"], first["offset"]) == ("buf", 1)
    assert (first["first"]["tid"], first["first"]["access"]) == (0, "read")
    assert (first["second"]["tid"], first["second"]["access"]) == (1, "write")
    assert len(r["races"]) == 9
    assert len(r["safeties"]) == 3
    for s in r["safeties"]:
        assert (s["kind"], s["tid"], s["array"]) == ("uninitialized-memory-read", 0, "buf")
    assert g["report"]["verdict"] == "kernel-B-error"


def test_warp_deadlock_report():
    g = _g(os.path.join(GOLDEN, "corpus_08_deadlock_warps__deadlock_warps__warps8"))
    d = g["run_a"]["deadlock"]
    assert g["run_a"]["outcome"] == "deadlock"
    assert d["conflict_tids"] == [4, 6]
    assert d["conflict_sets"] == [[4, 5, 6, 7], [0, 1, 2, 3, 4, 5, 6, 7]]


def test_workload_goldens_are_closed_forms():
    # C2: the reduction output is the Add of the CTA's 64 input symbols in
    # byte order of their names; both kernels agree (fast path)
    g = _g(os.path.join(GOLDEN, "wl_c2_reduce_b2"))
    assert g["report"]["verdict"] == "equivalent"
    fp = g["fast_path"]
    assert len(fp) == 1 and fp[0]["fast_equal"]


@pytest.mark.skipif(not os.path.exists(HARNESS), reason="oracle/_ref not built (make -C oracle)")
@pytest.mark.parametrize("d", golden_dirs("wl_"), ids=os.path.basename)
def test_oracle_reproduces_fixture(d):
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([HARNESS, "pair", tmp, os.path.join(d, "a.mk"), os.path.join(d, "b.mk"),
                        os.path.join(d, "cfg.cfg")], check=True, capture_output=True, timeout=300)
        assert json.load(open(os.path.join(tmp, "golden.json"))) == _g(d)
        for f in ("a.veqir", "b.veqir"):
            assert open(os.path.join(tmp, f), "rb").read() == open(os.path.join(d, f), "rb").read(), f


REF_TESTS = ["test_expr", "test_ir", "test_frontend", "test_symexec", "test_decide", "test_pipeline"]


@pytest.mark.skipif(not all(os.path.exists(os.path.join(REF, t)) for t in REF_TESTS),
                    reason="reference unit tests not built (make -C oracle tests)")
@pytest.mark.parametrize("t", REF_TESTS)
def test_reference_unit_suite(t):
    r = subprocess.run([os.path.join(REF, t)], capture_output=True, text=True, timeout=600, cwd=REF)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout
