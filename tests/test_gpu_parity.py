"""GPU parity: run() of every golden program through the C-ABI and compare
with the reference checker's own run() output (golden.json, produced by
oracle/_ref/ref_harness from the reference sources — tests/golden/make_golden.sh).

Compared exactly: steps, releases, outcome class, the ordered de-duplicated
race list (addresses, tids, access kinds, source locations, step numbers),
the safety list, the deadlock report, and — for fault-free runs — every
final shared-memory cell and every thread's final register file
(VEQ_OPT_KEEP_REGS) rendered by to_string of the canonical form.
"""
import json
import os

import pytest

from conftest import gen_dirs, golden_dirs
from paper_2511_12638_b200 import ir
from paper_2511_12638_b200.engine import Race, Safety

pytestmark = pytest.mark.gpu


def _race_j(r: Race):
    acc = lambda a: {"tid": a.tid, "access": a.access, "loc": {"line": a.loc[0], "col": a.loc[1]}, "step": a.step}
    return {"array": r.array, "offset": r.offset, "first": acc(r.first), "second": acc(r.second)}


def _safety_j(s: Safety):
    j = {"kind": s.kind, "tid": s.tid, "loc": {"line": s.loc[0], "col": s.loc[1]}}
    if s.array is not None:
        j["array"] = s.array
        j["offset"] = s.offset
    j.update({"reg": s.reg, "is_store": s.is_store, "detail": s.detail, "step": s.step})
    return j


def _strip(j, keys=("str",)):
    if isinstance(j, dict):
        return {k: _strip(v, keys) for k, v in j.items() if k not in keys}
    if isinstance(j, list):
        return [_strip(v, keys) for v in j]
    return j


def check_run(got, want, where):
    assert got.steps == want["steps"], where
    assert got.releases == want["releases"], where
    assert [_race_j(r) for r in got.races] == _strip(want["races"]), where
    assert [_safety_j(s) for s in got.safeties] == _strip(want["safeties"]), where
    wd = want["deadlock"]
    if wd is None:
        assert got.deadlock is None, where
    else:
        assert got.deadlock is not None, where
        gthreads = []
        for t in got.deadlock.threads:
            x = dict(t)
            if "loc" in x:
                x["loc"] = {"line": x["loc"][0], "col": x["loc"][1]}
            gthreads.append(x)
        assert gthreads == wd["threads"], where
        if "conflict_tids" in wd:
            assert list(got.deadlock.conflict_tids) == wd["conflict_tids"], where
            assert [list(x) for x in got.deadlock.conflict_sets] == wd["conflict_sets"], where
        else:
            assert got.deadlock.conflict_tids is None, where
    assert got.outcome == want["outcome"], where
    if want["outcome"] == "final":
        assert got.shared == want["shared"], where
        # Final register files (Outcome::regs, symexec.hpp:155-156), fixtures
        # of at most 256 threads
        if want.get("regs") and got.regs:
            assert got.regs == want["regs"], where


def _run_dir(session, d, sides):
    g = json.load(open(os.path.join(d, "golden.json")))
    if "elab_error" in g:
        pytest.skip("reference rejects this pair at elaboration")
    session.declare_inputs([(x["name"], x["size"]) for x in g["inputs"]])
    for side in sides:
        b = ir.load(os.path.join(d, f"{side}.veqir"))
        bid = session.load(b)
        (res,) = session.run_batch(bid)
        check_run(res, g[f"run_{side}"], f"{os.path.basename(d)}:{side}")


@pytest.mark.parametrize("d", golden_dirs("corpus_") + golden_dirs("extra_") + golden_dirs("wl_"), ids=os.path.basename)
def test_corpus_run_parity(session, d):
    _run_dir(session, d, ("a", "b"))


@pytest.mark.parametrize("d", gen_dirs(), ids=os.path.basename)
def test_generated_run_parity(session, d):
    _run_dir(session, d, ("a",))
