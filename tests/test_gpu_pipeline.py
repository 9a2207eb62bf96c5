"""GPU parity of the whole check (reference check_equivalence report,
pipeline.cpp:141-267) on the reference corpus (kernels/manifest.txt) and
extra pairs. Exact when the reference decides on the canonical fast path or
a kernel fails; for pairs the reference settles on its host slow path, the
per-VC fast-path bit (canonical forms identical) must match instead."""
import json
import os

import pytest

from conftest import golden_dirs
from paper_2511_12638_b200 import ir
from paper_2511_12638_b200.pipeline import check_batches
from test_gpu_parity import _race_j, _safety_j

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", golden_dirs("corpus_") + golden_dirs("extra_") + golden_dirs("wl_"), ids=os.path.basename)
def test_check_report_parity(session, d):
    g = json.load(open(os.path.join(d, "golden.json")))
    rep_ref = g["report"]
    if "elab_error" in g:
        pytest.skip("rejected by the reference frontend")
    session.declare_inputs([(x["name"], x["size"]) for x in g["inputs"]])
    a = ir.load(os.path.join(d, "a.veqir"))
    b = ir.load(os.path.join(d, "b.veqir"))
    (rep,) = check_batches(session, a, b)
    if rep_ref["verdict"] in ("kernel-A-error", "kernel-B-error"):
        assert rep.verdict == rep_ref["verdict"]
        assert [_race_j(r) for r in rep.races] == rep_ref.get("race", {}).get("pairs", [])
        want_s = rep_ref.get("safety", {}).get("faults", [])
        got_s = []
        for s in rep.safeties:
            j = _safety_j(s)
            # report_to_json omits empty reg/detail and is_store unless OOB
            if not j["reg"]:
                del j["reg"]
            if not j["detail"]:
                del j["detail"]
            if s.kind != "out-of-bounds":
                del j["is_store"]
            got_s.append(j)
        assert got_s == want_s
        return
    fp = g["fast_path"]
    assert len(rep.vcs) == len(fp)
    for v, w in zip(rep.vcs, fp):
        assert (v["array"], v["index"]) == (w["array"], w["index"])
        assert (v["verdict"] == "equal") == w["fast_equal"], (v, w)
    if all(w["fast_equal"] for w in fp):
        assert rep.verdict == rep_ref["verdict"]
        assert [x["verdict"] for x in rep.vcs] == [x["verdict"] for x in rep_ref["vcs"]]
        assert rep.side_conditions == rep_ref["side_conditions"]
    else:
        assert rep.verdict == "undecided"
