"""GPU parity of the benchmark workload families beyond the per-fixture
tests (test_gpu_parity / test_gpu_pipeline already run every wl_* golden):

* C5 as a batch: the reference matmul replicated against one program per
  mutated variant, all in ONE batch pair (the 1,000-variant configuration's
  shape), must give each pair the verdict and fault payload the reference
  gives that variant alone (golden wl_c5_*);
* grid workloads C2/C3/C4 elaborated by the product frontend for several
  CTAs in one batch must match the reference's per-CTA fixtures for the
  CTAs that have one (block index bound per CTA)."""
import json
import os
import re

import pytest

from conftest import GOLDEN, golden_dirs
from paper_2511_12638_b200 import frontend, ir, workloads
from paper_2511_12638_b200.pipeline import check_batches
from test_gpu_parity import _race_j

pytestmark = pytest.mark.gpu


def _golden(name):
    return json.load(open(os.path.join(GOLDEN, name, "golden.json")))


def test_c5_variant_batch(session):
    dirs = golden_dirs("wl_c5_")
    assert len(dirs) == len(workloads.C5_KINDS)
    As, Bs = [], []
    for d in dirs:
        As.append(ir.load(os.path.join(d, "a.veqir")))
        Bs.append(ir.load(os.path.join(d, "b.veqir")))
    g0 = json.load(open(os.path.join(dirs[0], "golden.json")))
    session.declare_inputs([(x["name"], x["size"]) for x in g0["inputs"]])
    reps = check_batches(session, ir.concat(As), ir.concat(Bs))
    assert len(reps) == len(dirs)
    for rep, d in zip(reps, dirs):
        want = json.load(open(os.path.join(d, "golden.json")))
        rv = want["report"]["verdict"]
        # not-equivalent mutants are settled by the slow path (veq_decide:
        # witnesses at the reference's own seeds and precisions)
        assert rep.verdict == rv, d
        if rv == "not-equivalent":
            assert [v["verdict"] for v in rep.vcs] == [v["verdict"] for v in want["report"]["vcs"]], d
        if rv == "kernel-B-error":
            assert [_race_j(r) for r in rep.races] == want["report"].get("race", {}).get("pairs", []), d


@pytest.mark.parametrize("name,w,blocks", [
    ("c2", workloads.c2_reduce(n_blocks=4, block=64), {2: "wl_c2_reduce_b2"}),
    ("c3", workloads.c3_conv(2, 2, 4, 4, 2, 2), {1: "wl_c3_conv_b1", 3: "wl_c3_conv_b3"}),
    ("c4", workloads.c4_attention(8, 4, 2, 2, 4), {1: "wl_c4_attn_b1"}),
])
def test_grid_matches_per_cta_fixtures(session, name, w, blocks):
    a, b, inputs = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, w.block_param, w.n_blocks)
    session.declare_inputs(inputs)
    reps = check_batches(session, a, b)
    assert len(reps) == w.n_blocks
    for blk, gname in blocks.items():
        g = _golden(gname)
        assert reps[blk].verdict == g["report"]["verdict"], (name, blk)
        assert [v["verdict"] == "equal" for v in reps[blk].vcs] == [v["fast_equal"] for v in g["fast_path"]]
        assert reps[blk].side_conditions == g["report"]["side_conditions"], (name, blk)
    assert all(r.verdict == "equivalent" for r in reps)
