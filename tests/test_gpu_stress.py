"""Repeatability of the concurrent evaluation (GPU): persistent warps claim
work dynamically, so the interleaving of term-table inserts differs from run
to run while the canonical results may not. Each workload is checked
several times from an empty table; verdicts and the rendered canonical form
of every output cell must be identical across repetitions (and, for the
C2 CTA with a golden fixture, equal to the reference's)."""
import json
import os

import pytest

from conftest import GOLDEN
from paper_2511_12638_b200 import frontend, native as N, workloads

pytestmark = pytest.mark.gpu


def _outputs(sess, b, bid):
    """to_string of every Out cell of every program of batch b."""
    roots = []
    for p in range(b.n_progs):
        pm = b.progs[p]
        for k in range(int(pm["n_arrays"])):
            ar = b.arrays[int(pm["array_off"]) + k]
            if int(ar["role"]) == N.ROLE_OUT:
                roots += [int(x) for x in sess.fetch_cells(bid, p, k, int(ar["size"]))]
    return sess.to_strings(roots)


@pytest.mark.parametrize("name,w", [
    ("c2", workloads.c2_reduce(n_blocks=32, block=256)),
    ("c4", workloads.c4_attention(16, 4, 4, 2, 4)),
    ("c3", workloads.c3_conv(2, 3, 8, 8, 4, 4)),
])
def test_repeat_identical(session, name, w):
    a, b, inputs = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, w.block_param, w.n_blocks)
    ref = None
    for rep in range(4):
        session.declare_inputs(inputs)
        ba, bb = session.load(a), session.load(b)
        ra, rb = session.run_pair_raw(ba, bb)
        assert ra.n_faults == 0 and rb.n_faults == 0
        vc = session.compare_raw(ba, bb, [k for k in range(int(a.progs[0]["n_arrays"]))
                                          if int(a.arrays[k]["role"]) == N.ROLE_OUT],
                                 [k for k in range(int(b.progs[0]["n_arrays"]))
                                  if int(b.arrays[k]["role"]) == N.ROLE_OUT])
        assert vc.n_equal == vc.n_vcs
        outs = (_outputs(session, a, ba), _outputs(session, b, bb))
        assert outs[0] == outs[1]
        if ref is None:
            ref = outs
        else:
            assert outs == ref, (name, rep)


def test_c2_matches_reference_form(session):
    d = os.path.join(GOLDEN, "wl_c2_reduce_b2")
    g = json.load(open(os.path.join(d, "golden.json")))
    w = workloads.c2_reduce(n_blocks=4, block=64)
    a, b, inputs = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, "B", 4)
    want = g["run_a"]["shared"]["y[0]"] if "y[0]" in g["run_a"]["shared"] else None
    for _ in range(3):
        session.declare_inputs(inputs)
        ba = session.load(a)
        session.run_raw(ba)
        got = _outputs(session, a, ba)[2]
        if want is not None:
            assert got == want
