"""The C-ABI verdict exchange (veq_comm_unique_id / veq_comm_init /
veq_comm_combine, NCCL loaded at run time) on one GPU: a single-rank NCCL
communicator must return exactly this ctx's own compare results — counters,
per-VC verdict bytes, side-condition (Merkle hash, discharged) pairs — and
folding them (dist.aggregate) must give the reference's report verdict.
Multi-rank folding is covered on CPU (tests/test_dist.py, gloo)."""
import ctypes as C
import json
import os

import pytest

from conftest import GOLDEN
from paper_2511_12638_b200 import dist as D
from paper_2511_12638_b200 import ir
from paper_2511_12638_b200 import native as N
from paper_2511_12638_b200.engine import Session

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["wl_c4_attn_l16_b2", "wl_c2_reduce_b2", "wl_c3_conv_b1"])
def test_single_rank_nccl_combine(name):
    d = os.path.join(GOLDEN, name)
    g = json.load(open(os.path.join(d, "golden.json")))
    s = Session(0, max_nodes=1 << 20, max_kid_words=1 << 22, scratch_bytes=256 << 20)
    try:
        L = N.lib()
        uid = C.create_string_buffer(128)
        assert L.veq_comm_unique_id(uid) == 0
        assert L.veq_comm_init(s.ctx, uid, 1, 0) == 0, L.veq_last_error(s.ctx).decode()
        s.declare_inputs([(x["name"], x["size"]) for x in g["inputs"]])
        a, b = ir.load(os.path.join(d, "a.veqir")), ir.load(os.path.join(d, "b.veqir"))
        ha, hb = s.load(a), s.load(b)
        s.run_pair_raw(ha, hb)
        o0 = int(a.progs[0]["array_off"])
        outs = [k for _, k in sorted((a.array_names[o0 + k], k) for k in range(int(a.progs[0]["n_arrays"]))
                                     if int(a.arrays[o0 + k]["role"]) == N.ROLE_OUT)]
        vc = s.compare_raw(ha, hb, outs, outs)
        local_eq = [int(vc.vcs[i].equal) for i in range(vc.n_vcs)]
        tot, ff, verdict, scs, voff = D.comm_combine(s, None)
        assert tot["equal"] == vc.n_equal and tot["vcs"] == vc.n_vcs
        assert list(voff) == [0, vc.n_vcs]
        assert verdict.tolist() == local_eq
        assert [d_ for _, d_ in scs] == [int(vc.sc_discharged[q]) for q in range(vc.n_sc)]
        assert ff is None
        assert D.aggregate(verdict.tolist(), scs) == g["report"]["verdict"]
    finally:
        s.close()
