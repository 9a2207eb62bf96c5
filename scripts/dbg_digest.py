"""Debug helper: one digest golden through the template or grid path, with
per-phase wall times (python scripts/dbg_digest.py DIR PATH [NODES KIDS])."""
import faulthandler
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from paper_2511_12638_b200 import frontend, ir  # noqa: E402
from paper_2511_12638_b200 import native as N  # noqa: E402
from paper_2511_12638_b200.engine import Session  # noqa: E402
import test_digest_parity as T  # noqa: E402

faulthandler.dump_traceback_later(int(os.environ.get("DBG_TIMEOUT", "170")), exit=True)
d, path = sys.argv[1], sys.argv[2]
t0 = time.time()
lap = lambda what: print(f"[{time.time() - t0:7.2f}s] {what}", flush=True)
g, ka, kb, cfg = T._load(d)
bp, base, nblk, me = T._grid_for(cfg)
if path == "template":
    a, b, inputs, da, db = frontend.elaborate_template(ka, kb, cfg, bp, nblk, block_base=base, want_names=False)
else:
    a, b, inputs = frontend.elaborate_pair(ka, kb, cfg, bp, nblk, block_base=base, want_names=False)
S = (len(a.stmts) + len(b.stmts)) * (nblk if path == "template" else 1)
nodes = int(sys.argv[3]) if len(sys.argv) > 3 else max(1 << 22, S)
kids = int(sys.argv[4]) if len(sys.argv) > 4 else (1 << 24) + 8 * S
lap(f"elaborated S={S}")
s = Session(0, max_nodes=nodes, max_kid_words=kids, scratch_bytes=8 << 30)
s.declare_inputs(inputs)
if path == "template":
    h = s.instantiate(s.load_template(ir.concat([a, b])), np.concatenate([da, db], axis=1))
else:
    h = s.load(ir.concat([a, b]))
lap("loaded")
N.lib().veq_set_timing(s.ctx, 1)
out = s.run_raw(h)
lap("ran: faults %d nodes %d work %d phases %s" % (out.n_faults, out.n_nodes, out.n_work,
                                                   [round(out.phase_ms[i], 2) for i in range(9)]))
pm = a.progs[0 if path == "template" else me]
o0 = int(pm["array_off"])
ks = [k for _, k in sorted((a.array_names[o0 + k], k) for k in range(int(pm["n_arrays"]))
                           if int(a.arrays[o0 + k]["role"]) == N.ROLE_OUT)]
P = nblk if path == "template" else a.n_progs
vc = s.compare_progs_raw(h, me, h, P + me, 1, ks, ks)
lap(f"compared: {vc.n_equal}/{vc.n_vcs} equal, {vc.n_sc} side conditions")
na = [vc.vcs[i].node_a for i in range(int(vc.n_vcs))]
dg = s.digests(na)
lap("digests")
ok = sum({"crc32": "%08x" % c, "len": l} == w["digest"] for (c, l), w in zip(dg, g["env_a"]))
lap(f"digest matches {ok}/{len(dg)}")
