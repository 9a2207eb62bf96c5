"""Debug helper: C2 grid of n_blocks CTA pairs of `block` elements through
the grid path (python scripts/dbg_c2.py BLOCK NBLOCKS)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_12638_b200 import frontend, ir, workloads  # noqa: E402
from paper_2511_12638_b200.engine import Session  # noqa: E402

bs, nb = int(sys.argv[1]), int(sys.argv[2])
w = workloads.c2_reduce(n_blocks=max(nb, 2), block=bs)
a, b, inputs = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, "B", nb, want_names=False)
s = Session(0, max_nodes=1 << 22, max_kid_words=1 << 25, scratch_bytes=8 << 30)
s.declare_inputs(inputs)
h = s.load(ir.concat([a, b]))
try:
    out = s.run_raw(h)
    print("bs", bs, "nb", nb, "ok nodes", out.n_nodes, "work", out.n_work, flush=True)
except Exception as e:
    print("bs", bs, "nb", nb, "FAIL", str(e)[-80:], flush=True)
