"""Debug/timing helper: C3 CTA pairs through the template path with the eval
profile (python scripts/dbg_c3.py NCTAS [CI CO])."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2511_12638_b200 import frontend, ir, workloads  # noqa: E402
from paper_2511_12638_b200 import native as N  # noqa: E402
from paper_2511_12638_b200.engine import Session  # noqa: E402

n = int(sys.argv[1])
ci = int(sys.argv[2]) if len(sys.argv) > 2 else 64
co = int(sys.argv[3]) if len(sys.argv) > 3 else 64
w = workloads.c3_conv(ci, co, 256, 256, 16, 16)
ta, tb, inputs, da, db = frontend.elaborate_template(w.kernel_a, w.kernel_b, w.cfg, "B", n, want_names=False)
S = (len(ta.stmts) + len(tb.stmts)) * n
s = Session(0, max_nodes=max(1 << 22, S // 5), max_kid_words=(1 << 24) + 4 * S, scratch_bytes=8 << 30)
s.declare_inputs(inputs)
t = s.load_template(ir.concat([ta, tb]))
for rep in range(2):
    N.lib().veq_clear_terms(s.ctx)
    h = s.instantiate(t, np.concatenate([da, db], axis=1))
    N.lib().veq_set_timing(s.ctx, 1)
    out = s.run_raw(h)
    print(f"run {rep}: nodes {out.n_nodes} work {out.n_work} phases", [round(out.phase_ms[i], 1) for i in range(9)],
          flush=True)
    s.drop(h)
