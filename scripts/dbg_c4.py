"""Debug/timing helper: C4 attention CTA pairs at a given size through the
template path (python scripts/dbg_c4.py SEQ D NCTAS)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2511_12638_b200 import frontend, ir, workloads  # noqa: E402
from paper_2511_12638_b200 import native as N  # noqa: E402
from paper_2511_12638_b200.engine import Session  # noqa: E402

L, D, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
w = workloads.c4_attention(L, D, 16, 16, 64)
t0 = time.time()
ta, tb, inputs, da, db = frontend.elaborate_template(w.kernel_a, w.kernel_b, w.cfg, "B", n, want_names=False)
S = (len(ta.stmts) + len(tb.stmts)) * n
print(f"elab {time.time() - t0:.1f}s S={S}", flush=True)
s = Session(0, max_nodes=min((1 << 31) - 1, max(1 << 22, S // 2)), max_kid_words=min((1 << 32) - 1, (1 << 24) + 4 * S),
            scratch_bytes=int(os.environ.get("DBG_SCRATCH_GB", "16")) << 30)
s.declare_inputs(inputs)
h = s.instantiate(s.load_template(ir.concat([ta, tb])), np.concatenate([da, db], axis=1))
N.lib().veq_set_timing(s.ctx, 1)
t1 = time.time()
out = s.run_raw(h)
print(f"run {time.time() - t1:.2f}s faults {out.n_faults} nodes {out.n_nodes} work {out.n_work} phases",
      [round(out.phase_ms[i], 1) for i in range(9)], flush=True)
o = [k for k in range(len(ta.arrays)) if int(ta.arrays[k]["role"]) == N.ROLE_OUT]
vc = s.compare_progs_raw(h, 0, h, n, n, o, o)
print(f"equal {vc.n_equal}/{vc.n_vcs} sc {vc.n_sc}", flush=True)
