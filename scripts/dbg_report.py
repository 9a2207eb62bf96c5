"""Debug helper: our report_to_json vs the reference's for golden dirs
(python scripts/dbg_report.py DIR...); prints the first difference."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_12638_b200 import ir  # noqa: E402
from paper_2511_12638_b200.engine import Session  # noqa: E402
from paper_2511_12638_b200.pipeline import check_batches, report_to_json  # noqa: E402

s = Session(0, max_nodes=1 << 20, max_kid_words=1 << 22, scratch_bytes=256 << 20)
for d in sys.argv[1:]:
    g = json.load(open(os.path.join(d, "golden.json")))
    want = dict(g["report"])
    want.pop("timings", None)
    s.declare_inputs([(x["name"], x["size"]) for x in g["inputs"]])
    (rep,) = check_batches(s, ir.load(os.path.join(d, "a.veqir")), ir.load(os.path.join(d, "b.veqir")))
    got = report_to_json(rep, want["kernels"]["a"], want["kernels"]["b"])
    a, b = json.dumps(got), json.dumps(want)
    if a == b:
        print("MATCH", d)
        continue
    k = next(i for i in range(min(len(a), len(b))) if a[i] != b[i]) if a[:min(len(a), len(b))] != b[:min(len(a), len(b))] else min(len(a), len(b))
    print("DIFF", d, "at", k)
    print("  got :", a[max(0, k - 300):k + 200])
    print("  want:", b[max(0, k - 300):k + 200])
