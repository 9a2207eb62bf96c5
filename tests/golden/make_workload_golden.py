"""Writes reduced-size instances of the benchmark workloads (our own kernels,
paper_2511_12638_b200/workloads.py) and runs the REFERENCE checker on them
(oracle/_ref/ref_harness pair) to produce golden fixtures. Build container
only. Usage: python tests/golden/make_workload_golden.py"""
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2511_12638_b200 import workloads  # noqa: E402

H = os.path.join(ROOT, "oracle", "_ref", "ref_harness")

CASES = [
    ("wl_c2_reduce_b2", workloads.c2_reduce(n_blocks=4, block=64), 2),
    ("wl_c2_reduce_b0", workloads.c2_reduce(n_blocks=2, block=128), 0),
    ("wl_c1_matmul_n8", workloads.c1_matmul(n=8, tk=2), None),
    ("wl_c1_matmul_n16", workloads.c1_matmul(n=16, tk=4), None),
]

for name, w, blk in CASES:
    d = os.path.join(HERE, name)
    os.makedirs(d, exist_ok=True)
    cfg = w.cfg
    if blk is not None:
        cfg = re.sub(r"params\.B = \d+", f"params.B = {blk}", cfg)
    for fn, text in (("a.mk", w.kernel_a), ("b.mk", w.kernel_b), ("cfg.cfg", cfg)):
        with open(os.path.join(d, fn), "w") as f:
            f.write(text)
    subprocess.check_call([H, "pair", d, os.path.join(d, "a.mk"), os.path.join(d, "b.mk"), os.path.join(d, "cfg.cfg")])
    print(name, "ok")
