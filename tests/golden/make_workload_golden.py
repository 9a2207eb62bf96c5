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
    # 1600 threads: exercises the block scheduler for CTAs above 1024 threads
    ("wl_c1_matmul_n33", workloads.c1_matmul(n=33, tk=11), None),
    # C3 conv at reduced shapes (CI, CO, H, W, tile)
    ("wl_c3_conv_b1", workloads.c3_conv(2, 2, 4, 4, 2, 2), 1),
    ("wl_c3_conv_b3", workloads.c3_conv(2, 2, 4, 4, 2, 2), 3),
    ("wl_c3_conv_c3_b2", workloads.c3_conv(3, 2, 8, 8, 4, 4), 2),
    # C4 attention at reduced shapes (L, D, rows, threads per row, key block)
    ("wl_c4_attn_b1", workloads.c4_attention(8, 4, 2, 2, 4), 1),
    ("wl_c4_attn_l16_b2", workloads.c4_attention(16, 4, 4, 2, 4), 2),
    ("wl_c4_attn_l12_b0", workloads.c4_attention(12, 2, 2, 1, 4), 0),
]
# C5: the first variant of every mutation kind of the seeded generator, N=4
_seen = {}
for _kind, _src, _cfg in workloads.c5_variants(400, 4):
    _seen.setdefault(_kind, (_src, _cfg))
C5 = [(f"wl_c5_{k}", _seen[k]) for k in workloads.C5_KINDS if k in _seen]


def _write(name, ka, kb, cfg):
    d = os.path.join(HERE, name)
    os.makedirs(d, exist_ok=True)
    for fn, text in (("a.mk", ka), ("b.mk", kb), ("cfg.cfg", cfg)):
        with open(os.path.join(d, fn), "w") as f:
            f.write(text)
    subprocess.check_call([H, "pair", d, os.path.join(d, "a.mk"), os.path.join(d, "b.mk"), os.path.join(d, "cfg.cfg")])
    print(name, "ok")


for name, (src, cfg) in C5:
    _write(name, workloads.c5_reference(4), src, cfg)

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
