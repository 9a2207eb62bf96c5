"""Digest goldens at (or near) the benchmarked sizes: the REFERENCE checker
(oracle/_ref/ref_harness digest) runs full-size CTA pairs of the benchmark
workloads and records its report, CRC-32 digests of every output's canonical
to_string for both kernels, and digests of its packed-IR elaboration. Build
container only (needs /root/reference). Usage:
  python tests/golden/make_digest_golden.py [name-prefix ...]"""
import gzip
import json
import os
import re
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2511_12638_b200 import workloads  # noqa: E402

H = os.path.join(ROOT, "oracle", "_ref", "ref_harness")

CASES = [
    # C2 at the bench's exact shape: CTA pairs 0 and 1023 of the 1024-block grid
    ("dg_c2_full_b0", workloads.c2_reduce(n_blocks=1024, block=1024), 0),
    ("dg_c2_full_b1023", workloads.c2_reduce(n_blocks=1024, block=1024), 1023),
    # C1 at full size (64x64x64, 4096 threads, TK=8)
    ("dg_c1_full", workloads.c1_matmul(n=64, tk=8), None),
    # C4 with the full per-CTA shape (16 rows, 16 threads per row, key blocks
    # of 64) at reduced sequence length / head dim (SURVEY 8d CPU plan)
    ("dg_c4_l64_d16_b3", workloads.c4_attention(64, 16, 16, 16, 64), 3),
    ("dg_c4_l128_d16_b0", workloads.c4_attention(128, 16, 16, 16, 64), 0),
    ("dg_c4_l128_d32_b5", workloads.c4_attention(128, 32, 16, 16, 64), 5),
    ("dg_c4_l256_d32_b1", workloads.c4_attention(256, 32, 16, 16, 64), 1),
    # C3: one full 16x16 tile CTA (256 threads, 3x3 filters) at 32 of the 64
    # input channels (K = 288) and 2 of the 64 output channels, on a 32x32
    # image (tile 3 = bottom right): the reference keeps every partial sum of
    # every output, so the full CTA does not fit host RAM
    ("dg_c3_cta_ci32_co2_b3", workloads.c3_conv(32, 2, 32, 32, 16, 16), 3),
]


def main(prefixes):
    for name, w, blk in CASES:
        if prefixes and not any(name.startswith(p) for p in prefixes):
            continue
        d = os.path.join(HERE, name)
        os.makedirs(d, exist_ok=True)
        cfg = w.cfg
        if blk is not None:
            cfg = re.sub(r"params\.B = \d+", f"params.B = {blk}", cfg)
        for fn, text in (("a.mk", w.kernel_a), ("b.mk", w.kernel_b), ("cfg.cfg", cfg)):
            with open(os.path.join(d, fn), "w") as f:
                f.write(text)
        t0 = time.time()
        subprocess.check_call([H, "digest", d, os.path.join(d, "a.mk"), os.path.join(d, "b.mk"),
                               os.path.join(d, "cfg.cfg")])
        print(f"{name} ok ({time.time() - t0:.1f} s)", flush=True)




def c5_cases(n_variants: int = 1000, n: int = 32):
    """C5 at full size: one digest golden per distinct (variant source,
    config) of the seeded 1,000-variant generator at N = 32."""
    seen = {}
    for kind, src, cfg in workloads.c5_variants(n_variants, n):
        key = (src, cfg)
        if key not in seen:
            tk = cfg.split("params.TK = ")[1].split()[0]
            seen[key] = f"dg_c5_{kind}_tk{tk}"
    return [(name, src, cfg) for (src, cfg), name in seen.items()]


def main_c5():
    ref = workloads.c5_reference(32)
    for name, src, cfg in c5_cases():
        d = os.path.join(HERE, name)
        if os.path.exists(os.path.join(d, "golden.json.gz")):
            continue
        os.makedirs(d, exist_ok=True)
        for fn, text in (("a.mk", ref), ("b.mk", src), ("cfg.cfg", cfg)):
            with open(os.path.join(d, fn), "w") as f:
                f.write(text)
        t0 = time.time()
        subprocess.check_call([H, "digest", d, os.path.join(d, "a.mk"), os.path.join(d, "b.mk"),
                               os.path.join(d, "cfg.cfg")])
        # race reports of the racy variants run to megabytes: stored compact
        # and gzipped (conftest.load_golden reads either form)
        p = os.path.join(d, "golden.json")
        g = json.load(open(p))
        with open(p + ".gz", "wb") as f:
            f.write(gzip.compress(json.dumps(g, separators=(",", ":")).encode(), 9, mtime=0))
        os.remove(p)
        print(f"{name} ok ({time.time() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["c5"]:
        main_c5()
    else:
        main(sys.argv[1:])
