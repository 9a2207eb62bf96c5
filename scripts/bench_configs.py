#!/usr/bin/env python3
"""Runs every BASELINE.json configuration family end to end on cuda:0 at a
moderate size (C1 at its full 64x64x64 size) through the public API — load,
both runs, compare — and prints one JSON line per configuration: verified
output elements per second (device steady state, inputs resident) and the
verdict census. The C2 headline is bench.py; this is coverage evidence.

  python scripts/bench_configs.py [--steps 3]
"""
import argparse
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_2511_12638_b200 import frontend, ir, workloads
    from paper_2511_12638_b200 import native as N
    from paper_2511_12638_b200.engine import Session
    from paper_2511_12638_b200.pipeline import check_batches

    cases = []
    w = workloads.c1_matmul(64, 8)
    cases.append(("C1 matmul 64x64x64 (4096 threads, naive vs smem-tiled TK=8)", w, None))
    w = workloads.c2_reduce(n_blocks=256, block=1024)
    cases.append(("C2 reduction, 256 CTA pairs x 1024", w, None))
    w = workloads.c3_conv(8, 8, 32, 32, 16, 16)
    cases.append(("C3 conv 3x3, 8->8 ch, 32x32, 16x16 tiles (4 CTAs x 256 threads)", w, None))
    w = workloads.c4_attention(128, 16, 16, 4, 32)
    cases.append(("C4 attention L=128 d=16, 16 rows x 4 threads per CTA, Bc=32 (8 CTAs)", w, None))
    variants = workloads.c5_variants(200, 16)
    cases.append(("C5 200 mutated 16x16x16 matmul variants vs the naive reference", None, variants))

    sess = Session(0, max_nodes=1 << 24, max_kid_words=1 << 27, scratch_bytes=4 << 30)
    L = N.lib()
    for name, w, var in cases:
        t0 = time.time()
        if var is None:
            a, b, inputs = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, w.block_param, w.n_blocks,
                                                   want_names=True)
        else:
            As, Bs, inputs = [], [], None
            ref = workloads.c5_reference(16)
            for kind, src, cfg in var:
                x, y, inputs = frontend.elaborate_pair(ref, src, cfg, want_names=True)
                As.append(x)
                Bs.append(y)
            a, b = ir.concat(As), ir.concat(Bs)
        t_elab = time.time() - t0
        sess.declare_inputs(inputs)
        reps = check_batches(sess, a, b)  # full report path once (verdicts)
        census = collections.Counter(r.verdict for r in reps)
        ba, bb = sess.load(a), sess.load(b)
        oa = [k for k in range(int(a.progs[0]["n_arrays"])) if int(a.arrays[k]["role"]) == N.ROLE_OUT]
        ob = [k for k in range(int(b.progs[0]["n_arrays"])) if int(b.arrays[k]["role"]) == N.ROLE_OUT]
        oa = [oa[0]] if len(oa) == 1 else oa
        ob = [ob[0]] if len(ob) == 1 else ob
        n_vcs = 0
        torch.cuda.synchronize()
        for i in range(args.steps + 1):
            if i == 1:
                torch.cuda.synchronize()
                t1 = time.perf_counter()
            assert L.veq_clear_terms(sess.ctx) == 0
            sess.run_pair_raw(ba, bb)
            vc = sess.compare_raw(ba, bb, oa, ob)
            n_vcs = vc.n_vcs
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t1) / args.steps
        print(json.dumps({"config": name, "programs": a.n_progs, "statements": int(len(a.stmts) + len(b.stmts)),
                          "output_elements": int(n_vcs), "ms_per_check": 1000 * dt,
                          "elements_per_s": n_vcs / dt if dt > 0 else None, "verdicts": dict(census),
                          "t_elaborate_s": t_elab}), flush=True)
    sess.close()


if __name__ == "__main__":
    main()
