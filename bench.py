#!/usr/bin/env python3
"""Benchmark: output elements verified per second per kernel pair.

Workload (BASELINE.json configs[1], the metric's config): warp-shuffle tree
reduction vs sequential sum over N = 2^20 inputs, as 1024 independent CTA
pairs of 1024 elements (each CTA pair is one reference
check_equivalence). A step = execute both kernels' CTAs (by default as one
merged batch: programs 0..P-1 are kernel A's, P..2P-1 kernel B's; --separate
runs two batches) and the per-VC canonical compare on the GPU (the
reference's t_exec_a + t_exec_b + t_decide), starting from an empty term
DAG, plus the cross-rank verdict all-reduce when N > 1. Packed IR is resident in HBM for `value`; `e2e`
re-uploads it from pinned host memory every step through the C-ABI and reads
the verdicts back.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: torchrun, one rank per GPU, weak scaling (each rank owns 1024 CTA
pairs of a world-sized input).
"""
from __future__ import annotations

import argparse
import json
import os
import re
import shutil
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "output elements verified/sec per kernel pair at 1/2/4/8 B200 vs CPU ref"
HBM_FALLBACK = 6650.0


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j.get("hbm_gbs", HBM_FALLBACK)), "measured"
    return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------
def ref_bench(workload, blocks, seconds, threads):
    """The reference checker (oracle/_ref, built from the reference sources)
    on a bounded sample of the workload's CTA pairs, all host threads."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
    if not os.path.exists(exe):
        return None, "oracle/_ref/ref_harness not built"
    d = tempfile.mkdtemp(prefix="veq_ref_")
    open(os.path.join(d, "a.mk"), "w").write(workload.kernel_a)
    open(os.path.join(d, "b.mk"), "w").write(workload.kernel_b)
    lst = []
    for b in blocks:
        p = os.path.join(d, f"cfg_{b}.cfg")
        open(p, "w").write(re.sub(r"params\.B = \d+", f"params.B = {b}", workload.cfg))
        lst.append(p)
    open(os.path.join(d, "list.txt"), "w").write("\n".join(lst) + "\n")
    out = subprocess.run([exe, "bench", os.path.join(d, "a.mk"), os.path.join(d, "b.mk"),
                          os.path.join(d, "list.txt"), str(threads), str(seconds)],
                         capture_output=True, text=True, timeout=seconds * 10 + 120)
    shutil.rmtree(d, ignore_errors=True)
    if out.returncode != 0:
        return None, out.stderr.strip()[-300:]
    return json.loads(out.stdout.strip().splitlines()[-1]), None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--blocks", type=int, default=1024, help="CTA pairs per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--separate", action="store_true",
                    help="load/run kernel A's and kernel B's CTAs as two batches (default: one merged batch)")
    args = ap.parse_args()

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    from paper_2511_12638_b200 import workloads
    from paper_2511_12638_b200.dist import combine_verdicts, shard_blocks
    W = workloads.c2_reduce(n_blocks=args.blocks * world, block=1024)
    cfg_json = {"workload": "C2 warp-shuffle tree reduction vs sequential sum, N=2^20 per GPU as "
                            f"{args.blocks} CTA pairs x 1024 elements",
                "kernel_a": "reduce_seq (1 thread)", "kernel_b": "reduce_shfl (1024 threads, warp 32)",
                "cta_pairs_per_gpu": args.blocks, "elements_per_step_per_gpu": args.blocks,
                "parallelism": f"dp{world} (CTA pairs sharded, verdict all-reduce)",
                "l2": "working set re-generated every step (term table cleared; IR > 126 MB L2)"}
    ncpu = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        per = max(1, args.steps)
        samples = []
        for s in range(args.warmup + per):
            blocks = list(range((s * 8) % args.blocks, (s * 8) % args.blocks + 8))
            r, err = ref_bench(W, blocks, max(2.0, args.cpu_seconds / per), ncpu)
            if r is None:
                print(json.dumps({"impl": "reference", "unavailable": err}))
                return
            if s >= args.warmup:
                samples.append(r)
        el = sum(r["elements"] for r in samples)
        busy = sum(r["busy_s"] for r in samples) / ncpu
        v = el / busy if busy > 0 else 0.0
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s", "n_gpus": world,
            "steps": per, "warmup": args.warmup, "ms_per_step": 1000.0 * busy / per if per else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "exact rational (int64/GMP)",
            "data": "synthetic", "config": cfg_json,
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": ncpu, "kind": "reference",
                             "sample": f"{el} CTA pairs (8 per step) of the C2 grid; exec+decide span timed"},
            "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import numpy as np
    import torch
    from paper_2511_12638_b200 import frontend, ir, native as N
    from paper_2511_12638_b200.engine import Session

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    t0 = time.time()
    # weak scaling: each rank owns a contiguous share of a world-sized grid
    base, nblk = shard_blocks(args.blocks * world, rank, world)
    a, b, inputs = frontend.elaborate_pair(W.kernel_a, W.kernel_b, W.cfg, "B", nblk, want_names=False,
                                           block_base=base)
    t_elab = time.time() - t0
    S = len(a.stmts) + len(b.stmts)
    sess = Session(local, max_nodes=max(1 << 22, 4 * S // 10), max_kid_words=(1 << 24) + 4 * S,
                   scratch_bytes=8 << 30)
    L = N.lib()
    sess.declare_inputs(inputs)
    oa, ob = [0], [0]  # y is the only Out array (array-name order)
    for k, name in enumerate(a.array_names[:int(a.progs[0]["n_arrays"])]):
        if int(a.arrays[k]["role"]) == N.ROLE_OUT:
            oa = [k]
    for k, name in enumerate(b.array_names[:int(b.progs[0]["n_arrays"])]):
        if int(b.arrays[k]["role"]) == N.ROLE_OUT:
            ob = [k]
    P = a.n_progs
    # default: both kernels' CTAs in ONE batch (programs 0..P-1 = kernel A,
    # P..2P-1 = kernel B): one run carries both, and program i of A is
    # compared with program P+i (veq_compare_progs)
    merged = None if args.separate else ir.concat([a, b])

    def load_all():
        if merged is not None:
            return (sess.load(merged),)
        return (sess.load(a), sess.load(b))

    def run_all(hs):
        if len(hs) == 1:
            return [sess.run_raw(hs[0])]
        return list(sess.run_pair_raw(hs[0], hs[1]))

    def compare_all(hs):
        if len(hs) == 1:
            return sess.compare_progs_raw(hs[0], 0, hs[0], P, P, oa, ob)
        return sess.compare_raw(hs[0], hs[1], oa, ob)

    hs = load_all()
    stream = torch.cuda.ExternalStream(L.veq_stream(sess.ctx))
    counters = torch.zeros(4, dtype=torch.float64, device="cuda")

    def step():
        st = L.veq_clear_terms(sess.ctx)
        assert st == 0
        rs = run_all(hs)
        vc = compare_all(hs)
        launches = sum(r.n_launches for r in rs) + 2
        if dist is not None:
            counters[0], counters[1] = float(vc.n_equal), float(vc.n_vcs)
            dist.all_reduce(counters)
        return rs, vc, launches

    # correctness gate: every VC equal, no faults, on every rank
    rs, vc, _ = step()
    nfaults = sum(r.n_faults for r in rs)
    tot, first_fail = combine_verdicts([vc.n_equal, vc.n_vcs, nfaults, vc.n_missing],
                                       None if vc.n_equal == vc.n_vcs else base, device="cuda" if dist else None)
    ok = tot["equal"] == tot["vcs"] == args.blocks * world and tot["faults"] == 0
    if not ok:
        print(f"[bench] rank {rank}: verification failed: {vc.n_equal}/{vc.n_vcs} equal, {nfaults} faults",
              file=sys.stderr)
        sys.exit(1)
    # instrumented pass: per-phase device time (CUDA events on the ctx stream;
    # one run at a time so each run's phase events are its own)
    L.veq_set_timing(sess.ctx, 1)
    assert L.veq_clear_terms(sess.ctx) == 0
    rs_t = [sess.run_raw(h) for h in hs]
    compare_all(hs)  # each bench step ends with a compare (profile step boundaries)
    L.veq_set_timing(sess.ctx, 0)
    phases = {}
    for i, name in enumerate(N.PHASES):
        phases[name] = sum(float(r.phase_ms[i]) for r in rs_t)

    for _ in range(args.warmup):
        step()

    def timed(fn, k):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launches = 0
        for _ in range(k):
            launches += fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches

    with ClockSampler(local) as clk:
        ms, launches = timed(lambda: step()[2], args.steps)
    ms_step = ms / args.steps
    elements_step = args.blocks * world
    value = elements_step / (ms_step / 1000.0)

    # e2e: public API from pinned host buffers each step (H2D IR, D2H verdicts)
    def pin(batch):
        import ctypes
        keep = []
        for f in ("progs", "thread_stmt", "thread_nregs", "stmts", "arrays", "consts", "syncsets", "set_words"):
            arr = getattr(batch, f)
            t = torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8)).pin_memory()
            keep.append(t)
            setattr(batch, f, t.numpy().view(arr.dtype))
        return keep

    keep = pin(merged) if merged is not None else pin(a) + pin(b)
    h2d = a.nbytes() + b.nbytes()
    d2h = elements_step // world * 24

    e2e_prof = os.environ.get("VEQ_E2E_PROF") == "1"

    def e2e_step():
        tt = [time.perf_counter()]
        if e2e_prof:
            L.veq_set_timing(sess.ctx, 1)
        sess.declare_inputs(inputs)
        tt.append(time.perf_counter())
        xs = load_all()
        tt.append(time.perf_counter())
        rs = run_all(xs)
        tt.append(time.perf_counter())
        vc = compare_all(xs)
        tt.append(time.perf_counter())
        if e2e_prof:
            print("[e2e] declare %.2f load %.2f run %.2f compare %.2f ms" %
                  tuple(1000 * (tt[k + 1] - tt[k]) for k in range(4)), "| phases",
                  " ".join("%s=%.2f" % (nm, rs[-1].phase_ms[i]) for i, nm in enumerate(N.PHASES)), file=sys.stderr)
        assert vc.n_equal == vc.n_vcs
        if dist is not None:
            counters[0], counters[1] = float(vc.n_equal), float(vc.n_vcs)
            dist.all_reduce(counters)
        return sum(r.n_launches for r in rs) + 2

    e2e_step()
    e2e_k = max(1, min(args.steps, 5))
    ms_e2e, _ = timed(e2e_step, e2e_k)
    e2e_value = elements_step / (ms_e2e / e2e_k / 1000.0)

    # roofline: dominant phase, algorithmic bytes:
    #   exec 16 B per executed statement; sort+memscan 32 B per access tuple;
    #   eval 2 x (16 + 4k) per created node (written once, read once)
    peak, peak_kind = peaks()
    S_exec = sum(r.n_stmts_executed for r in rs_t)
    R = sum(r.n_access for r in rs_t)
    U_bytes = 16 * sum(r.n_new_nodes for r in rs_t) + 4 * sum(r.n_new_kid_words for r in rs_t)
    alg = {"exec": 16 * S_exec, "sort": 16 * R, "memscan": 16 * R, "eval": 2 * U_bytes}
    dom = max(phases, key=lambda k: phases[k])
    dom_bytes = alg.get(dom, 0)
    achieved = dom_bytes / (phases[dom] / 1000.0) / 1e9 if phases[dom] > 0 else 0.0
    b_min = 16 * S_exec + 2 * U_bytes + 32 * R + 16 * elements_step // world
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dom)

    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "exact rational (int64 num/den), u32 term ids", "data": "synthetic",
        "config": cfg_json,
        "e2e": {"value": e2e_value, "unit": "elements/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "peak_kind": peak_kind, "alg_bytes_per_launch": dom_bytes},
        "step_roofline": {"b_min_bytes": b_min, "achieved_gbs": b_min / (ms_step / 1000.0) / 1e9,
                          "frac": b_min / (ms_step / 1000.0) / 1e9 / peak},
        "phases_ms": phases,
        "counts": {"S": S_exec, "R": R, "new_nodes": sum(r.n_new_nodes for r in rs_t),
                   "work_items": sum(r.n_work for r in rs_t), "t_elab_s": t_elab,
                   "batches": "merged (A and B CTAs in one batch)" if merged is not None else "separate"},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ncb = max(8, min(args.blocks, 64))
        r, err = ref_bench(W, list(range(ncb)), args.cpu_seconds, ncpu)
        if r is not None:
            busy = r["busy_s"] / ncpu
            line["cpu_baseline"] = {"value": r["elements"] / busy if busy else 0.0, "unit": "elements/s",
                                    "cores": ncpu, "kind": "reference",
                                    "sample": f"{r['pairs']} of the first {ncb} CTA pairs, "
                                              f"{args.cpu_seconds:.0f}s bound, exec+decide span"}
        else:
            line["cpu_baseline"] = {"value": None, "unit": "elements/s", "cores": ncpu, "kind": "reference",
                                    "sample": f"unavailable: {err}"}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    del keep
    sess.close()


if __name__ == "__main__":
    main()
