#!/usr/bin/env python3
"""Summarise the ncu evidence of one GPU round-trip (scripts/gpu_check.sh)
into profiles/: the per-kernel share of one bench step from the launch list,
the key counters of the full capture of the dominant kernel, and
profiles/traffic.json (DRAM bytes per launch, read by bench.py for the
roofline `traffic` field).

  python scripts/ncu_summary.py gpurun_out/launches.csv gpurun_out/prof.ncu-rep r02_c3 eval [c3]
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
            name = d["Kernel Name"].split("(")[0]
            if "<" in name:  # library templates: keep the kernel's own name
                name = name.split("<")[0] + "<...>"
            out.append((name, us))
    return out


def one_step(ls):
    """The launches of the device-timed bench step: bench.py --steps 1
    --warmup 0 runs a correctness step, an instrumented step, the timed step,
    then the e2e steps; each ends with k_compare. The timed step is the one
    after the second k_compare."""
    idx = [i for i, (k, _) in enumerate(ls) if k.endswith("k_compare")]
    if len(idx) >= 3:
        return ls[idx[1] + 1: idx[2] + 1]
    if len(idx) >= 2:
        return ls[idx[-2] + 1: idx[-1] + 1]
    return ls


def raw_metrics(rep):
    """One dict per captured launch: metric -> (unit, value)."""
    if rep.endswith(".csv"):  # raw page already exported on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [{k: (u, v) for k, u, v in zip(r[0], r[1], row)} for row in r[2:]]


def main():
    lpath, rep, tag, phase = sys.argv[1:5]
    wl = sys.argv[5] if len(sys.argv) > 5 else "c2"
    step = one_step(launches(lpath))
    agg = collections.OrderedDict()
    for k, us in step:
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values())
    lines = [f"# {tag}: kernel launches of the device-timed {wl.upper()} bench step (ncu --metrics gpu__time_duration.sum, "
             "--clock-control none; cold-cache, serialised: compare shares, not absolutes)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    lines.append(f"| **total** | {sum(n for n, _ in agg.values())} | {tot:.1f} | 100% |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")

    ms = raw_metrics(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct",
            "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
    lines = [f"# {tag}: ncu --set full of the dominant kernel ({phase}), {len(ms)} launch(es); "
             f"each launch is one {wl.upper()} bench step's {phase} (kernel A's and kernel B's CTAs in one merged batch)", "",
             "| metric | unit | " + " | ".join(f"launch {i}" for i in range(len(ms))) + " |",
             "|---|---|" + "---|" * len(ms)]
    for k in keys:
        if ms and k in ms[0]:
            lines.append(f"| `{k}` | {ms[0][k][0]} | " + " | ".join(m[k][1] for m in ms) + " |")
    for i, m in enumerate(ms):
        stalls = sorted(((k, v) for k, (u, v) in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                         and not k.endswith("not_issued")), key=lambda x: -float(x[1].replace(",", "") or 0))[:8]
        lines += ["", f"Top stall reasons, launch {i} (pc sampling):", ""] + [f"- `{k}`: {v}" for k, v in stalls]
    open(os.path.join(ROOT, "profiles", f"{tag}_{phase}_ncu.md"), "w").write("\n".join(lines) + "\n")

    def num(m, k):
        u, v = m.get(k, ("", "0"))
        v = float(v.replace(",", "") or 0)
        return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)
    # per launch (= per step with merged batches): mean over the captured launches
    # "--sum": the captured launches are the kernels of ONE step (e.g. both
    # evaluation passes), so their traffic adds up
    per_step = "--sum" in sys.argv
    traffic = sum(num(m, "dram__bytes_read.sum") + num(m, "dram__bytes_write.sum") for m in ms) / (
        1 if per_step else max(1, len(ms)))
    tp = os.path.join(ROOT, "profiles", f"traffic_{wl}.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    t[phase] = traffic
    t[f"{phase}_source"] = (f"profiles/{tag}_{phase}_ncu.md (dram__bytes_read.sum + dram__bytes_write.sum, "
                            + (f"summed over the {len(ms)} launches of one step)" if per_step
                               else f"per launch, mean of {len(ms)} launches)"))
    json.dump(t, open(tp, "w"), indent=1)
    print(open(os.path.join(ROOT, "profiles", f"{tag}_launches.md")).read())
    print(open(os.path.join(ROOT, "profiles", f"{tag}_{phase}_ncu.md")).read())


if __name__ == "__main__":
    main()
