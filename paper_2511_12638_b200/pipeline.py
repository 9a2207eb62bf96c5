"""check_equivalence over the C-ABI (mirror of proj/src/pipeline.cpp:141-267).

Given two packed-IR batches of equal length (program i of A is checked
against program i of B; one pair = one reference check_equivalence call),
runs both on the GPU, builds one VC per Out cell in array-name order
(pipeline.cpp:214-220), and assembles the reference's report: kernel errors
with their race/safety/deadlock payloads (harvest_errors, missing_output,
pipeline.cpp:62-87, 185-212), per-VC verdicts and the side-condition union
de-duplicated in VC order (pipeline.cpp:245-265).

Decision: the canonical fast path on the device (decide.cpp:765-768); a VC
whose canonical forms differ goes to the slow path (veq_decide: canonical
difference on the device, exp-polynomial zero test with opaque Max atoms,
MPFR witness search — decide.cpp:728-859), seeded with fnv1a of
"array[index]" as pipeline.cpp:18-25, 226 does. `report_to_json` renders a
report in the reference's JSON schema (pipeline.cpp:305-381, timings
omitted). The one verdict the reference cannot produce is "undecided": a VC
whose difference still needs the max case split (not restated).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import native as N
from .engine import RunResult, Safety, Session, build_results
from .ir import Batch


@dataclass
class PairReport:
    verdict: str
    vcs: List[dict] = field(default_factory=list)
    error_kernel: str = ""
    error_detail: str = ""
    races: list = field(default_factory=list)
    safeties: list = field(default_factory=list)
    deadlock: Optional[object] = None
    side_conditions: List[dict] = field(default_factory=list)


def out_array_pairs(a: Batch, b: Batch, p: int) -> Tuple[List[int], List[int], List[str]]:
    """Out arrays of program p in both batches, by ascending name."""
    def outs(bt: Batch):
        pm = bt.progs[p]
        o = int(pm["array_off"])
        return {bt.array_names[o + k]: k for k in range(int(pm["n_arrays"]))
                if int(bt.arrays[o + k]["role"]) == N.ROLE_OUT}
    oa, ob = outs(a), outs(b)
    names = sorted(oa)
    return [oa[n] for n in names], [ob.get(n, 0) for n in names], names


def signature_mismatch(a: Batch, b: Batch, p: int) -> Optional[str]:
    """In/Out declarations of program p must agree between the kernels
    (proj/src/pipeline.cpp:39-60): same count per role, then name and size of
    each array in ascending name order. Scratch layout is private."""
    def decls(bt: Batch, role: int):
        pm = bt.progs[p]
        o = int(pm["array_off"])
        return sorted((bt.array_names[o + k], int(bt.arrays[o + k]["size"])) for k in range(int(pm["n_arrays"]))
                      if int(bt.arrays[o + k]["role"]) == role)
    for role, rs in ((N.ROLE_IN, "in"), (N.ROLE_OUT, "out")):
        xs, ys = decls(a, role), decls(b, role)
        if len(xs) != len(ys):
            return f"kernels declare a different number of {rs} arrays"
        for (na, sa), (nb, sb) in zip(xs, ys):
            if na != nb:
                return f"{rs} array name mismatch: {na} vs {nb}"
            if sa != sb:
                return f"{rs} array {na} size mismatch: {sa} vs {sb}"
    return None


class _VcSnap:
    """Host copy of one veq_vc_out (its buffers are ctx-owned and reused by
    the next compare call)."""

    def __init__(self, v):
        n = int(v.n_vcs)
        self.n_vcs = n
        self.vcs = []
        for i in range(n):
            x = v.vcs[i]
            self.vcs.append(N.veq_vc(x.node_a, x.node_b, x.equal, x.sc_off, x.sc_n, 0))
        self.n_sc = int(v.n_sc)
        self.sc_node = [int(v.sc_node[i]) for i in range(self.n_sc)]
        self.sc_discharged = [int(v.sc_discharged[i]) for i in range(self.n_sc)]


def _failed(rr: RunResult) -> bool:
    return not (rr.outcome == "final" and not rr.races and not rr.safeties)


def fnv1a(text: str) -> int:
    """The VC seed of check_equivalence (pipeline.cpp:18-25; note the
    reference's offset basis 1469598103934665603, one digit short of the
    textbook FNV-1a 64 constant — reproduced as is)."""
    h = 1469598103934665603
    for c in text.encode():
        h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def check_batches(sess: Session, a: Batch, b: Batch, render_side_conditions: bool = True, slow_path: bool = True,
                  trials: int = 64) -> List[PairReport]:
    ba = sess.load(a)
    bb = sess.load(b)
    out_a, out_b = sess.run_pair_raw(ba, bb)
    ra = build_results(sess, ba, a, out_a, with_shared=False)
    rb = build_results(sess, bb, b, out_b, with_shared=False)
    reports: List[PairReport] = []
    mism = [signature_mismatch(a, b, p) for p in range(a.n_progs)]
    # Out layout (array-name order) per program pair; signatures agree for
    # every pair that is compared, so A's names index B's arrays
    layouts = [out_array_pairs(a, b, p) if mism[p] is None else None for p in range(a.n_progs)]
    ref = next((l for l in layouts if l is not None), None)
    vc_of: Dict[int, Tuple[object, int]] = {}  # program -> (vc_out, first VC index of the pair)
    if ref is not None and all(l is None or l == ref for l in layouts):
        vc = _VcSnap(sess.compare_raw(ba, bb, ref[0], ref[1]))
        n_per = vc.n_vcs // max(1, a.n_progs)
        outs = [vc] * a.n_progs
        for p in range(a.n_progs):
            vc_of[p] = (vc, p * n_per)
    else:
        outs = []
        for p in range(a.n_progs):
            if layouts[p] is not None:
                # per-pair compare when Out layouts differ between pairs
                v = _VcSnap(sess.compare_progs_raw(ba, p, bb, p, 1, layouts[p][0], layouts[p][1]))
                outs.append(v)
                vc_of[p] = (v, 0)
    sc_nodes = sorted({v.sc_node[i] for v in {id(x): x for x in outs}.values() for i in range(v.n_sc)}) \
        if outs else []
    sc_strs = dict(zip(sc_nodes, sess.to_strings(sc_nodes))) if (render_side_conditions and sc_nodes) else {}
    for p in range(a.n_progs):
        rep = PairReport(verdict="unknown")
        if mism[p] is not None:
            # signature_mismatch is checked before either run (pipeline.cpp:170-176)
            rep.verdict, rep.error_kernel, rep.error_detail = "kernel-B-error", "b", mism[p]
            reports.append(rep)
            continue
        oa, ob, names = layouts[p]
        o0 = int(a.progs[p]["array_off"])
        sizes = [int(a.arrays[o0 + k]["size"]) for k in oa]
        vc, base = vc_of[p]
        for side, rr in (("a", ra[p]), ("b", rb[p])):
            if _failed(rr):
                rep.verdict = f"kernel-{side.upper()}-error"
                rep.error_kernel = side
                rep.races, rep.safeties, rep.deadlock = rr.races, rr.safeties, rr.deadlock
                break
            # missing_output (pipeline.cpp:73-87): first unwritten Out cell
            off = 0
            miss = None
            for name, sz in zip(names, sizes):
                for i in range(sz):
                    v = vc.vcs[base + off + i]
                    node = v.node_a if side == "a" else v.node_b
                    if node == N.UNSET:
                        miss = (name, i)
                        break
                off += sz
                if miss:
                    break
            if miss:
                rep.verdict = f"kernel-{side.upper()}-error"
                rep.error_kernel = side
                rep.safeties = [Safety("uninitialized-memory-read", 0, (0, 0), miss[0], miss[1],
                                       detail="output element never written")]
                break
        if rep.error_kernel:
            reports.append(rep)
            continue
        seen = set()
        any_undecided = any_ne = any_unknown = False
        residual = False
        off = 0
        for name, sz in zip(names, sizes):
            for i in range(sz):
                v = vc.vcs[base + off + i]
                entry = {"array": name, "index": i, "verdict": "equal"}
                if not v.equal:
                    if slow_path:
                        entry.update(sess.decide(v.node_a, v.node_b, fnv1a(f"{name}[{i}]"), trials))
                    else:
                        entry.update({"verdict": "undecided", "reason": "slow path not run"})
                any_undecided |= entry["verdict"] == "undecided"
                any_ne |= entry["verdict"] == "not_equal"
                any_unknown |= entry["verdict"] == "unknown"
                rep.vcs.append(entry)
                for q in range(v.sc_off, v.sc_off + v.sc_n):
                    node = vc.sc_node[q]
                    key = sc_strs.get(node, node)
                    if key not in seen:
                        seen.add(key)
                        dis = bool(vc.sc_discharged[q])
                        rep.side_conditions.append({"denominator": sc_strs.get(node, f"#{node}"), "discharged": dis})
                        residual |= not dis
            off += sz
        # aggregation (pipeline.cpp:259-265)
        rep.verdict = ("not-equivalent" if any_ne else "undecided" if any_undecided
                       else "unknown" if (any_unknown or residual) else "equivalent")
        reports.append(rep)
    return reports


_SEEDS: Dict[Tuple[Tuple[str, int], ...], "np.ndarray"] = {}


def vc_seeds(names: Sequence[str], sizes: Sequence[int]):
    """fnv1a("array[index]") of every VC of one Out layout (pipeline.cpp:226)."""
    import numpy as np
    key = tuple(zip(names, sizes))
    if key not in _SEEDS:
        _SEEDS[key] = np.array([fnv1a(f"{n}[{i}]") for n, sz in key for i in range(sz)], dtype=np.uint64)
    return _SEEDS[key]


def fan_verdicts(sess: Session, h: int, prog_a: int, prog_b0: int, m: int, out_a: Sequence[int],
                 out_b: Sequence[int], names: Sequence[str], sizes: Sequence[int], run_out, trials: int = 64,
                 reports: bool = True, n_threads: int = 0, prof: bool = False) -> List[str]:
    """Report verdicts of m candidate programs (prog_b0 ..) against one
    reference program (prog_a) that ran in the same batch h — a batch of
    generated kernel variants checked against one reference (config C5) —
    with the aggregation of check_equivalence (pipeline.cpp:185-265):
    kernel errors of A, A's missing outputs, kernel errors of B, B's missing
    outputs, then every VC decided (device fast path; the differing ones in
    one veq_decide_batch call) and the verdict by precedence not-equivalent >
    undecided > unknown (or a residual side condition) > equivalent.
    `reports`: assemble each failing program's run report (veq_run_report,
    the Collector's ordering and de-duplication) as the reference does."""
    import ctypes as C
    import time
    import numpy as np
    L = N.lib()
    tt = [time.perf_counter()]
    vc = sess.compare_fan_raw(h, prog_a, h, prog_b0, m, out_a, out_b)
    tt.append(time.perf_counter())
    n = int(vc.n_vcs)
    per = n // max(1, m)
    raw = np.ctypeslib.as_array(C.cast(vc.vcs, C.POINTER(C.c_uint32)), shape=(max(1, n) * 6,))[:n * 6].reshape(n, 6)
    na, nb, eq = raw[:, 0].copy(), raw[:, 1].copy(), raw[:, 2] != 0
    sc_off, sc_n = raw[:, 3].astype(np.int64), raw[:, 4].astype(np.int64)
    n_sc = int(vc.n_sc)
    undis = (np.ctypeslib.as_array(vc.sc_discharged, shape=(n_sc,)) == 0) if n_sc else np.zeros(0, dtype=bool)
    cs = np.concatenate([[0], np.cumsum(undis, dtype=np.int64)])
    vc_resid = (sc_n > 0) & (cs[np.minimum(sc_off + sc_n, n_sc)] - cs[np.minimum(sc_off, n_sc)] > 0)
    progs = run_out.progs

    def failed(p):
        return progs[p].n_faults > 0 or progs[p].deadlocked != 0

    a_err = failed(prog_a)
    miss_a = (na.reshape(m, per) == N.UNSET).any(axis=1)
    miss_b = (nb.reshape(m, per) == N.UNSET).any(axis=1)
    verdict: List[Optional[str]] = [None] * m
    to_report = [prog_a] if a_err else []
    for j in range(m):
        if a_err or miss_a[j]:
            verdict[j] = "kernel-A-error"
        elif failed(prog_b0 + j):
            verdict[j] = "kernel-B-error"
            to_report.append(prog_b0 + j)
        elif miss_b[j]:
            verdict[j] = "kernel-B-error"
    if reports and to_report:
        # the failing programs' reports, assembled in parallel (veq_run_reports)
        ps = (C.c_uint32 * len(to_report))(*to_report)
        outs = (N.veq_report * len(to_report))()
        st = L.veq_run_reports(sess.ctx, h, ps, len(to_report), outs)
        if st != 0:
            raise N.VeqError(st, L.veq_last_error(sess.ctx).decode())
    tt.append(time.perf_counter())
    live = np.array([v is None for v in verdict], dtype=bool)
    idx = np.nonzero(~eq & np.repeat(live, per))[0]
    kinds = sess.decide_batch(na[idx], nb[idx], vc_seeds(names, sizes)[idx % per], trials, n_threads)
    tt.append(time.perf_counter())
    if prof:
        import sys
        print("[fan_verdicts] compare %.1f ms, errors/reports %.1f ms, decide_batch (%d VCs) %.1f ms" %
              (1000 * (tt[1] - tt[0]), 1000 * (tt[2] - tt[1]), len(idx), 1000 * (tt[3] - tt[2])), file=sys.stderr)
    flag = np.zeros((m, 4), dtype=bool)  # per pair: any kind 1..3 (not_equal, unknown, undecided)
    for k in (1, 2, 3):
        flag[idx[kinds == k] // per, k] = True
    resid = vc_resid.reshape(m, per).any(axis=1)
    for j in range(m):
        if verdict[j] is None:
            verdict[j] = ("not-equivalent" if flag[j, 1] else "undecided" if flag[j, 3]
                          else "unknown" if (flag[j, 2] or resid[j]) else "equivalent")
    return verdict


def _loc_j(loc):
    return {"line": loc[0], "col": loc[1]}


def report_to_json(rep: PairReport, kernel_a: str = "a", kernel_b: str = "b") -> dict:
    """The reference's JSON report (report_to_json, pipeline.cpp:305-381)
    without the timings block; dict key order matches, so json.dumps gives
    the reference's text."""
    j = {"verdict": rep.verdict, "kernels": {"a": kernel_a, "b": kernel_b}, "vcs": [dict(v) for v in rep.vcs]}
    if rep.error_detail:
        j["error"] = {"kernel": rep.error_kernel, "detail": rep.error_detail}
    if rep.races:
        acc = lambda x: {"tid": x.tid, "access": x.access, "loc": _loc_j(x.loc), "step": x.step}
        j["race"] = {"pairs": [{"array": r.array, "offset": r.offset, "first": acc(r.first), "second": acc(r.second)}
                               for r in rep.races]}
    if rep.deadlock is not None:
        d = {"threads": []}
        for t in rep.deadlock.threads:
            tj = {"tid": t["tid"], "state": t["state"]}
            if "waiting" in t:
                tj["waiting"] = t["waiting"]
            if t["state"] == "blocked":
                tj["loc"] = _loc_j(t["loc"])
            d["threads"].append(tj)
        if rep.deadlock.conflict_tids is not None:
            d["conflict_tids"] = list(rep.deadlock.conflict_tids)
            d["conflict_sets"] = [list(x) for x in rep.deadlock.conflict_sets]
        j["deadlock"] = d
    if rep.safeties:
        faults = []
        for s in rep.safeties:
            f = {"kind": s.kind, "tid": s.tid, "loc": _loc_j(s.loc)}
            if s.array is not None:
                f["array"], f["offset"] = s.array, s.offset
            if s.reg:
                f["reg"] = s.reg
            if s.kind == "out-of-bounds":
                f["is_store"] = s.is_store
            if s.detail:
                f["detail"] = s.detail
            f["step"] = s.step
            faults.append(f)
        j["safety"] = {"faults": faults}
    j["side_conditions"] = [{"denominator": c["denominator"], "discharged": c["discharged"]}
                            for c in rep.side_conditions]
    return j
