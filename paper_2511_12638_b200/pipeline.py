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
