"""check_equivalence over the C-ABI (mirror of proj/src/pipeline.cpp:141-267).

Given two packed-IR batches of equal length (program i of A is checked
against program i of B; one pair = one reference check_equivalence call),
runs both on the GPU, builds one VC per Out cell in array-name order
(pipeline.cpp:214-220), and assembles the reference's report: kernel errors
with their race/safety/deadlock payloads (harvest_errors, missing_output,
pipeline.cpp:62-87, 185-212), per-VC verdicts and the side-condition union
de-duplicated in VC order (pipeline.cpp:245-265).

Decision scope: the canonical fast path (decide.cpp:765-768). A VC whose
canonical forms differ is reported as "undecided" — the exp-polynomial slow
path and the MPFR witness search stay with the reference host code.
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


def _failed(rr: RunResult) -> bool:
    return not (rr.outcome == "final" and not rr.races and not rr.safeties)


def check_batches(sess: Session, a: Batch, b: Batch, render_side_conditions: bool = True) -> List[PairReport]:
    ba = sess.load(a)
    bb = sess.load(b)
    out_a, out_b = sess.run_pair_raw(ba, bb)
    ra = build_results(sess, ba, a, out_a, with_shared=False)
    rb = build_results(sess, bb, b, out_b, with_shared=False)
    reports: List[PairReport] = []
    # programs share Out array layout across the batch (same kernel pair)
    oa, ob, names = out_array_pairs(a, b, 0)
    vc = sess.compare_raw(ba, bb, oa, ob)
    n_per = vc.n_vcs // max(1, a.n_progs) if a.n_progs else 0
    sizes = []
    o0 = int(a.progs[0]["array_off"]) if a.n_progs else 0
    for k in oa:
        sizes.append(int(a.arrays[o0 + k]["size"]))
    sc_nodes = [vc.sc_node[i] for i in range(vc.n_sc)]
    uniq = sorted(set(sc_nodes))
    sc_strs = dict(zip(uniq, sess.to_strings(uniq))) if (render_side_conditions and uniq) else {}
    for p in range(a.n_progs):
        rep = PairReport(verdict="unknown")
        for side, rr in (("a", ra[p]), ("b", rb[p])):
            if _failed(rr):
                rep.verdict = f"kernel-{side.upper()}-error"
                rep.error_kernel = side
                rep.races, rep.safeties, rep.deadlock = rr.races, rr.safeties, rr.deadlock
                break
            # missing_output (pipeline.cpp:73-87): first unwritten Out cell
            base = p * n_per
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
        any_undecided = False
        residual = False
        off = 0
        base = p * n_per
        for name, sz in zip(names, sizes):
            for i in range(sz):
                v = vc.vcs[base + off + i]
                verdict = "equal" if v.equal else "undecided"
                any_undecided |= not v.equal
                rep.vcs.append({"array": name, "index": i, "verdict": verdict})
                for q in range(v.sc_off, v.sc_off + v.sc_n):
                    node = vc.sc_node[q]
                    key = sc_strs.get(node, node)
                    if key not in seen:
                        seen.add(key)
                        dis = bool(vc.sc_discharged[q])
                        rep.side_conditions.append({"denominator": sc_strs.get(node, f"#{node}"), "discharged": dis})
                        residual |= not dis
            off += sz
        rep.verdict = "undecided" if any_undecided else ("unknown" if residual else "equivalent")
        reports.append(rep)
    return reports
