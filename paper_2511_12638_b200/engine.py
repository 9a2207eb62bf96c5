"""Host-side mirror of the reference's run()/check interface over the C-ABI.

`Session` wraps one veq_ctx (one GPU). `run_batch` executes every program of
a batch on the device and rebuilds, per program, the reference's RunResult
(proj/include/ctaeq/symexec.hpp:214-225): ordered, de-duplicated race and
safety reports (Collector, symexec.cpp:308-328), the deadlock report
(make_deadlock_report, symexec.cpp:335-365), the outcome precedence
(symexec.cpp:838-845) and, for fault-free runs, the final shared memory with
canonical values rendered by the reference's to_string (expr.cpp:735-822).
All value computation happens on the GPU; this module only formats.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import native as N
from .ir import Batch

SAFETY_KIND = ["uninitialized-register-read", "uninitialized-memory-read", "out-of-bounds", "invalid-arithmetic"]
DETAIL = {
    N.DETAIL_NONE: "",
    N.DETAIL_NEGINF_ADD: "-inf is not a valid operand of Add",
    N.DETAIL_NEGINF_MUL: "-inf is not a valid operand of Mul",
    N.DETAIL_NEGINF_NEG: "-inf is not a valid operand of Neg",
    N.DETAIL_NEGINF_DIV: "-inf is not a valid operand of Div",
    N.DETAIL_NEGINF_EXP: "-inf is not a valid operand of Exp",
    N.DETAIL_ZERO_DEN: "zero denominator",
}


def _check(ctx, status: int):
    if status != 0:
        L = N.lib()
        msg = L.veq_last_error(ctx).decode() if ctx else ""
        raise N.VeqError(status, f"{L.veq_strerror(status).decode()}: {msg}")


@dataclass
class Access:
    tid: int
    access: str
    loc: Tuple[int, int]
    step: int


@dataclass
class Race:
    array: str
    offset: int
    first: Access
    second: Access


@dataclass
class Safety:
    kind: str
    tid: int
    loc: Tuple[int, int]
    array: Optional[str] = None
    offset: Optional[int] = None
    reg: str = ""
    is_store: bool = False
    detail: str = ""
    step: int = 0


@dataclass
class Deadlock:
    threads: List[dict]
    conflict_tids: Optional[Tuple[int, int]] = None
    conflict_sets: Optional[Tuple[List[int], List[int]]] = None


@dataclass
class RunResult:
    steps: int
    releases: int
    races: List[Race]
    safeties: List[Safety]
    deadlock: Optional[Deadlock]
    outcome: str
    shared: Dict[str, str] = field(default_factory=dict)       # addr -> to_string (Final only)
    cell_nodes: Dict[Tuple[int, int], int] = field(default_factory=dict)  # (array idx, offset) -> node


class Session:
    """One veq_ctx: a term table on one GPU plus its loaded batches."""

    def __init__(self, device: int = 0, max_nodes: int = 0, max_kid_words: int = 0, scratch_bytes: int = 0):
        L = N.lib()
        lim = N.veq_limits(max_nodes, max_kid_words, scratch_bytes)
        h = C.c_void_p()
        st = L.veq_open(device, C.byref(lim), C.byref(h))
        if st != 0:
            raise N.VeqError(st, L.veq_strerror(st).decode())
        self.ctx = h
        self.inputs: List[Tuple[str, int]] = []
        self._batches: List[Optional[Batch]] = []
        self._templates: List[Batch] = []

    def close(self):
        if self.ctx:
            N.lib().veq_close(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- session / batches
    def declare_inputs(self, inputs: Sequence[Tuple[str, int]]):
        arr = (N.veq_input_desc * max(1, len(inputs)))()
        keep = []
        for i, (name, size) in enumerate(inputs):
            b = name.encode()
            keep.append(b)
            arr[i].name = b
            arr[i].size = size
        _check(self.ctx, N.lib().veq_declare_inputs(self.ctx, arr, len(inputs)))
        self.inputs = list(inputs)
        self._batches = []
        self._templates = []

    def load(self, batch: Batch) -> int:
        d = batch.desc()
        h = C.c_uint32()
        _check(self.ctx, N.lib().veq_load_batch(self.ctx, C.byref(d), C.byref(h)))
        while len(self._batches) <= h.value:
            self._batches.append(None)
        self._batches[h.value] = batch
        return h.value

    def drop(self, bid: int):
        """Free a batch's device memory now (veq_drop_batch)."""
        _check(self.ctx, N.lib().veq_drop_batch(self.ctx, bid))
        self._batches[bid] = None

    def load_template(self, template: Batch) -> int:
        """Grid template to the device once (veq_load_template)."""
        d = template.desc()
        h = C.c_uint32()
        _check(self.ctx, N.lib().veq_load_template(self.ctx, C.byref(d), C.byref(h)))
        self._templates.append(template)
        return h.value

    def instantiate(self, tid: int, deltas: np.ndarray, meta: Optional[Batch] = None) -> int:
        """n_inst = deltas.shape[0] instances of template `tid` as one batch
        (veq_instantiate); deltas[i] holds instance i's shift of every
        template array. `meta` (optional) is a host Batch whose names and
        locations reports should use for the result."""
        dl = np.ascontiguousarray(deltas, dtype=np.int32)
        h = C.c_uint32()
        _check(self.ctx, N.lib().veq_instantiate(self.ctx, tid, dl.shape[0], dl.ctypes.data_as(C.POINTER(C.c_int32)),
                                                 C.byref(h)))
        while len(self._batches) <= h.value:
            self._batches.append(None)
        self._batches[h.value] = meta
        return h.value

    def run_raw(self, bid: int) -> N.veq_run_out:
        out = N.veq_run_out()
        _check(self.ctx, N.lib().veq_run(self.ctx, bid, C.byref(out)))
        return out

    def run_pair_raw(self, ba: int, bb: int) -> Tuple[N.veq_run_out, N.veq_run_out]:
        """Both runs of a check enqueued back to back (veq_run_start ×2, then
        veq_run_finish ×2): the device runs kernel B's batch right after
        kernel A's with no host round trip in between."""
        L = N.lib()
        oa, ob = N.veq_run_out(), N.veq_run_out()
        _check(self.ctx, L.veq_run_start(self.ctx, ba))
        st = L.veq_run_start(self.ctx, bb)
        ra = L.veq_run_finish(self.ctx, ba, C.byref(oa))
        if st == 0:
            _check(self.ctx, L.veq_run_finish(self.ctx, bb, C.byref(ob)))
        _check(self.ctx, ra)
        _check(self.ctx, st)
        return oa, ob

    def compare_progs_raw(self, ba: int, pa0: int, bb: int, pb0: int, n_pairs: int, out_a: Sequence[int],
                          out_b: Sequence[int]) -> N.veq_vc_out:
        n = len(out_a)
        A = (C.c_uint32 * max(1, n))(*out_a)
        B = (C.c_uint32 * max(1, n))(*out_b)
        out = N.veq_vc_out()
        _check(self.ctx, N.lib().veq_compare_progs(self.ctx, ba, pa0, bb, pb0, n_pairs, A, B, n, C.byref(out)))
        return out

    def compare_raw(self, ba: int, bb: int, out_a: Sequence[int], out_b: Sequence[int]) -> N.veq_vc_out:
        n = len(out_a)
        A = (C.c_uint32 * max(1, n))(*out_a)
        B = (C.c_uint32 * max(1, n))(*out_b)
        out = N.veq_vc_out()
        _check(self.ctx, N.lib().veq_compare(self.ctx, ba, bb, A, B, n, C.byref(out)))
        return out

    def fetch_cells(self, bid: int, prog: int, array: int, n: int) -> np.ndarray:
        out = np.empty(max(n, 1), dtype=np.uint32)
        _check(self.ctx, N.lib().veq_fetch_cells(self.ctx, bid, prog, array,
                                                 out.ctypes.data_as(C.POINTER(C.c_uint32)), n))
        return out[:n]

    # -- DAG export and rendering
    def to_strings(self, roots: Sequence[int]) -> List[str]:
        """to_string of each root (veq_render: C++ over the device DAG)."""
        if not roots:
            return []
        r = (C.c_uint32 * len(roots))(*roots)
        text = C.c_char_p()
        offs = C.POINTER(C.c_uint64)()
        _check(self.ctx, N.lib().veq_render(self.ctx, r, len(roots), C.byref(text), C.byref(offs)))
        n = len(roots)
        o = np.ctypeslib.as_array(offs, shape=(n + 1,)).copy()
        raw = C.string_at(text, int(o[n]))
        return [raw[int(o[i]):int(o[i + 1])].decode() for i in range(n)]

    def digests(self, roots: Sequence[int]) -> List[Tuple[int, int]]:
        """(CRC-32, byte length) of each root's to_string (veq_render_digest)."""
        n = len(roots)
        if not n:
            return []
        r = (C.c_uint32 * n)(*roots)
        crc = np.zeros(n, np.uint32)
        ln = np.zeros(n, np.uint64)
        _check(self.ctx, N.lib().veq_render_digest(self.ctx, r, n, crc.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                   ln.ctypes.data_as(C.POINTER(C.c_uint64))))
        return [(int(a), int(b)) for a, b in zip(crc, ln)]

    def to_strings_py(self, roots: Sequence[int]) -> List[str]:
        """Reference Python rendering over veq_export_dag (cross-check of veq_render)."""
        if not roots:
            return []
        L = N.lib()
        r = (C.c_uint32 * len(roots))(*roots)
        buf = N.veq_dag_buf()
        _check(self.ctx, L.veq_export_dag(self.ctx, r, len(roots), C.byref(buf)))
        nn, nk = buf.n_nodes, buf.n_kids
        nodes = (N.veq_dag_node * max(1, nn))()
        kids = (C.c_uint32 * max(1, nk))()
        ridx = (C.c_uint32 * len(roots))()
        buf.cap_nodes, buf.cap_kids = nn, nk
        buf.nodes, buf.kids, buf.root_index = nodes, kids, ridx
        _check(self.ctx, L.veq_export_dag(self.ctx, r, len(roots), C.byref(buf)))
        return render(nodes, kids, [ridx[i] for i in range(len(roots))], self.inputs)

    # -- run(): RunResult per program of a batch
    def run_batch(self, bid: int, with_shared: bool = True) -> List[RunResult]:
        b = self._batches[bid]
        out = self.run_raw(bid)
        return build_results(self, bid, b, out, with_shared)


# ---------------------------------------------------------------------------
def render(nodes, kids, roots: List[int], inputs: Sequence[Tuple[str, int]]) -> List[str]:
    """to_string of exported DAG nodes (expr.cpp:735-822)."""
    memo: Dict[Tuple[int, int], str] = {}

    def prec(k):
        return {N.K_ADD: 1, N.K_MUL: 2, N.K_DIV: 2, N.K_NEG: 3}.get(k, 4)

    def rat(num, den):
        return str(num) if den == 1 else f"{num}/{den}"

    def pr(i: int, ctx: int) -> str:
        key = (i, ctx)
        if key in memo:
            return memo[key]
        n = nodes[i]
        k = n.kind
        ks = [kids[n.kid_off + j] for j in range(n.nkids)]
        if k == N.K_CONST:
            s = rat(n.num, n.den)
        elif k == N.K_VAR:
            s = f"{inputs[n.var_input][0]}_{n.var_index}" if n.var_input >= 0 else f"!undef<{n.var_index:x}>"
        elif k == N.K_NEGINF:
            s = "-inf"
        elif k == N.K_ADD:
            s = " + ".join(pr(x, 2) for x in ks)
        elif k == N.K_MUL:
            s = "*".join(pr(x, 3) for x in ks)
        elif k == N.K_DIV:
            s = pr(ks[0], 3) + " / " + pr(ks[1], 3)
        elif k == N.K_NEG:
            s = "-" + pr(ks[0], 3)
        elif k == N.K_EXP:
            s = "exp(" + pr(ks[0], 0) + ")"
        elif k == N.K_MAX:
            s = "max(" + ", ".join(pr(x, 0) for x in ks) + ")"
        else:
            raise ValueError(f"bad kind {k}")
        if prec(k) < ctx:
            s = "(" + s + ")"
        memo[key] = s
        return s

    import sys
    sys.setrecursionlimit(max(10000, sys.getrecursionlimit()))
    return [pr(r, 0) for r in roots]


def _set_tids(b: Batch, s: int, n_threads: int) -> List[int]:
    if s >= len(b.syncsets):  # the device's full-set id (veq.h: n_syncsets)
        return list(range(n_threads))
    q = b.syncsets[s]
    if q["full"]:
        return list(range(n_threads))
    out = []
    for k in range(int(q["n_bits"])):
        if (int(b.set_words[int(q["word_off"]) + k // 64]) >> (k % 64)) & 1:
            out.append(int(q["lo"]) + k)
    return out


def build_results(sess: Session, bid: int, b: Batch, out: N.veq_run_out, with_shared: bool) -> List[RunResult]:
    nf = out.n_faults
    faults = np.ctypeslib.as_array(out.faults, shape=(nf,)).copy() if nf else []
    per_prog: Dict[int, list] = {}
    for f in faults:
        per_prog.setdefault(int(f["prog"]), []).append(f)
    results = []
    T = out.n_threads_total
    th_state = np.ctypeslib.as_array(out.thread_state, shape=(T,)).copy() if T else np.zeros(0, np.uint8)
    th_set = np.ctypeslib.as_array(out.thread_block_set, shape=(T,)).copy() if T else np.zeros(0, np.uint32)
    th_stmt = np.ctypeslib.as_array(out.thread_block_stmt, shape=(T,)).copy() if T else np.zeros(0, np.uint64)
    for p in range(out.n_progs):
        pr = out.progs[p]
        pm = b.progs[p]
        t_off, a_off = int(pm["thread_off"]), int(pm["array_off"])
        nthr = int(pm["n_threads"])
        aname = lambda a: b.array_names[a_off + int(a)]
        fl = sorted(per_prog.get(p, []), key=lambda f: (int(f["step"]), int(f["sub"])))
        races, safeties = [], []
        rkeys, skeys = set(), set()
        for f in fl:
            stmt = int(f["stmt"])
            if f["type"] == N.FAULT_RACE:
                first = Access(int(f["tid2"]), "write" if f["is_write2"] else "read", b.loc(int(f["stmt2"])),
                               int(f["step2"]))
                second = Access(int(f["tid"]), "write" if f["is_write"] else "read", b.loc(stmt), int(f["step"]))
                r = Race(aname(f["arr"]), int(f["offset"]), first, second)
                key = (r.array, r.offset, first.tid, first.access, first.loc, second.tid, second.access, second.loc)
                if key not in rkeys:
                    rkeys.add(key)
                    races.append(r)
            else:
                kind = int(f["kind"])
                st = b.stmts[stmt]
                gt = t_off + int(f["tid"])
                s = Safety(SAFETY_KIND[kind], int(f["tid"]), b.loc(stmt), step=int(f["step"]))
                if kind == N.SAFE_UNINIT_REG:
                    reg = int(st["b"]) if f["reg_slot"] == 1 else (int(st["dst"]) if st["kind"] == N.ST_STORE
                                                                     else int(st["a"]))
                    s.reg = b.reg_name(gt, reg)
                elif kind in (N.SAFE_UNINIT_MEM, N.SAFE_OOB):
                    s.array, s.offset = aname(f["arr"]), int(f["offset"])
                    s.is_store = bool(f["is_write"]) if kind == N.SAFE_OOB else False
                else:
                    s.reg = b.reg_name(gt, int(st["dst"]))
                    s.detail = DETAIL[int(f["detail"])]
                key = (s.kind, s.tid, s.loc, (s.array, s.offset) if s.array is not None else s.reg, s.is_store,
                       s.detail)
                if key not in skeys:
                    skeys.add(key)
                    safeties.append(s)
        dl = None
        if pr.deadlocked:
            threads = []
            for t in range(nthr):
                g = t_off + t
                state = {0: "runnable", 1: "blocked", 2: "returned"}[int(th_state[g])]
                tj = {"tid": t, "state": state}
                if state == "blocked":
                    tj["waiting"] = _set_tids(b, int(th_set[g]), nthr)
                    tj["loc"] = b.loc(int(th_stmt[g]))
                threads.append(tj)
            dl = Deadlock(threads)
            for a in range(nthr):
                if threads[a]["state"] != "blocked" or dl.conflict_tids:
                    continue
                for c in range(a + 1, nthr):
                    if threads[c]["state"] != "blocked":
                        continue
                    ia, ic = set(threads[a]["waiting"]), set(threads[c]["waiting"])
                    if ia != ic and a in ia and a in ic and c in ia and c in ic:
                        dl.conflict_tids = (a, c)
                        dl.conflict_sets = (sorted(ia), sorted(ic))
                        break
        outcome = "race" if races else ("safety" if safeties else ("deadlock" if dl else "final"))
        rr = RunResult(int(pr.steps), int(pr.releases), races, safeties, dl, outcome)
        if outcome == "final" and with_shared:
            cells: List[Tuple[str, int, int]] = []
            input_cells: List[Tuple[str, str]] = []
            for a in range(int(pm["n_arrays"])):
                ar = b.arrays[a_off + a]
                size = int(ar["size"])
                nodes = sess.fetch_cells(bid, p, a, size)
                for i in range(size):
                    if nodes[i] != N.UNSET:
                        cells.append((aname(a), i, int(nodes[i])))
                        rr.cell_nodes[(a, i)] = int(nodes[i])
                    elif int(ar["input"]) >= 0 and i < int(ar["seeded"]):
                        input_cells.append((f"{aname(a)}[{i}]", f"{sess.inputs[int(ar['input'])][0]}_{i}"))
            strs = sess.to_strings([c[2] for c in cells])
            for (an, i, _), s in zip(cells, strs):
                rr.shared[f"{an}[{i}]"] = s
            for k, v in input_cells:
                rr.shared[k] = v
        results.append(rr)
    return results
