"""Packed IR batches on the host (numpy mirror of include/veq_ir.hpp).

A Batch owns the SoA arrays a veq_batch_desc points at plus host-only report
metadata (names, register names, source locations). Batches are produced by
the product frontend (frontend.py) or read from VEQIR02 files.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import native as N

STMT_DT = np.dtype([("kind", "u1"), ("op", "u1"), ("arr", "<u2"), ("dst", "<u4"), ("a", "<u4"), ("b", "<u4")])
ARRAY_DT = np.dtype([("size", "<u8"), ("role", "<u4"), ("flags", "<u4"), ("input", "<i4"), ("seeded", "<u4")])
RAT_DT = np.dtype([("num", "<i8"), ("den", "<i8")])
SET_DT = np.dtype([("full", "<u4"), ("lo", "<u4"), ("n_bits", "<u4"), ("word_off", "<u4")])
PROG_DT = np.dtype([("n_threads", "<u4"), ("warp_size", "<u4"), ("thread_off", "<u4"), ("array_off", "<u4"),
                    ("n_arrays", "<u4"), ("pad", "<u4")])
LOC_DT = np.dtype([("line", "<u4"), ("col", "<u4")])
assert STMT_DT.itemsize == 16 and ARRAY_DT.itemsize == 24 and PROG_DT.itemsize == 24


@dataclass
class Batch:
    progs: np.ndarray
    thread_stmt: np.ndarray
    thread_nregs: np.ndarray
    stmts: np.ndarray
    arrays: np.ndarray
    consts: np.ndarray
    syncsets: np.ndarray
    set_words: np.ndarray
    prog_names: List[str] = field(default_factory=list)
    array_names: List[str] = field(default_factory=list)
    thread_reg_off: np.ndarray = None
    reg_names: List[str] = field(default_factory=list)
    locs: np.ndarray = None

    @property
    def n_progs(self) -> int:
        return len(self.progs)

    @property
    def n_threads(self) -> int:
        return len(self.thread_nregs)

    def desc(self) -> N.veq_batch_desc:
        """veq_batch_desc over this batch's buffers (they must stay alive)."""
        for name in ("progs", "thread_stmt", "thread_nregs", "stmts", "arrays", "consts", "syncsets", "set_words"):
            arr = getattr(self, name)
            if not arr.flags["C_CONTIGUOUS"]:
                setattr(self, name, np.ascontiguousarray(arr))
        d = N.veq_batch_desc()
        d.n_progs = len(self.progs)
        d.n_threads_total = len(self.thread_nregs)
        d.n_stmts = len(self.stmts)
        d.n_arrays_total = len(self.arrays)
        d.n_consts = len(self.consts)
        d.n_syncsets = len(self.syncsets)
        d.n_set_words = len(self.set_words)
        d.progs = self.progs.ctypes.data
        d.thread_stmt = self.thread_stmt.ctypes.data
        d.thread_nregs = self.thread_nregs.ctypes.data
        d.stmts = self.stmts.ctypes.data
        d.arrays = self.arrays.ctypes.data
        d.consts = self.consts.ctypes.data
        d.syncsets = self.syncsets.ctypes.data
        d.set_words = self.set_words.ctypes.data
        return d

    def nbytes(self) -> int:
        return sum(getattr(self, n).nbytes for n in ("progs", "thread_stmt", "thread_nregs", "stmts", "arrays",
                                                      "consts", "syncsets", "set_words"))

    # -- host metadata helpers
    def thread_of_stmt(self, s: int) -> int:
        return int(np.searchsorted(self.thread_stmt, s, side="right") - 1)

    def reg_name(self, thread: int, reg: int) -> str:
        lo, hi = int(self.thread_reg_off[thread]), int(self.thread_reg_off[thread + 1])
        if lo + int(reg) >= hi:  # elaborated without register names
            return f"r{int(reg)}"
        return self.reg_names[lo + int(reg)]

    def loc(self, s: int):
        if self.locs is None or len(self.locs) == 0:
            return (0, 0)
        r = self.locs[s]
        return (int(r["line"]), int(r["col"]))


def _rvec(buf: memoryview, pos: int, dt):
    (n,) = struct.unpack_from("<Q", buf, pos)
    pos += 8
    dt = np.dtype(dt)
    a = np.frombuffer(buf, dtype=dt, count=n, offset=pos).copy()
    return a, pos + n * dt.itemsize


def _rstrs(buf: memoryview, pos: int):
    (n,) = struct.unpack_from("<Q", buf, pos)
    pos += 8
    out = []
    for _ in range(n):
        (l,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        out.append(bytes(buf[pos:pos + l]).decode())
        pos += l
    return out, pos


def load(path: str) -> Batch:
    with open(path, "rb") as f:
        return loads(f.read(), path)


def loads(data: bytes, what: str = "<buffer>") -> Batch:
    if data[:8] != b"VEQIR02\0":
        raise ValueError(f"{what}: not a VEQIR02 image")
    buf = memoryview(data)
    pos = 8
    progs, pos = _rvec(buf, pos, PROG_DT)
    thread_stmt, pos = _rvec(buf, pos, "<u8")
    thread_nregs, pos = _rvec(buf, pos, "<u4")
    stmts, pos = _rvec(buf, pos, STMT_DT)
    arrays, pos = _rvec(buf, pos, ARRAY_DT)
    consts, pos = _rvec(buf, pos, RAT_DT)
    sets, pos = _rvec(buf, pos, SET_DT)
    words, pos = _rvec(buf, pos, "<u8")
    pnames, pos = _rstrs(buf, pos)
    anames, pos = _rstrs(buf, pos)
    reg_off, pos = _rvec(buf, pos, "<u8")
    rnames, pos = _rstrs(buf, pos)
    locs, pos = _rvec(buf, pos, LOC_DT)
    return Batch(progs, thread_stmt, thread_nregs, stmts, arrays, consts, sets, words, pnames, anames, reg_off,
                 rnames, locs)


def concat(batches: List[Batch]) -> Batch:
    """Concatenate batches into one (pool indices re-based)."""
    progs, ts, tn, st, ar, co, ss, sw = [], [np.zeros(1, "<u8")], [], [], [], [], [], []
    pn, an, ro, rn, lo = [], [], [np.zeros(1, "<u8")], [], []
    t0 = a0 = c0 = q0 = w0 = 0
    s0 = r0 = 0
    for b in batches:
        p = b.progs.copy()
        p["thread_off"] += t0
        p["array_off"] += a0
        progs.append(p)
        ts.append(b.thread_stmt[1:] + s0)
        tn.append(b.thread_nregs)
        s = b.stmts.copy()
        m = (s["kind"] == N.ST_SETCONST) & (s["op"] == 0)
        s["a"][m] += c0
        m = s["kind"] == N.ST_SYNC
        s["a"][m] += q0
        st.append(s)
        ar.append(b.arrays)
        co.append(b.consts)
        q = b.syncsets.copy()
        q["word_off"] += w0
        ss.append(q)
        sw.append(b.set_words)
        pn += b.prog_names
        an += b.array_names
        ro.append(b.thread_reg_off[1:] + r0)
        rn += b.reg_names
        lo.append(b.locs)
        t0 += b.n_threads
        a0 += len(b.arrays)
        c0 += len(b.consts)
        q0 += len(b.syncsets)
        w0 += len(b.set_words)
        s0 += len(b.stmts)
        r0 += len(b.reg_names)
    cat = np.concatenate
    return Batch(cat(progs), cat(ts), cat(tn), cat(st), cat(ar), cat(co), cat(ss), cat(sw), pn, an, cat(ro), rn,
                 cat(lo))


def instantiate(template: Batch, deltas: np.ndarray) -> Batch:
    """CTA instance of a one-program template (veqh_elaborate_template):
    every Load/Store offset on array a shifted by deltas[a]. Host-side
    mirror of the device expansion in veq_instantiate (tests compare it
    with per-CTA elaboration)."""
    assert template.n_progs == 1
    st = template.stmts.copy()
    m = (st["kind"] == N.ST_LOAD) | (st["kind"] == N.ST_STORE)
    d = np.asarray(deltas, dtype=np.int64)[st["arr"][m].astype(np.int64)]
    st["a"][m] = ((st["a"][m].astype(np.int64).astype(np.int32).astype(np.int64) + d) & 0xFFFFFFFF).astype(np.uint32)
    b = Batch(template.progs.copy(), template.thread_stmt, template.thread_nregs, st, template.arrays,
              template.consts, template.syncsets, template.set_words, list(template.prog_names),
              list(template.array_names), template.thread_reg_off, template.reg_names, template.locs)
    return b
