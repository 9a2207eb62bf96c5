"""Kernel-language frontend (binding of include/veq_host.h, libveq_host.so).

Parses and elaborates .mk kernels under a launch configuration into packed
IR batches, exactly as the reference frontend would (proj/src/frontend.cpp),
for one CTA or for a grid of CTAs (block index bound to a config param).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Tuple

from . import ir

_HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(_HERE, "libveq_host.so")


class FrontendError(RuntimeError):
    """Kernel/config rejected; `kernel` is "a", "b" or "config"."""

    def __init__(self, kernel: str, msg: str):
        super().__init__(msg)
        self.kernel = kernel


class TemplateUnsupported(RuntimeError):
    """The grid is not one template plus per-CTA array shifts (VEQH_E_TEMPLATE);
    elaborate it per CTA instead."""


class _Template(C.Structure):
    _fields_ = [("ir_a", C.POINTER(C.c_uint8)), ("ir_a_len", C.c_size_t), ("ir_b", C.POINTER(C.c_uint8)),
                ("ir_b_len", C.c_size_t), ("inputs", C.c_void_p), ("deltas_a", C.POINTER(C.c_int32)),
                ("deltas_b", C.POINTER(C.c_int32)), ("n_arrays_a", C.c_uint32), ("n_arrays_b", C.c_uint32),
                ("n_blocks", C.c_uint32)]


class _Pair(C.Structure):
    _fields_ = [("ir_a", C.POINTER(C.c_uint8)), ("ir_a_len", C.c_size_t), ("ir_b", C.POINTER(C.c_uint8)),
                ("ir_b_len", C.c_size_t), ("inputs", C.c_void_p)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(HOST_LIB):
            raise RuntimeError(f"{HOST_LIB} not built (run __graft_entry__.build())")
        L = C.CDLL(HOST_LIB)
        L.veqh_elaborate_grid.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_int, C.POINTER(_Pair), C.c_char_p, C.c_size_t]
        L.veqh_elaborate_grid.restype = C.c_int
        L.veqh_free.argtypes = [C.POINTER(_Pair)]
        L.veqh_free.restype = None
        L.veqh_elaborate_template.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int64,
                                              C.c_uint32, C.c_int, C.POINTER(_Template), C.c_char_p, C.c_size_t]
        L.veqh_elaborate_template.restype = C.c_int
        L.veqh_free_template.argtypes = [C.POINTER(_Template)]
        L.veqh_free_template.restype = None
        _lib = L
    return _lib


def elaborate_pair(kernel_a: str, kernel_b: str, cfg: str, block_param: Optional[str] = None, n_blocks: int = 1,
                   workers: int = 0, want_names: bool = True,
                   block_base: int = 0) -> Tuple[ir.Batch, ir.Batch, List[Tuple[str, int]]]:
    """Returns (batch A, batch B, input symbol table). With block_param, CTA k
    of the batch binds params.<block_param> = block_base + k."""
    L = _L()
    out = _Pair()
    err = C.create_string_buffer(4096)
    workers = workers or (os.cpu_count() or 1)
    st = L.veqh_elaborate_grid(kernel_a.encode(), kernel_b.encode(), cfg.encode(),
                               block_param.encode() if block_param else None, block_base, n_blocks, workers,
                               1 if want_names else 0, C.byref(out), err, len(err))
    if st != 0:
        raise FrontendError({1: "a", 2: "b", 3: "config"}.get(st, "arg"), err.value.decode())
    try:
        img_a = C.string_at(out.ir_a, out.ir_a_len)
        img_b = C.string_at(out.ir_b, out.ir_b_len)
        a = ir.loads(img_a)
        b = ir.loads(img_b)
        # the packed-IR byte images (digest parity with the reference's
        # elaboration, tests/test_digest_parity.py)
        a.image, b.image = img_a, img_b
        text = C.string_at(out.inputs).decode()
    finally:
        L.veqh_free(C.byref(out))
    inputs = []
    for line in text.splitlines():
        name, size = line.split("\t")
        inputs.append((name, int(size)))
    return a, b, inputs


def _parse_inputs(text: str) -> List[Tuple[str, int]]:
    out = []
    for line in text.splitlines():
        name, size = line.split("\t")
        out.append((name, int(size)))
    return out


def elaborate_template(kernel_a: str, kernel_b: str, cfg: str, block_param: str, n_blocks: int,
                       block_base: int = 0, want_names: bool = True):
    """One template program per kernel for blocks [block_base, block_base +
    n_blocks) plus per-CTA array shifts (veqh_elaborate_template). Returns
    (template A, template B, inputs, deltas A [n_blocks, n_arrays_a],
    deltas B [n_blocks, n_arrays_b]); raises TemplateUnsupported when the
    grid needs per-CTA elaboration."""
    import numpy as np
    L = _L()
    out = _Template()
    err = C.create_string_buffer(4096)
    st = L.veqh_elaborate_template(kernel_a.encode(), kernel_b.encode(), cfg.encode(), block_param.encode(),
                                   block_base, n_blocks, 1 if want_names else 0, C.byref(out), err, len(err))
    if st == 5:
        raise TemplateUnsupported(err.value.decode())
    if st != 0:
        raise FrontendError({1: "a", 2: "b", 3: "config"}.get(st, "arg"), err.value.decode())
    try:
        ta = ir.loads(C.string_at(out.ir_a, out.ir_a_len))
        tb = ir.loads(C.string_at(out.ir_b, out.ir_b_len))
        inputs = _parse_inputs(C.string_at(out.inputs).decode())
        da = np.ctypeslib.as_array(out.deltas_a, shape=(n_blocks * out.n_arrays_a,)).copy().reshape(
            n_blocks, out.n_arrays_a)
        db = np.ctypeslib.as_array(out.deltas_b, shape=(n_blocks * out.n_arrays_b,)).copy().reshape(
            n_blocks, out.n_arrays_b)
    finally:
        L.veqh_free_template(C.byref(out))
    return ta, tb, inputs, da, db
