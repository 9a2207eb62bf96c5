"""ctypes binding of the C-ABI in include/veq.h (libveq.so, built in-tree).

The product path has no CPU fallback: if the CUDA library cannot be loaded
or no device is visible, every entry point raises VeqError.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libveq.so")

u8, u16, u32, i32, u64, i64 = C.c_uint8, C.c_uint16, C.c_uint32, C.c_int32, C.c_uint64, C.c_int64
P = C.POINTER

# veq.h constants
ST_SETCONST, ST_BINOP, ST_UNOP, ST_COPY, ST_LOAD, ST_STORE, ST_SYNC = range(7)
BIN_ADD, BIN_MUL, BIN_DIV, BIN_MAX = range(4)
UN_NEG, UN_EXP = range(2)
ROLE_IN, ROLE_OUT, ROLE_SCRATCH = range(3)
ARR_STORED = 1
FAULT_RACE, FAULT_SAFETY = 1, 2
SAFE_UNINIT_REG, SAFE_UNINIT_MEM, SAFE_OOB, SAFE_INVALID_ARITH = range(4)
DETAIL_NONE, DETAIL_NEGINF_ADD, DETAIL_NEGINF_MUL, DETAIL_NEGINF_NEG, DETAIL_NEGINF_DIV, DETAIL_NEGINF_EXP, DETAIL_ZERO_DEN = range(7)
K_CONST, K_NEGINF, K_VAR, K_EXP, K_MAX, K_DIV, K_NEG, K_MUL, K_ADD = range(9)
UNSET = 0xFFFFFFFF


class veq_stmt(C.Structure):
    _fields_ = [("kind", u8), ("op", u8), ("arr", u16), ("dst", u32), ("a", u32), ("b", u32)]


class veq_array(C.Structure):
    _fields_ = [("size", u64), ("role", u32), ("flags", u32), ("input", i32), ("seeded", u32)]


class veq_rat(C.Structure):
    _fields_ = [("num", i64), ("den", i64)]


class veq_syncset(C.Structure):
    _fields_ = [("full", u32), ("lo", u32), ("n_bits", u32), ("word_off", u32)]


class veq_program_meta(C.Structure):
    _fields_ = [("n_threads", u32), ("warp_size", u32), ("thread_off", u32), ("array_off", u32),
                ("n_arrays", u32), ("pad", u32)]


class veq_batch_desc(C.Structure):
    _fields_ = [("n_progs", u32), ("n_threads_total", u32), ("n_stmts", u64), ("n_arrays_total", u32),
                ("n_consts", u32), ("n_syncsets", u32), ("n_set_words", u32),
                ("progs", C.c_void_p), ("thread_stmt", C.c_void_p), ("thread_nregs", C.c_void_p),
                ("stmts", C.c_void_p), ("arrays", C.c_void_p), ("consts", C.c_void_p),
                ("syncsets", C.c_void_p), ("set_words", C.c_void_p)]


class veq_input_desc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("size", u64)]


class veq_limits(C.Structure):
    _fields_ = [("max_nodes", u64), ("max_kid_words", u64), ("scratch_bytes", u64)]


class veq_fault(C.Structure):
    _fields_ = [("type", u8), ("kind", u8), ("sub", u8), ("detail", u8), ("is_write", u8), ("is_write2", u8),
                ("reg_slot", u8), ("pad", u8), ("prog", u32), ("tid", u32), ("stmt", u32), ("step", u32),
                ("tid2", u32), ("stmt2", u32), ("step2", u32), ("offset", i32), ("arr", u32)]


class veq_prog_result(C.Structure):
    _fields_ = [("steps", u64), ("releases", u32), ("n_faults", u32), ("deadlocked", u32), ("pad", u32)]


class veq_run_out(C.Structure):
    _fields_ = [("n_progs", u32), ("progs", P(veq_prog_result)), ("n_faults", u64), ("faults", P(veq_fault)),
                ("n_threads_total", u32), ("thread_state", P(u8)), ("thread_block_set", P(u32)),
                ("thread_block_stmt", P(u64)), ("n_nodes", u64), ("n_kid_words", u64), ("n_work", u64),
                ("n_access", u64), ("n_stmts_executed", u64), ("n_new_nodes", u64), ("n_new_kid_words", u64),
                ("n_launches", u32), ("n_phases", u32), ("phase_ms", C.c_float * 9)]


class veq_access(C.Structure):
    _fields_ = [("tid", u32), ("stmt", u32), ("step", u64), ("is_write", u32), ("pad", u32)]


class veq_race_report(C.Structure):
    _fields_ = [("arr", u32), ("offset", i32), ("first", veq_access), ("second", veq_access)]


class veq_safety_report(C.Structure):
    _fields_ = [("kind", u32), ("tid", u32), ("stmt", u32), ("detail", u32), ("step", u64), ("has_addr", u32),
                ("arr", u32), ("offset", i32), ("reg", u32), ("is_store", u32), ("pad", u32)]


class veq_thread_report(C.Structure):
    _fields_ = [("state", u32), ("set", u32), ("stmt", u32), ("pad", u32)]


class veq_report(C.Structure):
    _fields_ = [("outcome", u32), ("releases", u32), ("steps", u64), ("n_races", u64),
                ("races", P(veq_race_report)), ("n_safeties", u64), ("safeties", P(veq_safety_report)),
                ("deadlocked", u32), ("n_threads", u32), ("threads", P(veq_thread_report)),
                ("conflict_a", i32), ("conflict_b", i32), ("conflict_set_a", u32), ("conflict_set_b", u32)]


OUT_FINAL, OUT_RACE, OUT_DEADLOCK, OUT_SAFETY = range(4)
TS_RUNNABLE, TS_BLOCKED, TS_RETURNED = range(3)
OPT_KEEP_REGS = 1


class veq_combined(C.Structure):
    _fields_ = [("totals", u64 * 4), ("first_fail", u64), ("n_ranks", u32), ("pad", u32),
                ("rank_vc_off", P(u64)), ("verdict", P(u8)), ("rank_sc_off", P(u64)), ("sc_hash", P(u64)),
                ("sc_discharged", P(u8))]


class veq_decision(C.Structure):
    _fields_ = [("kind", u32), ("precision", u32), ("reason", C.c_char_p), ("n_assign", u32),
                ("names", P(C.c_char_p)), ("values", P(C.c_char_p)), ("f_enclosure", C.c_char_p),
                ("g_enclosure", C.c_char_p)]


VERDICT_KIND = ["equal", "not_equal", "unknown", "undecided"]


class veq_vc(C.Structure):
    _fields_ = [("node_a", u32), ("node_b", u32), ("equal", u32), ("sc_off", u32), ("sc_n", u32), ("pad", u32)]


class veq_vc_out(C.Structure):
    _fields_ = [("n_vcs", u64), ("vcs", P(veq_vc)), ("n_sc", u64), ("sc_node", P(u32)),
                ("sc_discharged", P(u8)), ("n_equal", u64), ("n_missing", u64)]


class veq_dag_node(C.Structure):
    _fields_ = [("kind", u32), ("nkids", u32), ("kid_off", u64), ("num", i64), ("den", i64),
                ("var_input", i64), ("var_index", u64)]


class veq_dag_buf(C.Structure):
    _fields_ = [("cap_nodes", u64), ("cap_kids", u64), ("nodes", P(veq_dag_node)), ("kids", P(u32)),
                ("root_index", P(u32)), ("n_nodes", u64), ("n_kids", u64)]


# status codes (include/veq.h)
OK, E_BUDGET, E_RATIONAL_OVERFLOW, E_OOM, E_INVALID_IR, E_CUDA, E_ARG, E_UNSUPPORTED, E_NO_DEVICE, E_SCRATCH = range(10)


class VeqError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"veq error {status}: {msg}")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    """Load libveq.so (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise VeqError(8, f"{LIB_PATH} not built (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.veq_open.argtypes = [C.c_int, P(veq_limits), P(vp)]
    L.veq_close.argtypes = [vp]
    L.veq_close.restype = None
    L.veq_strerror.argtypes = [C.c_int]
    L.veq_strerror.restype = C.c_char_p
    L.veq_last_error.argtypes = [vp]
    L.veq_last_error.restype = C.c_char_p
    L.veq_declare_inputs.argtypes = [vp, P(veq_input_desc), u32]
    L.veq_load_batch.argtypes = [vp, P(veq_batch_desc), P(u32)]
    L.veq_run.argtypes = [vp, u32, P(veq_run_out)]
    L.veq_run_start.argtypes = [vp, u32]
    L.veq_run_finish.argtypes = [vp, u32, P(veq_run_out)]
    L.veq_fetch_cells.argtypes = [vp, u32, u32, u32, P(u32), u64]
    L.veq_compare.argtypes = [vp, u32, u32, P(u32), P(u32), u32, P(veq_vc_out)]
    L.veq_compare_progs.argtypes = [vp, u32, u32, u32, u32, u32, P(u32), P(u32), u32, P(veq_vc_out)]
    L.veq_compare_fan.argtypes = [vp, u32, u32, u32, u32, u32, P(u32), P(u32), u32, P(veq_vc_out)]
    L.veq_export_dag.argtypes = [vp, P(u32), C.c_size_t, P(veq_dag_buf)]
    L.veq_verdict_counters.argtypes = [vp, P(u64)]
    L.veq_set_timing.argtypes = [vp, C.c_int]
    L.veq_stream.argtypes = [vp]
    L.veq_stream.restype = vp
    L.veq_clear_terms.argtypes = [vp]
    L.veq_drop_batch.argtypes = [vp, u32]
    L.veq_load_template.argtypes = [vp, P(veq_batch_desc), P(u32)]
    L.veq_instantiate.argtypes = [vp, u32, u32, P(i32), P(u32)]
    L.veq_drop_template.argtypes = [vp, u32]
    L.veq_render.argtypes = [vp, P(u32), C.c_size_t, P(C.c_char_p), P(P(u64))]
    L.veq_render_digest.argtypes = [vp, P(u32), C.c_size_t, P(u32), P(u64)]
    L.veq_batch_locs.argtypes = [vp, u32, P(u64)]
    L.veq_run_report.argtypes = [vp, u32, u32, P(veq_report)]
    L.veq_run_reports.argtypes = [vp, u32, P(u32), u32, P(veq_report)]
    L.veq_set_members.argtypes = [vp, u32, u32, u32, P(u32), u32, P(u32)]
    L.veq_set_option.argtypes = [vp, C.c_int, C.c_int]
    L.veq_fetch_regs.argtypes = [vp, u32, u32, u32, P(u32), u32, P(u32)]
    L.veq_comm_unique_id.argtypes = [C.c_char_p]
    L.veq_comm_init.argtypes = [vp, C.c_char_p, C.c_int, C.c_int]
    L.veq_comm_combine.argtypes = [vp, u64, P(veq_combined)]
    L.veq_decide.argtypes = [vp, u32, u32, u64, u64, P(veq_decision)]
    L.veq_decide_batch.argtypes = [vp, u64, P(u32), P(u32), P(u64), u64, u32, P(u32)]
    for f in ("veq_open", "veq_declare_inputs", "veq_load_batch", "veq_run", "veq_run_start", "veq_run_finish",
              "veq_fetch_cells", "veq_compare", "veq_compare_progs", "veq_compare_fan",
              "veq_export_dag", "veq_verdict_counters", "veq_set_timing", "veq_clear_terms"):
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


EXPORTED = ["veq_open", "veq_close", "veq_strerror", "veq_last_error", "veq_declare_inputs", "veq_load_batch",
            "veq_run", "veq_run_start", "veq_run_finish", "veq_fetch_cells", "veq_compare", "veq_compare_progs", "veq_export_dag", "veq_verdict_counters",
            "veq_set_timing", "veq_clear_terms", "veq_stream", "veq_drop_batch", "veq_load_template",
            "veq_instantiate", "veq_drop_template", "veq_render", "veq_render_digest", "veq_batch_locs",
            "veq_run_report", "veq_set_members", "veq_set_option", "veq_fetch_regs", "veq_comm_unique_id",
            "veq_comm_init", "veq_comm_combine", "veq_decide", "veq_compare_fan", "veq_decide_batch", "veq_run_reports"]
PHASES = ["schedule", "exec", "sort", "memscan", "resolve", "chains", "worklist", "eval", "finals"]
