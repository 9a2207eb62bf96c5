/* veq.h — C-ABI boundary of the B200-native equivalence-checker core.
 *
 * Replaces the hot section of the reference pipeline,
 *   ctaeq::check_equivalence  /root/reference/proj/src/pipeline.cpp:180-243
 * i.e. the two round-robin runs and the per-VC decision loop:
 *   ctaeq::run(const Program&, const SharedMem&, const SchedulePolicy&)
 *        proj/include/ctaeq/symexec.hpp:235-236, called at pipeline.cpp:183,199
 *   ctaeq::eq(const Expr&, const Expr&, ...) — fast path only (cf == cg plus
 *        side conditions), proj/src/decide.cpp:749-771, called at pipeline.cpp:227
 * Everything above (parse, elaborate, validate, signature check) and below
 * (aggregation, JSON, CLI) stays in host code. Plain C types only.
 *
 * Unit of work: a BATCH of independent CTA programs (one elaborated
 * ctaeq::Program each, proj/include/ctaeq/ir.hpp:148-156), packed SoA.
 * Threading: one veq_ctx per GPU; a ctx is not thread-safe; distinct ctxs
 * may be used concurrently. Ownership: input buffers are caller-owned and
 * copied; output buffers are ctx-owned and valid until the next call that
 * produces the same kind of output on that ctx.
 */
#ifndef VEQ_H
#define VEQ_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define VEQ_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------ */
enum {
  VEQ_OK = 0,
  VEQ_E_BUDGET = 1,            /* term-table / arena capacity exhausted      */
  VEQ_E_RATIONAL_OVERFLOW = 2, /* a coefficient left the exact int64 range   */
  VEQ_E_OOM = 3,               /* device allocation failed                   */
  VEQ_E_INVALID_IR = 4,        /* malformed batch                            */
  VEQ_E_CUDA = 5,              /* CUDA runtime error (see veq_last_error)    */
  VEQ_E_ARG = 6,               /* bad argument / handle                      */
  VEQ_E_UNSUPPORTED = 7,       /* input outside the supported envelope       */
  VEQ_E_NO_DEVICE = 8,         /* no CUDA device / extension unusable        */
  VEQ_E_SCRATCH = 9            /* per-node canonicalisation scratch overflow */
};

/* ---- packed IR ---------------------------------------------------------
 * Statement kinds/ops follow ctaeq::StmtKind / Bin / Un (ir.hpp:81-117). */
enum { VEQ_ST_SETCONST = 0, VEQ_ST_BINOP = 1, VEQ_ST_UNOP = 2, VEQ_ST_COPY = 3,
       VEQ_ST_LOAD = 4, VEQ_ST_STORE = 5, VEQ_ST_SYNC = 6 };
enum { VEQ_BIN_ADD = 0, VEQ_BIN_MUL = 1, VEQ_BIN_DIV = 2, VEQ_BIN_MAX = 3 };
enum { VEQ_UN_NEG = 0, VEQ_UN_EXP = 1 };
enum { VEQ_ROLE_IN = 0, VEQ_ROLE_OUT = 1, VEQ_ROLE_SCRATCH = 2 };

/* 16-byte statement.
 *  SETCONST: dst, a = const-pool index, op = 1 for NEG_INF (a ignored)
 *  BINOP:    dst, op, a, b (registers)      UNOP: dst, op, a
 *  COPY:     dst, a = src register
 *  LOAD:     dst, arr, a = (int32) offset   STORE: dst = SOURCE register, arr, a = offset
 *  SYNC:     a = sync-set pool index
 * Registers are dense PER THREAD (0 .. thread_nregs-1). */
typedef struct veq_stmt {
  uint8_t kind;
  uint8_t op;
  uint16_t arr;
  uint32_t dst;
  uint32_t a;
  uint32_t b;
} veq_stmt;

typedef struct veq_array {
  uint64_t size;      /* elements                                            */
  uint32_t role;      /* VEQ_ROLE_*                                          */
  uint32_t flags;     /* VEQ_ARR_STORED: some thread stores to it            */
  int32_t input;      /* index into the session's input table, or -1        */
  uint32_t seeded;    /* cells [0, seeded) start with input symbols          */
} veq_array;
#define VEQ_ARR_STORED 1u

/* Exact rational constant, canonical (den > 0, gcd 1). */
typedef struct veq_rat { int64_t num; int64_t den; } veq_rat;

/* Sync set. full = every thread of the program; otherwise the set lives in
 * one warp window: bit k of words[word_off ..] is thread lo + k, n_bits
 * valid bits (validate_structured, proj/src/ir.cpp:276-325). */
typedef struct veq_syncset {
  uint32_t full;
  uint32_t lo;
  uint32_t n_bits;
  uint32_t word_off;
} veq_syncset;

typedef struct veq_program_meta {
  uint32_t n_threads;
  uint32_t warp_size;  /* 0: none declared */
  uint32_t thread_off; /* first global thread index of this program */
  uint32_t array_off;  /* first array of this program in `arrays`   */
  uint32_t n_arrays;
  uint32_t pad;
} veq_program_meta;

/* A batch of n_progs programs. Global thread t of program p has statements
 * stmts[thread_stmt[t] .. thread_stmt[t+1]). All pools are batch-global. */
typedef struct veq_batch_desc {
  uint32_t n_progs;
  uint32_t n_threads_total;
  uint64_t n_stmts;
  uint32_t n_arrays_total;
  uint32_t n_consts;
  uint32_t n_syncsets;
  uint32_t n_set_words;
  const veq_program_meta *progs;     /* [n_progs]                 */
  const uint64_t *thread_stmt;       /* [n_threads_total + 1]     */
  const uint32_t *thread_nregs;      /* [n_threads_total]         */
  const veq_stmt *stmts;             /* [n_stmts]                 */
  const veq_array *arrays;           /* [n_arrays_total]          */
  const veq_rat *consts;             /* [n_consts]                */
  const veq_syncset *syncsets;       /* [n_syncsets]              */
  const uint64_t *set_words;         /* [n_set_words]             */
} veq_batch_desc;

/* ---- session inputs ----------------------------------------------------
 * The symbolic inputs of a check (ctaeq::make_symbolic_inputs,
 * pipeline.cpp:107-119): array `name` cell i holds Var("<name>_<i>").
 * Declaring them fixes the byte order of every input symbol (the order
 * Expr::compare uses for Vars, expr.cpp:120) and starts a new term table. */
typedef struct veq_input_desc {
  const char *name;
  uint64_t size;
} veq_input_desc;

typedef struct veq_limits {
  uint64_t max_nodes;      /* term-table node capacity (0: default)     */
  uint64_t max_kid_words;  /* kid arena capacity, u32 words (0: default) */
  uint64_t scratch_bytes;  /* canonicalisation scratch pool (0: default) */
} veq_limits;

typedef struct veq_ctx veq_ctx;

int veq_open(int device, const veq_limits *lim, veq_ctx **out);
void veq_close(veq_ctx *ctx);
const char *veq_strerror(int status);
const char *veq_last_error(veq_ctx *ctx);

/* Starts a new session: clears the term table and declares the inputs. */
int veq_declare_inputs(veq_ctx *ctx, const veq_input_desc *inputs, uint32_t n);

/* Copies a batch to the device; returns a batch handle (valid for the
 * session). Host buffers may be freed afterwards. */
int veq_load_batch(veq_ctx *ctx, const veq_batch_desc *desc, uint32_t *batch);

/* Frees a batch's device memory now (handle becomes invalid); a session's
 * batches are otherwise freed by the next veq_declare_inputs. */
int veq_drop_batch(veq_ctx *ctx, uint32_t batch);

/* ---- grid templates ----------------------------------------------------
 * A grid whose CTAs differ only by per-array offset shifts (veqh_elaborate_
 * template, include/veq_host.h) is loaded ONCE as a template (its programs
 * laid out in order) and expanded on the device into regular batches:
 * veq_instantiate makes n_inst instances; batch program q * n_inst + i is
 * template program q of instance i, with every Load/Store offset on the
 * program's array a shifted by deltas[i * n_arrays_total + array_off_q + a].
 * The result equals loading the per-CTA elaborations as one batch (the
 * instances share the template's constant and sync-set pools). */
int veq_load_template(veq_ctx *ctx, const veq_batch_desc *desc, uint32_t *tmpl);
int veq_instantiate(veq_ctx *ctx, uint32_t tmpl, uint32_t n_inst, const int32_t *deltas, uint32_t *batch);
int veq_drop_template(veq_ctx *ctx, uint32_t tmpl);

/* ---- run (K0 schedule, K3 executor, K4 race/uninit, K2 canonicalise) --- */
enum { VEQ_FAULT_RACE = 1, VEQ_FAULT_SAFETY = 2 };
enum { VEQ_SAFE_UNINIT_REG = 0, VEQ_SAFE_UNINIT_MEM = 1, VEQ_SAFE_OOB = 2,
       VEQ_SAFE_INVALID_ARITH = 3 }; /* ctaeq::SafetyKind order */
enum { VEQ_DETAIL_NONE = 0, VEQ_DETAIL_NEGINF_ADD, VEQ_DETAIL_NEGINF_MUL,
       VEQ_DETAIL_NEGINF_NEG, VEQ_DETAIL_NEGINF_DIV, VEQ_DETAIL_NEGINF_EXP,
       VEQ_DETAIL_ZERO_DEN };

/* One fault. Races: (tid,stmt,step,is_write) is the access whose check
 * failed ("second"); (tid2,stmt2,step2,is_write2) the recorded event
 * ("first"). Safeties use tid/stmt/step; reg_slot says which source
 * register (0 = a / store source, 1 = b) for uninitialised registers.
 * stmt indices are batch-global; order key is (prog, step, sub). */
typedef struct veq_fault {
  uint8_t type;
  uint8_t kind;     /* safety kind                                       */
  uint8_t sub;      /* order within one statement                        */
  uint8_t detail;   /* VEQ_DETAIL_*                                      */
  uint8_t is_write;
  uint8_t is_write2;
  uint8_t reg_slot;
  uint8_t pad;
  uint32_t prog;
  uint32_t tid;
  uint32_t stmt;
  uint32_t step;
  uint32_t tid2;
  uint32_t stmt2;
  uint32_t step2;
  int32_t offset;   /* memory faults: cell offset within `arr`           */
  uint32_t arr;     /* memory faults: program-local array index          */
} veq_fault;

/* Phases of veq_run, timed with CUDA events on the ctx stream when enabled. */
enum { VEQ_PH_SCHEDULE = 0, VEQ_PH_EXEC, VEQ_PH_SORT, VEQ_PH_MEMSCAN, VEQ_PH_RESOLVE, VEQ_PH_CHAINS,
       VEQ_PH_WORKLIST, VEQ_PH_EVAL, VEQ_PH_FINALS, VEQ_MAX_PHASES };
int veq_set_timing(veq_ctx *ctx, int on);
/* The CUDA stream (cudaStream_t) every kernel of this ctx is launched on,
 * for callers that time or order work around it. */
void *veq_stream(veq_ctx *ctx);
/* Resets the term table of the current session (declared inputs and loaded
 * batches stay valid): every run after it starts from an empty DAG. */
int veq_clear_terms(veq_ctx *ctx);

/* Per-program run summary (ctaeq::RunResult, symexec.hpp:214-225). */
typedef struct veq_prog_result {
  uint64_t steps;
  uint32_t releases;
  uint32_t n_faults;     /* faults (before host-side dedup)          */
  uint32_t deadlocked;   /* 1: run ended with a thread not returned  */
  uint32_t pad;
} veq_prog_result;

typedef struct veq_run_out {
  uint32_t n_progs;
  const veq_prog_result *progs;   /* [n_progs]                              */
  uint64_t n_faults;
  const veq_fault *faults;        /* unsorted; host sorts by (prog,step,sub) */
  /* final thread states, for deadlock reports (state: 0 runnable,
   * 1 blocked, 2 returned; blocked threads carry the sync set index and the
   * batch-global statement index of the blocking Sync) */
  uint32_t n_threads_total;
  const uint8_t *thread_state;
  const uint32_t *thread_block_set;
  const uint64_t *thread_block_stmt;
  /* device statistics of this call */
  uint64_t n_nodes;               /* term-table nodes after the run */
  uint64_t n_kid_words;
  uint64_t n_work;                /* canonicalised raw nodes         */
  uint64_t n_access;              /* race-check access tuples (R)    */
  uint64_t n_stmts_executed;      /* S: statements executed          */
  uint64_t n_new_nodes;           /* term nodes created by this run  */
  uint64_t n_new_kid_words;       /* kid words created by this run   */
  uint32_t n_launches;            /* device kernel launches (incl. library sort/scan) */
  uint32_t n_phases;
  float phase_ms[VEQ_MAX_PHASES]; /* per-phase device time when timing is on (veq_set_timing) */
} veq_run_out;

int veq_run(veq_ctx *ctx, uint32_t batch, veq_run_out *out);

/* veq_run in two halves: _start enqueues the whole run on the ctx stream and
 * returns without waiting; _finish waits for it and fills `out` (same
 * contents as veq_run). Several batches may be started before the first is
 * finished (they execute in start order), so the device never idles between
 * them. A batch cannot be started again before it is finished. */
int veq_run_start(veq_ctx *ctx, uint32_t batch);
int veq_run_finish(veq_ctx *ctx, uint32_t batch, veq_run_out *out);

/* ---- options -----------------------------------------------------------
 * VEQ_OPT_KEEP_REGS (0/1): runs started afterwards keep every thread's final
 * register file and canonicalise its values (veq_fetch_regs): the Final
 * outcome's register files (ctaeq::Outcome::regs, symexec.hpp:155-156)
 * that outcome_key and run()-level tests compare. Off by default: the
 * check pipeline only needs Out arrays (pipeline.cpp:214-220). */
enum { VEQ_OPT_KEEP_REGS = 1 };
int veq_set_option(veq_ctx *ctx, int option, int value);
/* Final register file of thread `tid` of program `prog`: canonical node per
 * thread-local register id (~0: never assigned); *n_regs = register count
 * (call with out_nodes NULL to size). Requires VEQ_OPT_KEEP_REGS at run. */
int veq_fetch_regs(veq_ctx *ctx, uint32_t batch, uint32_t prog, uint32_t tid, uint32_t *out_nodes, uint32_t n,
                   uint32_t *n_regs);

/* ---- run reports (ctaeq::RunResult, proj/include/ctaeq/symexec.hpp:214-225)
 * veq_run_report assembles one program's RunResult from the raw device
 * faults the way the reference's Collector does (symexec.cpp:308-328):
 * races and safety faults in execution order (step, then check order inside
 * a statement), de-duplicated by their identity without step numbers; the
 * deadlock report with every thread's final state and the first conflicting
 * pair (make_deadlock_report, symexec.cpp:335-365); and the outcome by
 * precedence race > safety > deadlock > final (symexec.cpp:838-845).
 * Statements are batch-global indices; the caller maps them to source
 * locations and register ids to names. Identity uses the per-statement
 * location keys given by veq_batch_locs (default: the statement index).
 * Output is ctx-owned, valid until the next veq_run_report on the batch. */
enum { VEQ_OUT_FINAL = 0, VEQ_OUT_RACE = 1, VEQ_OUT_DEADLOCK = 2, VEQ_OUT_SAFETY = 3 }; /* Outcome::Kind */
enum { VEQ_TS_RUNNABLE = 0, VEQ_TS_BLOCKED = 1, VEQ_TS_RETURNED = 2 };
typedef struct veq_access {
  uint32_t tid, stmt;
  uint64_t step;
  uint32_t is_write, pad;
} veq_access;
typedef struct veq_race_report {
  uint32_t arr;      /* program-local array index */
  int32_t offset;
  veq_access first;  /* the access recorded in the event context */
  veq_access second; /* the access whose check failed */
} veq_race_report;
typedef struct veq_safety_report {
  uint32_t kind;     /* VEQ_SAFE_* */
  uint32_t tid, stmt, detail;
  uint64_t step;
  uint32_t has_addr, arr;
  int32_t offset;
  uint32_t reg;      /* thread-local register id (register kinds), else ~0 */
  uint32_t is_store; /* out-of-bounds: write side */
  uint32_t pad;
} veq_safety_report;
typedef struct veq_thread_report {
  uint32_t state;    /* VEQ_TS_* */
  uint32_t set;      /* blocked: sync-set id (veq_set_members), else ~0 */
  uint32_t stmt;     /* blocked: the Sync statement, else ~0 */
  uint32_t pad;
} veq_thread_report;
typedef struct veq_report {
  uint32_t outcome;  /* VEQ_OUT_* */
  uint32_t releases;
  uint64_t steps;
  uint64_t n_races;
  const veq_race_report *races;
  uint64_t n_safeties;
  const veq_safety_report *safeties;
  uint32_t deadlocked;
  uint32_t n_threads; /* thread reports (deadlocked runs only) */
  const veq_thread_report *threads;
  int32_t conflict_a, conflict_b; /* -1: none */
  uint32_t conflict_set_a, conflict_set_b;
} veq_report;
int veq_batch_locs(veq_ctx *ctx, uint32_t batch, const uint64_t *loc_keys); /* [n_stmts] or NULL */
int veq_run_report(veq_ctx *ctx, uint32_t batch, uint32_t prog, veq_report *out);
/* The same for n programs at once, assembled in parallel on host threads:
 * outs[q] describes progs[q]; valid until the next veq_run_reports call on
 * the batch. */
int veq_run_reports(veq_ctx *ctx, uint32_t batch, const uint32_t *progs, uint32_t n, veq_report *outs);
/* Members (program-local tids, ascending) of a sync-set id of a report. */
int veq_set_members(veq_ctx *ctx, uint32_t batch, uint32_t prog, uint32_t set, uint32_t *tids, uint32_t cap,
                    uint32_t *n);

/* Final shared-memory contents after veq_run (the Final payload of
 * ctaeq::Outcome, symexec.hpp:155): canonical term node of each cell of
 * program `prog`'s array `array` (program-local index), or 0xFFFFFFFF when
 * the cell holds no value. Cells of read-only input arrays report
 * 0xFFFFFFFF too; they hold their input symbol by definition. */
int veq_fetch_cells(veq_ctx *ctx, uint32_t batch, uint32_t prog, uint32_t array,
                    uint32_t *out_nodes, uint64_t n);

/* ---- compare (K5) ------------------------------------------------------
 * Programs a.progs[i] and b.progs[i] are compared cell by cell over their
 * Out arrays in array-name order given by `out_order` (per program-pair,
 * the program-local Out array indices of A then of B, sorted by name).
 * One VC per Out cell; verdict bit: canonical forms identical (decide.cpp:
 * 765-768). Side conditions (decide.cpp:482-491, 306-333) are returned as
 * term-node ids with a positivity flag, in first-occurrence DFS order. */
typedef struct veq_vc {
  uint32_t node_a;       /* canonical node of kernel A's cell (or ~0: unset) */
  uint32_t node_b;
  uint32_t equal;        /* 1: structurally identical canonical forms        */
  uint32_t sc_off;       /* side conditions [sc_off, sc_off + sc_n)           */
  uint32_t sc_n;
  uint32_t pad;
} veq_vc;

typedef struct veq_vc_out {
  uint64_t n_vcs;
  const veq_vc *vcs;
  uint64_t n_sc;
  const uint32_t *sc_node;       /* denominator node ids                    */
  const uint8_t *sc_discharged;  /* positive_definite(denominator)          */
  uint64_t n_equal;              /* device-side count of equal VCs          */
  uint64_t n_missing;            /* Out cells never written (either side)   */
} veq_vc_out;

/* out_arrays: for program pair i, n_out_arrays[i] entries of
 * (array index in A's program, array index in B's program), already in
 * ascending array-name order (pipeline.cpp:128-131). */
int veq_compare(veq_ctx *ctx, uint32_t batch_a, uint32_t batch_b,
                const uint32_t *out_arrays_a, const uint32_t *out_arrays_b,
                uint32_t n_out_per_pair, veq_vc_out *out);

/* The same over program ranges: program prog_a0 + i of batch_a against
 * program prog_b0 + i of batch_b, i < n_pairs. The two ranges may lie in ONE
 * batch: loading and running both kernels' CTAs as a single batch lets one
 * set of launches carry both runs. */
int veq_compare_progs(veq_ctx *ctx, uint32_t batch_a, uint32_t prog_a0, uint32_t batch_b, uint32_t prog_b0,
                      uint32_t n_pairs, const uint32_t *out_arrays_a, const uint32_t *out_arrays_b,
                      uint32_t n_out_per_pair, veq_vc_out *out);

/* One reference program against many: program prog_a of batch_a against
 * program prog_b0 + i of batch_b, i < n_pairs (a batch of candidate kernels
 * checked against one reference kernel that ran once). VCs are laid out
 * pair-major as in veq_compare_progs. */
int veq_compare_fan(veq_ctx *ctx, uint32_t batch_a, uint32_t prog_a, uint32_t batch_b, uint32_t prog_b0,
                    uint32_t n_pairs, const uint32_t *out_arrays_a, const uint32_t *out_arrays_b,
                    uint32_t n_out_per_pair, veq_vc_out *out);

/* ---- slow path of the verdict API (ctaeq::eq, proj/src/decide.cpp:728-859)
 * For a VC whose canonical forms differ: d = canon(f - g) on the device; if
 * d is 0, or the exp-polynomial normal form of d's rationalized numerator
 * vanishes with every Max an opaque atom, the VC is equal; otherwise the
 * rigorous random witness search (MPFR intervals, libmpfr.so.6 loaded at run
 * time; same trials, seed and sampling as refute_random) looks for a
 * separating rational point: not-equal with the witness, else unknown with
 * the reference's reason text. A difference that still contains Max after
 * the opaque pass would need the max case split (split_max), which is not
 * restated: VEQ_UNDECIDED. Output strings are ctx-owned (next veq_decide). */
enum { VEQ_EQUAL = 0, VEQ_NOT_EQUAL = 1, VEQ_UNKNOWN = 2, VEQ_UNDECIDED = 3 };
typedef struct veq_decision {
  uint32_t kind;            /* VEQ_EQUAL .. VEQ_UNDECIDED (ctaeq::VerdictKind + undecided) */
  uint32_t precision;       /* witness: MPFR precision that separated                     */
  const char *reason;       /* unknown / undecided                                         */
  uint32_t n_assign;        /* witness assignment, variable-name order                     */
  const char *const *names;
  const char *const *values;
  const char *f_enclosure;  /* "[lo, hi]" as the reference prints it                       */
  const char *g_enclosure;
} veq_decision;
int veq_decide(veq_ctx *ctx, uint32_t node_f, uint32_t node_g, uint64_t seed, uint64_t trials, veq_decision *out);

/* veq_decide over n VCs at once (the decide loop of check_equivalence,
 * pipeline.cpp:222-243, with its OpenMP jobs): every difference canon(f - g)
 * in one device launch, one DAG export for all of them, then the host
 * decisions on n_threads threads (0: every hardware thread). kinds[i] is the
 * kind veq_decide returns for (f[i], g[i], seeds[i], trials); reasons and
 * witnesses are not kept — call veq_decide for a VC whose payload is
 * wanted. */
int veq_decide_batch(veq_ctx *ctx, uint64_t n, const uint32_t *node_f, const uint32_t *node_g, const uint64_t *seeds,
                     uint64_t trials, uint32_t n_threads, uint32_t *kinds);

/* ---- DAG export (host to_string / slow path / reports) -----------------
 * Exports the sub-DAG reachable from roots in canonical kid order. Nodes are
 * renumbered densely 0..n-1 in post-order (kids first); root_index maps each
 * root. Two-call protocol: call with buf->cap_* = 0 to size. */
enum { VEQ_K_CONST = 0, VEQ_K_NEGINF, VEQ_K_VAR, VEQ_K_EXP, VEQ_K_MAX,
       VEQ_K_DIV, VEQ_K_NEG, VEQ_K_MUL, VEQ_K_ADD }; /* ctaeq::Kind order */
typedef struct veq_dag_node {
  uint32_t kind;
  uint32_t nkids;
  uint64_t kid_off;   /* into kids[]                                      */
  int64_t num;        /* Const                                             */
  int64_t den;
  int64_t var_input;  /* Var: input table index, or -1 for an undefined symbol */
  uint64_t var_index; /* Var: cell index (input) or undef ordinal           */
} veq_dag_node;

typedef struct veq_dag_buf {
  uint64_t cap_nodes, cap_kids;
  veq_dag_node *nodes;   /* caller-allocated */
  uint32_t *kids;
  uint32_t *root_index;  /* [n_roots] */
  uint64_t n_nodes, n_kids;  /* filled */
} veq_dag_buf;

int veq_export_dag(veq_ctx *ctx, const uint32_t *roots, size_t n_roots,
                   veq_dag_buf *buf);

/* to_string (proj/src/expr.cpp:735-822) of term nodes, rendered on the host
 * from the device DAG: root i's text is text[offs[i] .. offs[i+1]). Output
 * is ctx-owned, valid until the next veq_render. */
int veq_render(veq_ctx *ctx, const uint32_t *roots, size_t n_roots, const char **text, const uint64_t **offs);
/* The same texts as CRC-32 (IEEE, as zlib.crc32) and byte length, streamed
 * without materialising them (digest comparison of very large forms). */
int veq_render_digest(veq_ctx *ctx, const uint32_t *roots, size_t n_roots, uint32_t *crc32, uint64_t *len);

/* ---- multi-GPU (one ctx per GPU, NCCL over NVLink / NVSwitch) ----------
 * CTA pairs, output elements and variants shard across GPUs with no data
 * exchange; each GPU keeps its own term table. The one exchange is the
 * verdict combine below. Rank 0 makes a unique id (veq_comm_unique_id, 128
 * bytes), the caller broadcasts it (any channel), every rank calls
 * veq_comm_init. NCCL is loaded at run time (libnccl.so.2). */
int veq_comm_unique_id(void *id_out);
int veq_comm_init(veq_ctx *ctx, const void *nccl_unique_id, int nranks, int rank);
typedef struct veq_combined {
  uint64_t totals[4];            /* summed over ranks: equal, vcs, faults, missing */
  uint64_t first_fail;           /* min over ranks of the caller's first failing global VC index */
  uint32_t n_ranks, pad;
  const uint64_t *rank_vc_off;   /* [n_ranks + 1]: rank r's VCs are verdict[off[r] .. off[r+1]) */
  const uint8_t *verdict;        /* per VC: 1 canonical forms equal                     */
  const uint64_t *rank_sc_off;   /* [n_ranks + 1]                                        */
  const uint64_t *sc_hash;       /* side-condition denominators: 64-bit Merkle hash      */
  const uint8_t *sc_discharged;
} veq_combined;
/* Called by every rank after its compare: all-reduce of the counters and of
 * the first failing index, all-gather of per-VC verdict bytes and
 * side-condition (hash, discharged) pairs in rank order (ctx-owned output,
 * valid until the next combine), so any rank can aggregate the report
 * (pipeline.cpp:245-266). Without veq_comm_init: this rank's own results. */
int veq_comm_combine(veq_ctx *ctx, uint64_t first_fail_local, veq_combined *out);
/* This ctx's counters of the last compare / run: equal, vcs, faults, missing. */
int veq_verdict_counters(veq_ctx *ctx, uint64_t out[4]);

#ifdef __cplusplus
}
#endif
#endif
