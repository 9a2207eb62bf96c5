// veq_kernels.cuh — the pipeline's shared device types and helpers, and the
// evaluator (compiled in veq_eval.cu under VEQ_TU_EVAL). The other kernels
// below are in veq_pipeline.cuh.
//
//   K0 k_schedule     round-robin control schedule (symexec.cpp:764-781,
//                     616-671): per program, step numbers of every executed
//                     segment and the release sequence. Control is value-
//                     independent, so this needs only the IR.
//   K3 k_exec         per-thread symbolic execution: registers hold value
//                     refs (raw statement ids or term ids), loads/stores emit
//                     access tuples, Add/Max chains are linked for fusion
//                     (step_impl, symexec.cpp:372-604).
//   K4 k_mem_scan     per-address scan of step-sorted access tuples: races,
//                     uninitialised reads, and load -> store value resolution
//                     (no_racing_rd/wr + sync_mem, symexec.cpp:22-69, 491-595).
//   K2 k_eval         canonicalises live raw nodes in step order with
//                     operand-ready spinning (persistent threads).
//   K5 k_compare      per-VC canonical id compare + side conditions.
#pragma once
#include <cooperative_groups.h>

#include "veq_warp.cuh"
#include "../../include/veq.h"

namespace cg = cooperative_groups;

namespace veqd {

constexpr uint8_t TS_RUN = 0, TS_BLOCK = 1, TS_RET = 2;
// deferred scaling (k_mark_defer, eval_add_deferred)
constexpr uint32_t USER_FINAL = 0xFFFFFFFEu;
constexpr uint8_t DF_LEAF = 1, DF_SUM = 2, DF_CHAIN = 4;  // deferred product / deferred sum / chain expands leaves
constexpr uint32_t DESC_DEFER = 1u << 16;                 // desc.w bit: the chain has deferred leaves
constexpr int E_DEFER = 11;

constexpr uint64_t UNSET64 = ~0ull;

struct Batch {
  uint32_t n_progs, n_threads;
  uint64_t n_stmts;
  const veq_program_meta *progs;
  const uint64_t *thread_stmt;
  const uint32_t *thread_prog;
  const veq_stmt *stmts;
  const veq_array *arrays;
  const uint64_t *arr_cell_base;  // per array: first global cell id, or UNSET64
  const uint32_t *const_node;
  const veq_syncset *sets;
  const uint64_t *set_words;
  const uint64_t *seg_off;    // [T+1]
  const uint64_t *seg_start;  // statement index of each segment start
  const uint32_t *seg_set;    // per segment: canonical set id of its ending Sync
  const uint64_t *rel_off;    // [P+1] release capacity per program
  const uint64_t *reg_off;    // [T+1]
  const uint32_t *prog_full_set;  // per program: set index of its full set, or UNSET
  uint64_t n_cells;
  uint32_t sched_on_chip;  // K0: capacity (threads) of its on-chip control state, 0 = global
  const uint32_t *long_threads;  // threads with >= EXEC_WARP_MIN statements (warp executor)
  uint32_t n_long;
  const uint64_t *prog_stmt;  // [P+1] first statement of each program when programs are laid out in order, else null
  uint32_t step_bits, prog_bits;  // widths of step / program fields in the sort keys
  const unsigned long long *set_chunk;  // per set: (32-thread chunk << 32) | member mask in it; ~0: not one chunk
  // run state
  uint32_t *seg_base;
  uint32_t *rel_step, *rel_set;
  uint32_t *prog_nrel;
  uint32_t *prog_dead;
  unsigned long long *prog_steps;
  uint8_t *th_state;
  uint32_t *th_seg, *th_bset;
  uint32_t *regfile;
  uint32_t *ref_a, *ref_b, *st_step, *canon;
  uint32_t *chain_head, *chain_pos, *chain_len, *uses;
  uint8_t *continued;
  // deferred scaling (k_mark_defer): the single consumer of a value used
  // once (USER_FINAL: a final memory cell), and per statement DF_* flags
  uint32_t *user;
  uint8_t *defer;
  uint32_t no_defer;  // 1: deferral disabled (VEQ_NO_DEFER, or the -inf fallback)
  // per program: the first step of an item that expands deferred leaves
  // (k_defer_split); items at or after it form the second eval pass
  uint32_t *prog_split;
  unsigned int *n_defer_chains;  // chains marked DF_CHAIN by k_mark_defer (0: no second pass)
  uint32_t keep_regs; // 1: final register files are kept and canonicalised (veq_fetch_regs)
  unsigned long long *tup_key, *tup_val;
  unsigned long long *n_tup;

  uint32_t *final_val, *final_node;
  veq_fault *faults;
  unsigned long long *n_faults;
  uint64_t fault_cap;
};

// Program of a batch-global statement: a search over the P+1 program
// boundaries (L1-resident), or over the thread table when programs are not
// laid out in order.
__device__ __forceinline__ uint32_t prog_of_stmt(const Batch &B, uint64_t i) {
  if (B.prog_stmt) {
    uint32_t lo = 0, hi = B.n_progs;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) / 2;
      if (__ldg(B.prog_stmt + mid) <= i) lo = mid;
      else hi = mid;
    }
    return lo;
  }
  uint32_t lo = 0, hi = B.n_threads;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) / 2;
    if (B.thread_stmt[mid] <= i) lo = mid;
    else hi = mid;
  }
  return B.thread_prog[lo];
}

// Program of statement i, starting from a program p0 known to hold a
// statement <= i (the block's first statement): a short forward walk over
// the program boundaries instead of a full search.
__device__ __forceinline__ uint32_t prog_walk(const Batch &B, uint32_t p0, uint64_t i) {
  if (!B.prog_stmt) return prog_of_stmt(B, i);
  uint32_t p = p0;
  while (p + 1 < B.n_progs && __ldg(B.prog_stmt + p + 1) <= i) p++;
  return p;
}

// Warp-aggregated slot allocation: one atomic per group of converged lanes.
__device__ __forceinline__ unsigned long long agg_inc(unsigned long long *ctr) {
  cg::coalesced_group g = cg::coalesced_threads();
  unsigned long long base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(ctr, (unsigned long long)g.size());
  return g.shfl(base, 0) + g.thread_rank();
}

// Block-wide append: every thread of the block calls it (no early exit) with
// its item count and gets its first output slot; one atomic per block, so a
// grid-wide stream compaction costs (items / block size) atomics instead of
// one per warp on a single contended address.
template <int NT>
__device__ __forceinline__ unsigned long long block_append(unsigned long long *ctr, uint32_t cnt) {
  static_assert(NT % 32 == 0 && NT <= 1024, "block size");
  __shared__ uint32_t s_w[NT / 32];
  __shared__ unsigned long long s_base;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) s_w[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = lane < NT / 32 ? s_w[lane] : 0;
    uint32_t z = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= (unsigned)o) z += y;
    }
    if (lane < NT / 32) s_w[lane] = z - v;
    if (lane == 31) s_base = z ? atomicAdd(ctr, (unsigned long long)z) : 0;
  }
  __syncthreads();
  return s_base + s_w[wid] + (x - cnt);
}
constexpr int APP_NT = 512, APP_ITEMS = 8;  // 4096 items per block

__device__ __forceinline__ void emit_fault(const Batch &B, const veq_fault &f) {
  unsigned long long i = agg_inc(B.n_faults);
  if (i < B.fault_cap) B.faults[i] = f;
}

// ---------------------------------------------------------------------------
// Batch preparation (veq_load_batch): control segments of every thread are
// cut at its Sync statements, and each Sync gets the canonical id of its set
// (content-equal sets share one id; a set covering every thread of the CTA
// is the full set, id = n_syncsets). Control is value-independent
// (symexec.cpp:764-781), so this needs only the IR.
struct PrepArgs {
  uint32_t n_progs, n_threads, n_syncsets, n_arrays_total;
  uint64_t n_stmts;
  const veq_program_meta *progs;
  const uint64_t *thread_stmt;
  const uint32_t *thread_prog;
  const veq_stmt *stmts;
  const veq_syncset *sets;
  const uint32_t *set_canon;  // pool index -> first pool index with equal content
  const uint32_t *set_pop;    // members per pool entry
  unsigned long long *cnt;    // per stmt: is_sync | is_access << 32 (then its exclusive scan)
  int *error;
  const uint64_t *set_words;
  unsigned int *sched_flags;  // bit 0: some sync set does not suit k_schedule_warp
  const veq_array *arrays;
  unsigned long long *n_arith;  // BinOp/UnOp statements: bound of the work list
};

__device__ __forceinline__ uint32_t thread_of_stmt(const uint64_t *thread_stmt, uint32_t n_threads, uint64_t i) {
  uint32_t lo = 0, hi = n_threads;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) / 2;
    if (thread_stmt[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}


// Template expansion (veq_instantiate): output statement o of template
// program q's instance i is template statement src0 + j with Load/Store
// offsets shifted by that instance's delta for the statement's array. One
// 16-byte read and write per statement (HBM-bound copy).
struct ExpandSeg {
  uint64_t out0;   // first output statement of this template program's instances
  uint64_t src0;   // first template statement of the program
  uint64_t len;    // statements per instance
  uint32_t array_off, pad;
};


// ---------------------------------------------------------------------------
// K0: schedule. One block per program, symbolic threads in contiguous chunks
// per CUDA thread so an ordered block scan gives round-robin step offsets.
constexpr int SCHED_BLOCK = 256;

__device__ inline bool set_contains(const Batch &B, uint32_t s, uint32_t tid) {
  veq_syncset q = B.sets[s];
  if (q.full) return true;
  if (tid < q.lo || tid >= q.lo + q.n_bits) return false;
  uint32_t k = tid - q.lo;
  return (B.set_words[q.word_off + k / 64] >> (k % 64)) & 1ull;
}
__device__ inline uint32_t set_min(const Batch &B, uint32_t s) {
  veq_syncset q = B.sets[s];
  if (q.full) return 0;
  for (uint32_t w = 0; w * 64 < q.n_bits; w++) {
    uint64_t x = B.set_words[q.word_off + w];
    if (x) return q.lo + w * 64 + __ffsll((long long)x) - 1;
  }
  return q.lo;
}

// Shared-memory variant of K0 (the one launched): per-thread control state
// lives in shared memory when the CTA has at most SCHED_SMEM_T threads, so a
// round costs a handful of block barriers and on-chip accesses.
constexpr uint32_t SCHED_SMEM_T = 8192;


// K0 for CTAs of at most 1024 threads: one CUDA thread per symbolic thread,
// control state in registers. A round is one block scan of the runnable
// threads' segment lengths (their step numbers) plus one release decision.
// Sets inside one 32-thread window are decided with warp votes: the lanes
// blocked on I are a __match_any_sync group, and I is releasable iff its
// members are all in that group or returned (releasable_syncs,
// symexec.cpp:616-654). The full set uses block counts; any other set is
// checked member by member from shared memory.
constexpr uint32_t TS_NONE = 3;  // lane beyond the CTA's thread count


// K0, one warp per CTA program (CTAs of at most 1024 threads whose sync
// sets are all the full set or windows inside one aligned 32-thread chunk).
// The round-robin loop (symexec.cpp:764-781) is emulated chunk by chunk:
// after a release only the released chunk's threads change state, so a
// round costs one chunk's scan plus a 32-way min over cached per-chunk
// release candidates, with no block barrier. Each thread's next segment
// end and set are prefetched when it blocks.
constexpr uint32_t SW_WARPS = 4;
struct SchedWarpSmem {
  // per thread: blocked set and its member mask (in the thread's chunk); the
  // segment to run next (index relative to the CTA's first segment), its
  // length, the set ending it and that set's mask
  uint32_t bs[1024], bm[1024], cj[1024], len[1024], nset[1024], nm[1024];
  uint8_t st[1024];
  unsigned long long cand[32];
};


// ---------------------------------------------------------------------------
// K3: per-thread symbolic execution over value refs.
__device__ __forceinline__ bool is_stmt_ref(uint32_t r) { return r < REF_NODE; }

// Threads with at least EXEC_WARP_MIN statements run on k_exec_warp.
constexpr uint64_t EXEC_WARP_MIN = 64;


// ---------------------------------------------------------------------------
// K3, warp-parallel: one warp per symbolic thread, 32 consecutive statements
// per step. Each lane owns one statement; a register read resolves to the
// last lane before it (in statement order) that defines the register — found
// with shuffles — else to the register file. Copies forward their source
// value; the first read of an uninitialised register faults and seeds it
// (symexec.cpp:390-408). Chain links are decided warp-uniformly in lane
// order. Semantics are identical to k_exec.
__device__ __forceinline__ bool defines_reg(uint8_t kind) {
  return kind == VEQ_ST_SETCONST || kind == VEQ_ST_BINOP || kind == VEQ_ST_UNOP || kind == VEQ_ST_COPY ||
         kind == VEQ_ST_LOAD;
}


// ---------------------------------------------------------------------------
// K4 helpers: "thread i is still pending in the event (owner j, step se) at
// step s" — no release (I, r) with se < r < s and {i, j} in I (sync_mem,
// symexec.cpp:48-69, folded over the release sequence).
__device__ inline uint32_t find_prog_of_thread(const Batch &B, uint32_t g) { return B.thread_prog[g]; }

__device__ inline bool pending(const Batch &B, uint32_t p, uint32_t j, uint32_t se, uint32_t i, uint32_t s) {
  const uint64_t r0 = B.rel_off[p];
  const uint32_t n = B.prog_nrel[p];
  // first release with step > se
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) / 2;
    if (B.rel_step[r0 + mid] <= se) lo = mid + 1;
    else hi = mid;
  }
  for (uint32_t k = lo; k < n; k++) {
    uint32_t rs = B.rel_step[r0 + k];
    if (rs >= s) break;
    uint32_t I = B.rel_set[r0 + k];
    if (set_contains(B, I, i) && set_contains(B, I, j)) return false;
  }
  return true;
}

struct Reader {
  uint32_t tid, step, stmt, pad;
};


// Follow load refs to the value they read (a load's ref_a holds the value
// of the store it observed, which may itself be a loaded value).
__device__ __forceinline__ uint32_t chase(const Batch &B, uint32_t r) {
  while (is_stmt_ref(r) && B.stmts[r].kind == VEQ_ST_LOAD) r = B.ref_a[r];
  return r;
}


__device__ __forceinline__ bool is_chain_op(const veq_stmt &st) {
  return st.kind == VEQ_ST_BINOP && (st.op == VEQ_BIN_ADD || st.op == VEQ_BIN_MAX);
}


// ---- deferred scaling ------------------------------------------------------
// A product M = X * c whose only use is as a LEAF of a fused Add chain, where
// X is the end of another fused Add chain used only by M, is never
// canonicalised on its own: the consuming chain expands it into X's leaves,
// each scaled by c (multiplied into any enclosing scale). canon_mul_kids
// distributes a sum term by term and canon_add_kids merges term multisets
// (proj/src/expr.cpp:415-481), and exp factors merge through the same
// multiset sum, so sum_y canon(y * S) collected equals canon(canon(sum_y y) * S)
// (SURVEY App. A.4): the canonical forms are unchanged, while the online-
// softmax rescale `acc = acc_prev * c` (C4) stops re-distributing every
// accumulated term once per key block. -inf anywhere in an expansion sets
// E_DEFER and the run is repeated without deferral (exact fault reports).

__device__ __forceinline__ bool is_add_chain_end(const Batch &B, uint32_t x) {
  if (!is_stmt_ref(x) || B.st_step[x] == UNSET) return false;
  const veq_stmt sx = B.stmts[x];
  return sx.kind == VEQ_ST_BINOP && sx.op == VEQ_BIN_ADD && !B.continued[x];
}


// A work item: every executed BinOp/UnOp except chain links absorbed by
// their successor, and deferred products and sums.
__device__ __forceinline__ bool is_work_item(const Batch &B, uint64_t i, const veq_stmt &st) {
  if (st.kind != VEQ_ST_BINOP && st.kind != VEQ_ST_UNOP) return false;
  if (is_chain_op(st) && B.continued[i] && B.uses[i] == 1) return false;
  return !(B.defer[i] & (DF_LEAF | DF_SUM));
}


// ---------------------------------------------------------------------------
// K2: persistent evaluation in (program, step) order.
__device__ __forceinline__ uint32_t wait_node(const Batch &B, uint32_t r) {
  if (!is_stmt_ref(r)) return r & ~REF_NODE;
  volatile uint32_t *c = B.canon + r;
  uint32_t v = *c;
  int spins = 0;
  while (v == UNSET) {
    if (++spins > 16) __nanosleep(spins > 1000 ? 1000 : 64);
    v = *c;
  }
  return v;
}

struct EvalCtx {
  const uint32_t *log, *log_stmt, *log_base;
  unsigned long long *prof;  // optional eval profile (VEQ_PROF=1), see veq_api.cu
  // path switches (VEQ_EVAL_OFF, diagnostics): 2 no smem path, 4 no lean
  // path. (Half-warp pairing of small sums was removed in round 2, see
  // profiles/r02_pairing.md; lane-parallel runs replace it.)
  uint32_t off;
  // memo of exp merges under deferred scales: key (exp node << 32 | scale
  // node) -> merged factor (veq_api.cu sizes and clears it per run)
  unsigned long long *mkeys;
  uint32_t *mvals;
  uint64_t mmask;
  uint32_t bucket_us;  // VEQ_PROF timeline bucket width
};

__device__ inline void arith_fault(const Batch &B, uint32_t stmt, uint8_t detail) {
  uint32_t lo = 0, hi = B.n_threads;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) / 2;
    if (B.thread_stmt[mid] <= stmt) lo = mid;
    else hi = mid;
  }
  uint32_t p = B.thread_prog[lo];
  veq_fault f{};
  f.type = VEQ_FAULT_SAFETY;
  f.kind = VEQ_SAFE_INVALID_ARITH;
  f.sub = 2;
  f.detail = detail;
  f.prog = p;
  f.tid = lo - B.progs[p].thread_off;
  f.stmt = stmt;
  f.step = B.st_step[stmt];
  emit_fault(B, f);
}

__device__ inline uint32_t eval_stmt(const Batch &B, const Table &T, Arena &A, const EvalCtx &E, uint32_t i) {
  const veq_stmt st = B.stmts[i];
  auto undef_of = [&](uint32_t s) { return intern_undef(T, 3, s >> 29, s); };
  if (st.kind == VEQ_ST_BINOP && (st.op == VEQ_BIN_ADD || st.op == VEQ_BIN_MAX)) {
    uint32_t h = B.chain_head[i], pos = B.chain_pos[i];
    uint32_t b = E.log_base[h], n = pos + 2;
    uint32_t *ids = A.get<uint32_t>(n);
    if (!ids) return T.id_zero;
    uint32_t start = 0;
    for (uint32_t k = 0; k < n; k++) ids[k] = wait_node(B, E.log[b + k]);
    if (st.op == VEQ_BIN_ADD) {
      // -inf operand: InvalidArithmetic at the chain statement that consumed
      // it (symexec.cpp:474-486); that statement's value is a fresh undefined
      // symbol and the chain continues from it, so everything up to and
      // including that statement's own leaves is replaced by the symbol.
      for (uint32_t k = 0; k < n; k++) {
        if (ids[k] == T.id_neginf) {
          uint32_t s = E.log_stmt[b + k];
          arith_fault(B, s, VEQ_DETAIL_NEGINF_ADD);
          uint32_t r = k < 1 ? 1 : k;  // the head statement owns leaves 0 and 1
          ids[r] = undef_of(s);
          start = r;
          if (k == 0) k = 1;
        }
      }
      return add_nary(T, A, ids + start, n - start);
    }
    return max_nary(T, A, ids, n);
  }
  if (st.kind == VEQ_ST_BINOP) {
    uint32_t a = wait_node(B, B.ref_a[i]), c = wait_node(B, B.ref_b[i]);
    if (st.op == VEQ_BIN_MUL) {
      if (a == T.id_neginf || c == T.id_neginf) {
        arith_fault(B, i, VEQ_DETAIL_NEGINF_MUL);
        return undef_of(i);
      }
      // product of two atoms (Var/Exp/Max/Div, at most one Exp): no
      // coefficient, no distribution, no exp merge, so canon_mul_kids
      // (expr.cpp:426-481) reduces to the two factors in canonical order
      const Node na = ld_node(T, a), nc = ld_node(T, c);
      auto atom = [](uint8_t k) { return k == K_VAR || k == K_EXP || k == K_MAX || k == K_DIV; };
      if (atom(na.kind) && atom(nc.kind) && !(na.kind == K_EXP && nc.kind == K_EXP)) {
        uint32_t f[2] = {a, c};
        if (cmp_pref(T, prefix_of(nc), c, prefix_of(na), a) < 0) {
          f[0] = c;
          f[1] = a;
        }
        return intern(T, K_MUL, 0, 0, f, 2);
      }
      uint32_t ops[2] = {a, c};
      return mul_canon(T, A, ops, 2);
    }
    // Div: div() smart constructor checks then canon_div (expr.cpp:237-245)
    if (a == T.id_neginf || c == T.id_neginf) {
      arith_fault(B, i, VEQ_DETAIL_NEGINF_DIV);
      return undef_of(i);
    }
    if (c == T.id_zero) {
      arith_fault(B, i, VEQ_DETAIL_ZERO_DEN);
      return undef_of(i);
    }
    Node na = ld_node(T, a), nc = ld_node(T, c);
    if (na.kind == K_CONST && nc.kind == K_CONST) return intern_const(T, rat_div(T, const_val(na), const_val(nc)));
    return canon_div(T, A, a, c);
  }
  // UnOp
  uint32_t a = wait_node(B, B.ref_a[i]);
  if (st.op == VEQ_UN_NEG) {
    if (a == T.id_neginf) {
      arith_fault(B, i, VEQ_DETAIL_NEGINF_NEG);
      return undef_of(i);
    }
    Node na = ld_node(T, a);
    if (na.kind == K_CONST) {
      Rat v = const_val(na);
      v.n = -v.n;
      return intern_const(T, v);
    }
    uint32_t ops[2] = {T.id_mone, a};
    return mul_canon(T, A, ops, 2);
  }
  if (a == T.id_neginf) {
    arith_fault(B, i, VEQ_DETAIL_NEGINF_EXP);
    return undef_of(i);
  }
  if (a == T.id_zero) return T.id_one;
  return intern(T, K_EXP, 0, 0, &a, 1);
}


__device__ __forceinline__ bool desc_is_add(const uint4 &d) {
  return (d.w & 0xff) == VEQ_ST_BINOP && ((d.w >> 8) & 0xff) == VEQ_BIN_ADD;
}

// Window evaluation. A warp claims a window of G consecutive items of the
// (step, program)-sorted work list and walks it in order:
//  * a fused Add chain runs warp-cooperatively (veq_warp.cuh): sums of at
//    most 32 terms in registers, larger ones in a shared-memory page pool
//    (one 32-warp block per SM, 54 x 4 KB pages; warp_add_smem), rare cases
//    (like terms, coefficients, -inf leaves, an exhausted pool) on exact
//    global-scratch paths;
//  * a maximal run of other items (Mul / Div / Neg / Exp / Max chains) runs
//    LANE-parallel, one item per lane (eval_stmt, veq_canon.cuh): products of
//    atoms — the bulk of C3/C4 — no longer leave 31 lanes idle. An item may
//    wait on an earlier item of its own run (another lane): diverged lanes
//    make independent progress, and nothing in eval_stmt synchronises the
//    warp.
// Every dependency of an item lies earlier in the sorted list, so windows
// claimed in list order always make progress. 64 registers/thread: 32
// resident warps per SM in one block sharing one 216 KB page pool.
constexpr uint32_t EVAL_BLOCK = 1024, EVAL_PAGES = 54;
// k_eval_warp is compiled in its own translation unit (veq_eval.cu) and
// launched through launch_eval_warp (parallel builds; the rest of the
// pipeline does not recompile when only the evaluator changes).
void eval_warp_config(int smem, int *per_sm);
void launch_eval_warp(uint32_t grid, uint32_t block, int smem, cudaStream_t s, const Batch &B, const Table &T,
                      const EvalCtx &E, const uint4 *desc, const unsigned long long *n_work_dev,
                      unsigned long long *cursor, char *pool, unsigned long long *pool_used, uint64_t pool_cap,
                      uint64_t chunk, bool defer);
#ifdef VEQ_TU_EVAL
// One fused Add chain, whole warp (lg: the chain's first 32 log entries,
// lane-indexed). Returns the canonical sum; `created` when this warp
// published a new node (its fence already ran).
__device__ inline uint32_t eval_add_warp(const Batch &B, const Table &T, const EvalCtx &E, Arena &A, WarpAlloc &W,
                                         const SmemPool &SP, const uint4 d, const uint32_t lg, bool &created,
                                         int &path, unsigned long long *prof_lean, unsigned long long *prof_smem,
                                         unsigned long long &prof_pool, unsigned long long &prof_pages) {
  const uint32_t lane = lane_id();
  const uint32_t b = d.y, n = d.z;
  uint32_t r = UNSET;
  created = false;
  path = 0;
  // operands ready, -inf check; sums of <= 32 terms finish in registers
  uint32_t leaf0 = lane < n ? wait_node(B, lg) : UNSET, m = 0;
  bool neg = leaf0 == T.id_neginf;
  for (uint32_t k = lane + 32; k < n; k += 32) neg |= wait_node(B, E.log[b + k]) == T.id_neginf;
  neg = __any_sync(kFull, neg);
  if (!neg) {
    bool counted = false;
    if (n <= 32 && !(E.off & 4)) {
      r = warp_add_lean(T, leaf0, n, m, &W, &created, prof_lean);
      counted = true;
      path = 1;
    }
    if (r == UNSET && (!counted || m > 32)) {
      if (!counted) {
        for (uint32_t k = lane; k < n; k += 32) m += n_terms_of(T, wait_node(B, E.log[b + k]));
        m = __reduce_add_sync(kFull, m);
      }
      // leaves with coefficient terms need the grouping region
      bool cleaf = false;
      for (uint32_t k = lane; k < n; k += 32) {
        const uint32_t fl = ld_node(T, wait_node(B, E.log[b + k])).flags;
        cleaf |= (fl & (F_COEF | F_ANYCOEF)) != 0;
      }
      cleaf = __any_sync(kFull, cleaf);
      const uint32_t pages = (uint32_t)((add_smem_bytes(n, m, cleaf) + SPAGE - 1) / SPAGE);
      const long long pa0 = E.prof ? clock64() : 0;
      const int first = (E.off & 2) ? -1 : pool_acquire(SP, pages);
      if (E.prof && lane == 0) {
        prof_pool += clock64() - pa0;
        prof_pages += pages;
      }
      if (first >= 0) {
        char *buf = SP.base + (uint64_t)first * SPAGE;
        uint32_t *lv = reinterpret_cast<uint32_t *>(buf);
        for (uint32_t k = lane; k < n; k += 32) lv[k] = wait_node(B, E.log[b + k]);
        __syncwarp();
        r = warp_add_smem(T, buf, n, m, &W, prof_smem, cleaf);
        pool_release(SP, first, pages);
        path = 2;
      }
    } else if (r == UNSET && n <= 32) {
      r = warp_add_small_reg(T, leaf0, n);  // like terms / coefficients
      path = 3;
    }
  }
  if (r == UNSET) {
    path = 4;
    uint32_t *ids = warp_get<uint32_t>(A, n);
    r = T.id_zero;
    if (ids) {
      for (uint32_t k = lane; k < n; k += 32) ids[k] = wait_node(B, E.log[b + k]);
      __syncwarp();
      uint32_t start = 0;
      if (neg) {
        // -inf operands: same restart rule as eval_stmt, sequentially
        if (lane == 0) {
          for (uint32_t k = 0; k < n; k++) {
            if (ids[k] != T.id_neginf) continue;
            uint32_t s = E.log_stmt[b + k];
            arith_fault(B, s, VEQ_DETAIL_NEGINF_ADD);
            uint32_t rr = k < 1 ? 1 : k;
            ids[rr] = intern_undef(T, 3, s >> 29, s);
            start = rr;
            if (k == 0) k = 1;
          }
        }
        start = __shfl_sync(kFull, start, 0);
        __syncwarp();
      }
      r = warp_add_small(T, ids + start, n - start);
      if (r == UNSET) r = warp_add_nary(T, A, ids + start, n - start);
    }
  }
  return r;
}

// ---- deferred scaling: expansion of a chain with deferred leaves ----------
// exp(a) * exp(s) -> exp(a + s) (merge_exp_factors, expr.cpp:371-391), memoised
// per (exp, scale): the online-softmax terms of one row share their merged
// exponents across every output column. Returns the merged factor (T.id_one
// when the exponents cancel). The first lane to claim a key computes it;
// others wait for the value.
constexpr unsigned long long MEMO_EMPTY = ~0ull;
VEQ_NOINLINE uint32_t merge_exp_pair(const Table &T, Arena &A, uint32_t e, uint32_t sc) {
  const Node ne = ld_node(T, e), ns = ld_node(T, sc);
  uint32_t args[2] = {ld_kid(T, ne.p0), ld_kid(T, ns.p0)};
  const uint32_t arg = add_nary(T, A, args, 2);
  return arg == T.id_zero ? T.id_one : intern(T, K_EXP, 0, 0, &arg, 1);
}
__device__ inline uint32_t memo_merge(const Table &T, const EvalCtx &E, Arena &A, uint32_t e, uint32_t sc) {
  if (!E.mkeys) return merge_exp_pair(T, A, e, sc);
  const unsigned long long key = ((unsigned long long)e << 32) | sc;
  uint64_t h = mix64(key) & E.mmask;
  for (uint64_t probes = 0; probes <= E.mmask; probes++, h = (h + 1) & E.mmask) {
    unsigned long long k = *((volatile unsigned long long *)(E.mkeys + h));
    if (k == MEMO_EMPTY) {
      k = atomicCAS(E.mkeys + h, MEMO_EMPTY, key);
      if (k == MEMO_EMPTY) {
        const uint32_t v = merge_exp_pair(T, A, e, sc);
        fence_acq_rel();
        atomicExch(E.mvals + h, v);
        return v;
      }
    }
    if (k == key) {
      volatile uint32_t *pv = E.mvals + h;
      uint32_t v = *pv;
      for (int spins = 0; v == UNSET; v = *pv)
        if (++spins > 16) __nanosleep(64);
      return v;
    }
  }
  return merge_exp_pair(T, A, e, sc);  // table full: compute without the memo
}

// canon(y * sc) for canonical y and scale sc (canon_mul_kids, expr.cpp:426-481)
// with a fast path for the common shapes: y an Exp, or a coefficient-free
// product with one Exp factor, and sc an Exp.
VEQ_NOINLINE uint32_t scaled_term(const Table &T, const EvalCtx &E, Arena &A, uint32_t y, uint32_t sc) {
  if (sc == T.id_one) return y;
  const Node ns = ld_node(T, sc), ny = ld_node(T, y);
  if (ns.kind == K_EXP) {
    if (ny.kind == K_EXP) return memo_merge(T, E, A, y, sc);
    if (ny.kind == K_MUL && ny.nkids <= 8) {
      uint32_t f[8];
      int ex = -1, nexp = 0;
      bool plain = true;
      for (uint32_t k = 0; k < ny.nkids; k++) {
        f[k] = ld_kid(T, ny.p0 + k);
        const uint8_t kk = ld_kind(T, f[k]);
        if (kk == K_EXP) {
          ex = (int)k;
          nexp++;
        }
        plain &= kk != K_CONST && kk != K_ADD && kk != K_MUL;
      }
      if (plain && nexp == 1) {
        const uint32_t m = memo_merge(T, E, A, f[ex], sc);
        uint32_t nf = 0, g[8];
        for (uint32_t k = 0; k < ny.nkids; k++)
          if ((int)k != ex) g[nf++] = f[k];
        if (m != T.id_one) g[nf++] = m;
        if (nf == 1) return g[0];
        // canonical factor order (insertion sort on order prefixes)
        uint64_t pk[8];
        for (uint32_t k = 0; k < nf; k++) pk[k] = prefix_id(T, g[k]);
        for (uint32_t k = 1; k < nf; k++) {
          const uint32_t x = g[k];
          const uint64_t px = pk[k];
          int q = (int)k - 1;
          while (q >= 0 && cmp_pref(T, px, x, pk[q], g[q]) < 0) {
            g[q + 1] = g[q];
            pk[q + 1] = pk[q];
            q--;
          }
          g[q + 1] = x;
          pk[q + 1] = px;
        }
        return intern(T, K_MUL, 0, 0, g, nf);
      }
    }
  }
  uint32_t ops[2] = {y, sc};
  return mul_canon(T, A, ops, 2);
}

// One fused Add chain whose leaves include deferred products M = X * c: the
// leaves are expanded (X's chain leaves, each under the scale c times the
// enclosing scale, recursively), every leaf is scaled lane-parallel, and the
// scaled terms are summed (canon_add_kids). Whole warp.
static __device__ __noinline__ uint32_t eval_add_deferred(const Batch &B, const Table &T, const EvalCtx &E, Arena &A,
                                             const uint4 d) {
  const uint32_t lane = lane_id();
  const long long c0 = E.prof ? clock64() : 0;
  uint32_t cap = d.z * 8 + 1024;
  uint32_t *ref = warp_get<uint32_t>(A, cap), *scl = warp_get<uint32_t>(A, cap);
  if (!ref || !scl) return T.id_zero;
  uint32_t total = 0;
  // job stack (lane 0): (log base, leaf count, scale)
  constexpr int MAXJ = 64;
  uint32_t jb[MAXJ], jn[MAXJ], js[MAXJ];
  int nj = 0;
  if (lane == 0) {
    jb[0] = d.y;
    jn[0] = d.z;
    js[0] = T.id_one;
    nj = 1;
  }
  for (;;) {
    nj = __shfl_sync(kFull, nj, 0);
    if (nj == 0) break;
    uint32_t base = 0, cnt = 0, scale = 0;
    if (lane == 0) {
      nj--;
      base = jb[nj];
      cnt = jn[nj];
      scale = js[nj];
    }
    base = __shfl_sync(kFull, base, 0);
    cnt = __shfl_sync(kFull, cnt, 0);
    scale = __shfl_sync(kFull, scale, 0);
    if (total + cnt > cap) {  // grow (bump arena; the old buffers die with the item)
      uint32_t ncap = 2 * (total + cnt);
      uint32_t *r2 = warp_get<uint32_t>(A, ncap), *s2 = warp_get<uint32_t>(A, ncap);
      if (!r2 || !s2) return T.id_zero;
      for (uint32_t k = lane; k < total; k += 32) {
        r2[k] = ref[k];
        s2[k] = scl[k];
      }
      ref = r2;
      scl = s2;
      cap = ncap;
    }
    for (uint32_t k = lane; k < cnt; k += 32) {
      const uint32_t v = __ldg(E.log + base + k);
      const bool dl = is_stmt_ref(v) && (B.defer[v] & DF_LEAF);
      ref[total + k] = dl ? UNSET : v;
      scl[total + k] = dl ? v : scale;  // a deferred product: its statement, expanded below
    }
    __syncwarp();
    // deferred products among the new entries become jobs (lane 0)
    if (lane == 0) {
      for (uint32_t k = 0; k < cnt; k++) {
        if (ref[total + k] != UNSET) continue;
        const uint32_t M = scl[total + k];
        const uint32_t a = B.ref_a[M], b = B.ref_b[M];
        const bool xa = is_stmt_ref(a) && (B.defer[a] & DF_SUM);
        const uint32_t X = xa ? a : b, c = xa ? b : a;
        const uint32_t cn = wait_node(B, c);
        uint32_t ns;
        if (cn == T.id_neginf || scale == T.id_neginf) {
          set_error(T, E_DEFER);
          ns = T.id_one;
        } else if (scale == T.id_one) {
          ns = cn;
        } else if (ld_kind(T, cn) == K_EXP && ld_kind(T, scale) == K_EXP) {
          ns = memo_merge(T, E, A, cn, scale);
        } else {
          uint32_t ops[2] = {cn, scale};
          ns = mul_canon(T, A, ops, 2);
        }
        if (nj >= MAXJ) {
          set_error(T, E_DEFER);
          break;
        }
        jb[nj] = E.log_base[B.chain_head[X]];
        jn[nj] = B.chain_pos[X] + 2;
        js[nj] = ns;
        nj++;
      }
    }
    total += cnt;
    __syncwarp();
  }
  const long long c1 = E.prof ? clock64() : 0;
  // scaled terms, lane-parallel; removed entries (expanded products) drop out
  uint32_t *out = warp_get<uint32_t>(A, total ? total : 1);
  if (!out) return T.id_zero;
  uint32_t m = 0;
  for (uint32_t k0 = 0; k0 < total; k0 += 32) {
    const uint32_t k = k0 + lane;
    uint32_t t = UNSET;
    if (k < total && ref[k] != UNSET) {
      const uint32_t y = wait_node(B, ref[k]);
      if (y == T.id_neginf) {
        set_error(T, E_DEFER);
        t = T.id_zero;
      } else {
        t = scaled_term(T, E, A, y, scl[k]);
      }
    }
    const uint32_t has = __ballot_sync(kFull, t != UNSET);
    if (t != UNSET) out[m + __popc(has & ((1u << lane) - 1))] = t;
    m += __popc(has);
  }
  __syncwarp();
  const long long c2 = E.prof ? clock64() : 0;
  uint32_t r = warp_add_small(T, out, m);
  if (r == UNSET) r = warp_add_nary(T, A, out, m);
  if (E.prof && lane == 0) {  // [24..27]: expand, scaled terms, sum cycles; items
    atomicAdd(E.prof + 24, (unsigned long long)(c1 - c0));
    atomicAdd(E.prof + 25, (unsigned long long)(c2 - c1));
    atomicAdd(E.prof + 26, (unsigned long long)(clock64() - c2));
    atomicAdd(E.prof + 27, 1ull);
  }
  return r;
}

// DEFER selects the pass (k_defer_split): n_work_dev = {items, pass-2 items};
// the sorted list holds pass 1 then pass 2, and only the pass-2 kernel
// carries the deferred expansion.
template <bool DEFER>
__global__ void __launch_bounds__(EVAL_BLOCK, 1) k_eval_warp(Batch B, Table T, EvalCtx E, const uint4 *desc,
                                                             const unsigned long long *n_work_dev,
                                                             unsigned long long *cursor, char *pool,
                                                             unsigned long long *pool_used, uint64_t pool_cap,
                                                             uint64_t chunk) {
  // work-list length and window size from the device (no host read-back): a
  // short list is claimed in small windows so it spreads over all warps
  const uint64_t n_all = n_work_dev[0], n_p2 = n_work_dev[1];
  const uint64_t n_work = DEFER ? n_p2 : n_all - n_p2;
  if (DEFER) desc += n_all - n_p2;
  const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint32_t G = n_work >= warps_total * 128 ? 32 : (n_work >= warps_total * 16 ? 8 : 1);
  extern __shared__ __align__(16) char eval_smem[];
  __shared__ unsigned long long s_mask;
  if (threadIdx.x == 0) s_mask = 0;
  __syncthreads();
  const SmemPool SP{&s_mask, eval_smem, EVAL_PAGES};
  Arena A{pool, pool_used, pool_cap, &T, nullptr, 0, 0, chunk, 0};
  WarpAlloc W{0, 0, 0, 0};
  const uint32_t lane = lane_id();
  // first window: fixed, interleaved across blocks (warp j of block b takes
  // window j * gridDim + b), so a short list spreads over every SM; later
  // windows come from the shared cursor
  const uint32_t wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const unsigned long long first_windows = (unsigned long long)gridDim.x * wpb;
  unsigned long long prof_wait = 0, prof_work[6] = {0, 0, 0, 0, 0, 0}, prof_n[6] = {0, 0, 0, 0, 0, 0},
                     prof_lean[3] = {0, 0, 0}, prof_pool = 0, prof_pages = 0, prof_smem[4] = {0, 0, 0, 0};
  unsigned long long t_k0 = 0;
  if (E.prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_k0));
  // VEQ_PROF timeline: items finished / smem items finished / warps done per
  // 400 us bucket since the kernel started (slots 32..127)
  auto tbucket = [&]() -> uint32_t {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long bk = (t - t_k0) / (1000ull * E.bucket_us);
    return (uint32_t)(bk < 31 ? bk : 31);
  };
  unsigned long long w0 = ((unsigned long long)wib * gridDim.x + blockIdx.x) * G;
  while (w0 < n_work) {
    const uint32_t cnt = (uint32_t)(n_work - w0 < G ? n_work - w0 : G);
    // the window's descriptors, one coalesced load; bit mask of Add chains
    const uint4 dl = lane < cnt ? __ldg(desc + w0 + lane) : make_uint4(0, 0, 0, 0xff);
    const uint32_t addm = __ballot_sync(kFull, lane < cnt && desc_is_add(dl));
    uint32_t j = 0;
    while (j < cnt) {
      if ((addm >> j) & 1u) {
        // ---- a fused Add chain: the whole warp
        const uint4 d = make_uint4(__shfl_sync(kFull, dl.x, j), __shfl_sync(kFull, dl.y, j),
                                   __shfl_sync(kFull, dl.z, j), __shfl_sync(kFull, dl.w, j));
        const uint32_t lg = lane < d.z ? __ldg(E.log + d.y + lane) : UNSET;
        A.item = d.x;
        const long long t0 = E.prof ? clock64() : 0;
        bool created = false;
        int path = 0;
        uint32_t r;
        if (d.w & DESC_DEFER) {
          if constexpr (DEFER) {
            r = arena_call(A, [&](Arena &a) { return eval_add_deferred(B, T, E, a, d); });
          } else {
            set_error(T, E_INTERNAL);  // k_defer_split puts every such chain in pass 2
            r = UNSET;
          }
          path = 4;
        } else {
          r = eval_add_warp(B, T, E, A, W, SP, d, lg, created, path, E.prof ? prof_lean : nullptr,
                            E.prof ? prof_smem : nullptr, prof_pool, prof_pages);
        }
        A.used = 0;  // items are independent: each lane reuses its current chunk
        if (lane == 0) {
          // a node this warp created was fenced before its slot was claimed;
          // anything else needs the fence for cumulativity
          if (!created) fence_acq_rel();
          atomicExch(B.canon + d.x, r);
          if (E.prof) {
            prof_work[path] += clock64() - t0;
            prof_n[path]++;
            const uint32_t tb = tbucket();
            atomicAdd(E.prof + 32 + tb, 1ull);
            if (path == 2) atomicAdd(E.prof + 64 + tb, 1ull);
          }
        }
        j++;
        continue;
      }
      // ---- a run of non-Add items [j, k): one per lane
      const uint32_t above = j + 1 < 32 ? (addm >> (j + 1)) << (j + 1) : 0u;
      const uint32_t k = above ? (uint32_t)(__ffs(above) - 1) : cnt;
      if (lane >= j && lane < k) {
        const uint32_t i = dl.x;
        A.item = i;
        const long long t0 = E.prof ? clock64() : 0;
        const uint32_t r = eval_stmt(B, T, A, E, i);
        A.used = 0;
        fence_acq_rel();
        atomicExch(B.canon + i, r);
        if (E.prof) {
          const long long dt = clock64() - t0;
          prof_work[0] += dt;
          prof_n[0]++;
          atomicAdd(E.prof + 32 + tbucket(), 1ull);
          // per operation: mul div max | neg exp (slots 128.., cycles 136..)
          const uint32_t kind = dl.w & 0xff, op = (dl.w >> 8) & 0xff;
          const uint32_t slot = kind == VEQ_ST_BINOP ? (op == VEQ_BIN_MUL ? 0 : op == VEQ_BIN_DIV ? 1 : 2)
                                                     : (op == VEQ_UN_NEG ? 3 : 4);
          atomicAdd(E.prof + 128 + slot, 1ull);
          atomicAdd(E.prof + 136 + slot, (unsigned long long)dt);
        }
      }
      __syncwarp();
      j = k;
    }
    // next window: the cursor counts windows claimed after the first ones
    unsigned long long x = 0;
    if (lane == 0) x = atomicAdd(cursor, 1ull);
    w0 = (__shfl_sync(kFull, x, 0) + first_windows) * G;
  }
  wa_flush(T, W);
  if (E.prof) {
    if (lane == 0) atomicAdd(E.prof + 96 + tbucket(), 1ull);
    // per-lane counters (lane-parallel runs) and lane 0's (warp items)
    atomicAdd(E.prof, prof_wait);
    for (int q = 0; q < 5; q++) {
      atomicAdd(E.prof + 1 + q, prof_work[q]);
      atomicAdd(E.prof + 6 + q, prof_n[q]);
    }
    if (lane == 0) {
      for (int q = 0; q < 3; q++) atomicAdd(E.prof + 11 + q, prof_lean[q]);
      atomicAdd(E.prof + 14, prof_pool);
      atomicAdd(E.prof + 15, prof_pages);
      for (int q = 0; q < 4; q++) atomicAdd(E.prof + 16 + q, prof_smem[q]);
    }
  }
}
#endif  // VEQ_TU_EVAL


// ---------------------------------------------------------------------------
// K5: compare. One thread per VC: id equality, then side conditions by an
// iterative pre-order DFS with a visited set (first-occurrence order of
// collect_side_conditions, decide.cpp:482-491).
struct CmpArgs {
  const uint32_t *cell_a, *cell_b;  // per VC: global cell ids (UNSET64 -> missing)
  uint64_t n_vcs;
  veq_vc *vcs;
  uint32_t *sc_node;
  uint8_t *sc_dis;
  unsigned long long *n_sc;
  uint64_t sc_cap;
  unsigned long long *n_equal, *n_missing;
};

// Overflowing any of the fixed per-VC sets is an error (E_SCRATCH), never a
// silent truncation: a dropped undischarged denominator would turn the
// reference's "unknown" into "equivalent".
__device__ inline void collect_sc(const Table &T, uint32_t root, uint32_t *seen_den, uint32_t &nseen,
                                  uint32_t cap, uint32_t *visited, uint32_t &nvis, uint32_t vcap, uint32_t *stack) {
  uint32_t sp = 0;
  stack[sp++] = root;
  while (sp) {
    uint32_t x = stack[--sp];
    Node n = ld_node(T, x);
    if (!(n.flags & F_HASDIV)) continue;
    bool vis = false;
    for (uint32_t q = 0; q < nvis; q++)
      if (visited[q] == x) {
        vis = true;
        break;
      }
    if (vis) continue;
    if (nvis >= vcap) {
      set_error(T, E_SCRATCH);
      return;
    }
    visited[nvis++] = x;
    if (n.kind == K_DIV) {
      uint32_t den = ld_kid(T, n.p0 + 1);
      bool dup = false;
      for (uint32_t q = 0; q < nseen; q++)
        if (seen_den[q] == den) dup = true;
      if (!dup) {
        if (nseen >= cap) {
          set_error(T, E_SCRATCH);
          return;
        }
        seen_den[nseen++] = den;
      }
    }
    for (int k = (int)n.nkids - 1; k >= 0; k--) {
      if (sp >= vcap) {
        set_error(T, E_SCRATCH);
        return;
      }
      stack[sp++] = ld_kid(T, n.p0 + k);
    }
  }
}


}  // namespace veqd
