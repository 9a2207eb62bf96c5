// veq_pipeline.cuh — the kernels of the per-batch pipeline other than the
// evaluator (prep, K0 schedule, K3 executors, race/memory scan, resolve,
// deferred marking, work list, finals, compare, slow-path differences).
// Included by veq_api.cu only; veq_eval.cu compiles k_eval_warp from
// veq_kernels.cuh, so the two translation units rebuild independently.
#pragma once
#include "veq_kernels.cuh"

namespace veqd {

__global__ void k_prep_thread_prog(PrepArgs A, uint32_t *thread_prog) {
  const uint32_t p = blockIdx.x;
  const veq_program_meta m = A.progs[p];
  for (uint32_t t = threadIdx.x; t < m.n_threads; t += blockDim.x) thread_prog[m.thread_off + t] = p;
}

// per statement: validation and the (sync, access) counts to scan
__global__ void k_prep_stmts(PrepArgs A) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool arith = i < A.n_stmts && (A.stmts[i].kind == VEQ_ST_BINOP || A.stmts[i].kind == VEQ_ST_UNOP);
  const int na = __syncthreads_count(arith);
  if (threadIdx.x == 0 && na) atomicAdd(A.n_arith, (unsigned long long)na);
  if (i >= A.n_stmts) return;
  const veq_stmt st = A.stmts[i];
  unsigned long long c = 0;
  if (st.kind > VEQ_ST_SYNC) {
    atomicCAS(A.error, 0, 1);
  } else if (st.kind == VEQ_ST_LOAD || st.kind == VEQ_ST_STORE) {
    const uint32_t t = thread_of_stmt(A.thread_stmt, A.n_threads, i);
    const veq_program_meta pm = A.progs[A.thread_prog[t]];
    if (st.arr >= pm.n_arrays) {
      atomicCAS(A.error, 0, 2);
    } else {
      // an access tuple is emitted by an in-bounds access to a checked
      // array; direct loads of never-stored inputs cannot race
      const veq_array ar = A.arrays[pm.array_off + st.arr];
      const int32_t off = (int32_t)st.a;
      const bool inb = off >= 0 && (uint64_t)off < ar.size;
      const bool direct = st.kind == VEQ_ST_LOAD && !(ar.flags & VEQ_ARR_STORED) && ar.input >= 0 &&
                          (uint32_t)off < ar.seeded;
      if (inb && !direct) c = 1ull << 32;
    }
  } else if (st.kind == VEQ_ST_SYNC) {
    c = 1;
    if (st.a >= A.n_syncsets) atomicCAS(A.error, 0, 3);
  }
  A.cnt[i] = c;
}

// per thread: segment offsets, first segment start, last segment's set
// (cnt has n_stmts + 1 entries after the scan: cnt[n_stmts] is the total)
__global__ void k_prep_threads(PrepArgs A, uint64_t *seg_off, uint64_t *seg_start, uint32_t *seg_set) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > A.n_threads) return;
  auto syncs_before = [&](uint64_t i) -> uint64_t { return A.cnt[i] & 0xffffffffull; };
  const uint64_t so = t + syncs_before(A.thread_stmt[t]);
  seg_off[t] = so;
  if (t == A.n_threads) return;
  seg_start[so] = A.thread_stmt[t];
  const uint64_t nsync = syncs_before(A.thread_stmt[t + 1]) - syncs_before(A.thread_stmt[t]);
  seg_set[so + nsync] = UNSET;  // the last segment ends the thread, not at a sync
}

// per Sync statement: canonical set id of the segment it ends, next start
__global__ void k_prep_syncs(PrepArgs A, uint64_t *seg_start, uint32_t *seg_set) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_stmts) return;
  const veq_stmt st = A.stmts[i];
  if (st.kind != VEQ_ST_SYNC || st.a >= A.n_syncsets) return;
  const uint32_t t = thread_of_stmt(A.thread_stmt, A.n_threads, i);
  const uint32_t p = A.thread_prog[t];
  const uint64_t j = t + (A.cnt[i] & 0xffffffffull);
  const bool full = A.sets[st.a].full || A.set_pop[st.a] == A.progs[p].n_threads;
  seg_set[j] = full ? A.n_syncsets : A.set_canon[st.a];
  seg_start[j + 1] = i + 1;
  if (!full && A.sched_flags) {
    // k_schedule_warp needs every window set inside one aligned 32-thread
    // chunk and every syncing thread to be a member of its set
    const veq_syncset q = A.sets[st.a];
    const uint32_t tid = t - A.progs[p].thread_off;
    const bool member = tid >= q.lo && tid < q.lo + q.n_bits &&
                        ((A.set_words[q.word_off + (tid - q.lo) / 64] >> ((tid - q.lo) % 64)) & 1ull);
    const bool chunk = q.n_bits == 0 || q.lo / 32 == (q.lo + q.n_bits - 1) / 32;
    if (!member || !chunk) atomicOr(A.sched_flags, 1u);
  }
}

// per sync set: the aligned 32-thread chunk holding its window and the
// member mask inside it (k_schedule_warp decides releases from it)
__global__ void k_prep_set_chunks(const veq_syncset *sets, const uint64_t *set_words, uint32_t n,
                                  unsigned long long *set_chunk) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  const veq_syncset q = sets[i];
  unsigned long long v = ~0ull;
  if (!q.full && q.n_bits && q.lo / 32 == (q.lo + q.n_bits - 1) / 32) {
    const uint64_t bits = set_words[q.word_off] & (q.n_bits >= 64 ? ~0ull : ((1ull << q.n_bits) - 1));
    v = ((unsigned long long)(q.lo / 32) << 32) | (uint32_t)(bits << (q.lo % 32));
  }
  set_chunk[i] = v;
}

// per program: sync count (release capacity) for the rel_off scan
__global__ void k_prep_progs(PrepArgs A, uint64_t *prog_sync, uint32_t *prog_full) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= A.n_progs) return;
  const veq_program_meta m = A.progs[p];
  auto syncs_before = [&](uint64_t i) -> uint64_t { return A.cnt[i] & 0xffffffffull; };
  prog_sync[p] = syncs_before(A.thread_stmt[m.thread_off + m.n_threads]) - syncs_before(A.thread_stmt[m.thread_off]);
  prog_full[p] = A.n_syncsets;
}

// threads with >= EXEC_WARP_MIN statements (they run on k_exec_warp)
__global__ void k_prep_long(PrepArgs A, uint32_t *longs, unsigned long long *n_long, uint64_t min_len) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.n_threads) return;
  if (A.thread_stmt[t + 1] - A.thread_stmt[t] >= min_len) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(n_long, (unsigned long long)g.size());
    longs[g.shfl(base, 0) + g.thread_rank()] = t;
  }
}

__global__ void k_expand_stmts(const veq_stmt *__restrict__ tmpl, const ExpandSeg *__restrict__ segs, uint32_t n_segs,
                               uint32_t n_inst, const int32_t *__restrict__ deltas, uint32_t n_arrays,
                               veq_stmt *__restrict__ out, uint64_t n_out) {
  const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_out) return;
  uint32_t q = 0;
  while (q + 1 < n_segs && segs[q + 1].out0 <= o) q++;
  const ExpandSeg sg = segs[q];
  const uint64_t r = o - sg.out0, i = r / sg.len, j = r - i * sg.len;
  veq_stmt st = tmpl[sg.src0 + j];
  if (st.kind == VEQ_ST_LOAD || st.kind == VEQ_ST_STORE)
    st.a = (uint32_t)((int32_t)st.a + __ldg(deltas + i * n_arrays + sg.array_off + st.arr));
  out[o] = st;
}

__global__ void __launch_bounds__(SCHED_BLOCK) k_schedule_smem(Batch B) {
  extern __shared__ uint8_t sched_smem[];
  const uint32_t p = blockIdx.x;
  const veq_program_meta pm = B.progs[p];
  const uint32_t T = pm.n_threads, t0 = pm.thread_off;
  const uint32_t cap = B.sched_on_chip;  // threads of on-chip state per block
  const bool on_chip = T <= cap;
  uint32_t *bs = on_chip ? reinterpret_cast<uint32_t *>(sched_smem) : B.th_bset + t0;
  uint32_t *sg = on_chip ? bs + cap : B.th_seg + t0;
  uint8_t *st = on_chip ? reinterpret_cast<uint8_t *>(sg + cap) : B.th_state + t0;
  const uint32_t chunk = (T + SCHED_BLOCK - 1) / SCHED_BLOCK;
  const uint32_t lo = threadIdx.x * chunk, hi = min(T, lo + chunk);
  __shared__ unsigned long long s_scan[SCHED_BLOCK];
  __shared__ unsigned long long s_step, s_best;
  __shared__ uint32_t s_ret, s_blkfull, s_nrel;
  __shared__ int s_released;
  const uint32_t full = B.prog_full_set[p];
  for (uint32_t t = lo; t < hi; t++) {
    uint32_t g = t0 + t;
    sg[t] = 0;
    st[t] = B.thread_stmt[g] == B.thread_stmt[g + 1] ? TS_RET : TS_RUN;
    bs[t] = UNSET;
  }
  if (threadIdx.x == 0) {
    s_step = 0;
    s_nrel = 0;
    s_ret = 0;
  }
  __syncthreads();
  {
    uint32_t c = 0;
    for (uint32_t t = lo; t < hi; t++) c += st[t] == TS_RET;
    if (c) atomicAdd(&s_ret, c);
  }
  __syncthreads();
  while (s_ret != T) {
    // ---- run phase
    unsigned long long mylen = 0;
    for (uint32_t t = lo; t < hi; t++) {
      if (st[t] != TS_RUN) continue;
      uint32_t g = t0 + t;
      uint64_t sj = B.seg_off[g] + sg[t];
      uint64_t end = (sj + 1 < B.seg_off[g + 1]) ? B.seg_start[sj + 1] : B.thread_stmt[g + 1];
      mylen += end - B.seg_start[sj];
    }
    // block exclusive scan (warp shuffles + one smem pass)
    unsigned long long x = mylen;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) s_scan[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long acc = 0;
      for (uint32_t w = 0; w < SCHED_BLOCK / 32; w++) {
        unsigned long long v = s_scan[w];
        s_scan[w] = acc;
        acc += v;
      }
      s_scan[SCHED_BLOCK / 32] = acc;
      s_best = ~0ull;
      s_blkfull = 0;
      s_released = 0;
    }
    __syncthreads();
    const unsigned long long total = s_scan[SCHED_BLOCK / 32];
    unsigned long long run = s_step + s_scan[wid] + x - mylen;
    uint32_t c_ret = 0, c_full = 0;
    for (uint32_t t = lo; t < hi; t++) {
      if (st[t] == TS_RUN) {
        uint32_t g = t0 + t;
        uint64_t sj = B.seg_off[g] + sg[t];
        bool last = sj + 1 >= B.seg_off[g + 1];
        uint64_t end = last ? B.thread_stmt[g + 1] : B.seg_start[sj + 1];
        B.seg_base[sj] = (uint32_t)run;
        run += end - B.seg_start[sj];
        if (last) {
          st[t] = TS_RET;
        } else {
          st[t] = TS_BLOCK;
          bs[t] = B.seg_set[sj];
        }
      }
      c_ret += st[t] == TS_RET;
      c_full += st[t] == TS_BLOCK && bs[t] == full;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_step += total;
      s_ret = 0;
    }
    __syncthreads();
    if (c_ret) atomicAdd(&s_ret, c_ret);
    if (c_full) atomicAdd(&s_blkfull, c_full);
    __syncthreads();
    // ---- release phase: the releasable set with the smallest min tid; a
    // set is checked once, by its first blocked member
    unsigned long long best = ~0ull;
    for (uint32_t t = lo; t < hi; t++) {
      if (st[t] != TS_BLOCK) continue;
      const uint32_t I = bs[t];
      bool ok;
      uint32_t mn;
      if (I == full) {
        ok = (s_blkfull + s_ret == T);
        mn = 0;
      } else {
        const veq_syncset q = B.sets[I];
        ok = true;
        mn = UNSET;
        bool skip = false;  // a smaller member blocked on I makes the same check
        for (uint32_t k = 0; k < q.n_bits; k++) {
          if (!((B.set_words[q.word_off + k / 64] >> (k % 64)) & 1ull)) continue;
          const uint32_t m = q.lo + k;
          if (mn == UNSET) mn = m;
          if (m >= T) {
            ok = false;
            break;
          }
          const uint8_t sm = st[m];
          if (sm == TS_BLOCK && bs[m] == I) {
            if (m < t) {
              skip = true;
              break;
            }
            continue;
          }
          if (sm == TS_RET) continue;
          ok = false;
          break;
        }
        if (skip) continue;
      }
      if (ok) {
        // releasable_syncs order (symexec.cpp:616-654): smallest min tid,
        // ties in discovery order = smallest blocked member (t checks I)
        unsigned long long key = ((unsigned long long)mn << 32) | t;
        best = key < best ? key : best;
      }
    }
    if (best != ~0ull) atomicMin(&s_best, best);
    __syncthreads();
    const unsigned long long sb = s_best;
    if (sb != ~0ull) {
      const uint32_t I = bs[(uint32_t)(sb & 0xffffffffu)];
      uint32_t c = 0;
      for (uint32_t t = lo; t < hi; t++) {
        if (st[t] != TS_BLOCK || bs[t] != I) continue;
        uint32_t g = t0 + t;
        uint32_t ns = sg[t] + 1;
        sg[t] = ns;
        uint64_t start = B.seg_start[B.seg_off[g] + ns];
        bool ret = start == B.thread_stmt[g + 1];
        st[t] = ret ? TS_RET : TS_RUN;
        c += ret;
      }
      if (c) atomicAdd(&s_ret, c);
      if (threadIdx.x == 0) {
        uint64_t r = B.rel_off[p] + s_nrel;
        if (r < B.rel_off[p + 1]) {
          B.rel_step[r] = (uint32_t)s_step;
          B.rel_set[r] = I;
        }
        s_nrel++;
        s_step += 1;
        s_released = 1;
      }
    }
    __syncthreads();
    if (total == 0 && !s_released) break;
  }
  // write back the final control state (deadlock reports) and the summary
  if (on_chip)
    for (uint32_t t = lo; t < hi; t++) {
      B.th_state[t0 + t] = st[t];
      B.th_seg[t0 + t] = sg[t];
      B.th_bset[t0 + t] = bs[t];
    }
  if (threadIdx.x == 0) {
    B.prog_nrel[p] = s_nrel;
    B.prog_steps[p] = s_step;
    B.prog_dead[p] = s_ret != T;
  }
}

__global__ void __launch_bounds__(1024, 2) k_schedule_lanes(Batch B) {
  __shared__ uint8_t s_st[1024];
  __shared__ uint32_t s_bs[1024];
  __shared__ unsigned long long s_scan[33];
  __shared__ unsigned long long s_best;
  __shared__ uint32_t s_blkfull;
  const uint32_t p = blockIdx.x, t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  const veq_program_meta pm = B.progs[p];
  const uint32_t T = pm.n_threads, full = B.prog_full_set[p];
  const uint32_t g = pm.thread_off + t;
  uint8_t st = TS_NONE;
  uint32_t bset = UNSET, nset = UNSET;
  uint64_t sj = 0, sj_end = 0, s_end = 0, cur_start = 0, next_start = 0, nword = 0;
  veq_syncset nq{};
  // the set ending the current segment and its descriptor are loaded when
  // the segment starts, off the critical path of the round that blocks
  auto prefetch = [&]() {
    next_start = sj + 1 < sj_end ? B.seg_start[sj + 1] : s_end;
    nset = sj + 1 < sj_end ? B.seg_set[sj] : UNSET;
    if (nset != UNSET && nset != full) {
      nq = B.sets[nset];
      nword = B.set_words[nq.word_off];
    }
  };
  if (t < T) {
    sj = B.seg_off[g];
    sj_end = B.seg_off[g + 1];
    s_end = B.thread_stmt[g + 1];
    cur_start = B.seg_start[sj];
    prefetch();
    st = cur_start == s_end ? TS_RET : TS_RUN;
  }
  s_st[t] = st;
  s_bs[t] = UNSET;
  unsigned long long step = 0;
  uint32_t nrel = 0;
  uint32_t ret_count = __syncthreads_count(st == TS_RET);
  while (ret_count != T) {
    // ---- run phase: every runnable thread executes its current segment;
    // an ordered block scan of the lengths gives round-robin step numbers
    const unsigned long long len = st == TS_RUN ? next_start - cur_start : 0;
    unsigned long long x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(kFull, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) s_scan[wid] = x;
    if (t == 0) {
      s_best = ~0ull;
      s_blkfull = 0;
    }
    __syncthreads();
    if (wid == 0) {
      const unsigned long long v = lane < nw ? s_scan[lane] : 0;
      unsigned long long z = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(kFull, z, o);
        if (lane >= (unsigned)o) z += y;
      }
      if (lane < nw) s_scan[lane] = z - v;
      if (lane == 31) s_scan[32] = z;
    }
    __syncthreads();
    const unsigned long long total = s_scan[32];
    if (st == TS_RUN) {
      B.seg_base[sj] = (uint32_t)(step + s_scan[wid] + x - len);
      if (sj + 1 >= sj_end) {
        st = TS_RET;
      } else {
        st = TS_BLOCK;
        bset = nset;
        s_bs[t] = bset;
      }
      s_st[t] = st;
    }
    step += total;
    {
      const uint32_t cf = __popc(__ballot_sync(kFull, st == TS_BLOCK && bset == full));
      if (lane == 0 && cf) atomicAdd(&s_blkfull, cf);
    }
    ret_count = __syncthreads_count(st == TS_RET);
    // ---- release phase: the releasable set with the smallest min tid, ties
    // in discovery order = smallest blocked member (releasable_syncs)
    const uint32_t blkd = __ballot_sync(kFull, st == TS_BLOCK);
    const uint32_t retm = __ballot_sync(kFull, st == TS_RET);
    if (st == TS_BLOCK) {
      const uint32_t grp = __match_any_sync(blkd, bset);
      if ((uint32_t)(__ffs(grp) - 1) == lane) {  // smallest lane blocked on I here
        bool ok;
        uint32_t mn, first = t;
        if (bset == full) {
          ok = s_blkfull + ret_count == T;
          mn = 0;
        } else {
          const veq_syncset q = nq;
          const uint32_t w0 = wid * 32;
          if (q.lo >= w0 && q.lo + q.n_bits <= w0 + 32) {
            // window inside this warp: one vote decides it (members beyond
            // the CTA are TS_NONE lanes, so they fail the test)
            const uint64_t bits = nword & (q.n_bits >= 64 ? ~0ull : ((1ull << q.n_bits) - 1));
            const uint32_t M = (uint32_t)(bits << (q.lo - w0));
            ok = M != 0 && (M & ~(grp | retm)) == 0;
            mn = M ? w0 + __ffs(M) - 1 : q.lo;
          } else {
            ok = true;
            mn = UNSET;
            for (uint32_t k = 0; k < q.n_bits; k++) {
              if (!((B.set_words[q.word_off + k / 64] >> (k % 64)) & 1ull)) continue;
              const uint32_t m = q.lo + k;
              if (mn == UNSET) mn = m;
              if (m >= T) {
                ok = false;
                break;
              }
              const uint8_t sm = s_st[m];
              if (sm == TS_RET) continue;
              if (sm == TS_BLOCK && s_bs[m] == bset) {
                first = m < first ? m : first;
                continue;
              }
              ok = false;
              break;
            }
            if (mn == UNSET) mn = q.lo;
          }
        }
        if (ok) atomicMin(&s_best, ((unsigned long long)mn << 32) | first);
      }
    }
    __syncthreads();
    const unsigned long long sb = s_best;
    const bool released = sb != ~0ull;
    if (released) {
      const uint32_t I = s_bs[(uint32_t)(sb & 0xffffffffu)];
      if (st == TS_BLOCK && bset == I) {
        sj++;
        cur_start = next_start;
        prefetch();
        st = cur_start == s_end ? TS_RET : TS_RUN;
        s_st[t] = st;
      }
      if (t == 0) {
        const uint64_t r = B.rel_off[p] + nrel;
        if (r < B.rel_off[p + 1]) {
          B.rel_step[r] = (uint32_t)step;
          B.rel_set[r] = I;
        }
      }
      nrel++;
      step += 1;
    }
    ret_count = __syncthreads_count(st == TS_RET);
    if (total == 0 && !released) break;
  }
  if (t < T) {
    B.th_state[g] = st;
    B.th_seg[g] = (uint32_t)(sj - B.seg_off[g]);
    B.th_bset[g] = st == TS_BLOCK ? bset : UNSET;
  }
  if (t == 0) {
    B.prog_nrel[p] = nrel;
    B.prog_steps[p] = step;
    B.prog_dead[p] = ret_count != T;
  }
}

__global__ void __launch_bounds__(SW_WARPS * 32) k_schedule_warp(Batch B) {
  extern __shared__ __align__(16) char swsm[];
  SchedWarpSmem &S = reinterpret_cast<SchedWarpSmem *>(swsm)[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t p = blockIdx.x * SW_WARPS + (threadIdx.x >> 5);
  if (p >= B.n_progs) return;
  const veq_program_meta pm = B.progs[p];
  const uint32_t T = pm.n_threads, full = B.prog_full_set[p], nch = (T + 31) / 32;
  const uint64_t seg0 = B.seg_off[pm.thread_off];
  // segment j (absolute) of thread g: length, ending set and its chunk mask
  auto seg_info = [&](uint32_t g, uint64_t j, uint32_t &ln, uint32_t &set, uint32_t &msk) {
    set = B.seg_set[j];
    const uint64_t start = B.seg_start[j];
    const uint64_t end = set == UNSET ? B.thread_stmt[g + 1] : B.seg_start[j + 1];
    ln = (uint32_t)(end - start);
    msk = (set != UNSET && set != full) ? (uint32_t)B.set_chunk[set] : 0u;
  };
  uint32_t ret = 0, blkfull = 0, fullmin = UNSET;
  for (uint32_t t = lane; t < nch * 32; t += 32) {
    uint8_t st = TS_NONE;
    if (t < T) {
      const uint32_t g = pm.thread_off + t;
      const uint64_t so = B.seg_off[g];
      uint32_t ln, set, msk;
      seg_info(g, so, ln, set, msk);
      S.cj[t] = (uint32_t)(so - seg0);
      S.len[t] = ln;
      S.nset[t] = set;
      S.nm[t] = msk;
      S.bs[t] = UNSET;
      S.bm[t] = 0;
      st = (set == UNSET && ln == 0) ? TS_RET : TS_RUN;
    }
    S.st[t] = st;
    ret += __popc(__ballot_sync(kFull, st == TS_RET));
  }
  for (uint32_t c = lane; c < 32; c += 32) S.cand[c] = ~0ull;
  __syncwarp();
  uint32_t dirty = nch >= 32 ? ~0u : ((1u << nch) - 1);
  unsigned long long step = 0;
  uint32_t nrel = 0;
  // next-segment loads of threads that block stay in registers and are
  // written to shared memory at the start of the next round, so the warp
  // does not wait for them inside the round that issued them (a released
  // thread is marked runnable; an empty last segment returns when it "runs")
  bool p_has = false;
  uint32_t p_t = 0, p_len = 0, p_set = 0, p_msk = 0;
  while (ret != T) {
    if (p_has) {
      S.len[p_t] = p_len;
      S.nset[p_t] = p_set;
      S.nm[p_t] = p_msk;
      p_has = false;
    }
    __syncwarp();
    const bool single = __popc(dirty) == 1;
    // ---- run phase over the dirty chunks, in tid order
    unsigned long long total = 0;
    for (uint32_t dm = dirty; dm; dm &= dm - 1) {
      const uint32_t c = __ffs(dm) - 1, t = c * 32 + lane;
      const bool run = S.st[t] == TS_RUN;
      const uint32_t ln = run ? S.len[t] : 0;
      uint32_t tot;
      const uint32_t ex = warp_excl_scan(ln, tot);
      bool newret = false, newfull = false;
      if (run) {
        const uint32_t cj = S.cj[t];
        B.seg_base[seg0 + cj] = (uint32_t)(step + total + ex);
        const uint32_t set = S.nset[t];
        if (set == UNSET) {
          S.st[t] = TS_RET;
          newret = true;
        } else {
          S.st[t] = TS_BLOCK;
          S.bs[t] = set;
          S.bm[t] = S.nm[t];
          newfull = set == full;
          // prefetch the segment after the sync: it runs when the set is
          // released, so these loads are off the critical path
          uint32_t ln2, set2, msk2;
          seg_info(pm.thread_off + t, seg0 + cj + 1, ln2, set2, msk2);
          S.cj[t] = cj + 1;
          if (single) {
            p_has = true;
            p_t = t;
            p_len = ln2;
            p_set = set2;
            p_msk = msk2;
          } else {
            S.len[t] = ln2;
            S.nset[t] = set2;
            S.nm[t] = msk2;
          }
        }
      }
      ret += __popc(__ballot_sync(kFull, newret));
      const uint32_t nf = __ballot_sync(kFull, newfull);
      blkfull += __popc(nf);
      if (nf) fullmin = min(fullmin, c * 32 + __ffs(nf) - 1);
      total += tot;
    }
    step += total;
    // ---- release candidates of the dirty chunks: a window set inside the
    // chunk is releasable iff every member is blocked on it or returned
    for (uint32_t dm = dirty; dm; dm &= dm - 1) {
      const uint32_t c = __ffs(dm) - 1, t = c * 32 + lane;
      const uint8_t st = S.st[t];
      const uint32_t bs = S.bs[t];
      const uint32_t retm = __ballot_sync(kFull, st == TS_RET);
      const uint32_t blk = __ballot_sync(kFull, st == TS_BLOCK && bs != full);
      unsigned long long key = ~0ull;
      if ((blk >> lane) & 1u) {
        const uint32_t grp = __match_any_sync(blk, bs);
        if ((uint32_t)(__ffs(grp) - 1) == lane) {
          const uint32_t M = S.bm[t];
          if (M != 0 && (M & ~(grp | retm)) == 0) key = ((unsigned long long)(c * 32 + __ffs(M) - 1) << 32) | t;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(kFull, key, o);
        key = y < key ? y : key;
      }
      if (lane == 0) S.cand[c] = key;
    }
    __syncwarp();
    // ---- the release: smallest (min tid, first blocked member)
    unsigned long long best = lane < nch ? S.cand[lane] : ~0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(kFull, best, o);
      best = y < best ? y : best;
    }
    if (blkfull && blkfull + ret == T) {
      const unsigned long long fk = (unsigned long long)fullmin;  // min tid 0
      best = fk < best ? fk : best;
    }
    if (best == ~0ull) {
      if (total == 0) break;  // nothing ran, nothing releasable: done or deadlock
      dirty = 0;
      continue;
    }
    const uint32_t I = S.bs[(uint32_t)(best & 0xffffffffu)];
    dirty = 0;
    if (I == full) {
      for (uint32_t c = 0; c < nch; c++) {
        const uint32_t t = c * 32 + lane;
        const bool rel = S.st[t] == TS_BLOCK && S.bs[t] == full;
        if (rel) S.st[t] = TS_RUN;
        if (__ballot_sync(kFull, rel)) dirty |= 1u << c;
      }
      blkfull = 0;
      fullmin = UNSET;
    } else {
      const uint32_t c = (uint32_t)(best & 0xffffffffu) / 32, t = c * 32 + lane;
      const bool rel = S.st[t] == TS_BLOCK && S.bs[t] == I;
      if (rel) S.st[t] = TS_RUN;
      dirty = 1u << c;
    }
    __syncwarp();
    if (lane == 0) {
      const uint64_t r = B.rel_off[p] + nrel;
      if (r < B.rel_off[p + 1]) {
        B.rel_step[r] = (uint32_t)step;
        B.rel_set[r] = I;
      }
    }
    nrel++;
    step += 1;
  }
  if (p_has) {
    S.len[p_t] = p_len;
    S.nset[p_t] = p_set;
    S.nm[p_t] = p_msk;
  }
  __syncwarp();
  for (uint32_t t = lane; t < T; t += 32) {
    const uint32_t g = pm.thread_off + t;
    const uint8_t st = S.st[t];
    B.th_state[g] = st;
    // blocked threads: the segment that ended at their sync
    B.th_seg[g] = S.cj[t] - (uint32_t)(B.seg_off[g] - seg0) - (st == TS_BLOCK ? 1u : 0u);
    B.th_bset[g] = st == TS_BLOCK ? S.bs[t] : UNSET;
  }
  if (lane == 0) {
    B.prog_nrel[p] = nrel;
    B.prog_steps[p] = step;
    B.prog_dead[p] = ret != T;
  }
}

__global__ void k_exec(Batch B, Table T) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= B.n_threads) return;
  if (B.thread_stmt[g + 1] - B.thread_stmt[g] >= EXEC_WARP_MIN) return;
  const uint32_t p = B.thread_prog[g];
  const veq_program_meta pm = B.progs[p];
  const uint32_t tid = g - pm.thread_off;
  // a short thread's register file lives in local memory (per-thread
  // interleaved, L1-resident) when it is small, else in the global file
  constexpr uint32_t LREG = 32;
  uint32_t lregs[LREG];
  const uint32_t nregs = (uint32_t)(B.reg_off[g + 1] - B.reg_off[g]);
  uint32_t *regs = B.regfile + B.reg_off[g];
  if (nregs <= LREG) {
#pragma unroll
    for (uint32_t k = 0; k < LREG; k++) lregs[k] = UNSET;
    regs = lregs;
  }
  const uint64_t s0 = B.thread_stmt[g], s1 = B.thread_stmt[g + 1];
  const uint64_t j0 = B.seg_off[g], j1 = B.seg_off[g + 1];
  for (uint64_t j = j0; j < j1; j++) {
    uint32_t base = B.seg_base[j];
    if (base == UNSET) break;  // segment never ran (deadlock)
    uint64_t start = B.seg_start[j], end = (j + 1 < j1) ? B.seg_start[j + 1] : s1;
    for (uint64_t i = start; i < end; i++) {
      const veq_stmt st = B.stmts[i];
      const uint32_t step = base + (uint32_t)(i - start);
      auto readreg = [&](uint32_t r, uint8_t slot) -> uint32_t {
        uint32_t v = regs[r];
        if (v == UNSET) {
          veq_fault f{};
          f.type = VEQ_FAULT_SAFETY;
          f.kind = VEQ_SAFE_UNINIT_REG;
          f.sub = slot;
          f.reg_slot = slot;
          f.prog = p;
          f.tid = tid;
          f.stmt = (uint32_t)i;
          f.step = step;
          emit_fault(B, f);
          v = REF_NODE | intern_undef(T, 0, g, r);
          regs[r] = v;
        }
        return v;
      };
      switch (st.kind) {
      case VEQ_ST_SETCONST:
        regs[st.dst] = REF_NODE | (st.op == 1 ? T.id_neginf : B.const_node[st.a]);
        break;
      case VEQ_ST_COPY: {
        uint32_t v = readreg(st.a, 0);
        regs[st.dst] = v;
        break;
      }
      case VEQ_ST_BINOP: {
        uint32_t va = readreg(st.a, 0);
        uint32_t vb = readreg(st.b, 1);
        B.st_step[i] = step;
        uint32_t ra = va, rb = vb;
        if (st.op == VEQ_BIN_ADD || st.op == VEQ_BIN_MAX) {
          // chain linking: continue a chain whose tail this thread holds
          auto tail = [&](uint32_t v) -> bool {
            if (!is_stmt_ref(v)) return false;
            if (v < s0 || v >= i) return false;
            veq_stmt sk = B.stmts[v];
            return sk.kind == VEQ_ST_BINOP && sk.op == st.op && !B.continued[v];
          };
          uint32_t k = UNSET, leaf = 0;
          if (tail(va)) {
            k = va;
            leaf = vb;
          } else if (tail(vb)) {
            k = vb;
            leaf = va;
          }
          if (k != UNSET) {
            uint32_t h = B.chain_head[k];
            uint32_t pos = B.chain_pos[k] + 1;
            B.continued[k] = 1;
            B.chain_head[i] = h;
            B.chain_pos[i] = pos;
            B.chain_len[h] = pos + 1;
            ra = k;
            rb = leaf;
          } else {
            B.chain_head[i] = (uint32_t)i;
            B.chain_pos[i] = 0;
            B.chain_len[i] = 1;
          }
        }
        B.ref_a[i] = ra;
        B.ref_b[i] = rb;
        regs[st.dst] = (uint32_t)i;
        break;
      }
      case VEQ_ST_UNOP: {
        uint32_t va = readreg(st.a, 0);
        B.st_step[i] = step;
        B.ref_a[i] = va;
        regs[st.dst] = (uint32_t)i;
        break;
      }
      case VEQ_ST_LOAD:
      case VEQ_ST_STORE: {
        const uint32_t ga = pm.array_off + st.arr;
        const veq_array arr = B.arrays[ga];
        const int32_t off = (int32_t)st.a;
        const bool is_store = st.kind == VEQ_ST_STORE;
        if (off < 0 || (uint64_t)off >= arr.size) {
          veq_fault f{};
          f.type = VEQ_FAULT_SAFETY;
          f.kind = VEQ_SAFE_OOB;
          f.sub = 2;
          f.is_write = is_store;
          f.prog = p;
          f.tid = tid;
          f.stmt = (uint32_t)i;
          f.step = step;
          f.arr = st.arr;
          f.offset = off;
          emit_fault(B, f);
          if (!is_store) regs[st.dst] = REF_NODE | intern_undef(T, 1, ga, (uint64_t)(uint32_t)off);
          break;
        }
        if (!is_store) {
          if (!(arr.flags & VEQ_ARR_STORED) && arr.input >= 0 && (uint32_t)off < arr.seeded) {
            regs[st.dst] = REF_NODE | B.canon[i];  // interned by k_pre_inputs
            break;
          }
          regs[st.dst] = (uint32_t)i;
        } else {
          uint32_t v = readreg(st.dst, 0);
          B.ref_a[i] = v;
        }
        B.st_step[i] = step;
        uint64_t cell = B.arr_cell_base[ga] + (uint64_t)off;
        // warp-aggregated slot (coalesced writes); unfilled slots keep key ~0
        const unsigned long long slot = agg_inc(B.n_tup);
        B.tup_key[slot] = (cell << B.step_bits) | step;
        B.tup_val[slot] = ((unsigned long long)i << 32) | tid;
        break;
      }
      case VEQ_ST_SYNC:
      default:
        break;
      }
    }
  }
  // the Final register file (Outcome::regs, symexec.hpp:155-156) when asked
  if (B.keep_regs && regs == lregs) {
    uint32_t *out = B.regfile + B.reg_off[g];
    for (uint32_t k = 0; k < nregs && k < LREG; k++) out[k] = lregs[k];
  }
}

// Per-warp shared table of the registers defined in the current
// 32-statement batch (at most 32, open addressing over 128 slots): register
// id -> mask of the defining lanes. The last earlier definition of an
// operand and the last definition of a register are then bit scans instead
// of 32-step shuffle loops, for any register count.
constexpr uint32_t EXEC_DEF_SLOTS = 128;

__global__ void __launch_bounds__(128) k_exec_warp(Batch B, Table T) {
  __shared__ uint32_t s_key[4][EXEC_DEF_SLOTS], s_mask[4][EXEC_DEF_SLOTS];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t *dkey = s_key[(threadIdx.x >> 5) & 3], *dmask = s_mask[(threadIdx.x >> 5) & 3];
  for (uint32_t r = lane; r < EXEC_DEF_SLOTS; r += 32) {
    dkey[r] = UNSET;
    dmask[r] = 0;
  }
  __syncwarp();
  if (w >= B.n_long) return;
  const uint32_t g = B.long_threads[w];
  const uint32_t p = B.thread_prog[g];
  const veq_program_meta pm = B.progs[p];
  const uint32_t tid = g - pm.thread_off;
  uint32_t *regs = B.regfile + B.reg_off[g];
  auto def_slot = [&](uint32_t r) { return (r * 0x9E3779B1u) >> 25; };  // 7 bits
  auto def_lanes = [&](uint32_t r) -> uint32_t {  // lanes of this batch defining r
    for (uint32_t sl = def_slot(r);; sl = (sl + 1) & (EXEC_DEF_SLOTS - 1)) {
      const uint32_t k = dkey[sl];
      if (k == r) return dmask[sl];
      if (k == UNSET) return 0u;
    }
  };
  const uint64_t s0 = B.thread_stmt[g], s1 = B.thread_stmt[g + 1];
  const uint64_t j0 = B.seg_off[g], j1 = B.seg_off[g + 1];
  // the previous batch's chain state, lane k describing statement
  // pv_bt + k: operator (0xFF: not a chain op), continued at batch end,
  // head and position. Links into the previous batch read these registers.
  uint64_t pv_bt = ~0ull;
  uint32_t pv_n = 0, pv_op = 0xFFu, pv_head = 0, pv_pos = 0;
  bool pv_cont = false;
  for (uint64_t j = j0; j < j1; j++) {
    const uint32_t base = B.seg_base[j];
    if (base == UNSET) break;  // segment never ran (deadlock)
    const uint64_t start = B.seg_start[j], end = (j + 1 < j1) ? B.seg_start[j + 1] : s1;
    for (uint64_t bt = start; bt < end; bt += 32) {
      const uint64_t i = bt + lane;
      const bool act = i < end;
      veq_stmt st;
      if (act) st = B.stmts[i];
      else {
        st.kind = VEQ_ST_SYNC;
        st.op = 0;
        st.arr = 0;
        st.dst = st.a = st.b = 0;
      }
      const uint32_t step = base + (uint32_t)(i - start);
      // ---- memory statements: bounds and direct input loads
      uint32_t ga = 0;
      veq_array arr{};
      int32_t off = 0;
      bool oob = false, direct = false, mem = act && (st.kind == VEQ_ST_LOAD || st.kind == VEQ_ST_STORE);
      if (mem) {
        ga = pm.array_off + st.arr;
        arr = B.arrays[ga];
        off = (int32_t)st.a;
        oob = off < 0 || (uint64_t)off >= arr.size;
        direct = !oob && st.kind == VEQ_ST_LOAD && !(arr.flags & VEQ_ARR_STORED) && arr.input >= 0 &&
                 (uint32_t)off < arr.seeded;
      }
      // a direct load's symbol (interned by k_pre_inputs), fetched early so
      // the load overlaps the bookkeeping below
      const uint32_t in_node = direct ? __ldcg(B.canon + i) : UNSET;
      const uint32_t def = (act && defines_reg(st.kind)) ? st.dst : UNSET;
      // operand registers (UNSET: none). An out-of-bounds store reads nothing.
      uint32_t ra = UNSET, rb = UNSET;
      if (act) {
        if (st.kind == VEQ_ST_COPY || st.kind == VEQ_ST_UNOP || st.kind == VEQ_ST_BINOP) ra = st.a;
        if (st.kind == VEQ_ST_BINOP) rb = st.b;
        if (st.kind == VEQ_ST_STORE && !oob) ra = st.dst;
      }
      // ---- last defining lane before me for each operand, and whether I
      // am the last definition of my register in this batch
      int la = -1, lb = -1;
      bool last_def = def != UNSET;
      {
        uint32_t my_slot = UNSET;
        if (def != UNSET) {
          for (uint32_t sl = def_slot(def);; sl = (sl + 1) & (EXEC_DEF_SLOTS - 1)) {
            const uint32_t prev = atomicCAS(dkey + sl, UNSET, def);
            if (prev == UNSET || prev == def) {
              atomicOr(dmask + sl, 1u << lane);
              my_slot = sl;
              break;
            }
          }
        }
        __syncwarp();
        const uint32_t below = (1u << lane) - 1u;
        if (ra != UNSET) {
          const uint32_t m = def_lanes(ra) & below;
          la = m ? 31 - __clz(m) : -1;
        }
        if (rb != UNSET) {
          const uint32_t m = def_lanes(rb) & below;
          lb = m ? 31 - __clz(m) : -1;
        }
        if (def != UNSET) last_def = (31 - __clz(dmask[my_slot])) == (int)lane;
        __syncwarp();
        if (my_slot != UNSET) {
          dkey[my_slot] = UNSET;
          dmask[my_slot] = 0;
        }
        __syncwarp();
      }
      // ---- register-file reads (operands with no earlier def in this batch)
      uint32_t fa = UNSET, fb = UNSET;
      if (ra != UNSET && la < 0) fa = regs[ra];
      if (rb != UNSET && lb < 0) fb = regs[rb];
      // uninitialised reads: the first read of a register in this batch faults
      const uint32_t ua = (ra != UNSET && la < 0 && fa == UNSET) ? ra : UNSET;
      const uint32_t ub = (rb != UNSET && lb < 0 && fb == UNSET) ? rb : UNSET;
      bool first_a = ua != UNSET, first_b = ub != UNSET && ub != ua;
      if (__any_sync(kFull, ua != UNSET || ub != UNSET)) {
        for (uint32_t k = 0; k < 32; k++) {
          uint32_t uak = __shfl_sync(kFull, ua, k), ubk = __shfl_sync(kFull, ub, k);
          if (k < lane) {
            if (ua != UNSET && (uak == ua || ubk == ua)) first_a = false;
            if (ub != UNSET && (uak == ub || ubk == ub)) first_b = false;
          }
        }
      }
      if (ua != UNSET) fa = REF_NODE | intern_undef(T, 0, g, ua);
      if (ub != UNSET) fb = REF_NODE | intern_undef(T, 0, g, ub);
      if (first_a || first_b) {
        veq_fault f{};
        f.type = VEQ_FAULT_SAFETY;
        f.kind = VEQ_SAFE_UNINIT_REG;
        f.prog = p;
        f.tid = tid;
        f.stmt = (uint32_t)i;
        f.step = step;
        if (first_a) {
          f.sub = 0;
          f.reg_slot = 0;
          emit_fault(B, f);
        }
        if (first_b) {
          f.sub = 1;
          f.reg_slot = 1;
          emit_fault(B, f);
        }
      }
      // ---- own value of each defining lane (copies resolved below)
      uint32_t val = UNSET;
      if (def != UNSET) {
        switch (st.kind) {
        case VEQ_ST_SETCONST: val = REF_NODE | (st.op == 1 ? T.id_neginf : B.const_node[st.a]); break;
        case VEQ_ST_BINOP:
        case VEQ_ST_UNOP: val = (uint32_t)i; break;
        case VEQ_ST_LOAD:
          if (oob) val = REF_NODE | intern_undef(T, 1, ga, (uint64_t)(uint32_t)off);
          else if (direct) val = REF_NODE | in_node;
          else val = (uint32_t)i;
          break;
        default: break;  // copy
        }
      }
      // ---- operand values; copies take their source's value (iterate until
      // every copy in the batch is resolved — chains are at most 31 long)
      uint32_t va = fa, vb = fb;
      bool pending_copy = st.kind == VEQ_ST_COPY && act;
      if (st.kind == VEQ_ST_COPY && act && la < 0) {
        val = va;
        pending_copy = false;
      }
      while (__any_sync(kFull, pending_copy)) {
        uint32_t src = __shfl_sync(kFull, val, la < 0 ? lane : (uint32_t)la);
        bool src_ready = __shfl_sync(kFull, !pending_copy, la < 0 ? lane : (uint32_t)la);
        if (pending_copy && src_ready) {
          val = src;
          pending_copy = false;
        }
      }
      {
        uint32_t x = __shfl_sync(kFull, val, la < 0 ? lane : (uint32_t)la);
        uint32_t y = __shfl_sync(kFull, val, lb < 0 ? lane : (uint32_t)lb);
        if (la >= 0) va = x;
        if (lb >= 0) vb = y;
      }
      if (st.kind == VEQ_ST_COPY && act) val = va;
      // ---- per-statement effects
      if (act) {
        if (mem && oob) {
          veq_fault f{};
          f.type = VEQ_FAULT_SAFETY;
          f.kind = VEQ_SAFE_OOB;
          f.sub = 2;
          f.is_write = st.kind == VEQ_ST_STORE;
          f.prog = p;
          f.tid = tid;
          f.stmt = (uint32_t)i;
          f.step = step;
          f.arr = st.arr;
          f.offset = off;
          emit_fault(B, f);
        } else if (mem && !direct) {
          if (st.kind == VEQ_ST_STORE) B.ref_a[i] = va;
          B.st_step[i] = step;
          uint64_t cell = B.arr_cell_base[ga] + (uint64_t)off;
          const unsigned long long slot = agg_inc(B.n_tup);  // coalesced; unfilled slots keep key ~0
          B.tup_key[slot] = (cell << B.step_bits) | step;
          B.tup_val[slot] = ((unsigned long long)i << 32) | tid;
        } else if (st.kind == VEQ_ST_BINOP || st.kind == VEQ_ST_UNOP) {
          B.st_step[i] = step;
          B.ref_a[i] = va;
          if (st.kind == VEQ_ST_BINOP) B.ref_b[i] = vb;
        }
      }
      // ---- chain links. In statement order, a chain op continues the
      // first of its operands that is a chain end of the same operator not
      // yet continued. Optimistically every lane decides at once against the
      // state before the batch; if no two lanes claim the same predecessor
      // that is exactly the sequential outcome, and heads and positions
      // follow by pointer jumping over the in-batch links. Otherwise the
      // lanes are decided one by one.
      const bool chain = act && st.kind == VEQ_ST_BINOP && (st.op == VEQ_BIN_ADD || st.op == VEQ_BIN_MAX);
      uint32_t my_head = 0, my_pos = 0;
      uint32_t cont_mask = 0;  // in-batch chain ops already continued
      uint32_t chain_lanes = __ballot_sync(kFull, chain);
      const uint32_t add_lanes = __ballot_sync(kFull, chain && st.op == VEQ_BIN_ADD);
      bool chains_done = false;
      if (chain_lanes) {
        const uint32_t same = chain ? (st.op == VEQ_BIN_ADD ? add_lanes : chain_lanes & ~add_lanes) : 0u;
        auto in_prev = [&](uint32_t v) { return is_stmt_ref(v) && pv_bt != ~0ull && v >= pv_bt && v < pv_bt + pv_n; };
        // the previous batch's state of both operands (all lanes shuffle)
        const uint32_t sa = in_prev(va) ? (uint32_t)(va - pv_bt) : lane, sb = in_prev(vb) ? (uint32_t)(vb - pv_bt) : lane;
        const uint32_t opa = __shfl_sync(kFull, pv_op, sa), opb = __shfl_sync(kFull, pv_op, sb);
        const bool cna = __shfl_sync(kFull, pv_cont, sa), cnb = __shfl_sync(kFull, pv_cont, sb);
        auto tail0 = [&](uint32_t v, uint32_t pop, bool pcont) -> bool {  // against the pre-batch state
          if (!is_stmt_ref(v) || v < s0 || v >= i) return false;
          if (v >= bt) return (same >> (uint32_t)(v - bt)) & 1u;
          if (in_prev(v)) return pop == st.op && !pcont;
          const veq_stmt sv = B.stmts[v];
          return sv.kind == VEQ_ST_BINOP && sv.op == st.op && !*((volatile uint8_t *)(B.continued + v));
        };
        uint32_t pred = UNSET, leaf = 0;
        if (chain) {
          if (tail0(va, opa, cna)) {
            pred = va;
            leaf = vb;
          } else if (tail0(vb, opb, cnb)) {
            pred = vb;
            leaf = va;
          }
        }
        // a predecessor claimed twice: fall back to the ordered decisions
        const uint32_t key = pred != UNSET ? pred : (0xFFFFFF00u | lane);
        const uint32_t peers = __match_any_sync(kFull, key);
        if (!__any_sync(kFull, __popc(peers) > 1)) {
          const bool in_b = pred != UNSET && pred >= bt;
          uint32_t anc = in_b ? (uint32_t)(pred - bt) : lane, dist = in_b ? 1u : 0u;
          uint32_t head0 = (uint32_t)i, pos0 = 0;
          const bool pp = chain && pred != UNSET && !in_b && in_prev(pred);
          const uint32_t sp = pp ? (uint32_t)(pred - pv_bt) : lane;
          const uint32_t ph = __shfl_sync(kFull, pv_head, sp), ppos = __shfl_sync(kFull, pv_pos, sp);
          if (chain && pred != UNSET && !in_b) {
            head0 = pp ? ph : B.chain_head[pred];
            pos0 = (pp ? ppos : B.chain_pos[pred]) + 1;
          }
#pragma unroll
          for (int r = 0; r < 5; r++) {
            dist += __shfl_sync(kFull, dist, anc);
            anc = __shfl_sync(kFull, anc, anc);
          }
          const uint32_t head = __shfl_sync(kFull, head0, anc);
          const uint32_t pos = __shfl_sync(kFull, pos0, anc) + dist;
          cont_mask = __reduce_or_sync(kFull, in_b ? 1u << (uint32_t)(pred - bt) : 0u);
          if (chain) {
            my_head = head;
            my_pos = pos;
            B.chain_head[i] = head;
            B.chain_pos[i] = pos;
            if (pred != UNSET) {
              B.ref_a[i] = pred;
              B.ref_b[i] = leaf;
              if (!in_b) B.continued[pred] = 1;
            }
          }
          // chain length: the last link of each head in this batch
          const uint32_t same_head = __match_any_sync(kFull, chain ? head : (0xFFFFFF00u | lane));
          if (chain && 31 - __clz(same_head) == (int)lane) B.chain_len[head] = pos + 1;
          chains_done = true;
        }
      }
      if (chains_done) chain_lanes = 0;
      while (chain_lanes) {
        const uint32_t k = __ffs(chain_lanes) - 1;
        chain_lanes &= chain_lanes - 1;
        const uint32_t vak = __shfl_sync(kFull, va, k), vbk = __shfl_sync(kFull, vb, k);
        const uint32_t opk = __shfl_sync(kFull, (uint32_t)st.op, k);
        const uint64_t ik = bt + k;
        // tail test for a candidate ref v (uniform across the warp)
        auto tail = [&](uint32_t v) -> bool {
          if (!is_stmt_ref(v) || v < s0 || v >= ik) return false;
          if (v >= bt) {
            uint32_t lv = (uint32_t)(v - bt);
            bool ch = (__ballot_sync(kFull, chain && st.op == opk) >> lv) & 1u;
            return ch && !((cont_mask >> lv) & 1u);
          }
          veq_stmt sv = B.stmts[v];
          return sv.kind == VEQ_ST_BINOP && sv.op == opk && !*((volatile uint8_t *)(B.continued + v));
        };
        uint32_t pred = UNSET, leaf = 0;
        bool ta = tail(vak);
        bool tb = !ta && tail(vbk);
        if (ta) {
          pred = vak;
          leaf = vbk;
        } else if (tb) {
          pred = vbk;
          leaf = vak;
        }
        uint32_t head, pos;
        if (pred != UNSET) {
          uint32_t hp, pp;
          if (pred >= bt) {
            hp = __shfl_sync(kFull, my_head, (uint32_t)(pred - bt));
            pp = __shfl_sync(kFull, my_pos, (uint32_t)(pred - bt));
            cont_mask |= 1u << (uint32_t)(pred - bt);
          } else {
            hp = B.chain_head[pred];
            pp = B.chain_pos[pred];
          }
          head = hp;
          pos = pp + 1;
          if (lane == 0) {
            if (pred < bt) B.continued[pred] = 1;
            B.chain_len[head] = pos + 1;
          }
        } else {
          head = (uint32_t)ik;
          pos = 0;
          if (lane == 0) B.chain_len[head] = 1;
        }
        if (lane == k) {
          my_head = head;
          my_pos = pos;
          B.chain_head[i] = head;
          B.chain_pos[i] = pos;
          if (pred != UNSET) {
            B.ref_a[i] = pred;
            B.ref_b[i] = leaf;
          }
        }
      }
      if ((cont_mask >> lane) & 1u) B.continued[i] = 1;
      pv_bt = bt;
      pv_n = (uint32_t)min((uint64_t)32, end - bt);
      pv_op = chain ? (uint32_t)st.op : 0xFFu;
      pv_cont = (cont_mask >> lane) & 1u;
      pv_head = my_head;
      pv_pos = my_pos;
      // ---- register file: seeds first, then the last def of each register
      if (first_a) regs[ua] = fa;
      if (first_b) regs[ub] = fb;
      __syncwarp();
      if (last_def) regs[def] = val;
      __syncwarp();
    }
  }
}

// One thread per address segment [s, e) of the (cell, step)-sorted tuples.
__global__ void k_mem_scan(Batch B, Table T, const unsigned long long *keys, const unsigned long long *vals,
                           const uint32_t *seg_starts, const unsigned long long *n_segs_dev, uint64_t n_tup,
                           Reader *rscratch) {
  const uint64_t n_segs = *n_segs_dev;  // device-side count: no host read-back
  uint32_t sidx = blockIdx.x * blockDim.x + threadIdx.x;
  if (sidx >= n_segs) return;
  const uint64_t s = seg_starts[sidx];
  const uint64_t cell = keys[s] >> B.step_bits;
  uint64_t e = s + 1;
  while (e < n_tup && (keys[e] >> B.step_bits) == cell) e++;
  // identify the array of this cell via the first tuple's statement
  const uint32_t stmt0 = (uint32_t)(vals[s] >> 32);
  const uint32_t tid0 = (uint32_t)(vals[s] & 0xffffffffu);
  (void)tid0;
  const veq_stmt st0 = B.stmts[stmt0];
  // program: thread of stmt0 -> binary search on thread_stmt
  uint32_t lo = 0, hi = B.n_threads;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) / 2;
    if (B.thread_stmt[mid] <= stmt0) lo = mid;
    else hi = mid;
  }
  const uint32_t p = B.thread_prog[lo];
  const veq_program_meta pm = B.progs[p];
  const uint32_t ga = pm.array_off + st0.arr;
  const veq_array arr = B.arrays[ga];
  const uint64_t offset = cell - B.arr_cell_base[ga];
  bool has = arr.input >= 0 && offset < arr.seeded;
  uint32_t value = has ? (REF_NODE | intern_input_var(T, (uint32_t)arr.input, offset)) : UNSET;
  bool w_valid = false;
  uint32_t w_tid = 0, w_step = 0, w_stmt = 0;
  Reader *rd = rscratch + s;
  uint32_t nrd = 0;
  for (uint64_t k = s; k < e; k++) {
    const uint32_t step = (uint32_t)(keys[k] & ((1ull << B.step_bits) - 1));
    const uint32_t stmt = (uint32_t)(vals[k] >> 32);
    const uint32_t tid = (uint32_t)(vals[k] & 0xffffffffu);
    const bool is_store = B.stmts[stmt].kind == VEQ_ST_STORE;
    if (!is_store) {
      if (w_valid && w_tid != tid && pending(B, p, w_tid, w_step, tid, step)) {
        veq_fault f{};
        f.type = VEQ_FAULT_RACE;
        f.sub = 0;
        f.prog = p;
        f.tid = tid;
        f.stmt = stmt;
        f.step = step;
        f.is_write = 0;
        f.tid2 = w_tid;
        f.stmt2 = w_stmt;
        f.step2 = w_step;
        f.is_write2 = 1;
        f.arr = st0.arr;
        f.offset = (int32_t)offset;
        emit_fault(B, f);
      }
      if (!has) {
        veq_fault f{};
        f.type = VEQ_FAULT_SAFETY;
        f.kind = VEQ_SAFE_UNINIT_MEM;
        f.sub = 2;
        f.prog = p;
        f.tid = tid;
        f.stmt = stmt;
        f.step = step;
        f.arr = st0.arr;
        f.offset = (int32_t)offset;
        emit_fault(B, f);
        value = REF_NODE | intern_undef(T, 2, cell >> 29, cell);
        has = true;
      }
      B.ref_a[stmt] = value;
      uint32_t q = 0;
      for (; q < nrd; q++)
        if (rd[q].tid == tid) break;
      rd[q] = Reader{tid, step, stmt, 0};
      if (q == nrd) nrd++;
    } else {
      uint32_t best = UNSET, bq = 0;
      for (uint32_t q = 0; q < nrd; q++) {
        if (rd[q].tid == tid || rd[q].tid >= best) continue;
        if (pending(B, p, rd[q].tid, rd[q].step, tid, step)) {
          best = rd[q].tid;
          bq = q;
        }
      }
      if (best != UNSET) {
        veq_fault f{};
        f.type = VEQ_FAULT_RACE;
        f.sub = 0;
        f.prog = p;
        f.tid = tid;
        f.stmt = stmt;
        f.step = step;
        f.is_write = 1;
        f.tid2 = best;
        f.stmt2 = rd[bq].stmt;
        f.step2 = rd[bq].step;
        f.is_write2 = 0;
        f.arr = st0.arr;
        f.offset = (int32_t)offset;
        emit_fault(B, f);
      }
      if (w_valid && w_tid != tid && pending(B, p, w_tid, w_step, tid, step)) {
        veq_fault f{};
        f.type = VEQ_FAULT_RACE;
        f.sub = 1;
        f.prog = p;
        f.tid = tid;
        f.stmt = stmt;
        f.step = step;
        f.is_write = 1;
        f.tid2 = w_tid;
        f.stmt2 = w_stmt;
        f.step2 = w_step;
        f.is_write2 = 1;
        f.arr = st0.arr;
        f.offset = (int32_t)offset;
        emit_fault(B, f);
      }
      w_valid = true;
      w_tid = tid;
      w_step = step;
      w_stmt = stmt;
      value = B.ref_a[stmt];
      has = true;
    }
  }
  B.final_val[cell] = has ? value : UNSET;
}

__global__ void __launch_bounds__(APP_NT) k_seg_heads(const unsigned long long *keys, uint64_t n, uint32_t *starts,
                                                     unsigned long long *n_starts, uint32_t step_bits) {
  // a head starts every run of equal cells; unfilled slots (key ~0, from
  // accesses that never executed) sort last and start nothing
  const uint64_t b0 = (uint64_t)blockIdx.x * APP_NT * APP_ITEMS + threadIdx.x;
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < APP_ITEMS; k++) {
    const uint64_t i = b0 + (uint64_t)k * APP_NT;
    if (i < n && keys[i] != ~0ull && (i == 0 || (keys[i] >> step_bits) != (keys[i - 1] >> step_bits)))
      mask |= 1u << k;
  }
  unsigned long long o = block_append<APP_NT>(n_starts, __popc(mask));
#pragma unroll
  for (int k = 0; k < APP_ITEMS; k++)
    if ((mask >> k) & 1u) starts[o++] = (uint32_t)(b0 + (uint64_t)k * APP_NT);
}

__global__ void k_resolve_finals(Batch B) {
  uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B.n_cells) return;
  uint32_t v = B.final_val[c];
  if (v == UNSET) return;
  v = chase(B, v);
  B.final_val[c] = v;
  if (is_stmt_ref(v)) {
    atomicAdd(B.uses + v, 1u);
    B.user[v] = USER_FINAL;
  }
}

// Final registers count as uses (and are never deferred) when kept: every
// register value is canonicalised like a final memory cell.
__global__ void k_resolve_regs(Batch B, uint64_t n_regs) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_regs) return;
  uint32_t v = B.regfile[k];
  if (v == UNSET) return;
  v = chase(B, v);
  B.regfile[k] = v;
  if (is_stmt_ref(v)) {
    atomicAdd(B.uses + v, 1u);
    B.user[v] = USER_FINAL;
  }
}

// Input symbols read by direct loads (never-stored input arrays) are
// interned in one parallel pass before execution; the executors read the
// node from canon[i].
// Direct input loads, in three passes so each input symbol is interned
// once: mark the cells the batch reads in the per-cell cache, intern every
// marked cell (one thread each, no contention on a key), then resolve every
// load from the cache.
constexpr uint32_t IN_NEEDED = 0xFFFFFFFEu;

__global__ void k_mark_inputs(Batch B, Table T) {
  __shared__ uint32_t s_p0;
  const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x;
  if (threadIdx.x == 0) s_p0 = prog_of_stmt(B, i0 < B.n_stmts ? i0 : B.n_stmts - 1);
  __syncthreads();
  const uint64_t i = i0 + threadIdx.x;
  if (i >= B.n_stmts) return;
  const veq_stmt st = B.stmts[i];
  if (st.kind != VEQ_ST_LOAD) return;
  const veq_program_meta pm = B.progs[prog_walk(B, s_p0, i)];
  const veq_array arr = B.arrays[pm.array_off + st.arr];
  const int32_t off = (int32_t)st.a;
  if (off < 0 || (uint64_t)off >= arr.size) return;
  if (!(arr.flags & VEQ_ARR_STORED) && arr.input >= 0 && (uint32_t)off < arr.seeded) {
    uint32_t *c = T.in_cache + T.in_base[arr.input] + (uint32_t)off;
    if (__ldcg(c) == UNSET) *c = IN_NEEDED;
  }
}

__global__ void k_intern_marked(Table T, uint64_t n_cells) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
       c += (uint64_t)gridDim.x * blockDim.x) {
    if (T.in_cache[c] != IN_NEEDED) continue;
    uint32_t j = 0;
    while (j + 1 < T.n_inputs && !(c >= T.in_base[j] && c < T.in_base[j] + T.in_size[j])) j++;
    const uint64_t cell = c - T.in_base[j];
    const uint64_t key = INPUT_KEY + T.in_base[j] + lexrank(cell, T.in_size[j]);
    T.in_cache[c] = intern(T, K_VAR, key, ((uint64_t)j << 40) | cell, nullptr, 0);
  }
}

__global__ void k_pre_inputs(Batch B, Table T) {
  __shared__ uint32_t s_p0;
  const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x;
  if (threadIdx.x == 0) s_p0 = prog_of_stmt(B, i0 < B.n_stmts ? i0 : B.n_stmts - 1);
  __syncthreads();
  const uint64_t i = i0 + threadIdx.x;
  if (i >= B.n_stmts) return;
  const veq_stmt st = B.stmts[i];
  if (st.kind != VEQ_ST_LOAD) return;
  const veq_program_meta pm = B.progs[prog_walk(B, s_p0, i)];
  const veq_array arr = B.arrays[pm.array_off + st.arr];
  const int32_t off = (int32_t)st.a;
  if (off < 0 || (uint64_t)off >= arr.size) return;
  if (!(arr.flags & VEQ_ARR_STORED) && arr.input >= 0 && (uint32_t)off < arr.seeded)
    B.canon[i] = intern_input_var(T, (uint32_t)arr.input, (uint64_t)off);
}

// One pass after the memory scan: operands resolved through loads, use
// counts, and the chain-log size of every chain head.
__global__ void k_resolve_all(Batch B, uint32_t *sz) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B.n_stmts) return;
  uint32_t v = 0;
  if (B.st_step[i] != UNSET) {
    const veq_stmt st = B.stmts[i];
    if (st.kind == VEQ_ST_BINOP) {
      const uint32_t a = chase(B, B.ref_a[i]), b = chase(B, B.ref_b[i]);
      B.ref_a[i] = a;
      B.ref_b[i] = b;
      // user[] is meaningful only where uses ends at 1 (a single writer)
      if (is_stmt_ref(a)) {
        atomicAdd(B.uses + a, 1u);
        B.user[a] = (uint32_t)i;
      }
      if (is_stmt_ref(b)) {
        atomicAdd(B.uses + b, 1u);
        B.user[b] = (uint32_t)i;
      }
      if ((st.op == VEQ_BIN_ADD || st.op == VEQ_BIN_MAX) && B.chain_head[i] == (uint32_t)i) v = B.chain_len[i] + 1;
    } else if (st.kind == VEQ_ST_UNOP) {
      const uint32_t a = chase(B, B.ref_a[i]);
      B.ref_a[i] = a;
      if (is_stmt_ref(a)) {
        atomicAdd(B.uses + a, 1u);
        B.user[a] = (uint32_t)i;
      }
    } else if (st.kind == VEQ_ST_STORE || st.kind == VEQ_ST_LOAD) {
      B.ref_a[i] = chase(B, B.ref_a[i]);
    }
  }
  sz[i] = v;
}

__global__ void k_mark_defer(Batch B) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // used-once first: loads, stores and syncs (uses 0) leave after one read
  if (i >= B.n_stmts || B.no_defer || B.uses[i] != 1 || B.st_step[i] == UNSET) return;
  const veq_stmt st = B.stmts[i];
  if (st.kind != VEQ_ST_BINOP || st.op != VEQ_BIN_MUL) return;
  const uint32_t u = B.user[i];
  if (u == USER_FINAL || u >= B.n_stmts) return;
  const veq_stmt su = B.stmts[u];
  if (su.kind != VEQ_ST_BINOP || su.op != VEQ_BIN_ADD) return;  // consumed as a chain leaf
  const uint32_t a = B.ref_a[i], b = B.ref_b[i];
  uint32_t X = UNSET;
  if (is_add_chain_end(B, a) && B.uses[a] == 1 && B.user[a] == (uint32_t)i) X = a;
  else if (is_add_chain_end(B, b) && B.uses[b] == 1 && B.user[b] == (uint32_t)i) X = b;
  if (X == UNSET) return;
  // flags of different statements share 32-bit words: set them atomically
  auto set_flag = [&](uint32_t x, uint8_t f) {
    atomicOr(reinterpret_cast<unsigned int *>(B.defer + (x & ~3u)), (unsigned)f << (8 * (x & 3u)));
  };
  set_flag((uint32_t)i, DF_LEAF);
  set_flag(X, DF_SUM);
  set_flag(B.chain_head[u], DF_CHAIN);
  atomicAdd(B.n_defer_chains, 1u);
}

// Two-pass evaluation: the deferred expansion (eval_add_deferred) needs a
// deep call stack that slows the whole evaluator down, so only the items
// from each program's first expanding chain onwards run in the kernel that
// carries it. Every dependency of an item is in its program at a smaller
// step, so pass 1 (steps below the split) never waits on pass 2.
__global__ void k_defer_split(Batch B) {
  if (*B.n_defer_chains == 0) return;  // nothing deferred: one pass
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B.n_stmts;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (B.st_step[i] == UNSET) continue;
    const veq_stmt st = B.stmts[i];
    if (!is_chain_op(st) || !(B.defer[B.chain_head[i]] & DF_CHAIN) || !is_work_item(B, i, st)) continue;
    atomicMin(B.prog_split + prog_of_stmt(B, i), B.st_step[i]);
  }
}

// One pass after the log scan: chain-log entries and the work list.
__global__ void __launch_bounds__(APP_NT) k_scatter_work(Batch B, const uint32_t *base, uint32_t *log,
                                                        uint32_t *log_stmt, unsigned long long *wkey, uint32_t *wval,
                                                        unsigned long long *n_work) {
  __shared__ uint32_t s_p0;
  const uint64_t blk0 = (uint64_t)blockIdx.x * APP_NT * APP_ITEMS;
  if (threadIdx.x == 0) s_p0 = prog_of_stmt(B, blk0 < B.n_stmts ? blk0 : B.n_stmts - 1);
  const uint64_t b0 = blk0 + threadIdx.x;
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < APP_ITEMS; k++) {
    const uint64_t i = b0 + (uint64_t)k * APP_NT;
    if (i >= B.n_stmts || B.st_step[i] == UNSET) continue;
    const veq_stmt st = B.stmts[i];
    if (is_chain_op(st)) {
      const uint32_t h = B.chain_head[i], pos = B.chain_pos[i];
      const uint32_t b = base[h];
      if (pos == 0) {
        log[b] = B.ref_a[i];
        log[b + 1] = B.ref_b[i];
        log_stmt[b] = (uint32_t)i;
        log_stmt[b + 1] = (uint32_t)i;
      } else {
        log[b + pos + 1] = B.ref_b[i];
        log_stmt[b + pos + 1] = (uint32_t)i;
      }
    }
    if (is_work_item(B, i, st)) mask |= 1u << k;
  }
  unsigned long long o = block_append<APP_NT>(n_work, __popc(mask));
#pragma unroll
  for (int k = 0; k < APP_ITEMS; k++) {
    if (!((mask >> k) & 1u)) continue;
    const uint64_t i = b0 + (uint64_t)k * APP_NT;
    // (step, program): every dependency of an item has a smaller step in the
    // same program, hence a smaller key, and all CTAs advance together
    const uint32_t p = prog_walk(B, s_p0, i);
    const unsigned long long pass2 = B.prog_split && B.st_step[i] >= B.prog_split[p];
    if (pass2) atomicAdd(n_work + 1, 1ull);
    wkey[o] = (pass2 << (B.prog_bits + B.step_bits)) | ((unsigned long long)B.st_step[i] << B.prog_bits) | p;
    wval[o] = (uint32_t)i;
    o++;
  }
}

// Work descriptor per sorted item: statement, chain-log base and leaf count
// (chain Adds), statement kind and op — one 16-byte load replaces the
// stmts -> chain_head/pos -> log_base chain of dependent reads.
__global__ void k_make_desc(Batch B, EvalCtx E, const uint32_t *work, const unsigned long long *n_work_dev,
                            uint4 *desc) {
  uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= *n_work_dev) return;
  const uint32_t i = work[w];
  const veq_stmt st = B.stmts[i];
  uint4 d{i, 0u, 0u, (uint32_t)st.kind | ((uint32_t)st.op << 8)};
  if (st.kind == VEQ_ST_BINOP && st.op == VEQ_BIN_ADD) {
    d.y = E.log_base[B.chain_head[i]];
    d.z = B.chain_pos[i] + 2;
    if (B.defer[B.chain_head[i]] & DF_CHAIN) d.w |= DESC_DEFER;
  }
  desc[w] = d;
}

// canon(a - b) (decide.cpp:779-787); ~0u: b is -inf (no Neg of -inf),
// ~1u: a is -inf (no Add with -inf)
__device__ __forceinline__ uint32_t canon_sub_one(const Table &T, Arena &A, uint32_t a, uint32_t b) {
  if (b == T.id_neginf) return ~0u;
  if (a == T.id_neginf) return ~1u;
  const Node nb = ld_node(T, b);
  uint32_t mb;
  if (nb.kind == K_CONST) {
    Rat v = const_val(nb);
    v.n = -v.n;
    mb = intern_const(T, v);
  } else {
    uint32_t ops[2] = {T.id_mone, b};
    mb = mul_canon(T, A, ops, 2);
  }
  uint32_t leaves[2] = {a, mb};
  return add_nary(T, A, leaves, 2);
}

__global__ void k_canon_sub(Table T, uint32_t a, uint32_t b, uint32_t *out, char *pool,
                            unsigned long long *pool_used, uint64_t pool_cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Arena A{pool, pool_used, pool_cap, &T, nullptr, 0, 0, 1ull << 20, 0};
  out[0] = canon_sub_one(T, A, a, b);
}

// veq_decide_batch: one difference per thread (equal pairs skipped)
__global__ void k_canon_sub_many(Table T, const uint32_t *fa, const uint32_t *gb, uint32_t *out, uint64_t n,
                                 char *pool, unsigned long long *pool_used, uint64_t pool_cap, uint64_t chunk) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t a = fa[i], b = gb[i];
  if (a == b) {
    out[i] = T.id_zero;
    return;
  }
  Arena A{pool, pool_used, pool_cap, &T, nullptr, 0, 0, chunk, i};
  out[i] = canon_sub_one(T, A, a, b);
}

// Fault order on the device (veq_run_finish): key (program, step, check
// order within the statement); the radix sort is stable, so equal keys keep
// their append order exactly as a host stable sort would.
__global__ void k_fault_keys(const veq_fault *f, uint64_t n, unsigned long long *key, uint32_t *idx) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const veq_fault x = f[i];
  key[i] = ((unsigned long long)x.prog << 40) | ((unsigned long long)x.step << 8) | x.sub;
  idx[i] = (uint32_t)i;
}
__global__ void k_fault_gather(const veq_fault *f, const uint32_t *idx, uint64_t n, veq_fault *out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = f[idx[i]];
}

__global__ void k_gather_stmts(const veq_stmt *stmts, const uint32_t *idx, uint64_t n, veq_stmt *out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = stmts[idx[i]];
}

__global__ void k_final_nodes(Batch B) {
  uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B.n_cells) return;
  uint32_t v = B.final_val[c];
  B.final_node[c] = (v == UNSET) ? UNSET : wait_node(B, v);
}

__global__ void k_intern_consts(Table T, const veq_rat *consts, uint32_t n, uint32_t *out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = intern_const(T, Rat{consts[i].num, consts[i].den});
}

__global__ void k_session_init(Table T, uint32_t *ids) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  ids[0] = intern(T, K_NEGINF, 0, 0, nullptr, 0);
  ids[1] = intern(T, K_CONST, 0, 1, nullptr, 0);
  ids[2] = intern(T, K_CONST, 1, 1, nullptr, 0);
  ids[3] = intern(T, K_CONST, (uint64_t)-1ll, 1, nullptr, 0);
}

__global__ void k_compare(Table T, const uint32_t *final_node_a, const uint32_t *final_node_b, CmpArgs C,
                          char *pool, unsigned long long *pool_used, uint64_t pool_cap, uint64_t chunk) {
  uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= C.n_vcs) return;
  Arena A{pool, pool_used, pool_cap, &T, nullptr, 0, 0, chunk, 0};
  uint32_t ca = C.cell_a[v], cb = C.cell_b[v];
  uint32_t na = ca == UNSET ? UNSET : final_node_a[ca];
  uint32_t nb = cb == UNSET ? UNSET : final_node_b[cb];
  veq_vc out{};
  out.node_a = na;
  out.node_b = nb;
  out.equal = (na != UNSET && na == nb);
  if (na == UNSET || nb == UNSET) atomicAdd(C.n_missing, 1ull);
  if (out.equal) atomicAdd(C.n_equal, 1ull);
  out.sc_n = 0;
  out.sc_off = 0;
  if (na != UNSET && nb != UNSET) {
    bool da = ld_node(T, na).flags & F_HASDIV, db = ld_node(T, nb).flags & F_HASDIV;
    if (da || db) {
      const uint32_t cap = 1024, vcap = 1u << 13;
      uint32_t *seen = A.get<uint32_t>(cap);
      uint32_t *visited = A.get<uint32_t>(vcap);
      uint32_t *stack = A.get<uint32_t>(vcap);  // shared by both roots
      if (seen && visited && stack) {
        uint32_t nseen = 0, nvis = 0;
        collect_sc(T, na, seen, nseen, cap, visited, nvis, vcap, stack);
        collect_sc(T, nb, seen, nseen, cap, visited, nvis, vcap, stack);
        unsigned long long off = atomicAdd(C.n_sc, (unsigned long long)nseen);
        if (off + nseen <= C.sc_cap) {
          for (uint32_t q = 0; q < nseen; q++) {
            C.sc_node[off + q] = seen[q];
            C.sc_dis[off + q] = (ld_node(T, seen[q]).flags & F_POSDEF) ? 1 : 0;
          }
          out.sc_off = (uint32_t)off;
          out.sc_n = nseen;
        }
      }
    }
  }
  C.vcs[v] = out;
}

}  // namespace veqd
