// veq_warp.cuh — warp-cooperative canonicalisation of sums (K1 + K2 hot path).
//
// One warp evaluates one fused Add node: the 32 lanes decompose the leaves'
// terms in parallel, group like terms with a bitonic sort on factor-vector
// hashes, rebuild the surviving terms, sort them into canonical order (order
// prefix, full Expr::compare on ties) and intern the result with a
// warp-reduced Merkle hash and a lane-parallel kid compare. Semantics are
// exactly add_nary's (canon_add_kids, proj/src/expr.cpp:415-424); the
// single-thread routines of veq_canon.cuh remain the fallback.
#pragma once
#include "veq_canon.cuh"

namespace veqd {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

template <class X> __device__ __forceinline__ X *warp_get(Arena &A, uint64_t n) {
  unsigned long long p = 0;
  if (lane_id() == 0) p = (unsigned long long)A.alloc(n * sizeof(X));
  p = __shfl_sync(kFull, p, 0);
  return reinterpret_cast<X *>(p);
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t &total) {
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane_id() >= (unsigned)o) x += y;
  }
  total = __shfl_sync(kFull, x, 31);
  return x - v;
}

// Per-warp bump allocation of node ids and kid words (held by lane 0):
// chunks come from the table's global counters, so the hot path issues no
// contended atomic per node. Unused chunk tails are holes, counted in
// counters[4] (ids) and counters[5] (kid words) when the warp exits.
struct WarpAlloc {
  uint64_t id_next, id_end, kid_next, kid_end;
};
constexpr uint64_t WA_IDS = 32, WA_KIDS = 2048;

// Lane 0 only. False when the table is full (E_BUDGET set).
__device__ inline bool wa_alloc(const Table &T, WarpAlloc &W, uint32_t nk, uint64_t &id, uint64_t &off) {
  const uint64_t ids_chunk = T.wa_ids ? T.wa_ids : WA_IDS, kids_chunk = T.wa_kids ? T.wa_kids : WA_KIDS;
  if (W.id_next == W.id_end) {
    unsigned long long b = atomicAdd(&T.counters[0], (unsigned long long)ids_chunk);
    W.id_next = b;
    W.id_end = b + ids_chunk;
  }
  if (W.kid_next + nk > W.kid_end) {
    const uint64_t want = nk > kids_chunk ? nk : kids_chunk;
    if (W.kid_end > W.kid_next) atomicAdd(&T.counters[5], (unsigned long long)(W.kid_end - W.kid_next));
    unsigned long long b = atomicAdd(&T.counters[1], (unsigned long long)want);
    W.kid_next = b;
    W.kid_end = b + want;
  }
  id = W.id_next++;
  off = W.kid_next;
  W.kid_next += nk;
  if (id >= T.max_nodes || off + nk > T.max_kids) {
    set_error(T, E_BUDGET);
    return false;
  }
  return true;
}
__device__ inline void wa_flush(const Table &T, WarpAlloc &W) {
  if (W.id_end > W.id_next) atomicAdd(&T.counters[4], (unsigned long long)(W.id_end - W.id_next));
  if (W.kid_end > W.kid_next) atomicAdd(&T.counters[5], (unsigned long long)(W.kid_end - W.kid_next));
  W.id_next = W.id_end = W.kid_next = W.kid_end = 0;
}
// an id / kid range allocated speculatively and then not published
__device__ inline void wa_waste(const Table &T, uint32_t nk) {
  atomicAdd(&T.counters[4], 1ull);
  atomicAdd(&T.counters[5], (unsigned long long)nk);
}

// Bitonic sort of n (key, val) pairs held in scratch; capacity must be the
// next power of two >= n (padding is filled here). less(ka, va, kb, vb).
template <class Less>
__device__ inline void warp_bitonic(uint64_t *key, uint32_t *val, uint32_t n, Less less) {
  uint32_t P = 1;
  while (P < n) P <<= 1;
  for (uint32_t i = n + lane_id(); i < P; i += 32) {
    key[i] = ~0ull;
    val[i] = UNSET;
  }
  __syncwarp();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane_id(); i < P; i += 32) {
        uint32_t l = i ^ j;
        if (l > i) {
          uint64_t ki = key[i], kl = key[l];
          uint32_t vi = val[i], vl = val[l];
          bool up = (i & k) == 0;
          bool sw = up ? less(kl, vl, ki, vi) : less(ki, vi, kl, vl);
          if (sw) {
            key[i] = kl;
            key[l] = ki;
            val[i] = vl;
            val[l] = vi;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Insert-or-find of a composite whose kids sit in scratch (all lanes call).
__device__ inline uint32_t warp_intern(const Table &T, uint8_t kind, const uint32_t *kids, uint32_t nk,
                                       WarpAlloc *W = nullptr) {
  const uint32_t lane = lane_id();
  uint64_t sum = 0, p1 = 0;
  bool any_pd = false, all_pd = true, any_div = false, k0c = false, any_cf = false;
#pragma unroll 4
  for (uint32_t i = lane; i < nk; i += 32) {
    Node kn = ld_node(T, kids[i]);
    sum += kid_term_k(kind, i, kn.hash);
    bool pd = kn.flags & F_POSDEF;
    any_pd |= pd;
    all_pd &= pd;
    any_div |= (kn.flags & F_HASDIV) != 0;
    any_cf |= (kn.flags & F_COEF) != 0;
    if (i == 0) {
      p1 = composite_prefix(kind, nk, prefix_of(kn));
      k0c = kn.kind == K_CONST;
    }
  }
  sum = warp_sum_u64(sum);
  p1 = __shfl_sync(kFull, p1, 0);
  k0c = __shfl_sync(kFull, k0c, 0);
  any_pd = __any_sync(kFull, any_pd);
  all_pd = __all_sync(kFull, all_pd);
  any_div = __any_sync(kFull, any_div);
  any_cf = __any_sync(kFull, any_cf);
  const uint64_t h = composite_hash(kind, nk, sum);
  const uint8_t flags = composite_flags(kind, any_pd, all_pd, any_div, k0c, any_cf);
  uint64_t slot = h & T.slot_mask;
  uint32_t mine = EMPTY;
  for (uint64_t probes = 0;; probes++) {
    if (probes > T.slot_mask) {
      if (lane == 0) set_error(T, E_BUDGET);
      return T.id_zero;
    }
    uint32_t cur = 0;
    if (lane == 0) cur = *((volatile uint32_t *)(T.slots + slot));
    cur = __shfl_sync(kFull, cur, 0);
    if (cur == EMPTY) {
      if (mine == EMPTY) {
        unsigned long long id = 0, off = 0;
        bool ok = true;
        if (lane == 0) {
          if (W) {
            ok = wa_alloc(T, *W, nk, (uint64_t &)id, (uint64_t &)off);
          } else {
            id = atomicAdd(&T.counters[0], 1ull);
            off = atomicAdd(&T.counters[1], (unsigned long long)nk);
          }
        }
        id = __shfl_sync(kFull, id, 0);
        off = __shfl_sync(kFull, off, 0);
        if (!__shfl_sync(kFull, ok, 0) || id >= T.max_nodes || off + nk > T.max_kids) {
          if (lane == 0) set_error(T, E_BUDGET);
          return T.id_zero;
        }
        for (uint32_t i = lane; i < nk; i += 32) T.kids[off + i] = kids[i];
        if (lane == 0) {
          Node n;
          n.kind = kind;
          n.flags = flags;
          n.pad = 0;
          n.nkids = nk;
          n.hash = h;
          n.p0 = off;
          n.p1 = p1;
          T.nodes[id] = n;
        }
        __syncwarp();
        fence_acq_rel();
        mine = (uint32_t)id;
      }
      uint32_t prev = 0;
      if (lane == 0) prev = atomicCAS(T.slots + slot, EMPTY, mine);
      prev = __shfl_sync(kFull, prev, 0);
      if (prev == EMPTY) return mine;
      cur = prev;
    }
    uint64_t ch = 0;
    if (lane == 0) ch = ld_hash(T, cur);
    ch = __shfl_sync(kFull, ch, 0);
    if (ch == h) {
      Node c = ld_node(T, cur);
      if (c.kind == kind && c.nkids == nk) {
        bool same = true;
        for (uint32_t i = lane; i < nk && same; i += 32) same = (ld_kid(T, c.p0 + i) == kids[i]);
        if (__all_sync(kFull, same)) return cur;
      }
    }
    slot = (slot + 1) & T.slot_mask;
  }
}

__device__ __forceinline__ bool canon_less(const Table &T, uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
  if (ka != kb) return ka < kb;
  if (va == vb || va == UNSET || vb == UNSET) return false;
  return cmp_nodes(T, va, vb) < 0;
}

// Sorts ids (scratch, n entries) into canonical order in place.
__device__ inline void warp_sort_canonical(const Table &T, Arena &A, uint32_t *ids, uint32_t n) {
  if (n < 2) return;
  uint32_t P = 1;
  while (P < n) P <<= 1;
  uint64_t *key = warp_get<uint64_t>(A, P);
  uint32_t *val = warp_get<uint32_t>(A, P);
  if (!key || !val) return;
  for (uint32_t i = lane_id(); i < n; i += 32) {
    key[i] = prefix_id(T, ids[i]);
    val[i] = ids[i];
  }
  warp_bitonic(key, val, n, [&](uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    return canon_less(T, ka, va, kb, vb);
  });
  for (uint32_t i = lane_id(); i < n; i += 32) ids[i] = val[i];
  __syncwarp();
}

// ---- register-only fast path: at most 32 terms, no like terms -------------
// One term per lane; both sorts are shuffle bitonic networks and the result
// is interned straight from registers (no scratch round trips).
template <class Less>
__device__ __forceinline__ void reg_bitonic(uint64_t &key, uint32_t &val, Less less) {
  const uint32_t lane = lane_id();
  for (uint32_t k = 2; k <= 32; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      uint64_t pk = __shfl_xor_sync(kFull, key, j);
      uint32_t pv = __shfl_xor_sync(kFull, val, j);
      bool up = (lane & k) == 0, lower = (lane & j) == 0;
      bool take = (up == lower) ? less(pk, pv, key, val) : less(key, val, pk, pv);
      if (take) {
        key = pk;
        val = pv;
      }
    }
  }
}

__device__ inline uint32_t warp_intern_regs_h(const Table &T, uint8_t kind, uint32_t kid, uint32_t m, uint64_t term,
                                              bool pd, bool dv, uint64_t p1, bool k0c, WarpAlloc *W = nullptr,
                                              bool *created = nullptr, bool cf = false);

// Interns a composite whose kid i is held by lane i (m <= 32 kids).
__device__ inline uint32_t warp_intern_regs(const Table &T, uint8_t kind, uint32_t kid, uint32_t m) {
  const uint32_t lane = lane_id();
  uint64_t term = 0, p1 = 0;
  bool pd = true, dv = false, k0c = false, cf = false;
  if (lane < m) {
    Node kn = ld_node(T, kid);
    term = kid_term_k(kind, lane, kn.hash);
    pd = kn.flags & F_POSDEF;
    dv = (kn.flags & F_HASDIV) != 0;
    cf = (kn.flags & F_COEF) != 0;
    if (lane == 0) {
      p1 = composite_prefix(kind, m, prefix_of(kn));
      k0c = kn.kind == K_CONST;
    }
  }
  return warp_intern_regs_h(T, kind, kid, m, term, pd, dv, __shfl_sync(kFull, p1, 0), __shfl_sync(kFull, k0c, 0),
                            nullptr, nullptr, cf);
}

// Same, with each lane's kid term hash (kid_term_k(kind, lane, hash)) and flags
// already known; p1 = composite prefix, k0c = kid 0 is a Const.
__device__ inline uint32_t warp_intern_regs_h(const Table &T, uint8_t kind, uint32_t kid, uint32_t m, uint64_t term,
                                              bool pd, bool dv, uint64_t p1, bool k0c, WarpAlloc *W,
                                              bool *created, bool cf) {
  const uint32_t lane = lane_id();
  if (lane >= m) {
    term = 0;
    pd = true;
    dv = false;
  }
  const uint64_t sum = warp_sum_u64(term);
  const bool any_pd = __any_sync(kFull, lane < m && pd), all_pd = __all_sync(kFull, pd);
  const bool any_div = __any_sync(kFull, dv);
  const bool any_cf = __any_sync(kFull, lane < m && cf);
  const uint64_t h = composite_hash(kind, m, sum);
  const uint8_t flags = composite_flags(kind, any_pd, all_pd, any_div, k0c, any_cf);
  uint64_t slot = h & T.slot_mask;
  uint32_t mine = EMPTY;
  if (W) {
    // speculative insert: write the node first, then claim the home slot
    // directly (one round trip fewer for the common new-node case)
    unsigned long long id = 0, off = 0;
    bool ok = true;
    if (lane == 0) ok = wa_alloc(T, *W, m, (uint64_t &)id, (uint64_t &)off);
    if (!__shfl_sync(kFull, ok, 0)) return T.id_zero;
    id = __shfl_sync(kFull, id, 0);
    off = __shfl_sync(kFull, off, 0);
    if (lane < m) T.kids[off + lane] = kid;
    if (lane == 0) {
      Node n;
      n.kind = kind;
      n.flags = flags;
      n.pad = 0;
      n.nkids = m;
      n.hash = h;
      n.p0 = off;
      n.p1 = p1;
      T.nodes[id] = n;
    }
    __syncwarp();
    fence_acq_rel();
    mine = (uint32_t)id;
  }
  for (uint64_t probes = 0;; probes++) {
    if (probes > T.slot_mask) {
      if (lane == 0) set_error(T, E_BUDGET);
      return T.id_zero;
    }
    uint32_t cur = EMPTY;
    if (mine == EMPTY) {
      if (lane == 0) cur = *((volatile uint32_t *)(T.slots + slot));
      cur = __shfl_sync(kFull, cur, 0);
    }
    if (cur == EMPTY) {
      if (mine == EMPTY) {
        unsigned long long id = 0, off = 0;
        if (lane == 0) {
          id = atomicAdd(&T.counters[0], 1ull);
          off = atomicAdd(&T.counters[1], (unsigned long long)m);
        }
        id = __shfl_sync(kFull, id, 0);
        off = __shfl_sync(kFull, off, 0);
        if (id >= T.max_nodes || off + m > T.max_kids) {
          if (lane == 0) set_error(T, E_BUDGET);
          return T.id_zero;
        }
        if (lane < m) T.kids[off + lane] = kid;
        if (lane == 0) {
          Node n;
          n.kind = kind;
          n.flags = flags;
          n.pad = 0;
          n.nkids = m;
          n.hash = h;
          n.p0 = off;
          n.p1 = p1;
          T.nodes[id] = n;
        }
        __syncwarp();
        fence_acq_rel();
        mine = (uint32_t)id;
      }
      uint32_t prev = 0;
      if (lane == 0) prev = atomicCAS(T.slots + slot, EMPTY, mine);
      prev = __shfl_sync(kFull, prev, 0);
      if (prev == EMPTY) {
        if (created) *created = true;
        return mine;
      }
      cur = prev;
    }
    Node c = ld_node(T, cur);
    bool same = c.hash == h && c.kind == kind && c.nkids == m;
    if (__all_sync(kFull, same)) {
      bool eq = lane >= m || ld_kid(T, c.p0 + lane) == kid;
      if (__all_sync(kFull, eq)) {
        if (W && lane == 0) wa_waste(T, m);
        return cur;
      }
    }
    slot = (slot + 1) & T.slot_mask;
  }
}

// Returns the canonical sum, or UNSET when the fast path does not apply
// (more than 32 terms, or like terms that must be merged).
__device__ inline uint32_t warp_add_small(const Table &T, const uint32_t *leaves, uint32_t n) {
  const uint32_t lane = lane_id();
  if (n > 32) return UNSET;
  uint32_t leaf = UNSET, c = 0, kind = 0;
  uint64_t p0 = 0;
  if (lane < n) {
    leaf = leaves[lane];
    Node ln = ld_node(T, leaf);
    kind = ln.kind;
    p0 = ln.p0;
    c = ln.kind == K_ADD ? ln.nkids : 1;
  }
  uint32_t m;
  const uint32_t ex = warp_excl_scan(c, m);
  if (m > 32) return UNSET;
  // the leaf holding term `lane`
  uint32_t src_leaf = 0;
  for (uint32_t l = 0; l < n; l++) {
    uint32_t el = __shfl_sync(kFull, ex, l), cl = __shfl_sync(kFull, c, l);
    if (cl && el <= lane) src_leaf = l;
  }
  const uint32_t lk = __shfl_sync(kFull, kind, src_leaf);
  const uint64_t lp = __shfl_sync(kFull, p0, src_leaf);
  const uint32_t lid = __shfl_sync(kFull, leaf, src_leaf);
  const uint32_t lex = __shfl_sync(kFull, ex, src_leaf);
  uint32_t term_node = UNSET;
  uint64_t key = ~0ull;
  bool real = false;  // a literal 0 term has coefficient 0 and is dropped
  if (lane < m) {
    term_node = lk == K_ADD ? ld_kid(T, lp + (lane - lex)) : lid;
    real = term_node != T.id_zero;
    if (real) key = decompose_one(T, term_node).fh;
  }
  const uint32_t m_all = m;
  m = __popc(__ballot_sync(kFull, real));
  (void)m_all;
  uint32_t val = lane;
  reg_bitonic(key, val, [](uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    return ka != kb ? ka < kb : va < vb;
  });
  const uint64_t prev = __shfl_up_sync(kFull, key, 1);
  if (__any_sync(kFull, lane > 0 && lane < m && key == prev)) return UNSET;  // like terms
  if (m == 0) return T.id_zero;
  if (m == 1) return __shfl_sync(kFull, term_node, __shfl_sync(kFull, val, 0) & 31);
  // no merges: the result's kids are the term nodes themselves
  uint32_t id = __shfl_sync(kFull, term_node, val & 31);
  uint64_t pk = lane < m ? prefix_id(T, id) : ~0ull;
  if (lane >= m) id = UNSET;
  reg_bitonic(pk, id, [&](uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) { return canon_less(T, ka, va, kb, vb); });
  return warp_intern_regs(T, K_ADD, id, m);
}

// Register-leaf variant of warp_add_small: lane i holds leaf i (n <= 32).
__device__ inline uint32_t warp_add_small_reg(const Table &T, uint32_t leaf_reg, uint32_t n) {
  const uint32_t lane = lane_id();
  uint32_t leaf = UNSET, c = 0, kind = 0;
  uint64_t p0 = 0;
  if (lane < n) {
    leaf = leaf_reg;
    Node ln = ld_node(T, leaf);
    kind = ln.kind;
    p0 = ln.p0;
    c = ln.kind == K_ADD ? ln.nkids : 1;
  }
  uint32_t m;
  const uint32_t ex = warp_excl_scan(c, m);
  if (m > 32) return UNSET;
  uint32_t src_leaf = 0;
  for (uint32_t l = 0; l < n; l++) {
    uint32_t el = __shfl_sync(kFull, ex, l), cl = __shfl_sync(kFull, c, l);
    if (cl && el <= lane) src_leaf = l;
  }
  const uint32_t lk = __shfl_sync(kFull, kind, src_leaf);
  const uint64_t lp = __shfl_sync(kFull, p0, src_leaf);
  const uint32_t lid = __shfl_sync(kFull, leaf, src_leaf);
  const uint32_t lex = __shfl_sync(kFull, ex, src_leaf);
  uint32_t term_node = UNSET;
  uint64_t key = ~0ull;
  bool real = false;
  if (lane < m) {
    term_node = lk == K_ADD ? ld_kid(T, lp + (lane - lex)) : lid;
    real = term_node != T.id_zero;
    if (real) key = decompose_one(T, term_node).fh;
  }
  m = __popc(__ballot_sync(kFull, real));
  uint32_t val = lane;
  reg_bitonic(key, val, [](uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    return ka != kb ? ka < kb : va < vb;
  });
  const uint64_t prev = __shfl_up_sync(kFull, key, 1);
  if (__any_sync(kFull, lane > 0 && lane < m && key == prev)) return UNSET;
  if (m == 0) return T.id_zero;
  if (m == 1) return __shfl_sync(kFull, term_node, __shfl_sync(kFull, val, 0) & 31);
  uint32_t id = __shfl_sync(kFull, term_node, val & 31);
  uint64_t pk = lane < m ? prefix_id(T, id) : ~0ull;
  if (lane >= m) id = UNSET;
  reg_bitonic(pk, id, [&](uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) { return canon_less(T, ka, va, kb, vb); });
  return warp_intern_regs(T, K_ADD, id, m);
}


// Register bitonic over a 64-bit key with a 32-bit payload, plain unsigned
// key order (ties keep an arbitrary order; callers detect them).
__device__ __forceinline__ void reg_bitonic_u64(uint64_t &key, uint32_t &val) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint64_t pk = __shfl_xor_sync(kFull, key, j);
      const uint32_t pv = __shfl_xor_sync(kFull, val, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      const bool take = (up == lower) ? (pk < key) : (key < pk);
      key = take ? pk : key;
      val = take ? pv : val;
    }
  }
}

// Register bitonic over (key, id) carrying one extra payload lane index.
template <class Less>
__device__ __forceinline__ void reg_bitonic3(uint64_t &key, uint32_t &val, uint32_t &aux, Less less) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      uint64_t pk = __shfl_xor_sync(kFull, key, j);
      uint32_t pv = __shfl_xor_sync(kFull, val, j);
      uint32_t pa = __shfl_xor_sync(kFull, aux, j);
      bool up = (lane & k) == 0, lower = (lane & j) == 0;
      bool take = (up == lower) ? less(pk, pv, key, val) : less(key, val, pk, pv);
      if (take) {
        key = pk;
        val = pv;
        aux = pa;
      }
    }
  }
}

// Lean register path for a sum of at most 32 terms (canon_add_kids,
// expr.cpp:415-424), lane k < n holding leaf k. Each term node is loaded
// once; its hash, flags and order prefix travel with it through the sort.
// Returns UNSET when the path does not apply: more than 32 terms (`m_out`
// then holds the term count), a term with a coefficient (F_COEF: like terms
// need factor-vector grouping), or like terms (equal ids after the sort).
__device__ inline uint32_t warp_add_lean(const Table &T, uint32_t leaf, uint32_t n, uint32_t &m_out, WarpAlloc *W,
                                       bool *created, unsigned long long *ph = nullptr) {
  const uint32_t lane = lane_id();
  long long c0 = ph ? clock64() : 0;
  uint32_t c = 0, kind = 0;
  uint64_t p0 = 0;
  if (lane < n) {
    const Node ln = ld_node(T, leaf);
    kind = ln.kind;
    p0 = ln.p0;
    c = ln.kind == K_ADD ? ln.nkids : 1;
  }
  uint32_t m;
  const uint32_t ex = warp_excl_scan(c, m);
  m_out = m;
  if (m > 32) return UNSET;
  // owning leaf of term `lane`: leaves with c >= 1 start at ex
  const uint32_t starts = __reduce_or_sync(kFull, (lane < n && c) ? (1u << ex) : 0u);
  const uint32_t src = __popc(starts & (lane == 31 ? ~0u : ((2u << lane) - 1))) - 1;
  const uint32_t lk = __shfl_sync(kFull, kind, src & 31);
  const uint64_t lp = __shfl_sync(kFull, p0, src & 31);
  const uint32_t lid = __shfl_sync(kFull, leaf, src & 31);
  const uint32_t lex = __shfl_sync(kFull, ex, src & 31);
  uint32_t id = UNSET;
  uint64_t key = ~0ull, hsh = 0;
  uint8_t fl = 0, tk = 0;
  Rat cv{0, 1};
  if (lane < m) {
    id = lk == K_ADD ? ld_kid(T, lp + (lane - lex)) : lid;
    Node tn = ld_node(T, id);
    key = prefix_of(tn);
    hsh = tn.hash;
    fl = tn.flags;
    tk = tn.kind;
    if (tk == K_CONST) cv = const_val(tn);
  }
  if (__any_sync(kFull, lane < m && tk == K_MUL && (fl & F_COEF))) return UNSET;
  long long c1 = ph ? clock64() : 0;
  // fold the Const terms into one (dropped when zero)
  const uint32_t cmask = __ballot_sync(kFull, lane < m && tk == K_CONST);
  if (cmask) {
    const uint32_t keep = __ffs(cmask) - 1;
    const bool keep_zero = __shfl_sync(kFull, (uint32_t)(cv.n == 0), keep);
    if (__popc(cmask) > 1 || keep_zero) {
      // exact sum over the Const lanes (lane order; rational addition is exact)
      Rat acc{0, 1};
      for (uint32_t mm = cmask; mm; mm &= mm - 1) {
        const uint32_t q = __ffs(mm) - 1;
        Rat v{(long long)__shfl_sync(kFull, (unsigned long long)cv.n, q),
              (long long)__shfl_sync(kFull, (unsigned long long)cv.d, q)};
        acc = rat_add(T, acc, v);
      }
      uint32_t cid = UNSET;
      if (lane == 0) cid = rat_is(acc, 0) ? UNSET : intern_const(T, acc);
      cid = __shfl_sync(kFull, cid, 0);
      if (lane < m && tk == K_CONST) {
        if (lane == keep && cid != UNSET) {
          id = cid;
          Node cn = ld_node(T, cid);
          hsh = cn.hash;
          fl = cn.flags;
          key = 0;
        } else {
          id = UNSET;
          key = ~0ull;
        }
      }
    }
  }
  // canonical order: bitonic on the 64-bit order prefix with the source
  // lane as payload (branch-free); equal prefixes need Expr::compare, so a
  // tie re-sorts with the full comparator
  const uint32_t real = __popc(__ballot_sync(kFull, id != UNSET));  // real terms sort first
  uint32_t aux = lane;
  reg_bitonic_u64(key, aux);
  {
    const uint64_t pk = __shfl_up_sync(kFull, key, 1);
    if (__any_sync(kFull, lane > 0 && lane < real && key == pk)) {
      id = __shfl_sync(kFull, id, aux & 31);
      uint32_t a2 = aux;
      reg_bitonic3(key, id, a2, [&](uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
        return canon_less(T, ka, va, kb, vb);
      });
      aux = a2;
    } else {
      id = __shfl_sync(kFull, id, aux & 31);
    }
  }
  // like terms (coefficient-free): equal ids, adjacent after the sort
  const uint32_t prev = __shfl_up_sync(kFull, id, 1);
  if (__any_sync(kFull, lane > 0 && lane < real && id == prev)) return UNSET;
  if (real == 0) return T.id_zero;
  if (real == 1) return __shfl_sync(kFull, id, 0);
  const uint64_t kh = __shfl_sync(kFull, hsh, aux & 31);
  const uint8_t kf = (uint8_t)__shfl_sync(kFull, (uint32_t)fl, aux & 31);
  const uint64_t k0p = __shfl_sync(kFull, key, 0);
  const bool k0c = __shfl_sync(kFull, (uint32_t)(key == 0), 0);
  long long c2 = ph ? clock64() : 0;
  const uint32_t res = warp_intern_regs_h(T, K_ADD, id, real, kid_term_k(K_ADD, lane, kh), kf & F_POSDEF, (kf & F_HASDIV) != 0,
                                          composite_prefix(K_ADD, real, k0p), k0c, W, created);
  if (ph && lane == 0) {
    long long c3 = clock64();
    ph[0] += c1 - c0;
    ph[1] += c2 - c1;
    ph[2] += c3 - c2;
  }
  return res;
}

// ---- shared-memory path for large sums -------------------------------------
// A block-wide pool of 4 KB shared-memory pages; a warp evaluating a sum with
// more than 32 terms takes a contiguous page run for its working set and
// returns it when the item completes (it never waits on other items while
// holding pages, so the pool cannot deadlock; if no run is free the item
// uses the global-scratch path instead).
constexpr uint32_t SPAGE = 4096;
struct SmemPool {
  unsigned long long *mask;  // bit i: page i taken (up to 64 pages)
  char *base;
  uint32_t npages;
};

__device__ inline int pool_acquire(const SmemPool &P, uint32_t k) {
  int got = -1;
  if (lane_id() == 0 && k <= P.npages) {
    const unsigned long long all = P.npages >= 64 ? ~0ull : ((1ull << P.npages) - 1);
    for (int tries = 0; tries < 4096 && got < 0; tries++) {
      const unsigned long long m = *(volatile unsigned long long *)P.mask;
      const unsigned long long fr = ~m & all;
      unsigned long long x = fr;
      for (uint32_t j = 1; j < k; j++) x &= fr >> j;
      if (!x) {
        __nanosleep(256);
        continue;
      }
      const int i = __ffsll((long long)x) - 1;
      const unsigned long long bits = (k >= 64 ? ~0ull : ((1ull << k) - 1)) << i;
      if (atomicCAS(P.mask, m, m | bits) == m) got = i;
    }
  }
  return __shfl_sync(kFull, got, 0);
}
__device__ inline void pool_release(const SmemPool &P, int first, uint32_t k) {
  __syncwarp();
  if (lane_id() == 0) atomicAnd(P.mask, ~((k >= 64 ? ~0ull : ((1ull << k) - 1)) << first));
}

// Working-set bytes of warp_add_smem for n leaves and m terms.
__device__ __forceinline__ uint32_t hash_slots(uint32_t m) {
  uint32_t H = 64;
  while (H < m + m / 2 + 1) H <<= 1;
  return H;
}
__device__ __forceinline__ uint32_t pz(uint32_t x) { return x + (x >> 5); }
__device__ __forceinline__ uint32_t smem_pad_len(uint32_t m) { return m + (m >> 5) + 1; }
__device__ __forceinline__ uint64_t add_smem_bytes(uint32_t n, uint32_t m, bool coef) {
  const uint64_t mp = smem_pad_len(m);
  uint64_t a = ((uint64_t)(2 * n + 1 + mp) * 4 + 7) & ~7ull;
  uint64_t y = coef ? 8ull * m + (uint64_t)hash_slots(m) * 4 : 0;  // coefficient grouping
  if (y < 12ull * mp) y = 12ull * mp;                               // merge ping-pong
  return a + 8ull * mp + y;
}

__device__ __forceinline__ bool pref_less(const Table &T, uint64_t pa, uint32_t a, uint64_t pb, uint32_t b) {
  if (pa != pb) return pa < pb;
  return cmp_nodes(T, a, b) < 0;
}

// canon_add_kids (expr.cpp:415-424) over n canonical leaves already stored in
// lv[] (shared memory, inside `buf`), m terms in total. Fast path: every
// non-constant term has a distinct factor vector (checked exactly via a
// shared-memory hash table on factor-vector hashes; any hash hit, true or
// false, defers to the exact global-scratch path by returning UNSET). Then
// the result's kids are the terms themselves plus at most one folded Const,
// and canonical order (Expr::compare) is produced by merging the leaves'
// already-sorted kid runs with warp-parallel merge-path passes.
__device__ inline uint32_t warp_add_smem(const Table &T, char *buf, uint32_t n, uint32_t m, WarpAlloc *W,
                                       unsigned long long *ph = nullptr, bool coef_room = true) {
  const uint32_t lane = lane_id();
  const long long c0 = ph ? clock64() : 0;
  long long c1 = 0, c2 = 0, c3 = 0;
  uint32_t *lv = reinterpret_cast<uint32_t *>(buf);
  uint32_t *rs = lv + n;  // run starts = leaf term offsets, n + 1 entries
  // term arrays are padded one slot per 32 (index pz(x)): lanes working on
  // neighbouring 32-element chunks then fall in different banks
  const uint32_t mp = smem_pad_len(m);
  uint32_t *idA = rs + n + 1;
  uint64_t *preA = reinterpret_cast<uint64_t *>(buf + (((uint64_t)(2 * n + 1 + mp) * 4 + 7) & ~7ull));
  char *Y = reinterpret_cast<char *>(preA + mp);
  const uint32_t H = hash_slots(m);
  uint64_t *preB = reinterpret_cast<uint64_t *>(Y);
  uint32_t *idB = reinterpret_cast<uint32_t *>(preB + mp);
  // 1. term offsets per leaf
  // (an Add leaf's slot in lv is replaced by its kid-arena offset: the
  // gather below then reads kid words without reloading the node)
  uint32_t run = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    uint32_t i = base + lane;
    uint32_t c = 0;
    if (i < n) {
      const Node ln = ld_node(T, lv[i]);
      c = ln.kind == K_ADD ? ln.nkids : 1;
      if (ln.kind == K_ADD) lv[i] = (uint32_t)ln.p0;
    }
    uint32_t tot;
    uint32_t ex = warp_excl_scan(c, tot);
    if (i < n) rs[i] = run + ex;
    run += tot;
  }
  if (lane == 0) rs[n] = run;
  __syncwarp();
  if (ph) c1 = clock64();
  // 2. gather terms and their order prefixes; note coefficient terms.
  // Two passes so each lane keeps several independent loads in flight:
  // term ids (kid words of Add leaves), then the term nodes.
  bool coef = false;
  uint32_t nconst = 0;
#pragma unroll 4
  for (uint32_t t = lane; t < m; t += 32) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) / 2;
      if (rs[mid] <= t) lo = mid;
      else hi = mid;
    }
    // a leaf with several terms is an Add (lv holds its kid offset); a
    // canonical Add has at least two kids, so a one-term leaf is the term
    const uint32_t nl = rs[lo + 1] - rs[lo];
    idA[pz(t)] = nl > 1 ? ld_kid(T, (uint64_t)lv[lo] + (t - rs[lo])) : lv[lo];
  }
  __syncwarp();
#pragma unroll 4
  for (uint32_t t = lane; t < m; t += 32) {
    const Node tn = ld_node(T, idA[pz(t)]);
    preA[pz(t)] = prefix_of(tn);
    nconst += tn.kind == K_CONST;
    coef |= tn.kind == K_MUL && (tn.flags & F_COEF);
  }
  nconst = __reduce_add_sync(kFull, nconst);
  coef = __any_sync(kFull, coef);
  __syncwarp();
  if (coef && !coef_room) return UNSET;  // sized without the grouping region
  if (coef) {
    // like terms may differ in id: exact grouping key = factor-vector hash
    // in a shared-memory table; any hit (true or a hash collision) defers to
    // the exact global-scratch path
    bool dup = false;
    uint64_t *fh = preB;  // Y is free until the sort
    uint32_t *hs2 = reinterpret_cast<uint32_t *>(Y + 8ull * m);
    for (uint32_t i = lane; i < H; i += 32) hs2[i] = EMPTY;
    __syncwarp();
    for (uint32_t t = lane; t < m; t += 32) {
      Term tm = decompose_one(T, idA[pz(t)]);
      if (tm.nf == 0) continue;
      const uint64_t h = tm.fh;
      fh[t] = h;
      __threadfence_block();  // publish the hash before the slot that names it
      uint32_t sl = (uint32_t)(h ^ (h >> 32)) & (H - 1);
      for (;;) {
        uint32_t prev = atomicCAS(hs2 + sl, EMPTY, t);
        if (prev == EMPTY) break;
        __threadfence_block();
        if (fh[prev] == h) {
          dup = true;
          break;
        }
        sl = (sl + 1) & (H - 1);
      }
    }
    __syncwarp();
    if (__any_sync(kFull, dup)) return UNSET;
  }
  if (ph) c2 = clock64();
  // 3b. the sum may already exist (the other kernel of the pair usually
  // built it): its hash depends only on the term multiset, so look it up
  // before sorting. A candidate matches when our terms are distinct and
  // every one of its m kids is among them.
  if (!coef && nconst == 0 && m >= 2) {
    uint64_t sum = 0;
    for (uint32_t t = lane; t < m; t += 32) sum += kid_term(0, ld_hash(T, idA[pz(t)]));
    const uint64_t h = composite_hash(K_ADD, m, warp_sum_u64(sum));
    uint32_t *set = reinterpret_cast<uint32_t *>(Y);
    for (uint32_t i = lane; i < H; i += 32) set[i] = EMPTY;
    __syncwarp();
    bool dup = false;
    for (uint32_t t = lane; t < m; t += 32) {
      const uint32_t id = idA[pz(t)];
      for (uint32_t sl = (uint32_t)mix64(id) & (H - 1);; sl = (sl + 1) & (H - 1)) {
        const uint32_t prev = atomicCAS(set + sl, EMPTY, id);
        if (prev == EMPTY) break;
        if (prev == id) {
          dup = true;
          break;
        }
      }
    }
    __syncwarp();
    if (!__any_sync(kFull, dup)) {
      uint64_t slot = h & T.slot_mask;
      for (uint64_t probes = 0; probes <= T.slot_mask; probes++) {
        uint32_t cur = EMPTY;
        uint64_t ch = 0;
        if (lane == 0) {
          cur = *((volatile uint32_t *)(T.slots + slot));
          if (cur != EMPTY) ch = ld_hash(T, cur);
        }
        cur = __shfl_sync(kFull, cur, 0);
        if (cur == EMPTY) break;
        if (__shfl_sync(kFull, ch, 0) == h) {
          const Node c = ld_node(T, cur);
          if (c.kind == K_ADD && c.nkids == m) {
            bool all_in = true;
            for (uint32_t k = lane; k < m && all_in; k += 32) {
              const uint32_t kid = ld_kid(T, c.p0 + k);
              bool in = false;
              for (uint32_t sl = (uint32_t)mix64(kid) & (H - 1);; sl = (sl + 1) & (H - 1)) {
                const uint32_t v = set[sl];
                if (v == kid) {
                  in = true;
                  break;
                }
                if (v == EMPTY) break;
              }
              all_in = in;
            }
            if (__all_sync(kFull, all_in)) return cur;
          }
        }
        slot = (slot + 1) & T.slot_mask;
      }
    }
    __syncwarp();
  }
  // 4. merge the sorted leaf runs pairwise until one run remains
  uint32_t R = n;
  uint64_t *ps = preA, *pd = preB;
  uint32_t *is = idA, *id_ = idB;
  const uint32_t E = (m + 31) / 32;
  while (R > 1) {
    const uint32_t npairs = (R + 1) / 2;
    uint32_t pos = min(lane * E, m), end = min(pos + E, m);
    while (pos < end) {
      // pair p holding output position pos: largest p with rs[2p] <= pos
      uint32_t lo = 0, hi = npairs;
      while (hi - lo > 1) {
        uint32_t mid = (lo + hi) / 2;
        if (rs[2 * mid] <= pos) lo = mid;
        else hi = mid;
      }
      const uint32_t a0 = rs[2 * lo], a1 = rs[min(2 * lo + 1, R)], b1 = rs[min(2 * lo + 2, R)];
      const uint32_t d = pos - a0, la = a1 - a0, lb = b1 - a1;
      // co-rank: i = number of A elements among the first d outputs
      uint32_t ilo = d > lb ? d - lb : 0, ihi = min(d, la);
      while (ilo < ihi) {
        uint32_t mid = (ilo + ihi) / 2;
        uint32_t bj = a1 + (d - mid - 1);
        if (pref_less(T, ps[pz(a0 + mid)], is[pz(a0 + mid)], ps[pz(bj)], is[pz(bj)])) ilo = mid + 1;
        else ihi = mid;
      }
      uint32_t i = a0 + ilo, j = a1 + (d - ilo);
      const uint32_t stop = min(end, b1);
      for (; pos < stop; pos++) {
        const uint32_t pi = pz(i), pj = pz(j);
        bool takeA;
        if (i >= a1) takeA = false;
        else if (j >= b1) takeA = true;
        else takeA = pref_less(T, ps[pi], is[pi], ps[pj], is[pj]);
        const uint32_t src = takeA ? pi : pj;
        pd[pz(pos)] = ps[src];
        id_[pz(pos)] = is[src];
        if (takeA) i++;
        else j++;
      }
    }
    __syncwarp();
    // run starts of the merged runs: rs'[p] = rs[2p]
    for (uint32_t base = 0; base <= npairs; base += 32) {
      uint32_t p = base + lane;
      uint32_t v = p <= npairs ? rs[min(2 * p, R)] : 0;
      __syncwarp();
      if (p <= npairs) rs[p] = v;
      __syncwarp();
    }
    R = npairs;
    uint64_t *tp = ps;
    ps = pd;
    pd = tp;
    uint32_t *ti = is;
    is = id_;
    id_ = ti;
  }
  if (ph) c3 = clock64();
  // like terms without coefficients are equal interned ids: adjacent now
  {
    bool dup = false;
    for (uint32_t t = lane + 1; t < m; t += 32) dup |= is[pz(t)] == is[pz(t - 1)];
    if (__any_sync(kFull, dup)) return UNSET;
  }
  // 5. fold the leading Const terms into one (dropped when zero)
  uint32_t first = 0;
  if (nconst) {
    uint32_t cid = 0;
    if (lane == 0) {
      Rat c{0, 1};
      for (uint32_t k = 0; k < nconst; k++) c = rat_add(T, c, const_val(ld_node(T, is[pz(k)])));
      cid = rat_is(c, 0) ? UNSET : intern_const(T, c);
      if (cid != UNSET) is[pz(nconst - 1)] = cid;
    }
    cid = __shfl_sync(kFull, cid, 0);
    first = cid == UNSET ? nconst : nconst - 1;
    __syncwarp();
  }
  const uint32_t nout = m - first;
  if (nout == 0) return T.id_zero;
  if (nout == 1) return is[pz(first)];
  // the kids, contiguous (unpadded) in the other id buffer
  for (uint32_t t = lane; t < nout; t += 32) id_[t] = is[pz(first + t)];
  __syncwarp();
  const uint32_t res = warp_intern(T, K_ADD, id_, nout, W);
  if (ph && lane == 0) {
    const long long c4 = clock64();
    ph[0] += c1 - c0;
    ph[1] += c2 - c1;
    ph[2] += c3 - c2;
    ph[3] += c4 - c3;
  }
  return res;
}

// canon_add_kids over n canonical leaves (scratch), warp-cooperative.
__device__ inline uint32_t warp_add_nary(const Table &T, Arena &A, const uint32_t *leaves, uint32_t n) {
  const uint32_t lane = lane_id();
  // 1. term offsets per leaf
  uint32_t *off = warp_get<uint32_t>(A, n + 1);
  if (!off) return T.id_zero;
  uint32_t run = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    uint32_t i = base + lane;
    uint32_t c = i < n ? n_terms_of(T, leaves[i]) : 0;
    uint32_t tot;
    uint32_t ex = warp_excl_scan(c, tot);
    if (i < n) off[i] = run + ex;
    run += tot;
  }
  if (lane == 0) off[n] = run;
  __syncwarp();
  const uint32_t m = run;
  if (m == 0) return T.id_zero;
  // 2. decompose terms in parallel
  Term *ts = warp_get<Term>(A, m);
  uint32_t P = 1;
  while (P < m) P <<= 1;
  uint64_t *key = warp_get<uint64_t>(A, P);
  uint32_t *val = warp_get<uint32_t>(A, P);
  if (!ts || !key || !val) return T.id_zero;
  for (uint32_t t = lane; t < m; t += 32) {
    uint32_t lo = 0, hi = n;  // leaf of term t: last leaf with off <= t
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) / 2;
      if (off[mid] <= t) lo = mid;
      else hi = mid;
    }
    uint32_t leaf = leaves[lo];
    Node ln = ld_node(T, leaf);
    uint32_t id = ln.kind == K_ADD ? ld_kid(T, ln.p0 + (t - off[lo])) : leaf;
    ts[t] = decompose_one(T, id);
    key[t] = ts[t].fh;
    val[t] = t;
  }
  __syncwarp();
  // 3. group like terms: sort by factor-vector hash (index breaks ties)
  warp_bitonic(key, val, m, [](uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    return ka != kb ? ka < kb : va < vb;
  });
  // 4. run heads combine their run (exact factor compare inside a hash run)
  uint32_t *out = warp_get<uint32_t>(A, m);
  uint32_t *cnt = warp_get<uint32_t>(A, m);
  if (!out || !cnt) return T.id_zero;
  uint32_t nout = 0;
  for (uint32_t base = 0; base < m; base += 32) {
    uint32_t p = base + lane;
    uint32_t made = 0;
    uint32_t local[4];
    bool overflow = false;
    if (p < m && (p == 0 || key[p] != key[p - 1])) {
      uint32_t q = p + 1;
      while (q < m && key[q] == key[p]) q++;
      for (uint32_t a = p; a < q; a++) {
        const Term &ta = ts[val[a]];
        bool dup = false;  // already merged into an earlier member of this run
        for (uint32_t b = p; b < a && !dup; b++) dup = term_key_cmp(ts[val[b]], ta) == 0;
        if (dup) continue;
        Rat c = ta.c;
        uint32_t nmerge = 1;
        for (uint32_t b = a + 1; b < q; b++)
          if (term_key_cmp(ts[val[b]], ta) == 0) {
            c = rat_add(T, c, ts[val[b]].c);
            nmerge++;
          }
        if (rat_is(c, 0)) continue;
        uint32_t r;
        if (nmerge == 1 && ta.src != UNSET) r = ta.src;
        else r = finish_term(T, A, c, ta);
        if (made < 4) local[made] = r;
        else overflow = true;
        made++;
      }
    }
    uint32_t tot;
    uint32_t ex = warp_excl_scan(made, tot);
    if (__any_sync(kFull, overflow)) {
      // a hash run with more than four distinct factor vectors: degenerate
      // collision pattern, handled by the single-thread path
      uint32_t r = 0;
      if (lane == 0) r = add_nary(T, A, leaves, n);
      return __shfl_sync(kFull, r, 0);
    }
    for (uint32_t k = 0; k < made; k++) out[nout + ex + k] = local[k];
    nout += tot;
  }
  __syncwarp();
  if (nout == 0) return T.id_zero;
  if (nout == 1) return out[0];
  // 5. canonical order, 6. intern
  warp_sort_canonical(T, A, out, nout);
  return warp_intern(T, K_ADD, out, nout);
}

}  // namespace veqd
