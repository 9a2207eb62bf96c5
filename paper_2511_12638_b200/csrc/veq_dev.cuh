// veq_dev.cuh — device-side term DAG (K1): hash-consed node table in HBM,
// exact rationals, and the canonical total order.
//
// Mirrors the reference term algebra (proj/include/ctaeq/expr.hpp:17-68,
// proj/src/expr.cpp:14-133) with one structural change: every node is
// interned (hash-consed) in an open-addressing table, so structural
// equality is id equality (expr.cpp:85-109 becomes `a == b`) and the
// reference's 64-bit node hash (expr.cpp:31-48) becomes a Merkle hash over
// kid hashes that doubles as the table key and a cross-GPU identity.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Routines of the rare paths (deferred-scaling expansion). Measured on C3:
// any out-of-line call in k_eval_warp costs the whole kernel ~2.7x (eval
// 31 ms -> 85 ms per 4 CTA pairs), so they are inlined like everything else;
// define VEQ_FAST_BUILD to outline them for quick development builds.
#ifdef VEQ_FAST_BUILD
#define VEQ_NOINLINE static __device__ __noinline__
#else
#define VEQ_NOINLINE static __device__ inline
#endif

namespace veqd {

// ctaeq::Kind order (expr.hpp:20): Const < NegInf < Var < Exp < Max < Div <
// Neg < Mul < Add. The numeric value is the compare rank.
enum Kind : uint8_t { K_CONST = 0, K_NEGINF, K_VAR, K_EXP, K_MAX, K_DIV, K_NEG, K_MUL, K_ADD };
// F_COEF: a Mul whose first kid is a Const (a term with coefficient != 1).
// Terms without it are determined by their factor vector, so two like terms
// of a sum without F_COEF terms are the same interned id.
// F_ANYCOEF: an Add with at least one F_COEF kid (tells a sum's consumer,
// before it gathers the terms, whether like terms may differ in id).
enum : uint8_t { F_HASDIV = 1, F_POSDEF = 2, F_COEF = 4, F_ANYCOEF = 8 };

// 32-byte node. Const: p0 = num, p1 = den. Var: p0 = order key, p1 =
// identity (input << 40 | cell, or the undef key). Composite: p0 = offset of
// the kid ids in the kid arena, p1 = 64-bit order prefix (see prefix_of).
struct __align__(16) Node {
  uint8_t kind, flags;
  uint16_t pad;
  uint32_t nkids;
  uint64_t hash;
  uint64_t p0;
  uint64_t p1;
};

constexpr uint32_t EMPTY = 0xFFFFFFFFu;
constexpr uint32_t UNSET = 0xFFFFFFFFu;
constexpr uint32_t REF_NODE = 0x80000000u;   // ref tag: term node id
constexpr uint64_t INPUT_KEY = 1ull << 62;    // Var keys >= this are input symbols

// error codes mirror veq.h
constexpr int E_BUDGET = 1, E_OVERFLOW = 2, E_SCRATCH = 9, E_INTERNAL = 10;

struct Table {
  Node *nodes;
  uint32_t *kids;
  uint32_t *slots;
  unsigned long long *counters;  // [0] nodes, [1] kid words, [2] scratch bytes
  uint64_t max_nodes, max_kids, slot_mask;
  int *error;
  unsigned long long *dbg;  // [0] failing request bytes, [1] pool offset, [2] item
  uint32_t id_neginf, id_zero, id_one, id_mone;
  const uint64_t *in_base;  // per declared input: first dense rank of its group
  const uint64_t *in_size;
  uint32_t n_inputs;
  uint32_t *in_cache;       // node id per input symbol (dense rank), UNSET = not yet interned
  uint32_t wa_ids, wa_kids; // per-warp allocation chunk sizes (set per launch from capacity and grid)
};

__device__ __forceinline__ void set_error(const Table &T, int code) { atomicCAS(T.error, 0, code); }

// Release/acquire fence at GPU scope: orders this thread's (and, after a
// __syncwarp, its warp's) prior writes before a later publishing store.
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ---- loads that bypass L1 (nodes are published by other SMs) -------------
__device__ __forceinline__ Node ld_node(const Table &T, uint32_t id) {
  const uint4 *p = reinterpret_cast<const uint4 *>(T.nodes + id);
  uint4 a = __ldcg(p), b = __ldcg(p + 1);
  Node n;
  n.kind = (uint8_t)(a.x & 0xff);
  n.flags = (uint8_t)((a.x >> 8) & 0xff);
  n.pad = 0;
  n.nkids = a.y;
  n.hash = ((uint64_t)a.w << 32) | a.z;
  n.p0 = ((uint64_t)b.y << 32) | b.x;
  n.p1 = ((uint64_t)b.w << 32) | b.z;
  return n;
}
__device__ __forceinline__ uint32_t ld_kid(const Table &T, uint64_t off) { return __ldcg(T.kids + off); }
__device__ __forceinline__ uint8_t ld_kind(const Table &T, uint32_t id) {
  return (uint8_t)(__ldcg(reinterpret_cast<const uint32_t *>(T.nodes + id)) & 0xff);
}
__device__ __forceinline__ uint64_t ld_hash(const Table &T, uint32_t id) {
  return __ldcg(reinterpret_cast<const unsigned long long *>(T.nodes + id) + 1);
}

// ---- hashing ----------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
__device__ __forceinline__ uint64_t hcomb(uint64_t h, uint64_t v) {
  return mix64(h ^ (v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2)));
}

// ---- exact rationals (Rat = mpq_class in the reference, expr.hpp:17) -----
// int64 num/den, canonical (den > 0, gcd 1). Intermediates in int128; a
// result outside int64 raises E_OVERFLOW (never rounds).
struct Rat {
  long long n, d;
};
__device__ __forceinline__ unsigned long long gcd64(unsigned long long a, unsigned long long b) {
  while (b) {
    unsigned long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}
__device__ __forceinline__ unsigned __int128 gcd128(unsigned __int128 a, unsigned __int128 b) {
  while (b) {
    if ((a >> 64) == 0 && (b >> 64) == 0) return gcd64((unsigned long long)a, (unsigned long long)b);
    unsigned __int128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
__device__ inline Rat rat_norm(const Table &T, __int128 n, __int128 d) {
  if (d < 0) {
    n = -n;
    d = -d;
  }
  if (n == 0) return Rat{0, 1};
  unsigned __int128 un = n < 0 ? (unsigned __int128)(-n) : (unsigned __int128)n;
  unsigned __int128 g = gcd128(un, (unsigned __int128)d);
  if (g > 1) {
    n /= (__int128)g;
    d /= (__int128)g;
  }
  const __int128 lim = (__int128)0x7fffffffffffffffLL;
  if (n > lim || n < -lim || d > lim) {
    set_error(T, E_OVERFLOW);
    return Rat{0, 1};
  }
  return Rat{(long long)n, (long long)d};
}
__device__ __forceinline__ Rat rat_add(const Table &T, Rat a, Rat b) {
  if (a.d == 1 && b.d == 1) {
    __int128 r = (__int128)a.n + b.n;
    if (r <= (__int128)0x7fffffffffffffffLL && r >= -(__int128)0x7fffffffffffffffLL) return Rat{(long long)r, 1};
  }
  return rat_norm(T, (__int128)a.n * b.d + (__int128)b.n * a.d, (__int128)a.d * b.d);
}
__device__ __forceinline__ Rat rat_mul(const Table &T, Rat a, Rat b) {
  if (a.d == 1 && b.d == 1) {
    __int128 r = (__int128)a.n * b.n;
    if (r <= (__int128)0x7fffffffffffffffLL && r >= -(__int128)0x7fffffffffffffffLL) return Rat{(long long)r, 1};
  }
  return rat_norm(T, (__int128)a.n * b.n, (__int128)a.d * b.d);
}
__device__ __forceinline__ Rat rat_div(const Table &T, Rat a, Rat b) {
  return rat_norm(T, (__int128)a.n * b.d, (__int128)a.d * b.n);
}
__device__ __forceinline__ int rat_cmp(Rat a, Rat b) {
  __int128 l = (__int128)a.n * b.d, r = (__int128)b.n * a.d;
  return l < r ? -1 : (l > r ? 1 : 0);
}
__device__ __forceinline__ bool rat_is(Rat a, long long v) { return a.d == 1 && a.n == v; }

// ---- order prefix ------------------------------------------------------------
// A 64-bit key monotone in Expr::compare (expr.cpp:111-133): prefix(a) <
// prefix(b) implies compare(a, b) < 0; equal prefixes fall back to the full
// structural compare. Layout: kind rank in bits 63..60. Var: input symbols
// carry their dense byte-order rank. Composites: kid count (12 bits, 4095
// saturates and drops the rest) then the top 48 bits of the first kid's
// prefix — the first kid decides the order among same-kind same-arity nodes.
__device__ __forceinline__ uint64_t var_prefix(uint64_t key) {
  uint64_t p = 2ull << 60;
  if (key >= INPUT_KEY) p |= (1ull << 59) | ((key - INPUT_KEY) << 16);
  return p;
}
__device__ __forceinline__ uint64_t prefix_of(const Node &n) {
  switch (n.kind) {
  case K_CONST: return 0;
  case K_NEGINF: return 1ull << 60;
  case K_VAR: return var_prefix(n.p0);
  default: return n.p1;
  }
}
__device__ __forceinline__ uint64_t prefix_id(const Table &T, uint32_t id) { return prefix_of(ld_node(T, id)); }

// Full canonical compare of two interned nodes. Interning makes id equality
// structural equality, so the recursive lexicographic kid walk of
// expr.cpp:123-131 becomes an iterative descent into the first differing kid.
__device__ inline int cmp_nodes(const Table &T, uint32_t a, uint32_t b) {
  while (a != b) {
    Node na = ld_node(T, a), nb = ld_node(T, b);
    if (na.kind != nb.kind) return na.kind < nb.kind ? -1 : 1;
    switch (na.kind) {
    case K_CONST: return rat_cmp(Rat{(long long)na.p0, (long long)na.p1}, Rat{(long long)nb.p0, (long long)nb.p1});
    case K_VAR: return na.p0 < nb.p0 ? -1 : (na.p0 > nb.p0 ? 1 : 0);
    case K_NEGINF: return 0;
    default: break;
    }
    if (na.nkids != nb.nkids) return na.nkids < nb.nkids ? -1 : 1;
    uint32_t i = 0;
    for (; i < na.nkids; i++) {
      uint32_t ka = ld_kid(T, na.p0 + i), kb = ld_kid(T, nb.p0 + i);
      if (ka != kb) {
        a = ka;
        b = kb;
        break;
      }
    }
    if (i == na.nkids) return 0;  // unreachable for distinct interned ids
  }
  return 0;
}
__device__ __forceinline__ int cmp_pref(const Table &T, uint64_t pa, uint32_t a, uint64_t pb, uint32_t b) {
  if (a == b) return 0;
  if (pa != pb) return pa < pb ? -1 : 1;
  return cmp_nodes(T, a, b);
}

// ---- interning (K1) ----------------------------------------------------------
// Lock-free insert-or-find. The node record and kid words are written and
// fenced before the slot CAS publishes the id; readers go through L2 (ldcg).
// Merkle hash of a composite: position-salted kid hashes summed, so a warp
// can compute it with one reduction (kid order still matters). A sum's kids
// are not salted: its hash is a function of the kid multiset, so a sum can
// be looked up before its terms are sorted (warp_add_smem).
__device__ __forceinline__ uint64_t kid_term(uint32_t i, uint64_t kid_hash) {
  return mix64(kid_hash + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ULL);
}
__device__ __forceinline__ uint64_t kid_term_k(uint8_t kind, uint32_t i, uint64_t kid_hash) {
  return kid_term(kind == K_ADD ? 0u : i, kid_hash);
}
__device__ __forceinline__ uint64_t composite_hash(uint8_t kind, uint32_t nk, uint64_t sum) {
  return mix64(hcomb(0x100001b3ULL, kind) ^ ((uint64_t)nk * 0xc2b2ae3d27d4eb4fULL) ^ sum);
}
__device__ __forceinline__ uint64_t composite_prefix(uint8_t kind, uint32_t nk, uint64_t kid0_prefix) {
  return ((uint64_t)kind << 60) | (nk >= 4095 ? (4095ull << 48) : (((uint64_t)nk << 48) | (kid0_prefix >> 16)));
}
// positive_definite (proj/src/decide.cpp:306-333) from kid flags
__device__ __forceinline__ uint8_t composite_flags(uint8_t kind, bool any_pd, bool all_pd, bool any_div,
                                                  bool kid0_const = false, bool any_coef = false) {
  uint8_t flags = (kind == K_MUL && kid0_const) ? F_COEF : 0;
  if (kind == K_ADD && any_coef) flags |= F_ANYCOEF;
  if (any_div || kind == K_DIV) flags |= F_HASDIV;
  if (kind == K_EXP) flags |= F_POSDEF;
  else if (kind == K_MAX && any_pd) flags |= F_POSDEF;
  else if ((kind == K_ADD || kind == K_MUL || kind == K_DIV) && all_pd) flags |= F_POSDEF;
  return flags;
}

__device__ inline uint32_t intern_meta(const Table &T, uint8_t kind, uint64_t p0, uint64_t p1, const uint32_t *kids,
                                       uint32_t nk, uint64_t h, uint8_t flags);

__device__ inline uint32_t intern(const Table &T, uint8_t kind, uint64_t p0, uint64_t p1, const uint32_t *kids,
                                  uint32_t nk) {
  uint64_t h = hcomb(0x100001b3ULL, kind);
  uint8_t flags = 0;
  if (kind == K_CONST) {
    h = hcomb(hcomb(h, p0), p1);
    if ((long long)p0 > 0) flags |= F_POSDEF;
  } else if (kind == K_VAR) {
    h = hcomb(h, p0);
  } else if (kind != K_NEGINF) {
    bool any_pd = false, all_pd = true, any_div = false, k0c = false, any_cf = false;
    uint64_t sum = 0;
    for (uint32_t i = 0; i < nk; i++) {
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
    h = composite_hash(kind, nk, sum);
    flags = composite_flags(kind, any_pd, all_pd, any_div, k0c, any_cf);
  }
  return intern_meta(T, kind, p0, p1, kids, nk, h, flags);
}

__device__ inline uint32_t intern_meta(const Table &T, uint8_t kind, uint64_t p0, uint64_t p1, const uint32_t *kids,
                                       uint32_t nk, uint64_t h, uint8_t flags) {
  uint64_t slot = h & T.slot_mask;
  uint32_t mine = EMPTY;
  for (uint64_t probes = 0;; probes++) {
    if (probes > T.slot_mask) {
      set_error(T, E_BUDGET);
      return T.id_zero;
    }
    uint32_t cur = *((volatile uint32_t *)(T.slots + slot));
    if (cur == EMPTY) {
      if (mine == EMPTY) {
        unsigned long long id = atomicAdd(&T.counters[0], 1ull);
        if (id >= T.max_nodes) {
          set_error(T, E_BUDGET);
          return T.id_zero;
        }
        uint64_t off = 0;
        if (nk) {
          off = atomicAdd(&T.counters[1], (unsigned long long)nk);
          if (off + nk > T.max_kids) {
            set_error(T, E_BUDGET);
            return T.id_zero;
          }
          for (uint32_t i = 0; i < nk; i++) T.kids[off + i] = kids[i];
        }
        Node n;
        n.kind = kind;
        n.flags = flags;
        n.pad = 0;
        n.nkids = nk;
        n.hash = h;
        n.p0 = (kind == K_CONST || kind == K_VAR || kind == K_NEGINF) ? p0 : off;
        n.p1 = p1;
        T.nodes[id] = n;
        fence_acq_rel();
        mine = (uint32_t)id;
      }
      uint32_t prev = atomicCAS(T.slots + slot, EMPTY, mine);
      if (prev == EMPTY) return mine;
      cur = prev;
    }
    if (ld_hash(T, cur) == h) {
      Node c = ld_node(T, cur);
      if (c.kind == kind && c.nkids == nk) {
        bool same;
        if (kind == K_CONST) same = (c.p0 == p0 && c.p1 == p1);
        else if (kind == K_VAR) same = (c.p0 == p0);
        else if (kind == K_NEGINF) same = true;
        else {
          same = true;
          for (uint32_t i = 0; i < nk && same; i++) same = (ld_kid(T, c.p0 + i) == kids[i]);
        }
        if (same) return cur;
      }
    }
    slot = (slot + 1) & T.slot_mask;
  }
}

__device__ __forceinline__ uint32_t intern_const(const Table &T, Rat r) {
  if (rat_is(r, 0)) return T.id_zero;
  if (rat_is(r, 1)) return T.id_one;
  if (rat_is(r, -1)) return T.id_mone;
  return intern(T, K_CONST, (uint64_t)r.n, (uint64_t)r.d, nullptr, 0);
}
__device__ __forceinline__ Rat const_val(const Node &n) { return Rat{(long long)n.p0, (long long)n.p1}; }

// Dense byte-order rank of the decimal string of i among the decimal strings
// of 0..n-1 ("x_10" < "x_2", the order std::string::compare gives the
// reference's Var names, expr.cpp:120 and pipeline.cpp:116).
__device__ inline uint64_t lexrank(uint64_t i, uint64_t n) {
  char s[24];
  int L = 0;
  {
    char tmp[24];
    uint64_t v = i;
    do {
      tmp[L++] = (char)('0' + v % 10);
      v /= 10;
    } while (v);
    for (int k = 0; k < L; k++) s[k] = tmp[L - 1 - k];
  }
  uint64_t count = 0, lo = 0, hi = 10;  // lengths k = 1..: [lo, hi)
  for (int k = 1; k <= 20 && lo < n; k++) {
    uint64_t top = hi < n ? hi : n;
    uint64_t bound;  // strings t of length k with t < s lexicographically: t < bound numerically
    if (k <= L) {
      uint64_t P = 0;
      for (int q = 0; q < k; q++) P = P * 10 + (uint64_t)(s[q] - '0');
      bound = P;
      uint64_t c = (bound > lo ? (bound < top ? bound : top) - lo : 0);
      count += c;
      if (k < L && P >= lo && P < top) count += 1;  // the proper prefix itself sorts first
    } else {
      unsigned __int128 B = 0;
      for (int q = 0; q < L; q++) B = B * 10 + (uint64_t)(s[q] - '0');
      for (int q = L; q < k; q++) B *= 10;
      uint64_t c = 0;
      if (B > lo) c = ((B < top ? (uint64_t)B : top) - lo);
      count += c;
    }
    lo = (k == 1) ? 10 : lo * 10;
    hi = hi * 10;
    if (k == 1) lo = 10;
  }
  return count;
}

// Input symbols are interned once per term table: a per-symbol cache (reset
// with the table) turns every later load of the same cell into one read.
__device__ __forceinline__ uint32_t intern_input_var(const Table &T, uint32_t input, uint64_t cell) {
  const uint64_t ci = T.in_base[input] + cell;  // dense and injective (cell < size)
  if (T.in_cache) {
    const uint32_t v = __ldcg(T.in_cache + ci);
    if (v != UNSET) return v;
  }
  uint64_t key = INPUT_KEY + T.in_base[input] + lexrank(cell, T.in_size[input]);
  const uint32_t v = intern(T, K_VAR, key, ((uint64_t)input << 40) | cell, nullptr, 0);
  if (T.in_cache) T.in_cache[ci] = v;
  return v;
}
// Undefined symbols (!undef<k>, symexec.cpp:316): their identity is a
// (class, a, b) triple; they sort before every input symbol, as '!' does.
__device__ __forceinline__ uint32_t intern_undef(const Table &T, uint32_t cls, uint64_t a, uint64_t b) {
  uint64_t key = ((uint64_t)cls << 58) | ((a & 0x1fffffffull) << 29) | (b & 0x1fffffffull);
  return intern(T, K_VAR, key, key, nullptr, 0);
}

}  // namespace veqd
