// veq_canon.cuh — AC-canonicalisation (K2) on the device.
//
// Each routine takes CANONICAL operands (interned ids) and returns the
// canonical id of the operation, reproducing the reference's
// canonicalize() rule set exactly (proj/src/expr.cpp:164-289 smart
// constructors, 291-640 CanonCtx). Because symbolic execution canonicalises
// after every statement (symexec.cpp:473), a statement's canonical value is a
// function of its canonical operands; these routines are that function.
//
//   add_nary   = canon_add_kids over all leaves of a fused Add chain
//                (expr.cpp:415-424; fusion is exact)
//   mul_canon  = canon_mul_kids (expr.cpp:426-481) incl. merge_exp_factors
//   canon_div  = canon_div + split_coeff (expr.cpp:497-559)
//   max_nary   = max_of (expr.cpp:254-289)
//
// Work buffers come from a per-thread bump arena carved out of a global
// scratch pool; one item's buffers die when the item completes (the lane's
// current chunk is reused from offset 0 by its next item, so the pool only
// grows when an item needs a larger chunk than any before it on that lane).
#pragma once
#include "veq_dev.cuh"

namespace veqd {

struct Arena {
  char *pool;
  unsigned long long *pool_used;
  uint64_t pool_cap;
  const Table *T;
  char *base;
  uint64_t cap, used;
  uint64_t chunk;  // bytes grabbed from the pool per refill
  uint64_t item;   // current work item (diagnostics)

  __device__ void *alloc(uint64_t bytes) {
    bytes = (bytes + 15) & ~15ull;
    if (used + bytes > cap) {
      uint64_t want = (bytes > chunk ? bytes : chunk);
      want = (want + 255) & ~255ull;  // keep every refill 256-B aligned
      unsigned long long off = atomicAdd(pool_used, (unsigned long long)want);
      if (off + want > pool_cap) {
        if (atomicCAS(T->dbg, 0ull, (unsigned long long)want) == 0ull) {
          T->dbg[1] = off;
          T->dbg[2] = item;
        }
        set_error(*T, E_SCRATCH);
        return nullptr;
      }
      base = pool + off;
      cap = want;
      used = 0;
    }
    void *p = base + used;
    used += bytes;
    return p;
  }
  template <class X> __device__ X *get(uint64_t n) { return reinterpret_cast<X *>(alloc(n * sizeof(X))); }
};

// Calls into the out-of-line routines go through a copy of the caller's
// arena: only the copy's address escapes, so a kernel's own arena stays in
// registers on its hot paths (the out-of-line call is the rare path).
template <class F>
__device__ __forceinline__ uint32_t arena_call(Arena &A, F f) {
  Arena a2 = A;
  const uint32_t r = f(a2);
  A = a2;
  return r;
}

// A term coeff * f[0] * ... * f[nf-1] (expr.cpp:296-300). Factors live in
// the kid arena of an existing Mul (read-only) or in scratch; a single
// factor is held inline.
struct Term {
  Rat c;
  uint64_t fh;
  const uint32_t *f;
  uint32_t nf;
  uint32_t inl;
  uint32_t src;  // canonical node this term was decomposed from (or UNSET)
  uint32_t pad;
};
__device__ __forceinline__ uint32_t tfac(const Term &t, uint32_t i) { return t.f ? __ldcg(t.f + i) : t.inl; }

__device__ inline uint64_t fac_hash(const Term &t) {
  uint64_t h = 0x84222325cbf29ce4ULL ^ t.nf;
  for (uint32_t i = 0; i < t.nf; i++) h = hcomb(h, tfac(t, i));
  return h;
}

// decompose_one (expr.cpp:348-368). A canonical Mul holds at most one Const
// kid and it sorts first.
__device__ inline Term decompose_one(const Table &T, uint32_t id) {
  Node n = ld_node(T, id);
  Term t;
  t.src = id;
  t.f = nullptr;
  t.inl = 0;
  if (n.kind == K_CONST) {
    t.c = const_val(n);
    t.nf = 0;
  } else if (n.kind == K_MUL) {
    uint32_t k0 = ld_kid(T, n.p0);
    Node n0 = ld_node(T, k0);
    if (n0.kind == K_CONST) {
      t.c = const_val(n0);
      t.f = T.kids + n.p0 + 1;
      t.nf = n.nkids - 1;
    } else {
      t.c = Rat{1, 1};
      t.f = T.kids + n.p0;
      t.nf = n.nkids;
    }
    if (t.nf == 1) {
      t.inl = __ldcg(t.f);
      t.f = nullptr;
    }
  } else {
    if (n.kind == K_ADD || n.kind == K_NEG) set_error(T, E_INTERNAL);
    t.c = Rat{1, 1};
    t.nf = 1;
    t.inl = id;
  }
  t.fh = fac_hash(t);
  return t;
}

__device__ __forceinline__ uint32_t n_terms_of(const Table &T, uint32_t id) {
  Node n = ld_node(T, id);
  return n.kind == K_ADD ? n.nkids : 1;
}
// decompose (expr.cpp:339-346)
__device__ inline uint32_t decompose_into(const Table &T, uint32_t id, Term *out) {
  Node n = ld_node(T, id);
  if (n.kind == K_ADD) {
    for (uint32_t i = 0; i < n.nkids; i++) out[i] = decompose_one(T, ld_kid(T, n.p0 + i));
    return n.nkids;
  }
  out[0] = decompose_one(T, id);
  return 1;
}

// Exact factor-vector equality and an arbitrary-but-fixed total order used
// only to group like terms (the TermMap of expr.cpp:302-313; its order does
// not reach the result because rebuild re-sorts through add()).
__device__ inline int term_key_cmp(const Term &a, const Term &b) {
  if (a.fh != b.fh) return a.fh < b.fh ? -1 : 1;
  if (a.nf != b.nf) return a.nf < b.nf ? -1 : 1;
  for (uint32_t i = 0; i < a.nf; i++) {
    uint32_t x = tfac(a, i), y = tfac(b, i);
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}

// ---- sorting (single thread; bottom-up merge sort, stable) ---------------
template <class Less>
__device__ inline void msort_u32(uint32_t *a, uint32_t n, uint32_t *tmp, Less less) {
  if (n < 2) return;
  for (uint32_t i = 1; i < n && n <= 16; i++) {  // insertion sort for tiny n
    uint32_t x = a[i];
    int j = (int)i - 1;
    while (j >= 0 && less(x, a[j])) {
      a[j + 1] = a[j];
      j--;
    }
    a[j + 1] = x;
  }
  if (n <= 16) return;
  uint32_t *src = a, *dst = tmp;
  for (uint32_t w = 1; w < n; w *= 2) {
    for (uint32_t lo = 0; lo < n; lo += 2 * w) {
      uint32_t mid = min(lo + w, n), hi = min(lo + 2 * w, n);
      uint32_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) dst[k++] = less(src[j], src[i]) ? src[j++] : src[i++];
      while (i < mid) dst[k++] = src[i++];
      while (j < hi) dst[k++] = src[j++];
    }
    uint32_t *t = src;
    src = dst;
    dst = t;
  }
  if (src != a)
    for (uint32_t i = 0; i < n; i++) a[i] = src[i];
}

// Sort node ids into canonical order (Expr::compare) using prefixes.
__device__ inline void sort_canonical(const Table &T, Arena &A, uint32_t *ids, uint32_t n) {
  if (n < 2) return;
  uint64_t *pre = A.get<uint64_t>(n);
  uint32_t *idx = A.get<uint32_t>(n), *tmp = A.get<uint32_t>(n), *out = A.get<uint32_t>(n);
  if (!pre || !idx || !tmp || !out) return;
  for (uint32_t i = 0; i < n; i++) {
    pre[i] = prefix_id(T, ids[i]);
    idx[i] = i;
  }
  msort_u32(idx, n, tmp, [&](uint32_t x, uint32_t y) { return cmp_pref(T, pre[x], ids[x], pre[y], ids[y]) < 0; });
  for (uint32_t i = 0; i < n; i++) out[i] = ids[idx[i]];
  for (uint32_t i = 0; i < n; i++) ids[i] = out[i];
}

// mul() smart constructor applied to non-Const, non-Mul, sorted factors
// plus coefficient c != 0 (expr.cpp:194-222; finish_term 393-400).
__device__ inline uint32_t finish_term(const Table &T, Arena &A, Rat c, const Term &t) {
  if (rat_is(c, 1)) {
    if (t.nf == 0) return T.id_one;
    if (t.nf == 1) return tfac(t, 0);
    if (t.src != UNSET && rat_is(t.c, 1) && t.f) {
      // the term is an existing canonical Mul without coefficient
      return t.src;
    }
  }
  uint32_t nk = t.nf + (rat_is(c, 1) ? 0 : 1);
  if (t.nf == 0) return intern_const(T, c);
  uint32_t *k = A.get<uint32_t>(nk);
  if (!k) return T.id_zero;
  uint32_t o = 0;
  if (!rat_is(c, 1)) k[o++] = intern_const(T, c);
  for (uint32_t i = 0; i < t.nf; i++) k[o++] = tfac(t, i);
  return intern(T, K_MUL, 0, 0, k, nk);
}

// Group like terms, drop zero coefficients, rebuild and add()
// (canon_add_kids tail + rebuild, expr.cpp:402-424).
__device__ inline uint32_t collect_terms(const Table &T, Arena &A, Term *ts, uint32_t n) {
  if (n == 0) return T.id_zero;
  uint32_t *idx = A.get<uint32_t>(n), *tmp = A.get<uint32_t>(n);
  if (!idx || !tmp) return T.id_zero;
  for (uint32_t i = 0; i < n; i++) idx[i] = i;
  msort_u32(idx, n, tmp, [&](uint32_t x, uint32_t y) { return term_key_cmp(ts[x], ts[y]) < 0; });
  uint32_t *out = A.get<uint32_t>(n);
  if (!out) return T.id_zero;
  uint32_t nout = 0;
  for (uint32_t i = 0; i < n;) {
    uint32_t j = i + 1;
    Rat c = ts[idx[i]].c;
    while (j < n && term_key_cmp(ts[idx[i]], ts[idx[j]]) == 0) {
      c = rat_add(T, c, ts[idx[j]].c);
      j++;
    }
    if (!rat_is(c, 0)) {
      const Term &t = ts[idx[i]];
      // reuse the source node when the coefficient is unchanged and it was
      // a single canonical term
      if (j == i + 1 && t.src != UNSET && c.n == t.c.n && c.d == t.c.d) out[nout++] = t.src;
      else out[nout++] = finish_term(T, A, c, t);
    }
    i = j;
  }
  if (nout == 0) return T.id_zero;
  if (nout == 1) return out[0];
  sort_canonical(T, A, out, nout);
  return intern(T, K_ADD, 0, 0, out, nout);
}

// canon_add_kids over canonical leaves (expr.cpp:415-424).
__device__ inline uint32_t add_nary(const Table &T, Arena &A, const uint32_t *leaves, uint32_t n) {
  uint32_t total = 0;
  for (uint32_t i = 0; i < n; i++) total += n_terms_of(T, leaves[i]);
  Term *ts = A.get<Term>(total ? total : 1);
  if (!ts) return T.id_zero;
  uint32_t o = 0;
  for (uint32_t i = 0; i < n; i++) o += decompose_into(T, leaves[i], ts + o);
  return collect_terms(T, A, ts, o);
}

// merge_exp_factors (expr.cpp:371-391) on a scratch factor vector; returns
// the new factor count (factors rewritten in place, sorted canonically).
__device__ inline uint32_t merge_exp_factors(const Table &T, Arena &A, uint32_t *f, uint32_t nf) {
  uint32_t nexp = 0;
  for (uint32_t i = 0; i < nf; i++) nexp += ld_kind(T, f[i]) == K_EXP;
  uint32_t nrest = 0;
  if (nexp > 1) {
    uint32_t *args = A.get<uint32_t>(nexp);
    if (!args) return 0;
    uint32_t a = 0;
    for (uint32_t i = 0; i < nf; i++) {
      Node n = ld_node(T, f[i]);
      if (n.kind == K_EXP) args[a++] = ld_kid(T, n.p0);
      else f[nrest++] = f[i];
    }
    uint32_t arg = add_nary(T, A, args, nexp);
    if (arg != T.id_zero) f[nrest++] = intern(T, K_EXP, 0, 0, &arg, 1);  // exp_e folds exp(0) = 1
  } else {
    nrest = nf;
  }
  sort_canonical(T, A, f, nrest);
  return nrest;
}

// canon_mul_kids over canonical operands (expr.cpp:426-481).
__device__ inline uint32_t mul_canon(const Table &T, Arena &A, const uint32_t *ops, uint32_t n) {
  Rat coeff{1, 1};
  uint32_t nfac = 0, nsum = 0;
  for (uint32_t i = 0; i < n; i++) {
    Node k = ld_node(T, ops[i]);
    if (k.kind == K_MUL) nfac += k.nkids;
    else if (k.kind == K_ADD) nsum++;
    else if (k.kind != K_CONST) nfac++;
  }
  uint32_t *fac = A.get<uint32_t>(nfac ? nfac : 1);
  const uint32_t **sums = A.get<const uint32_t *>(nsum ? nsum : 1);
  uint32_t *sumn = A.get<uint32_t>(nsum ? nsum : 1);
  if (!fac || !sums || !sumn) return T.id_zero;
  uint32_t f = 0, s = 0;
  for (uint32_t i = 0; i < n; i++) {
    Node k = ld_node(T, ops[i]);
    if (k.kind == K_CONST) coeff = rat_mul(T, coeff, const_val(k));
    else if (k.kind == K_ADD) {
      sums[s] = T.kids + k.p0;
      sumn[s++] = k.nkids;
    } else if (k.kind == K_MUL) {
      Term t = decompose_one(T, ops[i]);
      coeff = rat_mul(T, coeff, t.c);
      for (uint32_t j = 0; j < t.nf; j++) fac[f++] = tfac(t, j);
    } else if (k.kind == K_NEG) {
      set_error(T, E_INTERNAL);
    } else {
      fac[f++] = ops[i];
    }
  }
  if (rat_is(coeff, 0)) return T.id_zero;
  // cartesian distribution, left to right (expr.cpp:457-473)
  uint64_t nterms = 1;
  for (uint32_t i = 0; i < s; i++) nterms *= sumn[i];
  if (nterms > (1ull << 28)) {
    set_error(T, E_SCRATCH);
    return T.id_zero;
  }
  Term *acc = A.get<Term>(nterms);
  if (!acc) return T.id_zero;
  // each product term: coeff * fac * one term from each sum
  uint32_t *tmp_terms_n = A.get<uint32_t>(s ? s : 1);
  if (!tmp_terms_n) return T.id_zero;
  for (uint64_t t = 0; t < nterms; t++) {
    // decode mixed-radix index (first sum is the most significant digit so
    // the term order matches the nested loops; order is irrelevant anyway)
    uint64_t rem = t;
    Rat c = coeff;
    uint32_t cnt = f;
    // first pass: count factors
    uint64_t r2 = rem;
    for (int q = (int)s - 1; q >= 0; q--) {
      uint32_t pick = (uint32_t)(r2 % sumn[q]);
      r2 /= sumn[q];
      tmp_terms_n[q] = pick;
    }
    for (uint32_t q = 0; q < s; q++) {
      Term st = decompose_one(T, __ldcg(sums[q] + tmp_terms_n[q]));
      cnt += st.nf;
    }
    uint32_t *fv = A.get<uint32_t>(cnt ? cnt : 1);
    if (!fv) return T.id_zero;
    uint32_t o = 0;
    for (uint32_t j = 0; j < f; j++) fv[o++] = fac[j];
    for (uint32_t q = 0; q < s; q++) {
      Term st = decompose_one(T, __ldcg(sums[q] + tmp_terms_n[q]));
      c = rat_mul(T, c, st.c);
      for (uint32_t j = 0; j < st.nf; j++) fv[o++] = tfac(st, j);
    }
    uint32_t nf = merge_exp_factors(T, A, fv, o);
    Term &r = acc[t];
    r.c = c;
    r.src = UNSET;
    r.nf = nf;
    if (nf == 1) {
      r.f = nullptr;
      r.inl = fv[0];
    } else {
      r.f = fv;
      r.inl = 0;
    }
    r.fh = fac_hash(r);
  }
  // drop zero-coefficient products before collection (expr.cpp:477)
  uint32_t m = 0;
  for (uint64_t t = 0; t < nterms; t++)
    if (!rat_is(acc[t].c, 0)) acc[m++] = acc[t];
  return collect_terms(T, A, acc, m);
}

// split_coeff (expr.cpp:497-541).
__device__ inline uint32_t split_coeff(const Table &T, Arena &A, uint32_t e, Rat &content) {
  Node n = ld_node(T, e);
  if (n.kind == K_CONST) {
    content = const_val(n);
    return T.id_one;
  }
  if (n.kind == K_MUL) {
    Term t = decompose_one(T, e);
    content = t.c;
    if (t.nf == 0) return T.id_one;
    if (t.nf == 1) return tfac(t, 0);
    uint32_t *k = A.get<uint32_t>(t.nf);
    if (!k) return T.id_zero;
    for (uint32_t i = 0; i < t.nf; i++) k[i] = tfac(t, i);
    return intern(T, K_MUL, 0, 0, k, t.nf);
  }
  if (n.kind == K_ADD) {
    Term *ts = A.get<Term>(n.nkids);
    if (!ts) return T.id_zero;
    unsigned long long g = 0, l = 1;
    int mi = -1;
    for (uint32_t i = 0; i < n.nkids; i++) {
      ts[i] = decompose_one(T, ld_kid(T, n.p0 + i));
      unsigned long long an = (unsigned long long)(ts[i].c.n < 0 ? -ts[i].c.n : ts[i].c.n);
      g = gcd64(g, an);
      unsigned long long dd = (unsigned long long)ts[i].c.d;
      unsigned long long gg = gcd64(l, dd);
      unsigned __int128 L = (unsigned __int128)(l / gg) * dd;
      if (L > 0x7fffffffffffffffULL) {
        set_error(T, E_OVERFLOW);
        return T.id_zero;
      }
      l = (unsigned long long)L;
      // VecExprLess (expr.cpp:302-311): shorter first, then Expr::compare
      bool less = false;
      if (mi < 0) less = true;
      else if (ts[i].nf != ts[mi].nf) less = ts[i].nf < ts[mi].nf;
      else {
        for (uint32_t q = 0; q < ts[i].nf; q++) {
          uint32_t x = tfac(ts[i], q), y = tfac(ts[mi], q);
          if (x == y) continue;
          less = cmp_pref(T, prefix_id(T, x), x, prefix_id(T, y), y) < 0;
          break;
        }
      }
      if (less) mi = (int)i;
    }
    Rat cont = rat_norm(T, (__int128)g, (__int128)l);
    if (ts[mi].c.n < 0) cont.n = -cont.n;
    content = cont;
    if (rat_is(cont, 1)) return e;
    Rat inv = rat_div(T, Rat{1, 1}, cont);
    uint32_t *sc = A.get<uint32_t>(n.nkids);
    if (!sc) return T.id_zero;
    for (uint32_t i = 0; i < n.nkids; i++) {
      Rat c = rat_mul(T, ts[i].c, inv);
      Term t = ts[i];
      t.src = UNSET;
      sc[i] = finish_term(T, A, c, t);  // scale_term (expr.cpp:484-490)
    }
    // add(scaled): terms stay distinct; at most one Const
    sort_canonical(T, A, sc, n.nkids);
    return intern(T, K_ADD, 0, 0, sc, n.nkids);
  }
  content = Rat{1, 1};
  return e;
}

// canon_div (expr.cpp:543-559); den is not the literal 0 (checked by div()).
__device__ inline uint32_t canon_div(const Table &T, Arena &A, uint32_t num, uint32_t den) {
  Node dn = ld_node(T, den);
  if (dn.kind == K_CONST) {
    uint32_t ops[2] = {intern_const(T, rat_div(T, Rat{1, 1}, const_val(dn))), num};
    return mul_canon(T, A, ops, 2);
  }
  if (num == T.id_zero) return T.id_zero;
  Rat cn, cd;
  uint32_t nc = split_coeff(T, A, num, cn);
  uint32_t dc = split_coeff(T, A, den, cd);
  if (nc == dc) return intern_const(T, rat_div(T, cn, cd));
  uint32_t kids[2] = {nc, dc};
  uint32_t core = intern(T, K_DIV, 0, 0, kids, 2);
  if (cn.n == cd.n && cn.d == cd.d) return core;
  uint32_t ops[2] = {intern_const(T, rat_div(T, cn, cd)), core};
  return mul_canon(T, A, ops, 2);
}

// max_of over canonical leaves (expr.cpp:254-289): flatten Max kids, drop
// -inf, sort, dedup by structure, keep only the largest Const. A Max leaf's
// kids are already a sorted, duplicate-free run, so the result is a merge:
// the loose leaves are sorted on their own, then every run is merged in with
// binary-search insertion of the smaller side (the online-softmax chain
// max(m_prev, s_0..s_63) costs ~64 log n compares instead of a full
// n log n re-sort of m_prev's kids). Same result as sorting everything.
__device__ inline int mx_cmp(const Table &T, uint32_t a, uint64_t pa, uint32_t b, uint64_t pb) {
  return cmp_pref(T, pa, a, pb, b);
}
// first index in run[0..n) whose element is not less than x (lower bound)
__device__ inline uint32_t mx_lower(const Table &T, const uint32_t *run, uint32_t n, uint32_t x, uint64_t px) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) / 2;
    const uint32_t y = __ldcg(run + mid);
    if (mx_cmp(T, y, prefix_id(T, y), x, px) < 0) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ inline uint32_t max_nary(const Table &T, Arena &A, const uint32_t *leaves, uint32_t n) {
  uint32_t total = 0, nloose = 0;
  for (uint32_t i = 0; i < n; i++) {
    Node k = ld_node(T, leaves[i]);
    if (k.kind == K_MAX) total += k.nkids;
    else if (k.kind != K_NEGINF) {
      total++;
      nloose++;
    }
  }
  if (total == 0) return T.id_neginf;
  uint32_t *cur = A.get<uint32_t>(total), *tmp = A.get<uint32_t>(total), *loose = A.get<uint32_t>(nloose ? nloose : 1);
  if (!cur || !tmp || !loose) return T.id_zero;
  uint32_t m = 0;
  for (uint32_t i = 0; i < n; i++) {
    const uint8_t k = ld_kind(T, leaves[i]);
    if (k != K_MAX && k != K_NEGINF) loose[m++] = leaves[i];
  }
  sort_canonical(T, A, loose, nloose);
  uint32_t nc = 0;  // merged so far (in cur)
  for (uint32_t i = 0; i < nloose; i++)
    if (nc == 0 || cur[nc - 1] != loose[i]) cur[nc++] = loose[i];
  for (uint32_t i = 0; i < n; i++) {
    const Node k = ld_node(T, leaves[i]);
    if (k.kind != K_MAX) continue;
    // merge cur[0..nc) with the run kids[p0 .. p0 + nk): insert the smaller
    // side into the larger by lower-bound searches, copying the gaps
    const uint32_t *run = T.kids + k.p0;
    const uint32_t nk = k.nkids;
    const bool small_cur = nc <= nk;
    const uint32_t *big = small_cur ? run : cur, *sml = small_cur ? cur : run;
    const uint32_t nb = small_cur ? nk : nc, ns = small_cur ? nc : nk;
    uint32_t o = 0, bpos = 0;
    for (uint32_t j = 0; j < ns; j++) {
      const uint32_t x = small_cur ? sml[j] : __ldcg(sml + j);
      const uint64_t px = prefix_id(T, x);
      const uint32_t lb = bpos + mx_lower(T, big + bpos, nb - bpos, x, px);
      for (; bpos < lb; bpos++) tmp[o++] = small_cur ? __ldcg(big + bpos) : big[bpos];
      // equal elements (same interned id) appear once
      const bool dup = bpos < nb && (small_cur ? __ldcg(big + bpos) : big[bpos]) == x;
      if (!dup) tmp[o++] = x;
    }
    for (; bpos < nb; bpos++) tmp[o++] = small_cur ? __ldcg(big + bpos) : big[bpos];
    uint32_t *t = cur;
    cur = tmp;
    tmp = t;
    nc = o;
  }
  // keep only the largest Const (Consts sort first)
  uint32_t ncst = 0;
  while (ncst < nc && ld_kind(T, cur[ncst]) == K_CONST) ncst++;
  const uint32_t start = ncst > 1 ? ncst - 1 : 0;
  const uint32_t cnt = nc - start;
  if (cnt == 1) return cur[start];
  return intern(T, K_MAX, 0, 0, cur + start, cnt);
}

}  // namespace veqd
