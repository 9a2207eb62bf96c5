// decide.cpp — see decide.hpp.
#include "decide.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <functional>
#include <random>
#include <set>
#include <unordered_map>
#include <memory>
#include <stdexcept>

namespace veqdec {
namespace {

enum { K_CONST = 0, K_NEGINF, K_VAR, K_EXP, K_MAX, K_DIV, K_NEG, K_MUL, K_ADD };

// ---- exact rationals (int128, canonical; overflow is an error) ------------
using i128 = __int128;
i128 gcd128(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
struct Q {
  i128 n = 0, d = 1;
  Q() = default;
  Q(i128 a, i128 b = 1) : n(a), d(b) { norm(); }
  void norm() {
    if (d < 0) n = -n, d = -d;
    if (n == 0) {
      d = 1;
      return;
    }
    i128 g = gcd128(n, d);
    n /= g;
    d /= g;
    const i128 lim = (i128)1 << 100;
    if (n > lim || n < -lim || d > lim) throw DecideError("rational coefficient outside the exact range");
  }
  bool zero() const { return n == 0; }
  bool operator==(const Q &o) const { return n == o.n && d == o.d; }
  bool operator<(const Q &o) const { return n * o.d < o.n * d; }
};
Q operator+(const Q &a, const Q &b) { return Q(a.n * b.d + b.n * a.d, a.d * b.d); }
Q operator*(const Q &a, const Q &b) {
  const i128 g1 = gcd128(a.n, b.d), g2 = gcd128(b.n, a.d);
  return Q((a.n / (g1 ? g1 : 1)) * (b.n / (g2 ? g2 : 1)), (a.d / (g2 ? g2 : 1)) * (b.d / (g1 ? g1 : 1)));
}
Q neg(const Q &a) { return Q(-a.n, a.d); }

// ---- polynomials over opaque variables (decide.cpp Poly) -------------------
using Mono = std::vector<std::pair<uint32_t, uint32_t>>;  // (var id, exponent), var-sorted
struct MonoLess {
  bool operator()(const Mono &a, const Mono &b) const {
    const size_t n = std::min(a.size(), b.size());
    for (size_t i = 0; i < n; i++) {
      if (a[i].first != b[i].first) return a[i].first < b[i].first;
      if (a[i].second != b[i].second) return a[i].second < b[i].second;
    }
    return a.size() < b.size();
  }
};
Mono mono_mul(const Mono &a, const Mono &b) {
  Mono o;
  size_t i = 0, j = 0;
  while (i < a.size() && j < b.size()) {
    if (a[i].first == b[j].first) o.emplace_back(a[i].first, a[i].second + b[j].second), i++, j++;
    else if (a[i].first < b[j].first) o.push_back(a[i++]);
    else o.push_back(b[j++]);
  }
  for (; i < a.size(); i++) o.push_back(a[i]);
  for (; j < b.size(); j++) o.push_back(b[j]);
  return o;
}
struct Poly {
  std::map<Mono, Q, MonoLess> t;
  void add_term(const Mono &m, const Q &c) {
    if (c.zero()) return;
    auto [it, ins] = t.try_emplace(m, c);
    if (!ins) {
      it->second = it->second + c;
      if (it->second.zero()) t.erase(it);
    }
  }
  bool zero() const { return t.empty(); }
  Q constant() const {
    auto it = t.find(Mono{});
    return it == t.end() ? Q(0) : it->second;
  }
  Poly without_constant() const {
    Poly o = *this;
    o.t.erase(Mono{});
    return o;
  }
};
bool poly_less(const Poly &a, const Poly &b) {
  auto ia = a.t.begin(), ib = b.t.begin();
  MonoLess ml;
  for (; ia != a.t.end() && ib != b.t.end(); ++ia, ++ib) {
    if (ml(ia->first, ib->first)) return true;
    if (ml(ib->first, ia->first)) return false;
    if (ia->second < ib->second) return true;
    if (ib->second < ia->second) return false;
  }
  return ia == a.t.end() && ib != b.t.end();
}
Poly padd(const Poly &a, const Poly &b) {
  Poly o = a;
  for (auto &[m, c] : b.t) o.add_term(m, c);
  return o;
}
Poly pmul(const Poly &a, const Poly &b, uint64_t budget) {
  Poly o;
  for (auto &[ma, ca] : a.t)
    for (auto &[mb, cb] : b.t) {
      o.add_term(mono_mul(ma, mb), ca * cb);
      if (o.t.size() > budget) throw DecideError("monomial budget exceeded");
    }
  return o;
}
Poly pconst(const Q &c) {
  Poly p;
  p.add_term(Mono{}, c);
  return p;
}

// ---- exp-polynomial sums: sum of Poly * exp(poly + c) (ExpPolySum) --------
struct EKey {
  Poly p;
  Q c;
};
struct EKeyLess {
  bool operator()(const EKey &a, const EKey &b) const {
    if (poly_less(a.p, b.p)) return true;
    if (poly_less(b.p, a.p)) return false;
    return a.c < b.c;
  }
};
struct EPS {
  std::map<EKey, Poly, EKeyLess> t;
  void add_term(const EKey &k, const Poly &c) {
    if (c.zero()) return;
    auto [it, ins] = t.try_emplace(k, c);
    if (!ins) {
      for (auto &[m, q] : c.t) it->second.add_term(m, q);  // padd in place
      if (it->second.zero()) t.erase(it);
    }
  }
  bool zero() const { return t.empty(); }
  size_t monomials() const {
    size_t n = 0;
    for (auto &[k, c] : t) n += c.t.size();
    return n;
  }
};
EPS eps_const(const Q &c) {
  EPS s;
  s.add_term(EKey{Poly{}, Q(0)}, pconst(c));
  return s;
}
EPS eps_add(const EPS &a, const EPS &b) {
  EPS o = a;
  for (auto &[k, c] : b.t) o.add_term(k, c);
  return o;
}
EPS eps_neg(const EPS &a) {
  EPS o;
  for (auto &[k, c] : a.t) {
    Poly n;
    for (auto &[m, q] : c.t) n.t.emplace(m, neg(q));
    o.t.emplace(k, n);
  }
  return o;
}
EPS eps_mul(const EPS &a, const EPS &b, uint64_t budget) {
  EPS o;
  for (auto &[ka, ca] : a.t)
    for (auto &[kb, cb] : b.t) {
      o.add_term(EKey{padd(ka.p, kb.p), ka.c + kb.c}, pmul(ca, cb, budget));
      if (o.monomials() > budget) throw DecideError("monomial budget exceeded");
    }
  return o;
}
bool is_one(const EPS &s) {
  if (s.t.size() != 1) return false;
  auto &[k, c] = *s.t.begin();
  return k.p.zero() && k.c.zero() && c.t.size() == 1 && c.t.begin()->first.empty() && c.t.begin()->second == Q(1);
}
// a constant (no variables, no exp): its value
bool as_const(const EPS &s, Q &v) {
  if (s.t.empty()) {
    v = Q(0);
    return true;
  }
  if (s.t.size() != 1) return false;
  auto &[k, c] = *s.t.begin();
  if (!k.p.zero() || !k.c.zero()) return false;
  if (c.t.size() != 1 || !c.t.begin()->first.empty()) return false;
  v = c.t.begin()->second;
  return true;
}

// rationalize (decide.cpp:338-393) and eps_core (decide.cpp:408-453) fused:
// every node maps to (numerator, denominator) exp-polynomials of the same
// algebra; Max nodes are opaque atoms (the opaque-max pass).
struct Conv {
  const Dag &g;
  uint64_t budget;
  std::map<std::string, uint32_t> vars;
  std::map<uint32_t, std::pair<EPS, EPS>> memo;
  uint32_t var_id(const std::string &n) { return vars.emplace(n, (uint32_t)vars.size()).first->second; }
  // a * b; a product with the unit is the other factor (the accumulation in
  // eps_mul would rebuild it term by term and hit the same budget check)
  EPS mul(const EPS &a, const EPS &b) {
    const EPS *x = is_one(a) ? &b : is_one(b) ? &a : nullptr;
    if (!x) return eps_mul(a, b, budget);
    if (x->monomials() > budget) throw DecideError("monomial budget exceeded");
    return *x;
  }
  const std::pair<EPS, EPS> &ratio(uint32_t id) {
    if (auto it = memo.find(id); it != memo.end()) return it->second;
    const DNode &n = g.nodes[id];
    std::pair<EPS, EPS> r;
    const EPS one = eps_const(Q(1));
    switch (n.kind) {
    case K_CONST: r = {eps_const(Q(n.num, n.den)), one}; break;
    case K_NEGINF: throw DecideError("-inf is not an exp-polynomial");
    case K_VAR:
    case K_MAX: {  // a Max node is an opaque atom here
      EPS s;
      Poly p;
      p.add_term(Mono{{var_id(n.kind == K_VAR ? n.name : "!max#" + std::to_string(id)), 1}}, Q(1));
      s.add_term(EKey{Poly{}, Q(0)}, p);
      r = {s, one};
      break;
    }
    case K_NEG: {
      const auto &k = ratio(n.kids[0]);
      r = {eps_neg(k.first), k.second};
      break;
    }
    case K_ADD: {
      r = {eps_const(Q(0)), one};
      for (uint32_t k : n.kids) {
        const auto &x = ratio(k);
        if (is_one(r.second) && is_one(x.second)) {
          for (auto &[key, c] : x.first.t) r.first.add_term(key, c);  // eps_add in place
        } else {
          r.first = eps_add(mul(r.first, x.second), mul(x.first, r.second));
          r.second = mul(r.second, x.second);
        }
      }
      break;
    }
    case K_MUL: {
      r = {one, one};
      for (uint32_t k : n.kids) {
        const auto &x = ratio(k);
        r.first = mul(r.first, x.first);
        r.second = mul(r.second, x.second);
      }
      break;
    }
    case K_DIV: {
      const auto &a = ratio(n.kids[0]);
      const auto &b = ratio(n.kids[1]);
      r = {mul(a.first, b.second), mul(a.second, b.first)};
      break;
    }
    case K_EXP: {
      const auto &k = ratio(n.kids[0]);
      Q c;
      EPS arg = k.first;
      if (!is_one(k.second)) {
        if (!as_const(k.second, c)) throw DecideError("division inside an exponent");
        if (c.zero()) throw DecideError("zero denominator inside an exponent");
        arg = eps_mul(arg, eps_const(Q(c.d, c.n)), budget);
      }
      // the exponent must be a polynomial: one term with the zero key
      Poly p;
      if (!arg.t.empty()) {
        if (arg.t.size() != 1 || !arg.t.begin()->first.p.zero() || !arg.t.begin()->first.c.zero())
          throw DecideError("nested exponential");
        p = arg.t.begin()->second;
      }
      EPS s;
      s.add_term(EKey{p.without_constant(), p.constant()}, pconst(Q(1)));
      r = {s, one};
      break;
    }
    default: throw DecideError("unsupported expression");
    }
    return memo.emplace(id, std::move(r)).first->second;
  }
};

// ---- MPFR intervals (interval.cpp), libmpfr.so.6 loaded at run time ------
struct mpfr_s {
  long prec;
  int sign;
  long exp;
  void *d;
};
using mpfr_p = mpfr_s *;
using cmpfr_p = const mpfr_s *;
enum { RNDN = 0, RNDZ, RNDU, RNDD };
struct Mpfr {
  bool ok = false;
  void (*init2)(mpfr_p, long);
  void (*clear)(mpfr_p);
  int (*set)(mpfr_p, cmpfr_p, int);
  int (*set_si)(mpfr_p, long, int);
  int (*div_si)(mpfr_p, cmpfr_p, long, int);
  void (*set_inf)(mpfr_p, int);
  int (*add)(mpfr_p, cmpfr_p, cmpfr_p, int);
  int (*mul)(mpfr_p, cmpfr_p, cmpfr_p, int);
  int (*div)(mpfr_p, cmpfr_p, cmpfr_p, int);
  int (*neg)(mpfr_p, cmpfr_p, int);
  int (*exp)(mpfr_p, cmpfr_p, int);
  int (*max)(mpfr_p, cmpfr_p, cmpfr_p, int);
  int (*nan_p)(cmpfr_p);
  int (*sgn)(cmpfr_p);
  int (*less_p)(cmpfr_p, cmpfr_p);
  int (*greater_p)(cmpfr_p, cmpfr_p);
  int (*asprintf)(char **, const char *, ...);
  void (*free_str)(char *);
};
const Mpfr &mp() {
  static Mpfr m = [] {
    Mpfr x;
    void *h = dlopen("libmpfr.so.6", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
    bool ok = true;
    auto sym = [&](auto &f, const char *n) {
      f = (std::remove_reference_t<decltype(f)>)dlsym(h, n);
      ok &= f != nullptr;
    };
    sym(x.init2, "mpfr_init2");
    sym(x.clear, "mpfr_clear");
    sym(x.set, "mpfr_set");
    sym(x.set_si, "mpfr_set_si");
    sym(x.div_si, "mpfr_div_si");
    sym(x.set_inf, "mpfr_set_inf");
    sym(x.add, "mpfr_add");
    sym(x.mul, "mpfr_mul");
    sym(x.div, "mpfr_div");
    sym(x.neg, "mpfr_neg");
    sym(x.exp, "mpfr_exp");
    sym(x.max, "mpfr_max");
    sym(x.nan_p, "mpfr_nan_p");
    sym(x.sgn, "mpfr_sgn");
    sym(x.less_p, "mpfr_less_p");
    sym(x.greater_p, "mpfr_greater_p");
    sym(x.asprintf, "mpfr_asprintf");
    sym(x.free_str, "mpfr_free_str");
    x.ok = ok;
    return x;
  }();
  return m;
}

}  // namespace

bool mpfr_available() { return mp().ok; }

bool contains_max(const Dag &dag, uint32_t d) {
  std::set<uint32_t> seen;
  std::function<bool(uint32_t)> rec = [&](uint32_t x) -> bool {
    if (!seen.insert(x).second) return false;
    if (dag.nodes[x].kind == K_MAX) return true;
    for (uint32_t k : dag.nodes[x].kids)
      if (rec(k)) return true;
    return false;
  };
  return rec(d);
}

// d a sum of monomials (Add of Const / Var / Mul of Var and Const kids, or
// one such term): its expansion is those monomials with like terms
// collected, which is what the exp-polynomial conversion computes for this
// shape. handled = false for any other shape.
bool monomial_sum_zero(const Dag &dag, uint32_t d, bool &handled) {
  handled = false;
  const DNode &root = dag.nodes[d];
  std::vector<uint32_t> terms = root.kind == K_ADD ? root.kids : std::vector<uint32_t>{d};
  std::vector<std::pair<std::vector<uint32_t>, Q>> mono;
  mono.reserve(terms.size());
  for (uint32_t t : terms) {
    const DNode &n = dag.nodes[t];
    std::vector<uint32_t> vars;
    Q c(1);
    auto factor = [&](uint32_t x) {
      const DNode &k = dag.nodes[x];
      if (k.kind == K_VAR) vars.push_back(x);
      else if (k.kind == K_CONST) c = c * Q(k.num, k.den);
      else return false;
      return true;
    };
    if (n.kind == K_MUL) {
      for (uint32_t x : n.kids)
        if (!factor(x)) return false;
    } else if (!factor(t)) {
      return false;
    }
    std::sort(vars.begin(), vars.end());
    mono.emplace_back(std::move(vars), c);
  }
  handled = true;
  std::sort(mono.begin(), mono.end(), [](const auto &a, const auto &b) { return a.first < b.first; });
  for (size_t i = 0; i < mono.size();) {
    size_t j = i;
    Q sum(0);
    for (; j < mono.size() && mono[j].first == mono[i].first; j++) sum = sum + mono[j].second;
    if (!sum.zero()) return false;
    i = j;
  }
  return true;
}

bool zero_by_exp_poly(const Dag &dag, uint32_t d, uint64_t max_monomials) {
  bool handled = false;
  const bool z = monomial_sum_zero(dag, d, handled);
  if (handled) return z;
  Conv c{dag, max_monomials, {}, {}};
  return c.ratio(d).first.zero();
}

namespace {

// eval_numeric (interval.cpp:221-280) over closed intervals with directed-
// rounding MPFR endpoints, indeterminate absorbing: the sub-DAG under f and
// g in topological (index) order, kids folded left to right, evaluated into
// per-precision slot buffers without per-operation allocation. f and g share
// the memo (a node's enclosure depends only on the node).
struct SubDag {
  std::vector<uint32_t> ids;                 // reachable node ids, ascending
  std::vector<std::vector<uint32_t>> kids;   // local kid indices
  std::vector<int32_t> var;                  // Var: index into the sorted names
  uint32_t lf = 0, lg = 0;                   // local indices of f and g
  std::vector<std::string> names;            // free variables, sorted
};

SubDag make_sub(const Dag &g, uint32_t f, uint32_t h) {
  SubDag S;
  // per-thread node marks (generation stamps) instead of per-call sets
  thread_local std::vector<uint32_t> stamp, pos;
  thread_local uint32_t gen = 0;
  if (stamp.size() < g.nodes.size()) {
    stamp.assign(g.nodes.size(), 0);
    pos.resize(g.nodes.size());
    gen = 0;
  }
  if (++gen == 0) {
    std::fill(stamp.begin(), stamp.end(), 0);
    gen = 1;
  }
  std::vector<uint32_t> st{f, h}, seen;
  while (!st.empty()) {
    const uint32_t x = st.back();
    st.pop_back();
    if (stamp[x] == gen) continue;
    stamp[x] = gen;
    seen.push_back(x);
    for (uint32_t k : g.nodes[x].kids) st.push_back(k);
  }
  std::sort(seen.begin(), seen.end());  // post-order export: kids first
  S.ids = seen;
  for (uint32_t i = 0; i < seen.size(); i++) pos[seen[i]] = i;
  for (uint32_t x : seen)
    if (g.nodes[x].kind == K_VAR) S.names.push_back(g.nodes[x].name);
  std::sort(S.names.begin(), S.names.end());
  S.names.erase(std::unique(S.names.begin(), S.names.end()), S.names.end());
  S.kids.resize(seen.size());
  S.var.assign(seen.size(), -1);
  for (uint32_t i = 0; i < seen.size(); i++) {
    const DNode &n = g.nodes[seen[i]];
    S.kids[i].reserve(n.kids.size());
    for (uint32_t k : n.kids) S.kids[i].push_back(pos[k]);
    if (n.kind == K_VAR)
      S.var[i] = (int32_t)(std::lower_bound(S.names.begin(), S.names.end(), n.name) - S.names.begin());
  }
  S.lf = pos[f];
  S.lg = pos[h];
  return S;
}

// Integer polynomial sub-DAGs (integer Const, Var, Add, Mul, Neg) at an
// integer point: exact values while every intermediate stays below 2^63 in
// magnitude. Such values are exact at 64-bit MPFR precision, so the interval
// evaluation would return exactly these points: the exact evaluation is a
// shortcut with the same outcome. False: the sub-DAG is not of that shape,
// or a value left the range (the interval path then runs).
bool int_poly(const Dag &g, const SubDag &S) {
  for (uint32_t x : S.ids) {
    const DNode &n = g.nodes[x];
    if (!(n.kind == K_VAR || n.kind == K_ADD || n.kind == K_MUL || n.kind == K_NEG ||
          (n.kind == K_CONST && n.den == 1)))
      return false;
  }
  return true;
}
bool eval_int(const Dag &g, const SubDag &S, const std::vector<int64_t> &vals, std::vector<int64_t> &v) {
  const size_t n = S.ids.size();
  v.resize(n);
  const i128 lim = ((i128)1 << 63) - 1;
  for (size_t i = 0; i < n; i++) {
    const DNode &nd = g.nodes[S.ids[i]];
    const std::vector<uint32_t> &k = S.kids[i];
    i128 r;
    switch (nd.kind) {
    case K_CONST: r = nd.num; break;
    case K_VAR: r = vals[S.var[i]]; break;
    case K_NEG: r = -(i128)v[k[0]]; break;
    case K_ADD:
      r = v[k[0]];
      for (size_t q = 1; q < k.size(); q++) {
        r += v[k[q]];
        if (r > lim || r < -lim) return false;
      }
      break;
    default:  // K_MUL
      r = v[k[0]];
      for (size_t q = 1; q < k.size(); q++) {
        r *= v[k[q]];
        if (r > lim || r < -lim) return false;
      }
      break;
    }
    if (r > lim || r < -lim) return false;
    v[i] = (int64_t)r;
  }
  return true;
}


// Interval slots at one precision, grown on demand and reused by a thread.
struct IvBuf {
  unsigned prec = 0;
  std::vector<mpfr_s> lo, hi;
  std::vector<uint8_t> indet;
  mpfr_s t{}, nlo{}, nhi{};
  explicit IvBuf(unsigned p) : prec(p) {
    mp().init2(&t, p);
    mp().init2(&nlo, p);
    mp().init2(&nhi, p);
  }
  ~IvBuf() {
    for (auto &x : lo) mp().clear(&x);
    for (auto &x : hi) mp().clear(&x);
    mp().clear(&t);
    mp().clear(&nlo);
    mp().clear(&nhi);
  }
  void reserve(size_t n) {
    while (lo.size() < n) {
      lo.emplace_back();
      hi.emplace_back();
      mp().init2(&lo.back(), prec);
      mp().init2(&hi.back(), prec);
    }
    if (indet.size() < n) indet.resize(n);
  }
};

IvBuf &iv_buf(unsigned prec) {
  thread_local std::vector<std::unique_ptr<IvBuf>> bufs;
  for (auto &b : bufs)
    if (b->prec == prec) return *b;
  bufs.push_back(std::make_unique<IvBuf>(prec));
  return *bufs.back();
}

// iv_corners into (nlo, nhi) from slots a and b (r may alias a)
template <class Op>
bool corners(IvBuf &B, mpfr_s *alo, mpfr_s *ahi, const mpfr_s *blo, const mpfr_s *bhi, Op op) {
  const mpfr_s *as[2] = {alo, ahi}, *bs[2] = {blo, bhi};
  bool first = true, nan = false;
  for (int i = 0; i < 2; i++)
    for (int j = 0; j < 2; j++) {
      op(&B.t, as[i], bs[j], RNDD);
      if (mp().nan_p(&B.t)) nan = true;
      if (first || mp().less_p(&B.t, &B.nlo)) mp().set(&B.nlo, &B.t, RNDD);
      op(&B.t, as[i], bs[j], RNDU);
      if (mp().nan_p(&B.t)) nan = true;
      if (first || mp().greater_p(&B.t, &B.nhi)) mp().set(&B.nhi, &B.t, RNDU);
      first = false;
    }
  if (nan) return false;
  mp().set(alo, &B.nlo, RNDD);
  mp().set(ahi, &B.nhi, RNDU);
  return true;
}

void eval_sub(const Dag &g, const SubDag &S, const std::vector<int64_t> &vals, IvBuf &B) {
  const size_t n = S.ids.size();
  B.reserve(n);
  for (size_t i = 0; i < n; i++) {
    const DNode &nd = g.nodes[S.ids[i]];
    mpfr_s *lo = &B.lo[i], *hi = &B.hi[i];
    uint8_t &ind = B.indet[i];
    ind = 0;
    auto of_rat = [&](int64_t num, int64_t den) {
      mp().set_si(lo, (long)num, RNDD);
      mp().set_si(hi, (long)num, RNDU);
      if (den != 1) {
        mp().div_si(lo, lo, (long)den, RNDD);
        mp().div_si(hi, hi, (long)den, RNDU);
      }
    };
    const std::vector<uint32_t> &k = S.kids[i];
    switch (nd.kind) {
    case K_CONST: of_rat(nd.num, nd.den); break;
    case K_NEGINF:
      mp().set_inf(lo, -1);
      mp().set_inf(hi, -1);
      break;
    case K_VAR: of_rat(vals[S.var[i]], 1); break;
    case K_ADD:
    case K_MUL:
    case K_MAX: {
      ind = B.indet[k[0]];
      mp().set(lo, &B.lo[k[0]], RNDD);
      mp().set(hi, &B.hi[k[0]], RNDU);
      for (size_t q = 1; q < k.size() && !ind; q++) {
        const uint32_t c = k[q];
        if (B.indet[c]) {
          ind = 1;
          break;
        }
        if (nd.kind == K_ADD) {
          mp().add(lo, lo, &B.lo[c], RNDD);
          mp().add(hi, hi, &B.hi[c], RNDU);
          if (mp().nan_p(lo) || mp().nan_p(hi)) ind = 1;
        } else if (nd.kind == K_MUL) {
          if (!corners(B, lo, hi, &B.lo[c], &B.hi[c], mp().mul)) ind = 1;
        } else {
          mp().max(lo, lo, &B.lo[c], RNDD);
          mp().max(hi, hi, &B.hi[c], RNDU);
        }
      }
      break;
    }
    case K_NEG:
      ind = B.indet[k[0]];
      if (!ind) {
        mp().neg(lo, &B.hi[k[0]], RNDD);
        mp().neg(hi, &B.lo[k[0]], RNDU);
      }
      break;
    case K_DIV: {
      const uint32_t a = k[0], b = k[1];
      const bool bz = B.indet[b] || (mp().sgn(&B.lo[b]) <= 0 && mp().sgn(&B.hi[b]) >= 0);
      ind = B.indet[a] || bz;
      if (!ind) {
        mp().set(lo, &B.lo[a], RNDD);
        mp().set(hi, &B.hi[a], RNDU);
        if (!corners(B, lo, hi, &B.lo[b], &B.hi[b], mp().div)) ind = 1;
      }
      break;
    }
    case K_EXP:
      ind = B.indet[k[0]];
      if (!ind) {
        mp().exp(lo, &B.lo[k[0]], RNDD);
        mp().exp(hi, &B.hi[k[0]], RNDU);
      }
      break;
    default: ind = 1; break;
    }
  }
}

std::string slot_str(IvBuf &B, uint32_t i) {
  if (B.indet[i]) return "[indeterminate]";
  char *s = nullptr;
  mp().asprintf(&s, "[%.17Rg, %.17Rg]", &B.lo[i], &B.hi[i]);
  std::string o(s);
  mp().free_str(s);
  return o;
}

}  // namespace

bool refute_random(const Dag &dag, uint32_t f, uint32_t g, uint64_t trials, uint64_t seed, Result &w,
                   bool want_witness) {
  if (!mp().ok) return false;
  const SubDag S = make_sub(dag, f, g);
  const bool ipoly = int_poly(dag, S);
  std::vector<int64_t> vals(S.names.size()), iv;
  std::mt19937_64 rng(seed);
  for (uint64_t t = 0; t < trials; ++t) {
    const long box = 1 + (long)(t / 8);
    for (size_t v = 0; v < vals.size(); v++) {
      if (t == 0) {
        vals[v] = 0;
      } else {
        const unsigned long span = (unsigned long)(2 * box + 1);
        vals[v] = (long)(rng() % span) - box;
      }
    }
    if (ipoly && eval_int(dag, S, vals, iv)) {
      // exact values: equal ones are never separated at any precision;
      // different ones are separated at 64 bits (see int_poly). The interval
      // pass below still prints a witness (its points carry MPFR's signed
      // zeros).
      if (iv[S.lf] == iv[S.lg]) continue;
      if (!want_witness) {
        w.precision = 64;
        return true;
      }
    }
    for (unsigned prec : {64u, 128u, 192u, 256u}) {
      IvBuf &B = iv_buf(prec);
      eval_sub(dag, S, vals, B);
      const uint32_t a = S.lf, b = S.lg;
      if (B.indet[a] || B.indet[b]) continue;
      if (mp().less_p(&B.hi[a], &B.lo[b]) || mp().less_p(&B.hi[b], &B.lo[a])) {
        w.precision = prec;
        if (!want_witness) return true;
        w.assignment.clear();
        for (size_t v = 0; v < vals.size(); v++) w.assignment.emplace_back(S.names[v], std::to_string(vals[v]));
        w.f_enclosure = slot_str(B, a);
        w.g_enclosure = slot_str(B, b);
        return true;
      }
      // both enclosures are the same point: the true values are equal and
      // no higher precision can separate them
      auto point = [&](uint32_t x) { return !mp().less_p(&B.lo[x], &B.hi[x]); };
      if (point(a) && point(b) && !mp().less_p(&B.lo[a], &B.lo[b]) && !mp().less_p(&B.lo[b], &B.lo[a])) break;
    }
  }
  return false;
}

}  // namespace veqdec
