// decide.cpp — see decide.hpp.
#include "decide.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <functional>
#include <random>
#include <set>
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
      it->second = padd(it->second, c);
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
  std::pair<EPS, EPS> ratio(uint32_t id) {
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
      auto k = ratio(n.kids[0]);
      r = {eps_neg(k.first), k.second};
      break;
    }
    case K_ADD: {
      r = {eps_const(Q(0)), one};
      for (uint32_t k : n.kids) {
        auto x = ratio(k);
        if (is_one(r.second) && is_one(x.second)) {
          r.first = eps_add(r.first, x.first);
        } else {
          r.first = eps_add(eps_mul(r.first, x.second, budget), eps_mul(x.first, r.second, budget));
          r.second = eps_mul(r.second, x.second, budget);
        }
      }
      break;
    }
    case K_MUL: {
      r = {one, one};
      for (uint32_t k : n.kids) {
        auto x = ratio(k);
        r.first = eps_mul(r.first, x.first, budget);
        r.second = eps_mul(r.second, x.second, budget);
      }
      break;
    }
    case K_DIV: {
      auto a = ratio(n.kids[0]), b = ratio(n.kids[1]);
      r = {eps_mul(a.first, b.second, budget), eps_mul(a.second, b.first, budget)};
      break;
    }
    case K_EXP: {
      auto k = ratio(n.kids[0]);
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
    memo.emplace(id, r);
    return r;
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

// Closed interval with directed-rounding endpoints; indeterminate absorbs.
struct Iv {
  unsigned prec = 64;
  bool indet = true;
  mpfr_s lo{}, hi{};
  bool init = false;
  Iv() = default;
  explicit Iv(unsigned p) : prec(p), indet(false), init(true) {
    mp().init2(&lo, p);
    mp().init2(&hi, p);
  }
  Iv(const Iv &o) : prec(o.prec), indet(o.indet), init(o.init) {
    if (init) {
      mp().init2(&lo, prec);
      mp().init2(&hi, prec);
      mp().set(&lo, &o.lo, RNDD);
      mp().set(&hi, &o.hi, RNDU);
    }
  }
  Iv &operator=(const Iv &o) {
    if (this == &o) return *this;
    if (init) {
      mp().clear(&lo);
      mp().clear(&hi);
    }
    prec = o.prec;
    indet = o.indet;
    init = o.init;
    if (init) {
      mp().init2(&lo, prec);
      mp().init2(&hi, prec);
      mp().set(&lo, &o.lo, RNDD);
      mp().set(&hi, &o.hi, RNDU);
    }
    return *this;
  }
  ~Iv() {
    if (init) {
      mp().clear(&lo);
      mp().clear(&hi);
    }
  }
  static Iv of_rat(int64_t n, int64_t d, unsigned p) {
    Iv r(p);
    // n is exact at >= 64 bits; one correctly rounded division = set_q
    mp().set_si(&r.lo, (long)n, RNDD);
    mp().set_si(&r.hi, (long)n, RNDU);
    if (d != 1) {
      mp().div_si(&r.lo, &r.lo, (long)d, RNDD);
      mp().div_si(&r.hi, &r.hi, (long)d, RNDU);
    }
    return r;
  }
  bool contains_zero() const { return indet || (mp().sgn(&lo) <= 0 && mp().sgn(&hi) >= 0); }
};
Iv iv_add(const Iv &a, const Iv &b) {
  if (a.indet || b.indet) return Iv();
  Iv r(std::max(a.prec, b.prec));
  mp().add(&r.lo, &a.lo, &b.lo, RNDD);
  mp().add(&r.hi, &a.hi, &b.hi, RNDU);
  if (mp().nan_p(&r.lo) || mp().nan_p(&r.hi)) return Iv();
  return r;
}
template <class Op>
Iv iv_corners(const Iv &a, const Iv &b, Op op) {
  Iv r(std::max(a.prec, b.prec));
  mpfr_s t{};
  mp().init2(&t, r.prec);
  const mpfr_s *as[2] = {&a.lo, &a.hi}, *bs[2] = {&b.lo, &b.hi};
  bool first = true, nan = false;
  for (int i = 0; i < 2; i++)
    for (int j = 0; j < 2; j++) {
      op(&t, as[i], bs[j], RNDD);
      if (mp().nan_p(&t)) nan = true;
      if (first || mp().less_p(&t, &r.lo)) mp().set(&r.lo, &t, RNDD);
      op(&t, as[i], bs[j], RNDU);
      if (mp().nan_p(&t)) nan = true;
      if (first || mp().greater_p(&t, &r.hi)) mp().set(&r.hi, &t, RNDU);
      first = false;
    }
  mp().clear(&t);
  if (nan) return Iv();
  return r;
}
Iv iv_mul(const Iv &a, const Iv &b) {
  if (a.indet || b.indet) return Iv();
  return iv_corners(a, b, mp().mul);
}
Iv iv_div(const Iv &a, const Iv &b) {
  if (a.indet || b.indet || b.contains_zero()) return Iv();
  return iv_corners(a, b, mp().div);
}
Iv iv_neg(const Iv &a) {
  if (a.indet) return Iv();
  Iv r(a.prec);
  mp().neg(&r.lo, &a.hi, RNDD);
  mp().neg(&r.hi, &a.lo, RNDU);
  return r;
}
Iv iv_exp(const Iv &a) {
  if (a.indet) return Iv();
  Iv r(a.prec);
  mp().exp(&r.lo, &a.lo, RNDD);
  mp().exp(&r.hi, &a.hi, RNDU);
  return r;
}
Iv iv_max(const Iv &a, const Iv &b) {
  if (a.indet || b.indet) return Iv();
  Iv r(std::max(a.prec, b.prec));
  mp().max(&r.lo, &a.lo, &b.lo, RNDD);
  mp().max(&r.hi, &a.hi, &b.hi, RNDU);
  return r;
}
bool iv_disjoint(const Iv &a, const Iv &b) {
  if (a.indet || b.indet) return false;
  return mp().less_p(&a.hi, &b.lo) || mp().less_p(&b.hi, &a.lo);
}
std::string iv_str(const Iv &a) {
  if (a.indet) return "[indeterminate]";
  char *s = nullptr;
  mp().asprintf(&s, "[%.17Rg, %.17Rg]", &a.lo, &a.hi);
  std::string o(s);
  mp().free_str(s);
  return o;
}

// eval_numeric (interval.cpp:221-280): kids folded left to right, memoised
Iv eval(const Dag &g, uint32_t id, const std::map<std::string, int64_t> &as, unsigned prec,
        std::map<uint32_t, Iv> &memo) {
  if (auto it = memo.find(id); it != memo.end()) return it->second;
  const DNode &n = g.nodes[id];
  Iv r;
  switch (n.kind) {
  case K_CONST: r = Iv::of_rat(n.num, n.den, prec); break;
  case K_NEGINF:
    r = Iv(prec);
    mp().set_inf(&r.lo, -1);
    mp().set_inf(&r.hi, -1);
    break;
  case K_VAR: {
    auto it = as.find(n.name);
    if (it == as.end()) throw DecideError("eval_numeric: unassigned variable " + n.name);
    r = Iv::of_rat(it->second, 1, prec);
    break;
  }
  case K_ADD:
  case K_MUL:
  case K_MAX:
    r = eval(g, n.kids[0], as, prec, memo);
    for (size_t i = 1; i < n.kids.size(); i++) {
      const Iv k = eval(g, n.kids[i], as, prec, memo);
      r = n.kind == K_ADD ? iv_add(r, k) : n.kind == K_MUL ? iv_mul(r, k) : iv_max(r, k);
    }
    break;
  case K_NEG: r = iv_neg(eval(g, n.kids[0], as, prec, memo)); break;
  case K_DIV: r = iv_div(eval(g, n.kids[0], as, prec, memo), eval(g, n.kids[1], as, prec, memo)); break;
  case K_EXP: r = iv_exp(eval(g, n.kids[0], as, prec, memo)); break;
  default: break;
  }
  memo.emplace(id, r);
  return r;
}

void free_vars(const Dag &g, uint32_t id, std::set<std::string> &out, std::set<uint32_t> &seen) {
  if (!seen.insert(id).second) return;
  const DNode &n = g.nodes[id];
  if (n.kind == K_VAR) out.insert(n.name);
  for (uint32_t k : n.kids) free_vars(g, k, out, seen);
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

bool zero_by_exp_poly(const Dag &dag, uint32_t d, uint64_t max_monomials) {
  Conv c{dag, max_monomials, {}, {}};
  return c.ratio(d).first.zero();
}

bool refute_random(const Dag &dag, uint32_t f, uint32_t g, uint64_t trials, uint64_t seed, Result &w) {
  if (!mp().ok) return false;
  std::set<std::string> names;
  std::set<uint32_t> seen;
  free_vars(dag, f, names, seen);
  free_vars(dag, g, names, seen);
  std::mt19937_64 rng(seed);
  for (uint64_t t = 0; t < trials; ++t) {
    std::map<std::string, int64_t> a;
    const long box = 1 + (long)(t / 8);
    for (const std::string &n : names) {
      if (t == 0) {
        a[n] = 0;
      } else {
        const unsigned long span = (unsigned long)(2 * box + 1);
        a[n] = (long)(rng() % span) - box;
      }
    }
    for (unsigned prec : {64u, 128u, 192u, 256u}) {
      std::map<uint32_t, Iv> mf, mg;
      const Iv fi = eval(dag, f, a, prec, mf), gi = eval(dag, g, a, prec, mg);
      if (fi.indet || gi.indet) continue;
      if (iv_disjoint(fi, gi)) {
        w.assignment.clear();
        for (auto &[n, v] : a) w.assignment.emplace_back(n, std::to_string(v));
        w.f_enclosure = iv_str(fi);
        w.g_enclosure = iv_str(gi);
        w.precision = prec;
        return true;
      }
    }
  }
  return false;
}

}  // namespace veqdec
