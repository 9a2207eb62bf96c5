// Minimal gmpxx.h subset (mpz_class / mpq_class) for building the read-only
// reference as a parity oracle. TEST INFRASTRUCTURE ONLY: the real header is
// absent from this image; this one covers exactly the operations the
// reference sources use (arithmetic, comparison, gcd/lcm/abs/sgn/cmp,
// get_num/get_den/get_str/get_d, canonicalize) over the libgmp.so.10 ABI.
// Two-integer constructors do not canonicalize, as in GMP's gmpxx.
#ifndef VEQ_ORACLE_GMPXX_SHIM_H
#define VEQ_ORACLE_GMPXX_SHIM_H
#include <gmp.h>

#include <cstdlib>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

class mpz_class {
public:
  mpz_class() { mpz_init(z_); }
  mpz_class(const mpz_class &o) { mpz_init(z_); mpz_set(z_, o.z_); }
  mpz_class(mpz_class &&o) noexcept { mpz_init(z_); std::swap(z_[0], o.z_[0]); }
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  mpz_class(T v) {
    mpz_init(z_);
    if constexpr (std::is_signed_v<T>) mpz_set_si(z_, (long)v);
    else mpz_set_ui(z_, (unsigned long)v);
  }
  explicit mpz_class(const std::string &s, int base = 10) {
    mpz_init(z_);
    if (mpz_set_str(z_, s.c_str(), base) != 0) {
      mpz_clear(z_);
      throw std::invalid_argument("mpz_set_str");
    }
  }
  explicit mpz_class(const char *s, int base = 10) : mpz_class(std::string(s), base) {}
  explicit mpz_class(mpz_srcptr p) { mpz_init(z_); mpz_set(z_, p); }
  ~mpz_class() { mpz_clear(z_); }
  mpz_class &operator=(const mpz_class &o) { mpz_set(z_, o.z_); return *this; }
  mpz_class &operator=(mpz_class &&o) noexcept { std::swap(z_[0], o.z_[0]); return *this; }
  mpz_ptr get_mpz_t() { return z_; }
  mpz_srcptr get_mpz_t() const { return z_; }
  std::string get_str(int base = 10) const {
    char *s = mpz_get_str(nullptr, base, z_);
    std::string r(s);
    std::free(s);
    return r;
  }
  long get_si() const { return mpz_get_si(z_); }
  double get_d() const { return __gmpz_get_d(z_); }
  mpz_class &operator+=(const mpz_class &o) { mpz_add(z_, z_, o.z_); return *this; }
  mpz_class &operator-=(const mpz_class &o) { mpz_sub(z_, z_, o.z_); return *this; }
  mpz_class &operator*=(const mpz_class &o) { mpz_mul(z_, z_, o.z_); return *this; }
  mpz_class &operator/=(const mpz_class &o) { __gmpz_tdiv_q(z_, z_, o.z_); return *this; }
  mpz_class &operator%=(const mpz_class &o) { __gmpz_tdiv_r(z_, z_, o.z_); return *this; }
  mpz_class operator-() const { mpz_class r; mpz_neg(r.z_, z_); return r; }
  friend mpz_class operator+(mpz_class a, const mpz_class &b) { return a += b; }
  friend mpz_class operator-(mpz_class a, const mpz_class &b) { return a -= b; }
  friend mpz_class operator*(mpz_class a, const mpz_class &b) { return a *= b; }
  friend mpz_class operator/(mpz_class a, const mpz_class &b) { return a /= b; }
  friend mpz_class operator%(mpz_class a, const mpz_class &b) { return a %= b; }
  friend int cmp(const mpz_class &a, const mpz_class &b) { int c = mpz_cmp(a.z_, b.z_); return (c > 0) - (c < 0); }
  friend bool operator==(const mpz_class &a, const mpz_class &b) { return mpz_cmp(a.z_, b.z_) == 0; }
  friend bool operator!=(const mpz_class &a, const mpz_class &b) { return mpz_cmp(a.z_, b.z_) != 0; }
  friend bool operator<(const mpz_class &a, const mpz_class &b) { return mpz_cmp(a.z_, b.z_) < 0; }
  friend bool operator>(const mpz_class &a, const mpz_class &b) { return mpz_cmp(a.z_, b.z_) > 0; }
  friend bool operator<=(const mpz_class &a, const mpz_class &b) { return mpz_cmp(a.z_, b.z_) <= 0; }
  friend bool operator>=(const mpz_class &a, const mpz_class &b) { return mpz_cmp(a.z_, b.z_) >= 0; }
  friend int sgn(const mpz_class &a) { return mpz_sgn(a.z_); }
  friend mpz_class abs(const mpz_class &a) { mpz_class r; mpz_abs(r.z_, a.z_); return r; }
  friend mpz_class gcd(const mpz_class &a, const mpz_class &b) { mpz_class r; mpz_gcd(r.z_, a.z_, b.z_); return r; }
  friend mpz_class lcm(const mpz_class &a, const mpz_class &b) { mpz_class r; mpz_lcm(r.z_, a.z_, b.z_); return r; }
  friend std::ostream &operator<<(std::ostream &os, const mpz_class &a) { return os << a.get_str(); }
  friend bool mpz_fits_slong(const mpz_class &a) { return mpz_fits_slong_p(a.get_mpz_t()) != 0; }

private:
  mpz_t z_;
};

class mpq_class {
public:
  mpq_class() { mpq_init(q_); }
  mpq_class(const mpq_class &o) { mpq_init(q_); mpq_set(q_, o.q_); }
  mpq_class(mpq_class &&o) noexcept { mpq_init(q_); std::swap(q_[0], o.q_[0]); }
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  mpq_class(T v) {
    mpq_init(q_);
    if constexpr (std::is_signed_v<T>) mpz_set_si(mpq_numref(q_), (long)v);
    else mpz_set_ui(mpq_numref(q_), (unsigned long)v);
  }
  template <class T, class U,
            class = std::enable_if_t<std::is_integral_v<T> && std::is_integral_v<U>>>
  mpq_class(T n, U d) {
    mpq_init(q_);
    if constexpr (std::is_signed_v<T>) mpz_set_si(mpq_numref(q_), (long)n);
    else mpz_set_ui(mpq_numref(q_), (unsigned long)n);
    if constexpr (std::is_signed_v<U>) mpz_set_si(mpq_denref(q_), (long)d);
    else mpz_set_ui(mpq_denref(q_), (unsigned long)d);
  }
  mpq_class(const mpz_class &n, const mpz_class &d) {
    mpq_init(q_);
    mpz_set(mpq_numref(q_), n.get_mpz_t());
    mpz_set(mpq_denref(q_), d.get_mpz_t());
  }
  mpq_class(const mpz_class &n) {
    mpq_init(q_);
    mpz_set(mpq_numref(q_), n.get_mpz_t());
  }
  explicit mpq_class(const std::string &s, int base = 10) {
    mpq_init(q_);
    if (mpq_set_str(q_, s.c_str(), base) != 0) {
      mpq_clear(q_);
      throw std::invalid_argument("mpq_set_str");
    }
  }
  explicit mpq_class(const char *s, int base = 10) : mpq_class(std::string(s), base) {}
  ~mpq_class() { mpq_clear(q_); }
  mpq_class &operator=(const mpq_class &o) { mpq_set(q_, o.q_); return *this; }
  mpq_class &operator=(mpq_class &&o) noexcept { std::swap(q_[0], o.q_[0]); return *this; }
  mpq_ptr get_mpq_t() { return q_; }
  mpq_srcptr get_mpq_t() const { return q_; }
  // gmpxx hands out references to the embedded integers; the layout of
  // mpz_class is exactly one mpz_t, so the same cast is valid here.
  const mpz_class &get_num() const { return *reinterpret_cast<const mpz_class *>(mpq_numref(q_)); }
  const mpz_class &get_den() const { return *reinterpret_cast<const mpz_class *>(mpq_denref(q_)); }
  mpz_class &get_num() { return *reinterpret_cast<mpz_class *>(mpq_numref(q_)); }
  mpz_class &get_den() { return *reinterpret_cast<mpz_class *>(mpq_denref(q_)); }
  mpz_ptr get_num_mpz_t() { return mpq_numref(q_); }
  mpz_ptr get_den_mpz_t() { return mpq_denref(q_); }
  void canonicalize() { mpq_canonicalize(q_); }
  std::string get_str(int base = 10) const {
    char *s = mpq_get_str(nullptr, base, q_);
    std::string r(s);
    std::free(s);
    return r;
  }
  double get_d() const { return __gmpq_get_d(q_); }
  mpq_class &operator+=(const mpq_class &o) { mpq_add(q_, q_, o.q_); return *this; }
  mpq_class &operator-=(const mpq_class &o) { mpq_sub(q_, q_, o.q_); return *this; }
  mpq_class &operator*=(const mpq_class &o) { mpq_mul(q_, q_, o.q_); return *this; }
  mpq_class &operator/=(const mpq_class &o) { mpq_div(q_, q_, o.q_); return *this; }
  mpq_class operator-() const { mpq_class r; mpq_neg(r.q_, q_); return r; }
  mpq_class operator+() const { return *this; }
  friend mpq_class operator+(mpq_class a, const mpq_class &b) { return a += b; }
  friend mpq_class operator-(mpq_class a, const mpq_class &b) { return a -= b; }
  friend mpq_class operator*(mpq_class a, const mpq_class &b) { return a *= b; }
  friend mpq_class operator/(mpq_class a, const mpq_class &b) { return a /= b; }
  friend int cmp(const mpq_class &a, const mpq_class &b) { int c = mpq_cmp(a.q_, b.q_); return (c > 0) - (c < 0); }
  friend bool operator==(const mpq_class &a, const mpq_class &b) { return mpq_equal(a.q_, b.q_) != 0; }
  friend bool operator!=(const mpq_class &a, const mpq_class &b) { return mpq_equal(a.q_, b.q_) == 0; }
  friend bool operator<(const mpq_class &a, const mpq_class &b) { return mpq_cmp(a.q_, b.q_) < 0; }
  friend bool operator>(const mpq_class &a, const mpq_class &b) { return mpq_cmp(a.q_, b.q_) > 0; }
  friend bool operator<=(const mpq_class &a, const mpq_class &b) { return mpq_cmp(a.q_, b.q_) <= 0; }
  friend bool operator>=(const mpq_class &a, const mpq_class &b) { return mpq_cmp(a.q_, b.q_) >= 0; }
  friend int sgn(const mpq_class &a) { return mpq_sgn(a.q_); }
  friend mpq_class abs(const mpq_class &a) { mpq_class r; __gmpq_abs(r.q_, a.q_); return r; }
  friend std::ostream &operator<<(std::ostream &os, const mpq_class &a) { return os << a.get_str(); }

private:
  mpq_t q_;
};

#endif
