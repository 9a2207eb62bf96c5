/* Declaration-only GMP 6.3 shim for building the read-only reference
 * (/root/reference/proj) as a parity oracle. TEST INFRASTRUCTURE ONLY.
 * Struct layouts and the exported `__gmp*` symbols match libgmp.so.10
 * (GMP 6.3.0, x86_64 LP64); links against the runtime library by path. */
#ifndef VEQ_ORACLE_GMP_SHIM_H
#define VEQ_ORACLE_GMP_SHIM_H
#include <stddef.h>
#include <stdio.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef unsigned long mp_bitcnt_t;
typedef struct { int _mp_alloc; int _mp_size; mp_limb_t *_mp_d; } __mpz_struct;
typedef struct { __mpz_struct _mp_num; __mpz_struct _mp_den; } __mpq_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpq_struct mpq_t[1];
typedef __mpz_struct *mpz_ptr;
typedef const __mpz_struct *mpz_srcptr;
typedef __mpq_struct *mpq_ptr;
typedef const __mpq_struct *mpq_srcptr;

void __gmpz_init(mpz_ptr);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
int __gmpz_set_str(mpz_ptr, const char *, int);
char *__gmpz_get_str(char *, int, mpz_srcptr);
long __gmpz_get_si(mpz_srcptr);
double __gmpz_get_d(mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
void __gmpz_gcd(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_lcm(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_pow_ui(mpz_ptr, mpz_srcptr, unsigned long);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
mp_limb_t __gmpz_getlimbn(mpz_srcptr, mp_size_t);
size_t __gmpz_size(mpz_srcptr);
int __gmpz_fits_slong_p(mpz_srcptr);

void __gmpq_init(mpq_ptr);
void __gmpq_clear(mpq_ptr);
void __gmpq_set(mpq_ptr, mpq_srcptr);
void __gmpq_set_si(mpq_ptr, long, unsigned long);
void __gmpq_set_z(mpq_ptr, mpz_srcptr);
void __gmpq_set_num(mpq_ptr, mpz_srcptr);
void __gmpq_set_den(mpq_ptr, mpz_srcptr);
int __gmpq_set_str(mpq_ptr, const char *, int);
char *__gmpq_get_str(char *, int, mpq_srcptr);
double __gmpq_get_d(mpq_srcptr);
void __gmpq_canonicalize(mpq_ptr);
void __gmpq_add(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_sub(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_mul(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_div(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_neg(mpq_ptr, mpq_srcptr);
void __gmpq_abs(mpq_ptr, mpq_srcptr);
int __gmpq_cmp(mpq_srcptr, mpq_srcptr);
int __gmpq_equal(mpq_srcptr, mpq_srcptr);
#ifdef __cplusplus
}
#endif

#define mpz_init __gmpz_init
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_set_si __gmpz_set_si
#define mpz_set_ui __gmpz_set_ui
#define mpz_set_str __gmpz_set_str
#define mpz_get_str __gmpz_get_str
#define mpz_get_si __gmpz_get_si
#define mpz_cmp __gmpz_cmp
#define mpz_add __gmpz_add
#define mpz_sub __gmpz_sub
#define mpz_mul __gmpz_mul
#define mpz_neg __gmpz_neg
#define mpz_abs __gmpz_abs
#define mpz_gcd __gmpz_gcd
#define mpz_lcm __gmpz_lcm
#define mpz_pow_ui __gmpz_pow_ui
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_getlimbn __gmpz_getlimbn
#define mpz_fits_slong_p __gmpz_fits_slong_p
#define mpz_size(z) ((size_t)((z)->_mp_size < 0 ? -(z)->_mp_size : (z)->_mp_size))
#define mpz_sgn(z) ((z)->_mp_size < 0 ? -1 : (z)->_mp_size > 0)

#define mpq_init __gmpq_init
#define mpq_clear __gmpq_clear
#define mpq_set __gmpq_set
#define mpq_set_si __gmpq_set_si
#define mpq_set_str __gmpq_set_str
#define mpq_get_str __gmpq_get_str
#define mpq_canonicalize __gmpq_canonicalize
#define mpq_add __gmpq_add
#define mpq_sub __gmpq_sub
#define mpq_mul __gmpq_mul
#define mpq_div __gmpq_div
#define mpq_neg __gmpq_neg
#define mpq_cmp __gmpq_cmp
#define mpq_equal __gmpq_equal
#define mpq_numref(q) (&((q)->_mp_num))
#define mpq_denref(q) (&((q)->_mp_den))
#define mpq_sgn(q) mpz_sgn(mpq_numref(q))
#endif
