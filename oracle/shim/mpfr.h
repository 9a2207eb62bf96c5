/* Declaration-only MPFR 4.2 shim for building the read-only reference as a
 * parity oracle. TEST INFRASTRUCTURE ONLY. Layout and exported symbols
 * match libmpfr.so.6 (MPFR 4.2.1, x86_64 LP64). */
#ifndef VEQ_ORACLE_MPFR_SHIM_H
#define VEQ_ORACLE_MPFR_SHIM_H
#include <gmp.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;
typedef enum { MPFR_RNDN = 0, MPFR_RNDZ, MPFR_RNDU, MPFR_RNDD, MPFR_RNDA } mpfr_rnd_t;
typedef struct { mpfr_prec_t _mpfr_prec; mpfr_sign_t _mpfr_sign; mpfr_exp_t _mpfr_exp; mp_limb_t *_mpfr_d; } __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct *mpfr_ptr;
typedef const __mpfr_struct *mpfr_srcptr;
void mpfr_init2(mpfr_ptr, mpfr_prec_t);
void mpfr_clear(mpfr_ptr);
int mpfr_set(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_set_q(mpfr_ptr, mpq_srcptr, mpfr_rnd_t);
void mpfr_set_inf(mpfr_ptr, int);
int mpfr_sgn(mpfr_srcptr);
int mpfr_nan_p(mpfr_srcptr);
int mpfr_less_p(mpfr_srcptr, mpfr_srcptr);
int mpfr_lessequal_p(mpfr_srcptr, mpfr_srcptr);
int mpfr_greater_p(mpfr_srcptr, mpfr_srcptr);
void mpfr_swap(mpfr_ptr, mpfr_ptr);
int mpfr_neg(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_add(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_max(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_exp(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
double mpfr_get_d(mpfr_srcptr, mpfr_rnd_t);
int mpfr_asprintf(char **, const char *, ...);
void mpfr_free_str(char *);
#ifdef __cplusplus
}
#endif
#endif
