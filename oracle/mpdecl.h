/* Hand-declared ABI of the system GMP 6.3 / MPFR 4.2.1 / MPC 1.3.1 runtime
 * libraries (libgmp.so.10, libmpfr.so.6, libmpc.so.3).  The image ships the
 * shared objects but not their headers, so the few types and entry points
 * the oracle needs are restated here (x86-64 LP64 layout, validated by the
 * survey probes: SURVEY.md App. A items 1-2).
 *
 * TEST INFRASTRUCTURE ONLY: included by the oracle (the CPU checker), never
 * by the product path.
 */
#ifndef DSO_MPDECL_H
#define DSO_MPDECL_H

#include <stddef.h>

typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;
typedef unsigned long mp_limb_t;
typedef int mpfr_rnd_t;   /* enum; MPFR_RNDN == 0 */
#define MPFR_RNDN 0
#define MPC_RNDNN 0        /* MPC_RND(MPFR_RNDN, MPFR_RNDN) */

typedef struct {
  mpfr_prec_t _mpfr_prec;
  mpfr_sign_t _mpfr_sign;
  mpfr_exp_t _mpfr_exp;
  mp_limb_t *_mpfr_d;
} __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct *mpfr_ptr;
typedef const __mpfr_struct *mpfr_srcptr;

typedef struct {
  __mpfr_struct re;
  __mpfr_struct im;
} __mpc_struct;
typedef __mpc_struct mpc_t[1];
typedef __mpc_struct *mpc_ptr;
typedef const __mpc_struct *mpc_srcptr;

/* MPFR */
void mpfr_init2(mpfr_ptr, mpfr_prec_t);
void mpfr_clear(mpfr_ptr);
int mpfr_set(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
void mpfr_set_zero(mpfr_ptr, int);
int mpfr_setsign(mpfr_ptr, mpfr_srcptr, int, mpfr_rnd_t);
int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sub(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_add(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_neg(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_zero_p(mpfr_srcptr);
int mpfr_signbit(mpfr_srcptr);
int mpfr_number_p(mpfr_srcptr);
mpfr_exp_t mpfr_get_exp(mpfr_srcptr);

/* MPC */
void mpc_init2(mpc_ptr, mpfr_prec_t);
void mpc_clear(mpc_ptr);
int mpc_mul(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_sub(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_add(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_div(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_neg(mpc_ptr, mpc_srcptr, int);
int mpc_set(mpc_ptr, mpc_srcptr, int);

#endif
