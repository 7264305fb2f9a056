/* Hand-declared ABI of the system MPFR 4.2.1 / MPC 1.3.1 runtime libraries
 * (x86-64 LP64; the image ships the shared objects without headers).  Used by
 * hostgen.c (host-side input generation) only. */
#ifndef DS_MP_ABI_H
#define DS_MP_ABI_H
typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;
typedef unsigned long mp_limb_t;
typedef int mpfr_rnd_t;
#define MPFR_RNDN 0
#define MPFR_RNDZ 1
#define MPC_RNDNN 0
typedef struct { mpfr_prec_t _mpfr_prec; mpfr_sign_t _mpfr_sign; mpfr_exp_t _mpfr_exp; mp_limb_t *_mpfr_d; } __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct *mpfr_ptr;
typedef const __mpfr_struct *mpfr_srcptr;
typedef struct { __mpfr_struct re; __mpfr_struct im; } __mpc_struct;
typedef __mpc_struct mpc_t[1];
typedef __mpc_struct *mpc_ptr;
typedef const __mpc_struct *mpc_srcptr;
#define mpc_realref(x) (&((x)->re))
#define mpc_imagref(x) (&((x)->im))

void mpfr_init2(mpfr_ptr, mpfr_prec_t);
void mpfr_inits2(mpfr_prec_t, mpfr_ptr, ...);
void mpfr_clear(mpfr_ptr);
void mpfr_clears(mpfr_ptr, ...);
int mpfr_set(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_set_ui(mpfr_ptr, unsigned long, mpfr_rnd_t);
int mpfr_set_d(mpfr_ptr, double, mpfr_rnd_t);
int mpfr_set_str(mpfr_ptr, const char *, int, mpfr_rnd_t);
int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul_ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_mul_si(mpfr_ptr, mpfr_srcptr, long, mpfr_rnd_t);
int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div_ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_add_ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_add_d(mpfr_ptr, mpfr_srcptr, double, mpfr_rnd_t);
int mpfr_sub_d(mpfr_ptr, mpfr_srcptr, double, mpfr_rnd_t);
int mpfr_neg(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sqrt(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_exp(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_log(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sin_cos(mpfr_ptr, mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div_2ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_log2(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_const_pi(mpfr_ptr, mpfr_rnd_t);
int mpfr_fac_ui(mpfr_ptr, unsigned long, mpfr_rnd_t);
int mpfr_cmp(mpfr_srcptr, mpfr_srcptr);
int mpfr_zero_p(mpfr_srcptr);
int mpfr_signbit(mpfr_srcptr);
long mpfr_get_si(mpfr_srcptr, mpfr_rnd_t);
double mpfr_get_d(mpfr_srcptr, mpfr_rnd_t);
char *mpfr_get_str(char *, mpfr_exp_t *, int, size_t, mpfr_srcptr, mpfr_rnd_t);

void mpc_init2(mpc_ptr, mpfr_prec_t);
void mpc_clear(mpc_ptr);
int mpc_set(mpc_ptr, mpc_srcptr, int);
int mpc_set_fr(mpc_ptr, mpfr_srcptr, int);
int mpc_set_fr_fr(mpc_ptr, mpfr_srcptr, mpfr_srcptr, int);
int mpc_set_ui(mpc_ptr, unsigned long, int);
int mpc_set_ui_ui(mpc_ptr, unsigned long, unsigned long, int);
int mpc_set_d(mpc_ptr, double, int);
int mpc_add(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_sub(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_mul(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_div(mpc_ptr, mpc_srcptr, mpc_srcptr, int);
int mpc_abs(mpfr_ptr, mpc_srcptr, mpfr_rnd_t);
int mpc_log(mpc_ptr, mpc_srcptr, int);
int mpc_exp(mpc_ptr, mpc_srcptr, int);
#endif
