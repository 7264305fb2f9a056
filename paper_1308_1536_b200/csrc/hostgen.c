/* hostgen.c -- host-side input generation for the Artless-method beta matrix
 * (reference genmat.py:86-190, Eq. 9 of the paper), over the system
 * MPFR 4.2.1 / MPC 1.3.1 runtime (headers absent: ABI in mp_abi.h).
 *
 * This is INPUT GENERATION, not the elimination: it produces the N x N real
 * matrix a[n][j] = beta_n(gamma_j) in the ds SoA format, with exactly the
 * operation sequence and working precisions of the reference's beta_entry /
 * SpougeGamma.evaluate / SpougeGamma._coefficients, so the matrix is
 * bit-identical to the Python builders (checked by tests/test_hostgen.py
 * against genmat.beta_matrix and the reference golden fingerprint).  Work
 * that the reference recomputes per entry but that depends only on the
 * column (Gamma(1/4 - i t/2), the pi prefactor) is computed once per column.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

#include "mp_abi.h"
#include "../../include/detseries_b200.h"

#define RN MPFR_RNDN
#define RNN MPC_RNDNN

static void put_soa(ds_soa *s, int64_t idx, mpfr_srcptr x, int L) {
  if (mpfr_zero_p(x)) {
    for (int l = 0; l < L; l++) s->limbs[(int64_t)l * s->count + idx] = 0;
    s->exp[idx] = 0;
    s->cls[idx] = mpfr_signbit(x) ? DS_CLS_NZERO : DS_CLS_PZERO;
    return;
  }
  int n64 = (int)((x->_mpfr_prec + 63) / 64);
  int pad = 2 * n64 - L;
  for (int k = 0; k < n64; k++) {
    uint64_t v = x->_mpfr_d[k];
    int l0 = 2 * k - pad, l1 = 2 * k + 1 - pad;
    if (l0 >= 0) s->limbs[(int64_t)l0 * s->count + idx] = (uint32_t)v;
    if (l1 >= 0) s->limbs[(int64_t)l1 * s->count + idx] = (uint32_t)(v >> 32);
  }
  s->exp[idx] = (int32_t)x->_mpfr_exp;
  s->cls[idx] = mpfr_signbit(x) ? DS_CLS_NEG : DS_CLS_POS;
}


/* component c of element idx (complex SoA: c = 0 real, 1 imaginary) */
void dsh_put_soa(ds_soa *s, int c, int64_t idx, mpfr_srcptr x, int L) {
  ds_soa v = *s;
  v.limbs = s->limbs + (int64_t)c * L * s->count;
  v.exp = s->exp + (int64_t)c * s->count;
  v.cls = s->cls + (int64_t)c * s->count;
  put_soa(&v, idx, x, L);
}

/* Spouge coefficients at (a, work2): genmat.py:100-112 */
static void spouge_coeffs(mpfr_t *c, long a, long w) {
  mpfr_t pi, t, km, lg, s, f;
  mpfr_inits2(w, pi, t, km, lg, s, f, (mpfr_ptr)0);
  mpfr_const_pi(pi, RN);
  mpfr_mul_ui(t, pi, 2, RN);          /* 2 * const_pi() */
  mpfr_init2(c[0], w);
  mpfr_sqrt(c[0], t, RN);
  for (long k = 1; k < a; k++) {
    mpfr_set_ui(km, (unsigned long)k, RN);
    mpfr_sub_d(km, km, 0.5, RN);       /* k - mpfr(1)/2 (exact) */
    mpfr_set_ui(t, (unsigned long)(a - k), RN);
    mpfr_log(lg, t, RN);               /* log(a - k) */
    mpfr_mul(s, km, lg, RN);
    mpfr_add_ui(s, s, (unsigned long)(a - k), RN);
    mpfr_exp(t, s, RN);                /* mag */
    mpfr_fac_ui(f, (unsigned long)(k - 1), RN);
    mpfr_init2(c[k], w);
    mpfr_div(c[k], t, f, RN);
    if (k % 2 == 0) mpfr_neg(c[k], c[k], RN);
  }
  mpfr_clears(pi, t, km, lg, s, f, (mpfr_ptr)0);
}

/* Gamma(z) at precision `bits` (genmat.py:114-153); z exact at `bits`. */
static int spouge_gamma(mpc_ptr out, mpc_srcptr z, long bits, int guard) {
  long a = (long)((double)(bits + guard) / 2.65) + 5;
  double y = fabs(mpfr_get_d(mpc_imagref(z), RN));
  long w = bits + guard + (long)(0.45 * (double)a) + (long)(2.27 * y) + 32;
  for (int attempt = 0; attempt < 6; attempt++) {
    mpfr_t *c = (mpfr_t *)malloc(sizeof(mpfr_t) * a);
    spouge_coeffs(c, a, w);
    mpc_t x, acc, term, den, base, h, lb, m1, res, one;
    mpfr_t max_term, t, r1, q, l2;
    mpc_init2(x, w); mpc_init2(acc, w); mpc_init2(term, w); mpc_init2(den, w); mpc_init2(base, w);
    mpc_init2(h, w); mpc_init2(lb, w); mpc_init2(m1, w); mpc_init2(res, w); mpc_init2(one, w);
    mpfr_inits2(w, max_term, t, r1, q, l2, (mpfr_ptr)0);
    mpc_set(x, z, RNN);
    mpc_set_ui(one, 1, RNN);
    mpc_sub(x, x, one, RNN);                          /* x = mpc(zz) - 1 */
    mpc_set_fr(acc, c[0], RNN);                       /* acc = mpc(coeffs[0]) */
    mpc_abs(max_term, acc, RN);
    for (long k = 1; k < a; k++) {
      mpc_set_ui(den, (unsigned long)k, RNN);
      mpc_add(den, x, den, RNN);                      /* x + k */
      mpc_set_fr(term, c[k], RNN);
      mpc_div(term, term, den, RNN);                  /* coeffs[k] / (x + k) */
      mpc_abs(t, term, RN);
      if (mpfr_cmp(t, max_term) > 0) mpfr_set(max_term, t, RN);
      mpc_add(acc, acc, term, RNN);
    }
    mpc_set_ui(base, (unsigned long)a, RNN);
    mpc_add(base, x, base, RNN);                      /* base = x + a */
    mpc_set_d(h, 0.5, RNN);
    mpc_add(h, x, h, RNN);                            /* x + mpfr(1)/2 */
    mpc_log(lb, base, RNN);
    mpc_mul(m1, h, lb, RNN);
    mpc_sub(m1, m1, base, RNN);
    mpc_exp(m1, m1, RNN);
    mpc_mul(res, m1, acc, RNN);                       /* result */
    long cancelled;
    if (!(mpfr_zero_p(mpc_realref(acc)) && mpfr_zero_p(mpc_imagref(acc)))) {
      mpc_abs(r1, acc, RN);
      mpfr_div(q, max_term, r1, RN);
      mpfr_log2(l2, q, RN);
      cancelled = mpfr_get_si(l2, MPFR_RNDZ) + 1;     /* int(log2(...)) + 1 */
    } else {
      cancelled = w;
    }
    int ok = (w - cancelled >= bits + guard / 2);
    if (ok) mpc_set(out, res, RNN);                   /* mpc(result) at prec */
    for (long k = 0; k < a; k++) mpfr_clear(c[k]);
    free(c);
    mpc_clear(x); mpc_clear(acc); mpc_clear(term); mpc_clear(den); mpc_clear(base);
    mpc_clear(h); mpc_clear(lb); mpc_clear(m1); mpc_clear(res); mpc_clear(one);
    mpfr_clears(max_term, t, r1, q, l2, (mpfr_ptr)0);
    if (ok) return 0;
    w += (bits + guard - (w - cancelled)) + 128;
  }
  return -1;
}

/* a[n][j] = beta_n(gamma_j) for n, j = 1..N (genmat.py:156-190); zeros are
 * decimal strings parsed at precision p (load_zeros, genmat.py:40-73).
 * Returns 0, or -1 if a Gamma evaluation failed to stabilise. */
void dsh_get_soa(mpfr_ptr x, const ds_soa *s, int c, int64_t idx, int L) {
  uint8_t k = s->cls[c * s->count + idx];
  if (k >= DS_CLS_PZERO) {
    mpfr_set_ui(x, 0, RN);
    if (k == DS_CLS_NZERO) mpfr_neg(x, x, RN);
    return;
  }
  int n64 = (int)((x->_mpfr_prec + 63) / 64);
  int pad = 2 * n64 - L;
  for (int q = 0; q < n64; q++) {
    uint64_t lo = 0, hi = 0;
    int l0 = 2 * q - pad, l1 = 2 * q + 1 - pad;
    if (l0 >= 0) lo = s->limbs[((int64_t)c * L + l0) * s->count + idx];
    if (l1 >= 0) hi = s->limbs[((int64_t)c * L + l1) * s->count + idx];
    x->_mpfr_d[q] = lo | (hi << 32);
  }
  x->_mpfr_exp = s->exp[c * s->count + idx];
  x->_mpfr_sign = (k == DS_CLS_NEG) ? -1 : 1;
}

/* Gamma(1/4 - i gamma_j/2) at precision p + guard for every column (the
 * expensive, column-only part of beta_entry), as a complex ds SoA (count N).
 * Used to build the cached intermediates in data/. */
int dsh_beta_gammas(int N, long p, const char **zeros, int guard_bits, int nthreads, ds_soa *out) {
  const long work = p + guard_bits;
  const int L = (int)((work + 31) / 32);
  int failed = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
  for (int j = 0; j < N; j++) {
    mpfr_t tp, tt, ztmp, val;
    mpc_t z, g;
    mpfr_init2(tp, p);
    mpfr_set_str(tp, zeros[j], 10, RN);
    mpfr_inits2(work, tt, ztmp, val, (mpfr_ptr)0);
    mpc_init2(z, work);
    mpc_init2(g, work);
    mpfr_set(tt, tp, RN);
    mpfr_neg(ztmp, tt, RN);
    mpfr_div_ui(ztmp, ztmp, 2, RN);
    mpfr_set_d(val, 0.25, RN);
    mpc_set_fr_fr(z, val, ztmp, RNN);
    if (spouge_gamma(g, z, work, 64) != 0) failed = 1;
    ds_soa re = *out, im = *out;
    im.limbs = out->limbs + (int64_t)L * out->count;
    im.exp = out->exp + out->count;
    im.cls = out->cls + out->count;
    put_soa(&re, j, mpc_realref(g), L);
    put_soa(&im, j, mpc_imagref(g), L);
    mpfr_clears(tp, tt, ztmp, val, (mpfr_ptr)0);
    mpc_clear(z);
    mpc_clear(g);
  }
  return failed ? -1 : 0;
}

/* gammas: optional precomputed Gamma values (complex ds SoA, count >= N, at
 * precision p + guard_bits, from dsh_beta_gammas); NULL computes them. */
int dsh_beta_matrix_cols(int N, long p, const char **zeros, int guard_bits, int nthreads, ds_soa *out,
                         const ds_soa *gammas, int j0, int j1, int row0, int rstep);

int dsh_beta_matrix(int N, long p, const char **zeros, int guard_bits, int nthreads, ds_soa *out,
                    const ds_soa *gammas) {
  return dsh_beta_matrix_cols(N, p, zeros, guard_bits, nthreads, out, gammas, 0, N, 0, 1);
}

/* columns [j0, j1) and rows row0, row0 + rstep, ... only (a rank of the
 * row-cyclic layout builds just the rows it owns) */
int dsh_beta_matrix_cols(int N, long p, const char **zeros, int guard_bits, int nthreads, ds_soa *out,
                         const ds_soa *gammas, int j0, int j1, int row0, int rstep) {
  const long work = p + guard_bits;
  const int L = (int)((p + 31) / 32);
  int failed = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
  for (int j = j0; j < j1; j++) {
    mpfr_t tp, tt, pi, lp, A, lnn, val, outp, ztmp;
    mpc_t I, z, g, v, w2, pref, pAg, u, e, npow, den, term, four, half, tmpc;
    mpfr_init2(tp, p);
    mpfr_set_str(tp, zeros[j], 10, RN);              /* gamma_j at prec */
    mpfr_inits2(work, tt, pi, lp, A, lnn, val, ztmp, (mpfr_ptr)0);
    mpfr_init2(outp, p);
    mpc_init2(I, work); mpc_init2(z, work); mpc_init2(g, work); mpc_init2(v, work); mpc_init2(w2, work);
    mpc_init2(pref, work); mpc_init2(pAg, work); mpc_init2(u, work); mpc_init2(e, work); mpc_init2(npow, work);
    mpc_init2(den, work); mpc_init2(term, work); mpc_init2(four, work); mpc_init2(half, work);
    mpc_init2(tmpc, work);
    mpfr_set(tt, tp, RN);                             /* tt = mpfr(t) */
    mpc_set_ui_ui(I, 0, 1, RNN);                      /* i = mpc(0, 1) */
    mpfr_const_pi(pi, RN);
    /* g = Gamma(mpc(1/4, -tt/2)) at work */
    mpfr_neg(ztmp, tt, RN);
    mpfr_div_ui(ztmp, ztmp, 2, RN);
    mpfr_set_d(val, 0.25, RN);
    mpc_set_fr_fr(z, val, ztmp, RNN);
    if (gammas) {
      int Lw = (int)((work + 31) / 32);
      dsh_get_soa(mpc_realref(g), gammas, 0, j, Lw);
      dsh_get_soa(mpc_imagref(g), gammas, 1, j, Lw);
    } else if (spouge_gamma(g, z, work, 64) != 0) {
      failed = 1;
    }
    /* pref = exp((mpfr(-1)/4 + i*tt/2) * log(pi)) */
    mpc_set_fr(tmpc, tt, RNN);
    mpc_mul(v, I, tmpc, RNN);                          /* i * tt */
    mpc_set_ui(tmpc, 2, RNN);
    mpc_div(v, v, tmpc, RNN);                          /* / 2 */
    mpc_set_d(tmpc, -0.25, RNN);
    mpc_add(w2, tmpc, v, RNN);                         /* mpfr(-1)/4 + ... */
    mpfr_log(lp, pi, RN);
    mpc_set_fr(tmpc, lp, RNN);
    mpc_mul(w2, w2, tmpc, RNN);
    mpc_exp(pref, w2, RNN);
    /* A = tt*tt + mpfr(1)/4 ; pAg = (pref * A) * g */
    mpfr_mul(A, tt, tt, RN);
    mpfr_add_d(A, A, 0.25, RN);
    mpc_set_fr(tmpc, A, RNN);
    mpc_mul(pAg, pref, tmpc, RNN);
    mpc_mul(pAg, pAg, g, RNN);
    /* u = mpfr(1)/2 - i*tt (per entry in the reference; identical per column) */
    mpc_set_fr(tmpc, tt, RNN);
    mpc_mul(v, I, tmpc, RNN);
    mpc_set_d(half, 0.5, RNN);
    mpc_sub(u, half, v, RNN);
    mpc_set_ui(four, 4, RNN);
    for (int n = 1 + row0; n <= N; n += rstep) {
      mpfr_set_ui(lnn, (unsigned long)n, RN);
      mpfr_log(lnn, lnn, RN);                          /* log(mpfr(n)) */
      mpc_set_fr(tmpc, lnn, RNN);
      mpc_mul(e, u, tmpc, RNN);
      mpc_exp(npow, e, RNN);
      mpc_mul(den, four, npow, RNN);                   /* 4 * npow */
      mpc_div(term, pAg, den, RNN);
      mpfr_mul_si(val, mpc_realref(term), -2, RN);     /* -2 * term.real */
      mpfr_set(outp, val, RN);                         /* mpfr(val) at prec */
      /* full N x N output, or only rows row0, row0 + rstep, ... (count nloc * N) */
      const int64_t ridx = out->count == (int64_t)N * N ? (int64_t)(n - 1) : (int64_t)((n - 1 - row0) / rstep);
      put_soa(out, ridx * N + j, outp, L);
    }
    mpfr_clears(tp, tt, pi, lp, A, lnn, val, ztmp, outp, (mpfr_ptr)0);
    mpc_clear(I); mpc_clear(z); mpc_clear(g); mpc_clear(v); mpc_clear(w2); mpc_clear(pref); mpc_clear(pAg);
    mpc_clear(u); mpc_clear(e); mpc_clear(npow); mpc_clear(den); mpc_clear(term); mpc_clear(four);
    mpc_clear(half); mpc_clear(tmpc);
  }
  return failed ? -1 : 0;
}


/* ---- the Artless zero-power matrix (reference genmat.py:193-223) ----------
 * (2M+1) x (2M+1) complex; row 1 = 1; row n >= 2 holds, at the work precision
 * w = p + guard (genmat power_matrix):
 *     ln_n = log(mpfr(n)),  r = exp(-ln_n / 2),
 *     for m < M: theta = gamma_m * ln_n, c = r*cos(theta), s = r*sin(theta),
 *                entries (c, s), (c, -s);
 *     last: theta_t = mpfr(t) * ln_n, entry (r*cos(theta_t), -r*sin(theta_t)),
 * each op correctly rounded at w (cos and sin from mpfr_sin_cos, which rounds
 * both exactly as mpfr_cos / mpfr_sin do), then every component rounded to p
 * (mpc(x) in the p context).  gamma_m are the zeros file's tokens rounded at
 * zero_prec (load_zeros' precision) and t the token t_str at t_prec, as the
 * reference's callers pass them.  Rows row0, row0 + rstep, ... only, into a full
 * (count N*N) or owned-rows (count nloc*N) complex SoA. */
int dsh_power_matrix(int M, long p, const char **zeros, long zero_prec, const char *t_str, long t_prec,
                     int guard_bits, int nthreads, ds_soa *out, int row0, int rstep) {
  const int N = 2 * M + 1;
  const long work = p + guard_bits;
  const int L = (int)((p + 31) / 32);
  const int full = out->count == (int64_t)N * N;
  mpfr_t *g = (mpfr_t *)malloc(sizeof(mpfr_t) * (M > 0 ? M : 1));
  mpfr_t t;
  for (int m = 0; m < M; m++) {
    mpfr_init2(g[m], zero_prec);
    mpfr_set_str(g[m], zeros[m], 10, RN);
  }
  mpfr_init2(t, t_prec);
  mpfr_set_str(t, t_str, 10, RN);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
  for (int n = 1 + row0; n <= N; n += rstep) {
    const int64_t ridx = full ? (int64_t)(n - 1) : (int64_t)((n - 1 - row0) / rstep);
    mpfr_t lnn, r, th, c, sn, cc, ss, tw, o;
    mpfr_inits2(work, lnn, r, th, c, sn, cc, ss, tw, (mpfr_ptr)0);
    mpfr_init2(o, p);
    if (n == 1) {
      for (int j = 0; j < N; j++) {
        mpfr_set_ui(o, 1, RN);
        dsh_put_soa(out, 0, ridx * N + j, o, L);
        mpfr_set_ui(o, 0, RN);
        dsh_put_soa(out, 1, ridx * N + j, o, L);
      }
    } else {
      mpfr_set_ui(lnn, (unsigned long)n, RN);
      mpfr_log(lnn, lnn, RN);                      /* ln_n = log(mpfr(n)) */
      mpfr_neg(r, lnn, RN);
      mpfr_div_2ui(r, r, 1, RN);                   /* -ln_n / 2 (exact) */
      mpfr_exp(r, r, RN);                          /* r */
      for (int m = 0; m < M; m++) {
        mpfr_mul(th, g[m], lnn, RN);               /* theta = gamma_m * ln_n */
        mpfr_sin_cos(sn, cc, th, RN);
        mpfr_mul(c, r, cc, RN);                    /* r * cos(theta) */
        mpfr_mul(ss, r, sn, RN);                   /* r * sin(theta) */
        const int64_t e0 = ridx * N + 2 * m;
        mpfr_set(o, c, RN);
        dsh_put_soa(out, 0, e0, o, L);
        dsh_put_soa(out, 0, e0 + 1, o, L);
        mpfr_set(o, ss, RN);
        dsh_put_soa(out, 1, e0, o, L);
        mpfr_neg(o, o, RN);                        /* mpc(c, -s): -RN(s) = RN(-s) */
        dsh_put_soa(out, 1, e0 + 1, o, L);
      }
      mpfr_set(tw, t, RN);                         /* mpfr(t) at work */
      mpfr_mul(th, tw, lnn, RN);                   /* theta_t */
      mpfr_sin_cos(sn, cc, th, RN);
      mpfr_mul(c, r, cc, RN);
      mpfr_mul(ss, r, sn, RN);
      mpfr_neg(ss, ss, RN);                        /* -r * sin(theta_t) */
      mpfr_set(o, c, RN);
      dsh_put_soa(out, 0, ridx * N + 2 * M, o, L);
      mpfr_set(o, ss, RN);
      dsh_put_soa(out, 1, ridx * N + 2 * M, o, L);
    }
    mpfr_clears(lnn, r, th, c, sn, cc, ss, tw, o, (mpfr_ptr)0);
  }
  for (int m = 0; m < M; m++) mpfr_clear(g[m]);
  free(g);
  mpfr_clear(t);
  return 0;
}
