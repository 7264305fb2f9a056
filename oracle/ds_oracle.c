/*
 * ds_oracle.c -- CPU ORACLE (test infrastructure, NOT the product).
 *
 * A plain-C restatement of the reference hot path over the system
 * MPFR/MPC libraries that gmpy2 wraps (gmpy2 itself is absent here; the
 * reference's arithmetic is exactly mpfr_mul/sub/div and mpc_mul/sub/div at
 * round-to-nearest).  It follows, line for line:
 *
 *   elim.py:37-53    apply_pivot_to_row  -> dso_apply_row
 *   elim.py:56-61    minors_row_from_l   -> emit_minors
 *   elim.py:138-155  normalize_minors / _attach_normalized -> emit_minors
 *   elim.py:203-228  eliminate step loop -> dso_pivot_stage + dso_step
 *   parexec.py:244-287 / 290-333  row-cyclic shards, owner broadcasts the
 *                    unnormalized pivot row, every worker recomputes the det
 *                    chain -> the rank/world arguments of dso_create
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load it -- as the checker and as the timed CPU baseline, never as
 * the shipped path.  The scalar format is the ds SoA format of
 * include/detseries_b200.h.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <omp.h>

#include "mpdecl.h"
#include "../include/detseries_b200.h"

#define MPFR_EXP_ZERO_FIELD (-0x7fffffffffffffffL) /* 0 - LONG_MAX: mpfr zero marker */

/* ---------------------------------------------------------------- format */

static inline int nlimbs32(long prec) { return (int)((prec + 31) / 32); }

/* x <- SoA element (component c, index idx); x already has precision prec. */
static void soa_get(mpfr_ptr x, const ds_soa *s, int c, int64_t idx, int L) {
  uint8_t k = s->cls[c * s->count + idx];
  if (k == DS_CLS_PZERO || k == DS_CLS_NZERO) {
    mpfr_set_zero(x, k == DS_CLS_NZERO ? -1 : 1);
    return;
  }
  int n64 = (int)((x->_mpfr_prec + 63) / 64);
  /* 64*n64 >= 32*L; the extra (64*n64 - 32*L) low bits are zero */
  int pad = 2 * n64 - L; /* 0 or 1 leading-zero 32-bit limbs at the bottom */
  for (int k64 = 0; k64 < n64; k64++) {
    uint64_t lo = 0, hi = 0;
    int l0 = 2 * k64 - pad, l1 = 2 * k64 + 1 - pad;
    if (l0 >= 0) lo = s->limbs[((int64_t)c * L + l0) * s->count + idx];
    if (l1 >= 0) hi = s->limbs[((int64_t)c * L + l1) * s->count + idx];
    x->_mpfr_d[k64] = lo | (hi << 32);
  }
  x->_mpfr_exp = s->exp[c * s->count + idx];
  x->_mpfr_sign = (k == DS_CLS_NEG) ? -1 : 1;
}

static void soa_put(ds_soa *s, int c, int64_t idx, mpfr_srcptr x, int L) {
  if (mpfr_zero_p(x)) {
    for (int l = 0; l < L; l++) s->limbs[((int64_t)c * L + l) * s->count + idx] = 0;
    s->exp[c * s->count + idx] = 0;
    s->cls[c * s->count + idx] = mpfr_signbit(x) ? DS_CLS_NZERO : DS_CLS_PZERO;
    return;
  }
  int n64 = (int)((x->_mpfr_prec + 63) / 64);
  int pad = 2 * n64 - L;
  for (int k64 = 0; k64 < n64; k64++) {
    uint64_t v = x->_mpfr_d[k64];
    int l0 = 2 * k64 - pad, l1 = 2 * k64 + 1 - pad;
    if (l0 >= 0) s->limbs[((int64_t)c * L + l0) * s->count + idx] = (uint32_t)v;
    if (l1 >= 0) s->limbs[((int64_t)c * L + l1) * s->count + idx] = (uint32_t)(v >> 32);
  }
  s->exp[c * s->count + idx] = (int32_t)x->_mpfr_exp;
  s->cls[c * s->count + idx] = mpfr_signbit(x) ? DS_CLS_NEG : DS_CLS_POS;
}

/* A scalar slot: real uses re only; complex uses re + im (mpc_t layout). */
typedef __mpc_struct scal;

static void scal_init(scal *x, long prec, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_init2(x, prec);
  else mpfr_init2(&x->re, prec);
}
static void scal_clear(scal *x, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_clear(x);
  else mpfr_clear(&x->re);
}
static void scal_get(scal *x, const ds_soa *s, int64_t idx, int L, int kind) {
  soa_get(&x->re, s, 0, idx, L);
  if (kind == DS_KIND_COMPLEX) soa_get(&x->im, s, 1, idx, L);
}
static void scal_put(ds_soa *s, int64_t idx, const scal *x, int L, int kind) {
  soa_put(s, 0, idx, &x->re, L);
  if (kind == DS_KIND_COMPLEX) soa_put(s, 1, idx, &x->im, L);
}
static int scal_is_zero(const scal *x, int kind) {
  if (kind == DS_KIND_COMPLEX) return mpfr_zero_p(&x->re) && mpfr_zero_p(&x->im);
  return mpfr_zero_p(&x->re);
}
static void s_mul(scal *r, const scal *a, const scal *b, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_mul(r, a, b, MPC_RNDNN);
  else mpfr_mul(&r->re, &a->re, &b->re, MPFR_RNDN);
}
static void s_sub(scal *r, const scal *a, const scal *b, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_sub(r, a, b, MPC_RNDNN);
  else mpfr_sub(&r->re, &a->re, &b->re, MPFR_RNDN);
}
static void s_add(scal *r, const scal *a, const scal *b, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_add(r, a, b, MPC_RNDNN);
  else mpfr_add(&r->re, &a->re, &b->re, MPFR_RNDN);
}
static void s_div(scal *r, const scal *a, const scal *b, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_div(r, a, b, MPC_RNDNN);
  else mpfr_div(&r->re, &a->re, &b->re, MPFR_RNDN);
}
static void s_neg(scal *r, const scal *a, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_neg(r, a, MPC_RNDNN);
  else mpfr_neg(&r->re, &a->re, MPFR_RNDN);
}
static void s_set(scal *r, const scal *a, int kind) {
  if (kind == DS_KIND_COMPLEX) mpc_set(r, a, MPC_RNDNN);
  else mpfr_set(&r->re, &a->re, MPFR_RNDN);
}

/* ------------------------------------------------------- scalar conformance */

int dso_scalar_op(int op, int kind, long prec, const ds_soa *a, const ds_soa *b,
                  ds_soa *out) {
  int L = nlimbs32(prec);
  int rc = DS_OK;
#pragma omp parallel
  {
    scal x, y, r;
    scal_init(&x, prec, kind);
    scal_init(&y, prec, kind);
    scal_init(&r, prec, kind);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < a->count; i++) {
      scal_get(&x, a, i, L, kind);
      scal_get(&y, b, i, L, kind);
      switch (op) {
        case 0: s_mul(&r, &x, &y, kind); break;
        case 1: s_sub(&r, &x, &y, kind); break;
        case 2: s_div(&r, &x, &y, kind); break;
        default: s_add(&r, &x, &y, kind); break;
      }
      scal_put(out, i, &r, L, kind);
    }
    scal_clear(&x, kind);
    scal_clear(&y, kind);
    scal_clear(&r, kind);
  }
  return rc;
}

/* ------------------------------------------------------------ elimination */

typedef struct dso_ctx {
  int n, kind, L, rank, world, nloc, nthreads;
  long prec;
  scal *rows;      /* [nloc][n] owned rows (global row = rank + k*world) */
  scal *prow;      /* [n] unpacked pivot row */
  scal det;        /* running det of this rank (parexec.py:266-268) */
  int have_det;
  scal *tmp_z, *tmp_t; /* per-thread temporaries */
  int failed_step;
  /* broadcast buffer in the ds pivot-buffer format */
  uint8_t *pbuf;
  size_t pbuf_bytes;
  /* accumulated host results (trace + owned minors rows) */
  scal *pivots, *dets; /* [n] */
  scal *sig, *nrm;     /* [n][n] lower triangle, only owned rows used */
  uint8_t *row_flags;  /* [n] */
} dso_ctx;

/* pivot buffer layout: limbs[ncomp][L][n] u32 | exp[ncomp][n] i32 |
 * cls[ncomp][n] u8 (padded to 4 bytes).  Same bytes as the device buffer. */
static ds_soa pbuf_view(uint8_t *p, int n, int L, int ncomp) {
  ds_soa s;
  s.limbs = (uint32_t *)p;
  s.exp = (int32_t *)(p + (size_t)4 * ncomp * L * n);
  s.cls = (uint8_t *)(p + (size_t)4 * ncomp * L * n + (size_t)4 * ncomp * n);
  s.count = n;
  return s;
}

static size_t pbuf_size(int n, int L, int ncomp) {
  return (size_t)4 * ncomp * L * n + (size_t)4 * ncomp * n + (((size_t)ncomp * n + 3) & ~(size_t)3);
}

dso_ctx *dso_create(int n, long prec, int kind, int rank, int world, int nthreads) {
  if (n < 1 || prec < 64 || world < 1 || rank < 0 || rank >= world) return NULL;
  dso_ctx *c = (dso_ctx *)calloc(1, sizeof(dso_ctx));
  c->n = n; c->kind = kind; c->prec = prec; c->L = nlimbs32(prec);
  c->rank = rank; c->world = world;
  c->nloc = (n - rank + world - 1) / world;
  c->nthreads = nthreads > 0 ? nthreads : omp_get_max_threads();
  int ncomp = kind == DS_KIND_COMPLEX ? 2 : 1;
  c->rows = (scal *)calloc((size_t)c->nloc * n, sizeof(scal));
  for (int64_t k = 0; k < (int64_t)c->nloc * n; k++) scal_init(&c->rows[k], prec, kind);
  c->prow = (scal *)calloc(n, sizeof(scal));
  c->pivots = (scal *)calloc(n, sizeof(scal));
  c->dets = (scal *)calloc(n, sizeof(scal));
  for (int k = 0; k < n; k++) {
    scal_init(&c->prow[k], prec, kind);
    scal_init(&c->pivots[k], prec, kind);
    scal_init(&c->dets[k], prec, kind);
  }
  c->sig = (scal *)calloc((size_t)n * n, sizeof(scal));
  c->nrm = (scal *)calloc((size_t)n * n, sizeof(scal));
  c->row_flags = (uint8_t *)calloc(n, 1);
  scal_init(&c->det, prec, kind);
  c->tmp_z = (scal *)calloc(c->nthreads, sizeof(scal));
  c->tmp_t = (scal *)calloc(c->nthreads, sizeof(scal));
  for (int t = 0; t < c->nthreads; t++) {
    scal_init(&c->tmp_z[t], prec, kind);
    scal_init(&c->tmp_t[t], prec, kind);
  }
  c->pbuf_bytes = pbuf_size(n, c->L, ncomp);
  c->pbuf = (uint8_t *)calloc(c->pbuf_bytes, 1);
  c->failed_step = -1;
  return c;
}

void dso_destroy(dso_ctx *c) {
  if (!c) return;
  int n = c->n, kind = c->kind;
  for (int64_t k = 0; k < (int64_t)c->nloc * n; k++) scal_clear(&c->rows[k], kind);
  for (int k = 0; k < n; k++) {
    scal_clear(&c->prow[k], kind);
    scal_clear(&c->pivots[k], kind);
    scal_clear(&c->dets[k], kind);
  }
  for (int64_t k = 0; k < (int64_t)n * n; k++) {
    if (c->sig[k].re._mpfr_d) scal_clear(&c->sig[k], kind);
    if (c->nrm[k].re._mpfr_d) scal_clear(&c->nrm[k], kind);
  }
  for (int t = 0; t < c->nthreads; t++) {
    scal_clear(&c->tmp_z[t], kind);
    scal_clear(&c->tmp_t[t], kind);
  }
  scal_clear(&c->det, kind);
  free(c->rows); free(c->prow); free(c->pivots); free(c->dets); free(c->sig);
  free(c->nrm); free(c->row_flags); free(c->tmp_z); free(c->tmp_t); free(c->pbuf);
  free(c);
}

static inline int owns(const dso_ctx *c, int row) { return row % c->world == c->rank; }
static inline scal *lrow(dso_ctx *c, int row) { return &c->rows[(size_t)(row / c->world) * c->n]; }

int dso_load(dso_ctx *c, const ds_soa *a) {
  for (int r = c->rank; r < c->n; r += c->world)
    for (int k = 0; k < c->n; k++)
      scal_get(&lrow(c, r)[k], a, (int64_t)r * c->n + k, c->L, c->kind);
  return DS_OK;
}

int dso_fetch(dso_ctx *c, ds_soa *a) {
  for (int r = c->rank; r < c->n; r += c->world)
    for (int k = 0; k < c->n; k++)
      scal_put(a, (int64_t)r * c->n + k, &lrow(c, r)[k], c->L, c->kind);
  return DS_OK;
}

void *dso_pivot_buffer(dso_ctx *c, size_t *bytes) {
  *bytes = c->pbuf_bytes;
  return c->pbuf;
}

/* owner(i) packs its unnormalized row i (parexec.py:307-309) */
int dso_pivot_stage(dso_ctx *c, int i) {
  if (!owns(c, i)) return DS_INVALID;
  ds_soa v = pbuf_view(c->pbuf, c->n, c->L, c->kind == DS_KIND_COMPLEX ? 2 : 1);
  scal *row = lrow(c, i);
  for (int k = 0; k < c->n; k++) scal_put(&v, k, &row[k], c->L, c->kind);
  return DS_OK;
}

/* elim.py:37-53, verbatim op order: z = row[i]/piv; L slots k<i ascending
 * (only when collecting minors); U slots k>i ascending; row[i] = -z. */
static void dso_apply_row(scal *row, const scal *prow, int i, int n, int collect_minors,
                          scal *z, scal *t, int kind) {
  s_div(z, &row[i], &prow[i], kind);
  if (collect_minors)
    for (int k = 0; k < i; k++) {
      s_mul(t, z, &prow[k], kind);
      s_sub(&row[k], &row[k], t, kind);
    }
  for (int k = i + 1; k < n; k++) {
    s_mul(t, z, &prow[k], kind);
    s_sub(&row[k], &row[k], t, kind);
  }
  s_neg(&row[i], z, kind);
}

/* minors_row_from_l + _attach_normalized for leading size m = i+2 from this
 * rank's copy of row i+1 after step i (elim.py:220-226, parexec.py:458-462). */
static void emit_minors(dso_ctx *c, int i) {
  int m = i + 2, kind = c->kind;
  scal *row = lrow(c, i + 1);
  scal *sig = &c->sig[(size_t)(m - 1) * c->n];
  scal *nrm = &c->nrm[(size_t)(m - 1) * c->n];
  for (int k = 0; k < m; k++) {
    if (!sig[k].re._mpfr_d) scal_init(&sig[k], c->prec, kind);
    if (!nrm[k].re._mpfr_d) scal_init(&nrm[k], c->prec, kind);
  }
  for (int k = 0; k < m - 1; k++) s_mul(&sig[k], &c->det, &row[k], kind); /* det_prev * v */
  s_set(&sig[m - 1], &c->det, kind);                                      /* append det_prev */
  uint8_t fl = 1;
  if (!scal_is_zero(&sig[0], kind)) {                                     /* lead == 0 -> None */
    for (int k = 0; k < m; k++) s_div(&nrm[k], &sig[k], &sig[0], kind);
    fl |= 2;
  }
  c->row_flags[m - 1] = fl;
}

/* one pivot step on this rank from the (broadcast) pivot buffer */
int dso_step(dso_ctx *c, int i, int collect_minors, int series) {
  if (c->failed_step >= 0) return DS_ZERO_PIVOT;
  int n = c->n, kind = c->kind;
  ds_soa v = pbuf_view(c->pbuf, n, c->L, kind == DS_KIND_COMPLEX ? 2 : 1);
  for (int k = 0; k < n; k++) scal_get(&c->prow[k], &v, k, c->L, kind);
  if (scal_is_zero(&c->prow[i], kind)) { /* elim.py:209-212: exact zero only */
    c->failed_step = i;
    return DS_ZERO_PIVOT;
  }
  /* det = piv if det is None else det * piv   (elim.py:213-215) */
  if (!c->have_det) { s_set(&c->det, &c->prow[i], kind); c->have_det = 1; }
  else s_mul(&c->det, &c->det, &c->prow[i], kind);
  s_set(&c->pivots[i], &c->prow[i], kind);
  s_set(&c->dets[i], &c->det, kind);
  /* rows j > i owned by this rank (elim.py:216-218, parexec.py:318-321) */
  int first = i + 1;
  int k0 = (first - c->rank + c->world - 1) / c->world; /* first local index >= i+1 */
  if (k0 < 0) k0 = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(c->nthreads)
  for (int k = k0; k < c->nloc; k++) {
    int t = omp_get_thread_num();
    dso_apply_row(&c->rows[(size_t)k * n], c->prow, i, n, collect_minors, &c->tmp_z[t],
                  &c->tmp_t[t], kind);
  }
  if (collect_minors && i + 1 < n) {
    int m = i + 2;
    if ((series || m == n) && owns(c, i + 1)) emit_minors(c, i);
  }
  return DS_OK;
}

int dso_set_det(dso_ctx *c, const ds_soa *d) {
  scal_get(&c->det, d, 0, c->L, c->kind);
  c->have_det = 1;
  return DS_OK;
}

int dso_status(dso_ctx *c, int *failed_step) {
  *failed_step = c->failed_step;
  return DS_OK;
}

/* trace for steps [0, upto) and owned minors rows into host SoA buffers */
int dso_results_fetch(dso_ctx *c, int upto, ds_results *r) {
  int n = c->n, L = c->L, kind = c->kind;
  for (int i = 0; i < upto && i < n; i++) {
    if (r->pivots.limbs) scal_put(&r->pivots, i, &c->pivots[i], L, kind);
    if (r->dets.limbs) scal_put(&r->dets, i, &c->dets[i], L, kind);
  }
  for (int m = 2; m <= n; m++) {
    if (!c->row_flags[m - 1]) continue;
    if (r->row_flags) r->row_flags[m - 1] = c->row_flags[m - 1];
    for (int k = 0; k < m; k++) {
      int64_t idx = (int64_t)(m - 1) * n + k;
      if (r->signed_minors.limbs)
        scal_put(&r->signed_minors, idx, &c->sig[(size_t)(m - 1) * n + k], L, kind);
      if (r->normalized.limbs && (c->row_flags[m - 1] & 2))
        scal_put(&r->normalized, idx, &c->nrm[(size_t)(m - 1) * n + k], L, kind);
    }
  }
  return DS_OK;
}

/* Serial convenience (world must be 1): steps [start, stop). */
int dso_run(dso_ctx *c, int collect_minors, int series, int start, int stop, int *steps_done) {
  for (int i = start; i < stop; i++) {
    dso_pivot_stage(c, i);
    int rc = dso_step(c, i, collect_minors, series);
    if (rc != DS_OK) { *steps_done = i; return rc; }
  }
  *steps_done = stop;
  return DS_OK;
}

/* ------------------------------------------------ CPU baseline primitive */

/* Time-able form of the hot loop: apply step i of prow (count n) to `nrows`
 * full-width rows (count nrows*n, row-major), elim.py:37-53, on nthreads. */
int dso_apply_pivot_rows(int n, long prec, int kind, int i, int collect_minors,
                         const ds_soa *prow_soa, ds_soa *rows_soa, int nrows, int nthreads) {
  int L = nlimbs32(prec);
  scal *prow = (scal *)calloc(n, sizeof(scal));
  scal *rows = (scal *)calloc((size_t)nrows * n, sizeof(scal));
  for (int k = 0; k < n; k++) { scal_init(&prow[k], prec, kind); scal_get(&prow[k], prow_soa, k, L, kind); }
  for (int64_t k = 0; k < (int64_t)nrows * n; k++) { scal_init(&rows[k], prec, kind); scal_get(&rows[k], rows_soa, k, L, kind); }
#pragma omp parallel num_threads(nthreads)
  {
    scal z, t;
    scal_init(&z, prec, kind);
    scal_init(&t, prec, kind);
#pragma omp for schedule(dynamic, 1)
    for (int r = 0; r < nrows; r++) dso_apply_row(&rows[(size_t)r * n], prow, i, n, collect_minors, &z, &t, kind);
    scal_clear(&z, kind);
    scal_clear(&t, kind);
  }
  for (int64_t k = 0; k < (int64_t)nrows * n; k++) { scal_put(rows_soa, k, &rows[k], L, kind); scal_clear(&rows[k], kind); }
  for (int k = 0; k < n; k++) scal_clear(&prow[k], kind);
  free(prow); free(rows);
  return DS_OK;
}

/* Same as above but only the update loop is timed internally (conversion
 * excluded); returns seconds. */
double dso_time_apply_pivot_rows(int n, long prec, int kind, int i, int collect_minors,
                                 const ds_soa *prow_soa, ds_soa *rows_soa, int nrows,
                                 int nthreads) {
  int L = nlimbs32(prec);
  scal *prow = (scal *)calloc(n, sizeof(scal));
  scal *rows = (scal *)calloc((size_t)nrows * n, sizeof(scal));
  for (int k = 0; k < n; k++) { scal_init(&prow[k], prec, kind); scal_get(&prow[k], prow_soa, k, L, kind); }
  for (int64_t k = 0; k < (int64_t)nrows * n; k++) { scal_init(&rows[k], prec, kind); scal_get(&rows[k], rows_soa, k, L, kind); }
  double t0 = omp_get_wtime();
#pragma omp parallel num_threads(nthreads)
  {
    scal z, t;
    scal_init(&z, prec, kind);
    scal_init(&t, prec, kind);
#pragma omp for schedule(dynamic, 1)
    for (int r = 0; r < nrows; r++) dso_apply_row(&rows[(size_t)r * n], prow, i, n, collect_minors, &z, &t, kind);
    scal_clear(&z, kind);
    scal_clear(&t, kind);
  }
  double t1 = omp_get_wtime();
  for (int64_t k = 0; k < (int64_t)nrows * n; k++) { scal_put(rows_soa, k, &rows[k], L, kind); scal_clear(&rows[k], kind); }
  for (int k = 0; k < n; k++) scal_clear(&prow[k], kind);
  free(prow); free(rows);
  return t1 - t0;
}

const char *dso_version(void) { return "ds_oracle 1 (MPFR 4.2.1 / MPC 1.3.1, restated elim.py)"; }
