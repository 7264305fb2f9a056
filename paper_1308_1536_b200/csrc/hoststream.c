/* hoststream.c -- native consumer of the minors stream (ds_stream_minors) for the
 * drop-in eliminate() (elim.py:158-229, rows reach the sink as they finalise).
 *
 * dsh_rowq_cb is passed to ds_stream_minors as the ds_rows_cb.  It runs on the
 * thread that drives ds_run, holds no Python lock, and turns each delivered batch
 * of plane-major staging rows into ready mpfr_t structs: the limbs of every
 * emitted row are transposed into an element-major pool (n64 words per scalar,
 * the L limbs right-aligned -- the layout MPFR reads) and the struct fields are
 * set, rows in parallel.  The batch is queued; the Python thread pops it
 * (dsh_rowq_pop blocks with the GIL released) and only wraps the structs in
 * scalar objects.  So the device never waits for scalar conversion and the
 * issuing thread never waits for the interpreter.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#include "mp_abi.h"
#include "../../include/detseries_b200.h"

void mpfr_set_zero(mpfr_ptr, int);

typedef struct dsh_rowbatch {
  /* read by the Python side (hostgen.py mirrors the leading fields) */
  int32_t g0, stride, nrows, ncomp;
  int32_t *m;              /* [nrows] leading size of row r, 0 when the row was not emitted */
  uint8_t *flags;          /* [nrows] row_flags (bit0 emitted, bit1 normalized defined) */
  int64_t *off;            /* [nrows] element offset of row r in the struct arrays */
  __mpfr_struct *sg[2];    /* [comp][E] signed minors */
  __mpfr_struct *nm[2];    /* [comp][E] normalized minors (rows with bit1 only) */
  int64_t nel;             /* E */
  /* private */
  uint64_t *pool;
  struct dsh_rowbatch *next;
} dsh_rowbatch;

typedef struct dsh_rowq {
  pthread_mutex_t mu;
  pthread_cond_t cv;
  dsh_rowbatch *head, *tail;
  int closed, failed;
  int n, ncomp, L, n64;
  long prec;
  int nthreads;
} dsh_rowq;

dsh_rowq *dsh_rowq_create(int n, int ncomp, int L, long prec, int nthreads) {
  if (n < 1 || ncomp < 1 || ncomp > 2 || L < 1 || prec < 1) return NULL;
  const int n64 = (int)((prec + 63) / 64);
  if (2 * n64 < L) return NULL;
  dsh_rowq *q = (dsh_rowq *)calloc(1, sizeof(dsh_rowq));
  if (!q) return NULL;
  pthread_mutex_init(&q->mu, NULL);
  pthread_cond_init(&q->cv, NULL);
  q->n = n;
  q->ncomp = ncomp;
  q->L = L;
  q->n64 = n64;
  q->prec = prec;
  q->nthreads = nthreads > 0 ? nthreads : omp_get_max_threads();
  return q;
}

void dsh_rowbatch_free(dsh_rowbatch *b) {
  if (!b) return;
  free(b->m);
  free(b->flags);
  free(b->off);
  for (int c = 0; c < 2; c++) {
    free(b->sg[c]);
    free(b->nm[c]);
  }
  free(b->pool);
  free(b);
}

/* one row of one component of one output: planes [r*n, r*n + m) -> pool + structs */
static void fill_row(const dsh_rowq *q, const ds_soa *s, int c, int64_t cnt, int64_t e0, int m,
                     __mpfr_struct *out, uint64_t *pool) {
  const int L = q->L, W = 2 * q->n64, pad = W - L;
  const uint32_t *limbs = s->limbs + (int64_t)c * L * cnt + e0;
  const int32_t *ex = s->exp + (int64_t)c * cnt + e0;
  const uint8_t *cl = s->cls + (int64_t)c * cnt + e0;
  uint32_t *p32 = (uint32_t *)pool;
  for (int k0 = 0; k0 < m; k0 += 32) {
    const int nb = m - k0 < 32 ? m - k0 : 32;
    uint32_t *dst = p32 + (int64_t)k0 * W;
    for (int kk = 0; kk < nb; kk++)
      for (int j = 0; j < pad; j++) dst[kk * W + j] = 0;
    for (int j = 0; j < L; j++) {
      const uint32_t *src = limbs + (int64_t)j * cnt + k0;
      for (int kk = 0; kk < nb; kk++) dst[kk * W + pad + j] = src[kk];
    }
  }
  for (int k = 0; k < m; k++) {
    __mpfr_struct *x = &out[k];
    x->_mpfr_prec = q->prec;
    x->_mpfr_d = (mp_limb_t *)(pool + (int64_t)k * q->n64);
    if (cl[k] >= DS_CLS_PZERO) {
      mpfr_set_zero(x, cl[k] == DS_CLS_NZERO ? -1 : 1);
      continue;
    }
    x->_mpfr_exp = ex[k];
    x->_mpfr_sign = cl[k] == DS_CLS_NEG ? -1 : 1;
  }
}

/* the ds_rows_cb (include/detseries_b200.h): row r has leading size g0 + r*stride + 1
 * and its entries at [r*n, r*n + m) of the staging SoAs (count = plane stride) */
void dsh_rowq_cb(int g0, int stride, int nrows, const ds_soa *sg, const ds_soa *nm, const uint8_t *flags,
                 void *user) {
  dsh_rowq *q = (dsh_rowq *)user;
  if (!q || nrows <= 0) return;
  dsh_rowbatch *b = (dsh_rowbatch *)calloc(1, sizeof(dsh_rowbatch));
  if (!b) goto oom;
  b->g0 = g0;
  b->stride = stride;
  b->nrows = nrows;
  b->ncomp = q->ncomp;
  b->m = (int32_t *)malloc(sizeof(int32_t) * nrows);
  b->flags = (uint8_t *)malloc(nrows);
  b->off = (int64_t *)malloc(sizeof(int64_t) * nrows);
  if (!b->m || !b->flags || !b->off) goto oom;
  memcpy(b->flags, flags, nrows);
  int64_t E = 0;
  for (int r = 0; r < nrows; r++) {
    b->m[r] = (flags[r] & 1) ? g0 + r * stride + 1 : 0;
    b->off[r] = E;
    E += b->m[r];
  }
  b->nel = E;
  const int nc = q->ncomp;
  const int64_t per = (int64_t)E * q->n64;  /* pool words of one (output, component) */
  if (E > 0) {
    for (int c = 0; c < nc; c++) {
      b->sg[c] = (__mpfr_struct *)malloc(sizeof(__mpfr_struct) * E);
      b->nm[c] = (__mpfr_struct *)malloc(sizeof(__mpfr_struct) * E);
      if (!b->sg[c] || !b->nm[c]) goto oom;
    }
    b->pool = (uint64_t *)malloc(sizeof(uint64_t) * per * 2 * nc);
    if (!b->pool) goto oom;
    const int64_t cnt = sg->count;
    const int tasks = nrows * 2 * nc;
#pragma omp parallel for schedule(dynamic, 1) num_threads(q->nthreads)
    for (int t = 0; t < tasks; t++) {
      const int r = t / (2 * nc), v = (t / nc) & 1, c = t % nc;
      const int m = b->m[r];
      if (m == 0 || (v == 1 && !(b->flags[r] & 2))) continue;
      const int64_t o = b->off[r];
      uint64_t *pool = b->pool + (int64_t)(v * nc + c) * per + o * q->n64;
      fill_row(q, v ? nm : sg, c, cnt, (int64_t)r * q->n, m, (v ? b->nm[c] : b->sg[c]) + o, pool);
    }
  }
  pthread_mutex_lock(&q->mu);
  if (q->tail) q->tail->next = b; else q->head = b;
  q->tail = b;
  pthread_cond_signal(&q->cv);
  pthread_mutex_unlock(&q->mu);
  return;
oom:
  dsh_rowbatch_free(b);
  pthread_mutex_lock(&q->mu);
  q->failed = 1;
  pthread_cond_signal(&q->cv);
  pthread_mutex_unlock(&q->mu);
}

/* producer finished (normally or not): pop returns NULL once the queue is drained */
void dsh_rowq_close(dsh_rowq *q) {
  pthread_mutex_lock(&q->mu);
  q->closed = 1;
  pthread_cond_broadcast(&q->cv);
  pthread_mutex_unlock(&q->mu);
}

/* next batch in delivery order (blocks); NULL when closed and drained.  *failed is
 * set when a batch could not be allocated (the caller raises MemoryError). */
dsh_rowbatch *dsh_rowq_pop(dsh_rowq *q, int *failed) {
  pthread_mutex_lock(&q->mu);
  while (!q->head && !q->closed && !q->failed) pthread_cond_wait(&q->cv, &q->mu);
  dsh_rowbatch *b = q->head;
  if (b) {
    q->head = b->next;
    if (!q->head) q->tail = NULL;
    b->next = NULL;
  }
  if (failed) *failed = q->failed;
  pthread_mutex_unlock(&q->mu);
  return b;
}

void dsh_rowq_destroy(dsh_rowq *q) {
  if (!q) return;
  dsh_rowbatch *b = q->head;
  while (b) {
    dsh_rowbatch *nx = b->next;
    dsh_rowbatch_free(b);
    b = nx;
  }
  pthread_mutex_destroy(&q->mu);
  pthread_cond_destroy(&q->cv);
  free(q);
}
