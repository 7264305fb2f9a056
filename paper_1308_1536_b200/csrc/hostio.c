/* hostio.c -- native output path: the reference CLI's result files written
 * straight from the ds SoA results, many files in parallel.
 *
 *   dets.txt        "<i> <det_i>\n" for i = 1..count          (cli.py:218-221)
 *   minors_<m>.txt  "<k+1> <signed_k> <normalized_k | undefined>\n"
 *                   for every emitted size m, k = 0..m-1       (cli.py:224-232)
 *
 * Scalars are formatted exactly like format_scalar (scalars.py:89-104):
 * mpfr_get_str(base 10, `digits` digits, RNDN) -- the call behind gmpy2's
 * mpfr.digits -- then "<sign>0.<digits>e<exp10>", or "<sign>0" when every
 * digit is 0; complex scalars are "<re> <im>".  The Python writer
 * (paper_1308_1536_b200/output.py) restates the same loops over scalar
 * objects; tests/test_output.py checks both byte-for-byte against files the
 * reference wrote.
 */
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#include "mp_abi.h"
#include "../../include/detseries_b200.h"

void dsh_get_soa(mpfr_ptr x, const ds_soa *s, int c, int64_t idx, int L);

typedef struct {
  char *p;
  size_t n, cap;
} obuf;

static int ob_reserve(obuf *b, size_t more) {
  if (b->n + more <= b->cap) return 0;
  size_t cap = b->cap ? b->cap : 1 << 16;
  while (cap < b->n + more) cap *= 2;
  char *q = (char *)realloc(b->p, cap);
  if (!q) return -ENOMEM;
  b->p = q;
  b->cap = cap;
  return 0;
}

/* one real component, format_scalar semantics; dbuf holds digits + 2 bytes */
static void fmt_real(obuf *b, mpfr_ptr x, int digits, char *dbuf) {
  mpfr_exp_t e10 = 0;
  mpfr_get_str(dbuf, &e10, 10, (size_t)digits, x, MPFR_RNDN);
  const char *d = dbuf;
  int neg = 0;
  if (*d == '-') {
    neg = 1;
    d++;
  }
  int allz = 1;
  for (const char *q = d; *q; q++)
    if (*q != '0') {
      allz = 0;
      break;
    }
  size_t dl = strlen(d);
  char *o = b->p + b->n;
  if (neg) *o++ = '-';
  if (allz) {
    *o++ = '0';
  } else {
    *o++ = '0';
    *o++ = '.';
    memcpy(o, d, dl);
    o += dl;
    o += sprintf(o, "e%ld", (long)e10);
  }
  b->n = (size_t)(o - b->p);
}

static void fmt_scalar(obuf *b, mpfr_ptr x, const ds_soa *s, int ncomp, int64_t idx, int L, int digits,
                       char *dbuf) {
  for (int c = 0; c < ncomp; c++) {
    if (c) b->p[b->n++] = ' ';
    dsh_get_soa(x, s, c, idx, L);
    fmt_real(b, x, digits, dbuf);
  }
}

static int write_file(const char *path, const obuf *b) {
  FILE *f = fopen(path, "wb");
  if (!f) return -errno;
  size_t w = fwrite(b->p, 1, b->n, f);
  int rc = (w == b->n) ? 0 : -EIO;
  if (fclose(f) != 0 && rc == 0) rc = -EIO;
  return rc;
}

/* worst-case text bytes of one formatted component */
static size_t comp_bytes(int digits) { return (size_t)digits + 32; }

int dsh_write_dets(const char *path, int count, int kind, int L, long p, const ds_soa *dets, int digits) {
  const int ncomp = kind == DS_KIND_COMPLEX ? 2 : 1;
  obuf b = {0, 0, 0};
  mpfr_t x;
  mpfr_init2(x, p);
  char *dbuf = (char *)malloc((size_t)digits + 2);
  int rc = dbuf ? 0 : -ENOMEM;
  for (int i = 0; i < count && rc == 0; i++) {
    if ((rc = ob_reserve(&b, 24 + ncomp * comp_bytes(digits))) != 0) break;
    b.n += (size_t)sprintf(b.p + b.n, "%d ", i + 1);
    fmt_scalar(&b, x, dets, ncomp, i, L, digits, dbuf);
    b.p[b.n++] = '\n';
  }
  if (rc == 0) rc = write_file(path, &b);
  mpfr_clear(x);
  free(dbuf);
  free(b.p);
  return rc;
}

/* flags[m-1]: 0 = size m not emitted, 1 = emitted with normalized None
 * (leading signed minor zero), 3 = emitted with normalized values.  Row m-1
 * of sig / nrm (count n*n) holds the m entries of size m. */
int dsh_write_minors(const char *outdir, int n, int kind, int L, long p, const ds_soa *sig, const ds_soa *nrm,
                     const uint8_t *flags, int digits, int nthreads) {
  const int ncomp = kind == DS_KIND_COMPLEX ? 2 : 1;
  int err = 0;
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
  {
    obuf b = {0, 0, 0};
    mpfr_t x;
    mpfr_init2(x, p);
    char *dbuf = (char *)malloc((size_t)digits + 2);
    char path[4096];
#pragma omp for schedule(dynamic, 1)
    for (int m = n; m >= 2; m--) {  /* large files first */
      if (!flags[m - 1] || err) continue;
      int rc = dbuf ? 0 : -ENOMEM;
      b.n = 0;
      const int64_t row = (int64_t)(m - 1) * n;
      for (int k = 0; k < m && rc == 0; k++) {
        if ((rc = ob_reserve(&b, 48 + 2 * ncomp * comp_bytes(digits))) != 0) break;
        b.n += (size_t)sprintf(b.p + b.n, "%d ", k + 1);
        fmt_scalar(&b, x, sig, ncomp, row + k, L, digits, dbuf);
        b.p[b.n++] = ' ';
        if (flags[m - 1] == 1) {
          memcpy(b.p + b.n, "undefined", 9);
          b.n += 9;
        } else {
          fmt_scalar(&b, x, nrm, ncomp, row + k, L, digits, dbuf);
        }
        b.p[b.n++] = '\n';
      }
      if (rc == 0) {
        snprintf(path, sizeof(path), "%s/minors_%d.txt", outdir, m);
        rc = write_file(path, &b);
      }
      if (rc != 0) {
#pragma omp critical
        err = rc;
      }
    }
    mpfr_clear(x);
    free(dbuf);
    free(b.p);
  }
  return err;
}

/* ---------------------------------------------------------------- MPMAT
 * MatrixBuffer.save / load (matrix.py:109-140): header
 * "MPMAT 1 <kind> <n> <bits>\n", then the n*n scalars row-major, one per line,
 * format_scalar with its default digits int(bits*log10(2)) + 3 -- the text
 * round-trips bit-exactly through parse_scalar (mpfr from the decimal token,
 * RNDN at bits).  The reference's checkpoints (cli.py:110-120) are this
 * file plus state.txt. */
int mpfr_set_str(mpfr_ptr, const char *, int, mpfr_rnd_t);
void dsh_put_soa(ds_soa *s, int c, int64_t idx, mpfr_srcptr x, int L);

static int default_digits(long p) { return (int)((double)p * 0.30102999566398120) + 3; }

int dsh_write_mpmat(const char *path, int n, int kind, int L, long p, const ds_soa *m, int nthreads) {
  const int ncomp = kind == DS_KIND_COMPLEX ? 2 : 1;
  const int digits = default_digits(p);
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  FILE *f = fopen(path, "wb");
  if (!f) return -errno;
  int rc = fprintf(f, "MPMAT 1 %s %d %ld\n", kind == DS_KIND_COMPLEX ? "complex" : "real", n, p) > 0 ? 0 : -EIO;
  const int64_t total = (int64_t)n * n, chunk = 512;
  const int R = 4 * nthreads;  /* chunks per round */
  obuf *bufs = (obuf *)calloc((size_t)R, sizeof(obuf));
  if (!bufs) rc = -ENOMEM;
  /* rounds of R chunks: formatted in parallel (any thread count), written in order */
  for (int64_t base = 0; base < total && rc == 0; base += (int64_t)R * chunk) {
    int err = 0;
#pragma omp parallel num_threads(nthreads)
    {
      mpfr_t x;
      mpfr_init2(x, p);
      char *dbuf = (char *)malloc((size_t)digits + 2);
#pragma omp for schedule(dynamic, 1)
      for (int c = 0; c < R; c++) {
        obuf *b = &bufs[c];
        b->n = 0;
        const int64_t i0 = base + (int64_t)c * chunk;
        for (int64_t i = i0; i < i0 + chunk && i < total; i++) {
          if (!dbuf || ob_reserve(b, 8 + ncomp * comp_bytes(digits)) != 0) {
#pragma omp critical
            err = -ENOMEM;
            break;
          }
          fmt_scalar(b, x, m, ncomp, i, L, digits, dbuf);
          b->p[b->n++] = '\n';
        }
      }
      mpfr_clear(x);
      free(dbuf);
    }
    for (int c = 0; c < R && !err; c++)
      if (bufs[c].n && fwrite(bufs[c].p, 1, bufs[c].n, f) != bufs[c].n) err = -EIO;
    rc = err;
  }
  for (int q = 0; bufs && q < R; q++) free(bufs[q].p);
  free(bufs);
  if (fclose(f) != 0 && rc == 0) rc = -EIO;
  return rc;
}

/* [-+]?[0-9]+(\.[0-9]+)?([eE][-+]?[0-9]+)?  (scalars.py:32) over [s, e) */
static int real_token_ok(const char *s, const char *e) {
  if (s < e && (*s == '-' || *s == '+')) s++;
  const char *d = s;
  while (s < e && *s >= '0' && *s <= '9') s++;
  if (s == d) return 0;
  if (s < e && *s == '.') {
    s++;
    d = s;
    while (s < e && *s >= '0' && *s <= '9') s++;
    if (s == d) return 0;
  }
  if (s < e && (*s == 'e' || *s == 'E')) {
    s++;
    if (s < e && (*s == '-' || *s == '+')) s++;
    d = s;
    while (s < e && *s >= '0' && *s <= '9') s++;
    if (s == d) return 0;
  }
  return s == e;
}

/* MatrixBuffer.load: parse into `out` (ncomp x L x n*n, caller-allocated for
 * the header values read by dsh_mpmat_header).  Returns 0, -1 malformed
 * header/token, -2 truncated, or -errno. */
int dsh_mpmat_header(const char *path, int *n, int *kind, long *bits) {
  FILE *f = fopen(path, "rb");
  if (!f) return -errno;
  char kbuf[16] = {0};
  int ver = 0;
  int got = fscanf(f, "MPMAT %d %15s %d %ld", &ver, kbuf, n, bits);
  fclose(f);
  if (got != 4 || ver != 1) return -1;
  if (!strcmp(kbuf, "real")) *kind = DS_KIND_REAL;
  else if (!strcmp(kbuf, "complex")) *kind = DS_KIND_COMPLEX;
  else return -1;
  return 0;
}

int dsh_read_mpmat(const char *path, int n, int kind, int L, long p, ds_soa *out, int nthreads) {
  const int ncomp = kind == DS_KIND_COMPLEX ? 2 : 1;
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  FILE *f = fopen(path, "rb");
  if (!f) return -errno;
  if (fseek(f, 0, SEEK_END) != 0) {
    fclose(f);
    return -EIO;
  }
  long sz = ftell(f);
  rewind(f);
  char *buf = (char *)malloc((size_t)sz + 1);
  if (!buf) {
    fclose(f);
    return -ENOMEM;
  }
  size_t rd = fread(buf, 1, (size_t)sz, f);
  fclose(f);
  buf[rd] = 0;
  const int64_t total = (int64_t)n * n;
  char **lines = (char **)malloc(sizeof(char *) * (size_t)(total + 1));
  int rc = lines ? 0 : -ENOMEM;
  /* line starts (first line = header) */
  char *q = strchr(buf, '\n');
  int64_t cnt = 0;
  while (rc == 0 && q && cnt < total) {
    q++;
    if (!*q) break;
    lines[cnt++] = q;
    q = strchr(q, '\n');
  }
  if (rc == 0 && cnt < total) rc = -2;
  if (rc == 0) {
    int err = 0;
#pragma omp parallel num_threads(nthreads)
    {
      mpfr_t x;
      mpfr_init2(x, p);
      char *tok = (char *)malloc(65536);
      size_t tcap = 65536;
#pragma omp for schedule(static)
      for (int64_t i = 0; i < total; i++) {
        if (err) continue;
        char *s = lines[i];
        char *e = strchr(s, '\n');
        if (!e) e = s + strlen(s);
        for (int c = 0; c < ncomp; c++) {
          while (s < e && (*s == ' ' || *s == '\t' || *s == '\r')) s++;
          char *t = s;
          while (t < e && *t != ' ' && *t != '\t' && *t != '\r') t++;
          size_t len = (size_t)(t - s);
          if (!real_token_ok(s, t)) {
#pragma omp critical
            err = -1;
            break;
          }
          if (len + 1 > tcap) {
            char *nt = (char *)realloc(tok, len + 1);
            if (!nt) {
              err = -ENOMEM;
              break;
            }
            tok = nt;
            tcap = len + 1;
          }
          memcpy(tok, s, len);
          tok[len] = 0;
          mpfr_set_str(x, tok, 10, MPFR_RNDN);
          dsh_put_soa(out, c, i, x, L);
          s = t;
        }
        if (!err) {  /* nothing but blanks may follow */
          while (s < e && (*s == ' ' || *s == '\t' || *s == '\r')) s++;
          if (s != e) err = -1;
        }
      }
      mpfr_clear(x);
      free(tok);
    }
    rc = err;
  }
  free(lines);
  free(buf);
  return rc;
}

/* ---- boundary conversion: ds SoA -> mpfr_t (batch) ----------------------
 * Initialise `count` caller-allocated mpfr_t structs at precision p from the
 * SoA elements [start, start + count) of component c (exact copies of the
 * limbs, exponent and sign class).  The Python scalar objects (mp.mpfr) wrap
 * these structs, so one call replaces count per-scalar ctypes round trips
 * when the drop-in eliminate() hands rows to its caller. */
int dsh_soa_to_mpfr(__mpfr_struct *out, const ds_soa *s, int c, int64_t start, int64_t count, int L, long p) {
  for (int64_t k = 0; k < count; k++) {
    mpfr_init2(&out[k], p);
    dsh_get_soa(&out[k], s, c, start + k, L);
  }
  return 0;
}

void mpfr_set_zero(mpfr_ptr, int);

/* Pooled variant: the mpfr_t structs point into one caller-owned limb pool
 * (n64 = ceil(p/64) words per scalar, element-major) instead of a malloc per
 * scalar -- the same representation mpfr_custom_init_set builds (regular
 * numbers: precision, sign, exponent, significand pointer; zeros through
 * mpfr_set_zero).  The Python wrappers keep the pool alive and never call
 * mpfr_clear on these structs. */
int dsh_soa_to_mpfr_pool(__mpfr_struct *out, uint64_t *pool, const ds_soa *s, int c, int64_t start, int64_t count,
                         int L, long p) {
  const int n64 = (int)((p + 63) / 64), pad = 2 * n64 - L;
  const uint32_t *base = s->limbs + (int64_t)c * L * s->count;
  for (int64_t k = 0; k < count; k++) {
    const int64_t idx = start + k;
    __mpfr_struct *x = &out[k];
    uint64_t *d = pool + k * n64;
    x->_mpfr_prec = p;
    x->_mpfr_d = (mp_limb_t *)d;
    const uint8_t cl = s->cls[(int64_t)c * s->count + idx];
    if (cl >= DS_CLS_PZERO) {
      for (int q = 0; q < n64; q++) d[q] = 0;
      mpfr_set_zero(x, cl == DS_CLS_NZERO ? -1 : 1);
      continue;
    }
    for (int q = 0; q < n64; q++) {
      const int l0 = 2 * q - pad, l1 = 2 * q + 1 - pad;
      const uint64_t lo = l0 >= 0 ? base[(int64_t)l0 * s->count + idx] : 0u;
      const uint64_t hi = l1 >= 0 ? base[(int64_t)l1 * s->count + idx] : 0u;
      d[q] = lo | (hi << 32);
    }
    x->_mpfr_exp = s->exp[(int64_t)c * s->count + idx];
    x->_mpfr_sign = cl == DS_CLS_NEG ? -1 : 1;
  }
  return 0;
}

/* Fastest form: the limb pool is already element-major (n64 words per scalar,
 * built by one numpy transpose of the SoA row); only the struct fields are set. */
int dsh_mpfr_structs(__mpfr_struct *out, uint64_t *pool, const int32_t *ex, const uint8_t *cl, int64_t count,
                     int n64, long p) {
  for (int64_t k = 0; k < count; k++) {
    __mpfr_struct *x = &out[k];
    x->_mpfr_prec = p;
    x->_mpfr_d = (mp_limb_t *)(pool + k * n64);
    if (cl[k] >= DS_CLS_PZERO) {
      mpfr_set_zero(x, cl[k] == DS_CLS_NZERO ? -1 : 1);
      continue;
    }
    x->_mpfr_exp = ex[k];
    x->_mpfr_sign = cl[k] == DS_CLS_NEG ? -1 : 1;
  }
  return 0;
}

/* Same, from the plane-major SoA limbs directly: the transpose into the
 * element-major pool (2*n64 words per scalar, the L limbs right-aligned) is done
 * here in 32-element blocks so each block's pool rows stay in L1. */
int dsh_mpfr_structs_planes(__mpfr_struct *out, uint32_t *pool, const uint32_t *limbs, int64_t plane_stride, int L,
                            const int32_t *ex, const uint8_t *cl, int64_t count, int n64, long p) {
  const int W = 2 * n64, pad = W - L;
  if (pad < 0) return -1;
  const int64_t nblk = (count + 31) / 32;
#pragma omp parallel for schedule(static) if (count >= 1024)
  for (int64_t b = 0; b < nblk; b++) {
    const int64_t k0 = b * 32;
    const int64_t nb = count - k0 < 32 ? count - k0 : 32;
    uint32_t *dst = pool + k0 * W;
    for (int64_t kk = 0; kk < nb; kk++)
      for (int j = 0; j < pad; j++) dst[kk * W + j] = 0;
    for (int j = 0; j < L; j++) {
      const uint32_t *src = limbs + (int64_t)j * plane_stride + k0;
      for (int64_t kk = 0; kk < nb; kk++) dst[kk * W + pad + j] = src[kk];
    }
  }
  return dsh_mpfr_structs(out, (uint64_t *)pool, ex, cl, count, n64, p);
}

