/*
 * detseries_b200.h -- C ABI of the B200 (sm_100a) hot path of arXiv:1308.1536:
 * arbitrary-precision, unpivoted Gaussian elimination on [A | I] returning all
 * leading principal minors (running product of pivots) and, for every leading
 * size m = 2..n, the signed and normalized minors of column m.
 *
 * The ABI is plain C: pointers, sizes and integer codes, no torch/CUDA types.
 * Each entry point names the reference interface it replaces (paths are
 * relative to the reference package root pkg/src/detseries/).
 *
 * ---------------------------------------------------------------------------
 * Scalar format ("ds SoA").  Precision p bits, L = ceil(p/32) limbs.
 * A real scalar x != 0 is  x = (-1)^s * M * 2^(e - 32L),  M an integer with
 * 2^(32L-1) <= M < 2^(32L) whose low 32L-p bits are zero (the MPFR
 * convention 0.5 <= |x| / 2^e < 1, scalars.py:129-145 canonical form).
 * M is stored as L little-endian 32-bit limbs (limb L-1 holds the MSB).
 * cls holds the sign class, with the same codes as the reference wire
 * format's sign byte (parexec.py:36): 0 = positive, 1 = negative, 2 = +0,
 * 3 = -0.  Zeros have all limbs 0 and e = 0.
 *
 * An array of `count` scalars is structure-of-arrays, limb-plane major:
 *     limbs[(c*L + l)*count + idx],  exp[c*count + idx],  cls[c*count + idx]
 * where c is the component (0 = real part; complex scalars have c = 1 for
 * the imaginary part).  A matrix is count = n*n with idx = row*n + col.
 * ---------------------------------------------------------------------------
 */
#ifndef DETSERIES_B200_H
#define DETSERIES_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes (mapped to detseries.errors by the Python layer) */
#define DS_OK 0
#define DS_ZERO_PIVOT 1          /* errors.ZeroPivot          (errors.py:16-28) */
#define DS_PRECISION_MISMATCH 2  /* errors.PrecisionMismatch  (errors.py:12-13) */
#define DS_INVALID 3             /* ValueError                                   */
#define DS_CUDA 4                /* errors.WorkerFailure      (errors.py:55-60) */
#define DS_NCCL 5                /* errors.WorkerFailure                         */
#define DS_OOM 6                 /* MemoryError                                  */
#define DS_OVERFLOW 7            /* exponent left MPFR's default range           */

#define DS_KIND_REAL 0
#define DS_KIND_COMPLEX 1

#define DS_CLS_POS 0
#define DS_CLS_NEG 1
#define DS_CLS_PZERO 2
#define DS_CLS_NZERO 3

/* MPFR default exponent range (emin/emax = -/+ (2^30 - 1)) */
#define DS_EMAX 1073741823
#define DS_EMIN (-1073741823)

typedef struct ds_soa {
  uint32_t *limbs; /* [ncomp][L][count] */
  int32_t *exp;    /* [ncomp][count]    */
  uint8_t *cls;    /* [ncomp][count]    */
  int64_t count;
} ds_soa;

/* Result buffers of one elimination run (host memory, caller-owned).
 *   pivots, dets : count >= n   (trace.pivots / trace.det_series,
 *                                elim.py:64-89)
 *   signed_minors, normalized : count >= n*n; the minors of leading size m
 *                                live in row m-1, columns 0..m-1
 *                                (MinorRow.signed / .normalized,
 *                                elim.py:92-99)
 *   row_flags[m-1] : bit0 = row m emitted, bit1 = normalized defined
 *                    (normalized is None when signed[0] == 0, elim.py:151-155)
 * Any pointer may be NULL to skip that output. */
typedef struct ds_results {
  ds_soa pivots;
  ds_soa dets;
  ds_soa signed_minors;
  ds_soa normalized;
  uint8_t *row_flags;
} ds_results;

typedef struct ds_ctx ds_ctx;

/* Library version string. */
const char *ds_version(void);

/* Create a context for an n x n elimination at `prec_bits` (>= 64,
 * scalars.py:37-54) of `kind` on CUDA `device`.  The matrix is sharded
 * row-cyclically over `world` ranks and this context holds the rows r with
 * r % world == rank (parexec.py:39-55, WorkerTopology.owner); world = 1 is
 * the serial engine (elim.eliminate, elim.py:158).  Replaces the allocation
 * of MatrixBuffer (matrix.py:24-51) on the device. */
int ds_create(ds_ctx **out, int n, long prec_bits, int kind, int device, int rank,
              int world);
void ds_destroy(ds_ctx *ctx);

/* Row-block context for the panel-paged executor (out-of-core, SURVEY 8(f)
 * rank 4; the reference's blockpager.py:224-241 / 505-529 role): it holds the
 * consecutive rows [row0, row0 + nrows) of an n x n matrix at full width.
 * Steps i < row0 take their (final) pivot row from the host (ds_pivot_load);
 * steps row0 <= i < row0 + nrows stage it from the block (ds_pivot_stage).
 * Every element sees the in-core op sequence, so results are bit-identical
 * (the prefix / left-looking order of elim.py:203-218).  ds_load / ds_fetch /
 * ds_results_fetch take the block's rows (count nrows*n) or the full matrix. */
int ds_create_block(ds_ctx **out, int n, long prec_bits, int kind, int device, int row0, int nrows);
/* Copy a final pivot row (host SoA of count n) into the pivot buffer for step
 * `step` (elim.py:216-218 with prow = rows[step]), instead of ds_pivot_stage. */
int ds_pivot_load(ds_ctx *ctx, int step, const ds_soa *row);

/* Copy the rows this rank owns into HBM.  The host matrix is either the full
 * n x n matrix (count = n*n; global row r at idx r*n + col) or only this
 * rank's rows (count = nloc*n with nloc = #{r < n : r % world == rank}; local
 * row jl = global row rank + jl*world at idx jl*n + col), so a rank of a
 * sharded run never needs host memory for the other ranks' rows.  Replaces
 * the initial row scatter of parexec.py:367-368. */
int ds_load(ds_ctx *ctx, const ds_soa *host_matrix);

/* Copy host rows into HBM like ds_load but keep the run state (det chain,
 * emitted rows, abort flag): a step_hook that edited the in-place buffer
 * mid-run (elim.py:227-228) hands its rows back before the next step. */
int ds_update_rows(ds_ctx *ctx, const ds_soa *host_matrix);

/* Device-side builder (no host matrix): fill this rank's rows with family
 * `family` -- DS_FAMILY_RANDOM_UNIFORM: x = 2U - 1, U a p-bit uniform
 * (genmat.synth_matrix("random_uniform"), genmat.py:242-246) -- drawn from
 * the counter-based "ds-splitmix" generator (element (row, col)
 * is a pure function of seed, row, col and p, so every rank count and the
 * host twin synth.counter_uniform_soa give the same matrix).  The bits differ
 * from gmpy2's Mersenne-twister stream; the distribution is the reference's.
 * Resets the run state like ds_load.  Real matrices only. */
#define DS_FAMILY_RANDOM_UNIFORM 0
int ds_generate(ds_ctx *ctx, int family, uint64_t seed);

/* Copy the rows this rank owns back into a host matrix -- full (count n*n)
 * or owned rows only (count nloc*n), as for ds_load: the in-place L\U state
 * (elim.py:19-22; parexec.py:395-398). */
int ds_fetch(ds_ctx *ctx, ds_soa *host_matrix);

/* Serial engine (world == 1): run pivot steps [start_step, stop_step) of
 * elim.eliminate (elim.py:203-228) entirely on the device, then copy the
 * trace and minors into `res`.  For a resumed run (start_step > 0) res->dets
 * must hold det_series[start_step-1] (elim.py:201).  On an exact zero pivot
 * returns DS_ZERO_PIVOT with *steps_done = the 0-based failing step
 * (ZeroPivot.step - 1, elim.py:209-212) and the partial results copied. */
int ds_run(ds_ctx *ctx, int collect_minors, int series, int start_step, int stop_step,
           ds_results *res, int *steps_done);

/* pivot_mode of elim.eliminate (elim.py:159, 184-208): mode 0 = "none",
 * mode 1 = "partial" -- before each step of ds_run, the first row j >= i of
 * maximal |a_ji| (exact magnitude comparison, elim.py:205) is swapped with
 * row i on the device (elim.py:206-207).  Serial real engine only (world 1,
 * kind real; complex abs() is a rounded modulus); ds_run rejects
 * collect_minors with DS_INVALID (elim.py:186-187). */
int ds_set_pivot_mode(ds_ctx *ctx, int mode);
/* swapped[i] = 1 when step i swapped rows (the det sign flips, elim.py:207,
 * 216), for steps [0, upto_step).  Synchronises the context stream. */
int ds_swaps_fetch(ds_ctx *ctx, int upto_step, uint8_t *swapped);

/* --- sharded engine building blocks (world > 1; the caller broadcasts) ---
 * Per step i: the owner of row i calls ds_pivot_stage (copies the
 * unnormalized row i into the pivot buffer: parexec.py:307-309), every rank
 * broadcasts the pivot buffer from that owner (ncclBroadcast through
 * torch.distributed), then every rank calls ds_step (det chain, update of
 * its own rows, minor emission for the row it owns: parexec.py:312-325). */
int ds_pivot_buffer(ds_ctx *ctx, void **device_ptr, size_t *bytes);
int ds_pivot_stage(ds_ctx *ctx, int step);
int ds_step(ds_ctx *ctx, int step, int collect_minors, int series);
/* Status of the device abort flag: *failed_step = -1 when no zero pivot was
 * seen, else the 0-based step.  Synchronises the context stream. */
int ds_status(ds_ctx *ctx, int *failed_step);
/* Copy trace (replicated on every rank) and the minors rows this rank owns
 * (row m-1 owned when (m-1) % world == rank) into `res`; the minors buffers
 * are full (count n*n) or owned rows only (count nloc*n), as for ds_load. */
int ds_results_fetch(ds_ctx *ctx, int upto_step, ds_results *res);
/* Incremental form of ds_results_fetch for a serial context (world 1):
 * trace entries [t0, t1) (pivots / det_series) and the minors rows of leading
 * sizes [m0, m1) (row m-1, its first m entries, plus row_flags[m-1]) into the
 * same positions of `res` (counts n and n*n).  Lets the drop-in eliminate()
 * hand each MinorRow to its sink as the row finalises (elim.py:220-226)
 * instead of after the whole run.  Synchronises the context streams. */
int ds_results_fetch_range(ds_ctx *ctx, int t0, int t1, int m0, int m1, ds_results *res);
/* Streaming of the minors rows to the host (the output
 * volume equals the matrix, ~416 GB at config 5, so it cannot stay resident).
 * After ds_stream_minors(ctx, batch_steps, cb, user) the context keeps only a
 * ring of minors rows in HBM (3 flush intervals) and every flush -- ds_run
 * calls it every batch_steps steps and at its end, a multi-rank driver calls
 * it itself at least every batch_steps steps -- copies the owned rows
 * finalised since the previous flush into pinned staging on the side stream
 * and hands the PREVIOUS batch to cb (so the copy overlaps the caller's
 * work).  cb(g0, stride, nrows, signed, normalized, flags, user): rows of
 * leading sizes m_r = g0 + r*stride + 1 (r < nrows; g is the global row,
 * stride = world) hold their m_r entries at [r*n, r*n + m_r) of signed /
 * normalized (ds SoA, valid only during the call); flags[r] = row_flags of
 * that size (bit0 emitted, bit1 normalized defined).  Rows arrive in
 * increasing size, like sink calls (elim.py:220-226).  batch_steps <= 0 turns
 * streaming off (minors resident again, fetched by ds_results_fetch).
 * final = 1 waits for and delivers everything up to upto_step. */
typedef void (*ds_rows_cb)(int g0, int stride, int nrows, const ds_soa *signed_rows,
                           const ds_soa *normalized_rows, const uint8_t *flags, void *user);
int ds_stream_minors(ds_ctx *ctx, int batch_steps, ds_rows_cb cb, void *user);
int ds_stream_flush(ds_ctx *ctx, int upto_step, int final);
/* Seed the device det chain (resume, elim.py:201): det = host scalar. */
int ds_set_det(ds_ctx *ctx, const ds_soa *det1);

/* CUDA stream the context launches on (cudaStream_t as void*). */
void *ds_stream(ds_ctx *ctx);
/* Launch on the caller's stream from now on (e.g. torch's current stream, so
 * the NCCL broadcast of the pivot buffer is stream-ordered with the kernels
 * without host synchronisation).  NULL restores the context's own stream. */
int ds_set_stream(ds_ctx *ctx, void *stream);
/* Use caller-owned device memory of >= the ds_pivot_buffer size as the
 * pivot buffer (e.g. a torch tensor that torch.distributed broadcasts in
 * place).  NULL restores the internal buffer. */
int ds_use_pivot_buffer(ds_ctx *ctx, void *device_ptr, size_t bytes);
/* In-process broadcast for virtual shards (par_eliminate transport="local"):
 * copy src's pivot buffer into dst's, ordered after src's pending work. */
int ds_pivot_copy(ds_ctx *dst, ds_ctx *src);
/* Number of kernel launches issued by this context since creation. */
int64_t ds_launch_count(ds_ctx *ctx);
/* Device-side snapshot of this rank's rows: save = 1 copies them to a
 * backup buffer in HBM, save = 0 restores them and resets the run state
 * (abort flag, det chain, emitted-row flags).  Lets a caller re-run the
 * elimination on resident inputs (benchmarks, checkpoint/resume). */
int ds_snapshot(ds_ctx *ctx, int save);
/* Update-kernel profiling: while enabled, every update launch (digit prep +
 * fused update) is bracketed by CUDA events on the context stream.
 * ds_profile_read synchronises, returns the summed kernel time (ms), the
 * number of launches and their algorithmic work in schoolbook limb-MACs
 * (rows * cols * L^2, x4 for complex), then clears the counters. */
int ds_profile(ds_ctx *ctx, int enable);
int ds_profile_read(ds_ctx *ctx, double *update_ms, int64_t *launches, double *limb_macs);
/* Multi-rank lookahead (one process per GPU): with ds_lookahead_enable(ctx,
 * limit) the TC update of step i (i + 1 < limit) runs the column tile that
 * holds column i+1 first, on the context's lookahead stream
 * (ds_lookahead_stream).  The caller then, on that stream: lets the owner of
 * row i+1 stage a_{i+1,i+1} into a (4L + 8)-byte exchange buffer
 * (ds_lookahead_pivot), broadcasts the buffer from that owner, and launches
 * step i+1's multipliers from it (ds_lookahead_mult); ds_step(i+1) then uses
 * them.  Same results as without lookahead; parexec.py:290-333 exchange
 * order is kept (every rank issues the same broadcasts in the same order).
 * limit <= 0 disables. */
int ds_lookahead_enable(ds_ctx *ctx, int limit);
int ds_lookahead_stream(ds_ctx *ctx, void **stream);
int ds_lookahead_pivot(ds_ctx *ctx, int i1, void *buf);
int ds_lookahead_mult(ds_ctx *ctx, int i1, const void *buf);

/* Internal engine counters (observability; no reference counterpart):
 * out[0] = elements the tensor-core update handed to the exact fallback
 * (short product undecided / normalisation uncertain), out[1] = 1 if the
 * tensor-core update engine is active, out[2] = 1 if the DFMA engine is,
 * out[3] = elements whose predicted normalisation (single-pass rounding) was
 * wrong and which went to the exact fallback, out[4] / out[5] = bytes copied
 * host->device / device->host by this context's ABI calls since creation
 * (ds_load, ds_fetch, results; the e2e accounting).  Writes min(n, 6) values. */
int ds_counters(ds_ctx *ctx, int64_t *out, int n);

/* Last error message of this context (or of the last failed ds_create when
 * ctx is NULL). */
const char *ds_last_error(ds_ctx *ctx);

/* ---- correctly-rounded scalar kernels (conformance surface) ----
 * Element-wise RN(a op b) over `count` real (kind 0) or complex (kind 1)
 * scalars at precision prec_bits, computed on `device`.  op: 0 = mul,
 * 1 = sub, 2 = div, 3 = add.  Host buffers.  These are the device routines
 * k_update / k_mult / k_emit use; they stand in for mpfr_mul/sub/div and
 * mpc_mul/sub/div. */
int ds_scalar_op(int op, int kind, long prec_bits, int device, const ds_soa *a,
                 const ds_soa *b, ds_soa *out);

#ifdef __cplusplus
}
#endif

#endif /* DETSERIES_B200_H */
