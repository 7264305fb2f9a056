// ds_update.cu -- fused real update kernel of the elimination step
// (elim.py:49-52; the reference's hot loop):
//
//     a_jk <- RN_p( a_jk - RN_p( z_j * b_k ) )      for this rank's rows j > i,
//                                                   all columns k != i
//
// Two roundings per element, exactly as mpfr_mul then mpfr_sub; the fusion is
// of memory traffic only, never of numerics.
//
// B200 mapping.  B200 has a full-rate FP64 pipe (64 DFMA/clk/SM, measured in
// tools/microbench/imad_tput.cu) next to the INT32 IMAD pipe, whose 32x32->64
// carry chains reach only ~18 limb-products/clk/SM.  A DFMA is an EXACT
// multiply-accumulate of balanced 24-bit digits (|d| <= 2^23, |d*d'| <= 2^46)
// as long as an accumulator stays below 2^53, so the mantissa product runs on
// the FP64 pipe at 576 bit^2 per instruction:
//   * prep kernels convert z_j (per row) and b_k (per pivot-row column) once
//     per step into balanced radix-2^24 digits held as doubles (O(p) each);
//   * the CTA stages TR rows of z digits and TC = 32 columns of b digits in
//     shared memory (one warp = 32 consecutive columns of one row: z digits are
//     warp broadcasts, b digits consecutive 8-byte words);
//   * each thread owns one element and computes its product by column blocks
//     of W output digits with a register-rotated sliding window of b digits:
//     per s-step 1 broadcast LDS + 1 LDS + W independent DFMAs, carries flushed
//     every 64 steps (exactness bound |acc| < 2^53);
//   * SHORT PRODUCT: only digit columns >= c_lo = floor((p-2)/24) - 4 are
//     computed (~p^2/1152 DFMAs instead of p^2/576).  The omitted low part is
//     bounded, |E| < Db * 2^22 units of 2^(24 c_lo); if the computed bits
//     between 24 c_lo + eps and the round bit are neither all-zero nor
//     all-one, the rounding of z*b is provably decided (inc = round bit);
//     otherwise the element recomputes the FULL product (exact round/sticky).
//     Probability of the fallback on non-exact data ~2^-60;
//   * digits stream low -> high into the rounded p-bit t, which streams into
//     the exact aligned a -/+ t window (guard limb + sticky, borrow trick),
//     written in place into a's own limb slots; a final pass normalises,
//     rounds to nearest-even and writes the result.  No scratch memory.
// Normalisation of z*b (top bit at 2p-1 or 2p-2) is predicted from the
// leading 64 bits of each operand and only trusted with a 2^-43 margin; the
// rare undecided case runs an exact dry product first.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <string>

#include "../../include/detseries_b200.h"
#include "ds_mp.cuh"
#include "ds_update.cuh"
#include "ds_stream.cuh"

namespace {

using namespace dss;

constexpr int TC = 32;        // columns per CTA (one warp row)
constexpr int GUARD = 4;      // guard digits of the short product
constexpr int FLUSH = 64;     // s-steps between carry flushes (64 * 2^46 < 2^53)
constexpr double R24 = 1.0 / 16777216.0;
constexpr double B24 = 16777216.0;

// Generic fused product / update over a tile of (rows r) x (columns c):
//   mode 0 (update): out[r,c] <- RN(out[r,c] - RN(z_r * b_c))   (elim.py:50-52)
//   mode 1 (mul)   : out[r,c] <- RN(z_r * b_c)                  (elim.py:59, 214)
// z_r: digits zdig[r*Db + s], meta zexp/zcls/zf[r]
// b_c: column k = bmap(c): digits bdig[s*bstride + k], meta bexp/bcls/bf[k]
// out: element index (orow0 + r) * ostride + ocol(c), limb planes o_count apart
struct UArgs {
  int p, L, Db, zb, mode;
  int nrows, ncols;
  int c_lo, cmax, eps;
  const double* zdig;
  const double* zf;
  const int32_t* zexp;
  const uint8_t* zcls;
  const double* bdig;
  const double* bf;
  const int32_t* bexp;
  const uint8_t* bcls;
  int64_t bstride;
  int col_off;   // k = c + col_off
  int skip_col;  // column k == skip_col is left untouched (the pivot column)
  int ocol_off;  // output column = (o_same ? k : c + ocol_off)
  int o_same;
  uint32_t* o_limbs;
  int32_t* o_exp;
  uint8_t* o_cls;
  int64_t o_count, ostride, orow0;
  int32_t* status;
  int step;  // skip when a zero pivot was seen at a step <= this one
};

__device__ __forceinline__ void cp_async4(uint32_t* smem_dst, const uint32_t* gsrc) {
  unsigned int d = (unsigned int)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc));
}
// 8-byte async copy with zero fill when !valid (src-size 0)
__device__ __forceinline__ void cp_async8z(double* smem_dst, const double* gsrc, bool valid) {
  unsigned int d = (unsigned int)__cvta_generic_to_shared(smem_dst);
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(n));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// ------------------------------------------------------------ prep kernels
// Balanced radix-2^24 digits of the p-bit integer mantissa m = M >> (32L-p):
// with u_s the unsigned 24-bit digits and c_s = [u_{s-1} >= 2^23],
//     d_s = u_s + c_s - 2^24 [u_s >= 2^23]   in [-2^23, 2^23],
// which telescopes to sum d_s 2^(24s) = m with no carry chain, so every
// digit is computed independently (one thread per (element, digit)).
// Element e (limbs src[e + l*count]) -> dig[e*es + s*ds]; topf[e] = leading
// 64 bits as a double in [1, 2).
__device__ __forceinline__ uint32_t udigit(ds::CPtr M, int L, int p, int zb, int s) {
  if (s < 0 || 24 * s >= p) return 0u;
  return ds::bits32(M, L, (int64_t)24 * s + zb) & 0xFFFFFFu;
}

__global__ void k_prep_digits(const uint32_t* src, int64_t count, int64_t num, int L, int p, int Db, double* dig,
                              int64_t es, int64_t ds_, double* topf) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= num * Db) return;
  // consecutive threads -> consecutive elements when ds_ == 1 is not the
  // layout: choose the mapping that makes the digit stores coalesced
  int64_t e, s;
  if (es == 1) {  // dig[s*ds + e]: element-fastest
    e = t % num;
    s = t / num;
  } else {        // dig[e*es + s]: digit-fastest
    e = t / Db;
    s = t % Db;
  }
  ds::CPtr M{src + e, count};
  int zb = 32 * L - p;
  uint32_t u = udigit(M, L, p, zb, (int)s);
  uint32_t up = udigit(M, L, p, zb, (int)s - 1);
  int d = (int)u + (up >= (1u << 23) ? 1 : 0) - (u >= (1u << 23) ? (1 << 24) : 0);
  dig[e * es + s * ds_] = (double)d;
  if (s == 0) {
    uint64_t top = ((uint64_t)M[L - 1] << 32) | M[L - 2];
    topf[e] = (double)top * 0x1p-63;
  }
}

static inline void prep_launch(const uint32_t* src, int64_t count, int64_t num, int L, int p, int Db, double* dig,
                               int64_t es, int64_t ds_, double* topf, cudaStream_t s) {
  int64_t tot = num * Db;
  k_prep_digits<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(src, count, num, L, p, Db, dig, es, ds_, topf);
}

// ------------------------------------------------------------ the product
// Accumulators of output digit columns [c0, c0+W) (+ the overflow slot acc[W])
// of P = sum_c col_c 2^(24c), col_c = sum_{s+t=c} z_s b_t, starting from zero.
// z digits zrow[s] (padded by W zeros), b digits bcol[(t + 2W) * BS]
// (padded by 2W below and W above).  Every partial sum is an exact integer
// below 2^53 (carries flushed every FLUSH steps).
template <int W, int BS>
__device__ __forceinline__ void block_accumulate(const double* __restrict__ zrow, const double* __restrict__ bcol,
                                                 int Db, int c0, double (&acc)[W + 1]) {
#pragma unroll
  for (int w = 0; w <= W; w++) acc[w] = 0.0;
  int s_lo = c0 - (Db - 1);
  if (s_lo < 0) s_lo = 0;
  int s_hi = c0 + W - 1;
  if (s_hi > Db - 1) s_hi = Db - 1;
  if (s_lo > s_hi) return;
  double ph[W];
#pragma unroll
  for (int w = 0; w < W; w++) ph[w] = bcol[(c0 + w - s_lo + 2 * W) * BS];
  int ngroups = (s_hi - s_lo + W) / W;
  int s = s_lo;
  for (int g = 0; g < ngroups; g++) {
#pragma unroll
    for (int u = 0; u < W; u++) {
      double zv = zrow[s + u];
#pragma unroll
      for (int w = 0; w < W; w++) acc[w] = fma(zv, ph[(w - u + W) % W], acc[w]);
      ph[(2 * W - 1 - u) % W] = bcol[(c0 - (s + u) - 1 + 2 * W) * BS];
    }
    s += W;
    if (((g + 1) & (FLUSH / W - 1)) == 0) {
#pragma unroll
      for (int w = 0; w < W; w++) {
        double q = rint(acc[w] * R24);
        acc[w] = fma(-q, B24, acc[w]);
        acc[w + 1] += q;
      }
    }
  }
}

// Final normalisation of one block (c0 = 0 mod 4) with the incoming carry;
// packs the W nonnegative 24-bit digits into 3W/4 whole limbs of P (limb
// index 3*c0/4) and feeds them to `cons`; false if the consumer aborted.
template <int W, class C>
__device__ __forceinline__ bool block_emit(double (&acc)[W + 1], double& carry, int c0, C& cons) {
  acc[0] += carry;
  uint32_t dg[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    double q = floor(acc[w] * R24);
    acc[w] = fma(-q, B24, acc[w]);
    acc[w + 1] += q;
    dg[w] = (uint32_t)(int)acc[w];
  }
  carry = acc[W];
  const int g0 = (3 * c0) >> 2;
  uint32_t P[3 * W / 4];
#pragma unroll
  for (int k = 0; k < W / 4; k++) {
    uint32_t d0 = dg[4 * k], d1 = dg[4 * k + 1], d2 = dg[4 * k + 2], d3 = dg[4 * k + 3];
    P[3 * k] = d0 | (d1 << 24);
    P[3 * k + 1] = (d1 >> 8) | (d2 << 16);
    P[3 * k + 2] = (d2 >> 16) | (d3 << 8);
  }
  return cons.block(g0, P);
}

// P = sum_c col_c 2^(24c) for columns c >= c_start, streamed low -> high as
// nonnegative digits to `cons` (one thread).
template <int W, int BS, class C>
__device__ __forceinline__ bool product(const double* __restrict__ zrow, const double* __restrict__ bcol, int Db,
                                        int c_start, int cmax, C& cons) {
  double carry = 0.0;
  for (int c0 = c_start; c0 <= cmax; c0 += W) {
    double acc[W + 1];
    block_accumulate<W, BS>(zrow, bcol, Db, c0, acc);
    if (!block_emit<W>(acc, carry, c0, cons)) return false;
  }
  return cons.finish(carry);
}

// ------------------------------------------------------------ element
// The whole element: sign/zero logic, normalisation prediction, product
// (short, exact fallback), streamed rounding into the S window, final RN.
// SPLIT: lanes of the warp compute disjoint column blocks in parallel and
// lane 0 consumes them (pure products of the det chain / minors emission).
template <int W, int BS, bool SPLIT>
__device__ void fused_element(const UArgs& a, const double* zrow, const double* bcol, uint32_t* Sw, int nth, int r,
                              int k, int64_t oidx, double* blk) {
  const int L = a.L, p = a.p;
  uint8_t cz = a.zcls[r];
  uint8_t cb = a.bcls[k];
  int st = (cz & 1) ^ (cb & 1);
  bool mul = a.mode == 1;
  uint8_t ca = mul ? DS_CLS_PZERO : a.o_cls[oidx];
  bool za = ca >= DS_CLS_PZERO;
  int sa = ca & 1;
  if (cz >= DS_CLS_PZERO || cb >= DS_CLS_PZERO) {  // t = (-1)^st 0
    if (mul) {
      for (int l = 0; l < L; l++) a.o_limbs[(int64_t)l * a.o_count + oidx] = 0u;
      a.o_exp[oidx] = 0;
      a.o_cls[oidx] = st ? DS_CLS_NZERO : DS_CLS_PZERO;
      return;
    }
    if (!za) return;  // a - 0 = a
    a.o_cls[oidx] = (sa && !st) ? DS_CLS_NZERO : DS_CLS_PZERO;
    return;
  }
  int32_t ea = za ? 0 : a.o_exp[oidx];
  double pr = a.zf[r] * a.bf[k];
  int norm = pr >= 2.0 ? 1 : 0;
  bool confident = fabs(pr - 2.0) > 0x1p-42;
  int64_t ebase = (int64_t)a.zexp[r] + a.bexp[k];
  if (!za && (int64_t)ea - (ebase - 1) >= (int64_t)p + 3) return;  // a dominates whatever the norm
  if (!confident) {
    DryTop dt;
    dt.bitpos = 2 * p - 1;
    dt.top = 0;
    if (!SPLIT || (threadIdx.x & 31) == 0) product<W, BS>(zrow, bcol, a.Db, 0, a.cmax, dt);
    norm = dt.top;
    if (SPLIT) norm = __shfl_sync(0xffffffffu, norm, 0);
  }
  int64_t et = ebase - (norm ? 0 : 1);
  int64_t d = za ? -(int64_t)(1 << 30) : (int64_t)ea - et;
  if (!za && d >= (int64_t)p + 2) return;  // RN(a - t) = a
  bool xa = !za && d >= 0;
  bool sub = !za && (sa == st);           // a + (-t): magnitudes subtract iff sign(a) == sign(t)
  int neg = mul ? st : (xa ? sa : (st ^ 1));
  int64_t E = xa ? ea : et;

  const int lane = threadIdx.x & 31;
  SWin S;
  S.base(Sw, nth);
  Emit em;
  bool done = false;
  for (int attempt = 0; attempt < 2 && !done; attempt++) {
    bool exact = attempt == 1 || a.c_lo == 0;
    if (!SPLIT || lane == 0) S.init(L, xa, sub, za, xa ? d : (za ? 0 : -d));
    em.S = &S;
    em.r = norm ? p : p - 1;
    em.zb = a.zb; em.p = p; em.L = L;
    em.exact = exact;
    em.onesided = false;
    em.lo_chk = 24 * a.c_lo + a.eps;
    em.hi_chk = em.r - 2;
    em.allz = true; em.allo = true; em.sticky = false; em.decided = false;
    em.rbit = 0; em.tcarry = 0; em.tl = 0; em.excess = false;
    em.setup<3 * W / 4>();
    if (SPLIT && !exact) {
      // lanes accumulate disjoint column blocks; lane 0 normalises and rounds
      const int c_start = a.c_lo;
      const int nb = (a.cmax - c_start) / W + 1;
      for (int b = lane; b < nb; b += 32) {
        double acc[W + 1];
        block_accumulate<W, BS>(zrow, bcol, a.Db, c_start + b * W, acc);
#pragma unroll
        for (int w = 0; w <= W; w++) blk[b * (W + 1) + w] = acc[w];
      }
      __syncwarp();
      bool ok = true;
      if (lane == 0) {
        double carry = 0.0;
        for (int b = 0; b < nb && ok; b++) {
          double acc[W + 1];
#pragma unroll
          for (int w = 0; w <= W; w++) acc[w] = blk[b * (W + 1) + w];
          ok = block_emit<W>(acc, carry, c_start + b * W, em);
        }
        if (ok) ok = em.finish(carry);
      }
      done = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
    } else {
      if (!SPLIT || lane == 0) done = product<W, BS>(zrow, bcol, a.Db, exact ? 0 : a.c_lo, a.cmax, em);
      if (SPLIT) done = __shfl_sync(0xffffffffu, done ? 1 : 0, 0) != 0;
    }
  }
  if (SPLIT && lane != 0) return;
  if (em.excess) atomicAdd(&a.status[4], 1);  // normalisation misprediction (must never happen)

  round_write(S, neg, E, L, p, a.zb, a.o_limbs + oidx, a.o_count, a.o_exp + oidx, a.o_cls + oidx, a.status);
}

template <int W, int TCc>
__global__ void __launch_bounds__(256) k_fused(UArgs a, int TR) {
  extern __shared__ double sm[];
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  const int Db = a.Db, L = a.L;
  const int ZP = Db + W;
  const int BP = Db + 3 * W;
  double* zs = sm;
  double* bs = sm + TR * ZP;
  uint32_t* Sw = (uint32_t*)(bs + BP * TCc);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int col0 = blockIdx.x * TCc, row0 = blockIdx.y * TR;
  const int tid = ty * TCc + tx, nth = TCc * TR;
  const int r = row0 + ty, cc = col0 + tx;
  const bool active = r < a.nrows && cc < a.ncols && (cc + a.col_off) != a.skip_col;
  const int k = cc + a.col_off;
  const int64_t oidx = (a.orow0 + r) * a.ostride + (a.o_same ? k : cc + a.ocol_off);
  // prefetch a's limbs into the S window (slots 1..L) while the operands stage
  if (a.mode == 0 && active) {
    const uint32_t* A = a.o_limbs + oidx;
    for (int l = 0; l < L; l++) cp_async4(Sw + (l + 1) * nth + tid, A + (int64_t)l * a.o_count);
  }
  {  // operand staging: warp ty loads z row ty; b digits column tx, rows strided by TR
    const bool zrow_ok = row0 + ty < a.nrows;
    const double* zsrc = a.zdig + (int64_t)(zrow_ok ? row0 + ty : 0) * Db;
    for (int s = tx; s < ZP; s += TCc) cp_async8z(zs + ty * ZP + s, zsrc + (s < Db ? s : 0), zrow_ok && s < Db);
    const bool col_ok = col0 + tx < a.ncols;
    const double* bsrc = a.bdig + (col_ok ? col0 + tx + a.col_off : 0);
    for (int tt = ty; tt < BP; tt += TR) {
      int t = tt - 2 * W;
      bool ok = col_ok && t >= 0 && t < Db;
      cp_async8z(bs + tt * TCc + tx, bsrc + (int64_t)(ok ? t : 0) * a.bstride, ok);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (!active) return;
  fused_element<W, TCc, false>(a, zs + ty * ZP, bs + tx, Sw + tid, nth, r, k, oidx, nullptr);
}

// One warp per product (mode 1): the det chain (1 element per step, on the
// critical path) and the signed-minor row (i+1 elements).
template <int W>
__global__ void __launch_bounds__(128) k_mul_split(UArgs a, int nbs) {
  extern __shared__ double sm[];
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  const int Db = a.Db, L = a.L;
  const int WPB = blockDim.x >> 5;
  const int ZP = Db + W, BP = Db + 3 * W;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xs = sm;
  double* ys = xs + ZP + (ZP & 1);
  double* blk = ys + WPB * BP;
  uint32_t* Sw = (uint32_t*)(blk + WPB * nbs * (W + 1));
  for (int e = threadIdx.x; e < ZP; e += blockDim.x) xs[e] = e < Db ? a.zdig[e] : 0.0;
  const int c = blockIdx.x * WPB + warp;
  double* yw = ys + warp * BP;
  for (int tt = lane; tt < BP; tt += 32) {
    int t = tt - 2 * W;
    yw[tt] = (c < a.ncols && t >= 0 && t < Db) ? a.bdig[(int64_t)t * a.bstride + c + a.col_off] : 0.0;
  }
  __syncthreads();
  if (c >= a.ncols) return;
  const int k = c + a.col_off;
  const int64_t oidx = a.orow0 * a.ostride + (a.o_same ? k : c + a.ocol_off);
  fused_element<W, 1, true>(a, xs, yw, Sw + warp * (L + 2), 1, 0, k, oidx, blk + warp * nbs * (W + 1));
}

// highest digit column of z*b that can be nonzero: P < 2^(2p) needs columns
// <= (2p-1)/24, but when p = 0 mod 24 the balanced top digit d_{D-1} (the
// borrow of u_{D-2} >= 2^23) can be 1 and its column 2D-2 must be summed too
// (it cancels the -1 carry out of the column below).
static int top_column(int p) {
  int D = (p + 23) / 24 + 1;
  return p % 24 == 0 ? 2 * D - 2 : (2 * p - 1) / 24;
}

static int split_smem(int W, int Db, int L, int cmax, int c_lo, int wpb) {
  int nbs = (cmax - c_lo) / W + 1;
  return 8 * ((Db + W + 1) + wpb * (Db + 3 * W) + wpb * nbs * (W + 1)) + 4 * wpb * (L + 2);
}

int fused_smem(int W, int TR, int Db, int L, int tc = TC) {
  return 8 * (TR * (Db + W) + (Db + 3 * W) * tc) + 4 * (L + 2) * TR * tc;
}

std::string g_err;

}  // namespace

// ---------------------------------------------------------------- host API
struct UpdateWork {
  double* zdig;   // [nloc][Db] multipliers of the current step
  double* bdig;   // [Db][n] pivot row
  double* zf;
  double* bf;
  double* ddig;   // [Db] det
  double* df;
  double* edig;   // [Db][n] row i+1 (minors emission)
  double* ef;
  int nloc;
};

// per-context side-stream workspaces for mul_row_launch: digits + topf
size_t mul_ws_doubles(const UpdatePlan* plan, int count) { return (size_t)plan->D * count + count + 8; }

static int pick_tr(int W, int Db, int L, int maxsm) {
  int TR = 8;
  while (TR > 1 && fused_smem(W, TR, Db, L) > maxsm) TR /= 2;
  return fused_smem(W, TR, Db, L) <= maxsm ? TR : 0;
}

int update_plan_init(UpdatePlan* plan, int n, int p, int device) {
  plan->enabled = 0;
  plan->fused = 0;
  plan->n = n;
  plan->p = p;
  plan->L = (p + 31) / 32;
  plan->D = (p + 23) / 24 + 1;
  plan->device = device;
  plan->workspace = nullptr;
  if (getenv("DS_DISABLE_DFMA")) return DS_OK;
  int W = plan->D <= 24 ? 8 : 16;  // W = 32 measured slower (corner waste (W-1)/Db)
  if (const char* ew = getenv("DS_FUSED_W")) {  // tuning override: 8 / 16 / 32
    int w = atoi(ew);
    if (w == 8 || w == 16 || w == 32) W = w;
  }
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int TR = pick_tr(W, plan->D, plan->L, maxsm);
  int tc = TC;
  if (TR == 0) {  // wide precisions (~16K bits): 16-column CTAs with fewer rows
    tc = 16;
    TR = 8;
    while (TR > 1 && fused_smem(W, TR, plan->D, plan->L, 16) > maxsm) TR /= 2;
    // too wide for one CTA: no fused update (the wide tensor-core engine or the
    // general engine updates), the row products still run here
    if (fused_smem(W, TR, plan->D, plan->L, 16) > maxsm) TR = 0;
  }
  int smsm = 0;  // shared memory per SM
  cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  // two independent 16-column CTAs per SM desynchronise the warps' epilogues
  // (one 256-thread CTA runs all its warps in lockstep phases)
  if (TR && fused_smem(W, 8, plan->D, plan->L, 16) * 2 + 2048 <= smsm && !getenv("DS_FUSED_TC32")) {
    tc = 16;
    TR = 8;
  }
  plan->w = W;
  plan->tr = TR;
  plan->tc = tc;
  plan->smem = fused_smem(W, TR, plan->D, plan->L, tc);
  cudaDeviceGetAttribute(&plan->sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e1 = cudaFuncSetAttribute(k_fused<8, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  if (e1 == cudaSuccess) e1 = cudaFuncSetAttribute(k_fused<8, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  cudaError_t e2 = cudaFuncSetAttribute(k_fused<16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  if (e2 == cudaSuccess) e2 = cudaFuncSetAttribute(k_fused<16, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  if (e2 == cudaSuccess) e2 = cudaFuncSetAttribute(k_fused<32, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  cudaError_t e3 = cudaFuncSetAttribute(k_mul_split<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) return DS_CUDA;
  {
    int clo = ((p - 2) / 24 - GUARD) & ~3;
    if (clo < 0) clo = 0;
    if (split_smem(4, plan->D, plan->L, top_column(p), clo, 4) > maxsm) return DS_OK;
  }
  plan->fused = TR > 0 ? 1 : 0;
  plan->enabled = 1;
  return DS_OK;
}

void update_plan_free(UpdatePlan* plan) {
  if (plan->workspace) {
    UpdateWork* w = (UpdateWork*)plan->workspace;
    double* ptrs[] = {w->zdig, w->bdig, w->zf, w->bf, w->ddig, w->df, w->edig, w->ef};
    for (double* q : ptrs)
      if (q) cudaFree(q);
    delete w;
    plan->workspace = nullptr;
  }
}

static int ensure_work(UpdatePlan* plan, int nloc) {
  if (plan->workspace) return DS_OK;
  UpdateWork* w = new UpdateWork();
  memset(w, 0, sizeof(*w));
  w->nloc = nloc;
  size_t D = plan->D, nl = nloc > 0 ? nloc : 1, n = plan->n;
  bool ok = cudaMalloc(&w->zdig, sizeof(double) * D * nl) == cudaSuccess &&
            cudaMalloc(&w->bdig, sizeof(double) * D * n) == cudaSuccess &&
            cudaMalloc(&w->zf, sizeof(double) * nl) == cudaSuccess &&
            cudaMalloc(&w->bf, sizeof(double) * n) == cudaSuccess &&
            cudaMalloc(&w->ddig, sizeof(double) * D) == cudaSuccess &&
            cudaMalloc(&w->df, sizeof(double) * 1) == cudaSuccess &&
            cudaMalloc(&w->edig, sizeof(double) * D * n) == cudaSuccess &&
            cudaMalloc(&w->ef, sizeof(double) * n) == cudaSuccess;
  plan->workspace = w;
  return ok ? DS_OK : DS_OOM;
}

static void base_args(UpdatePlan* plan, UArgs& a, int32_t* status) {
  const int p = plan->p;
  a.p = p; a.L = plan->L; a.Db = plan->D; a.zb = 32 * plan->L - p;
  int clo = ((p - 2) / 24 - GUARD) & ~3;  // blocks start on whole limbs
  a.c_lo = clo > 0 ? clo : 0;
  a.cmax = top_column(p);
  int lg = 0;
  while ((1 << lg) < plan->D) lg++;
  a.eps = 23 + lg;
  a.status = status;
}

static cudaError_t launch_fused(UpdatePlan* plan, const UArgs& a, int TR, cudaStream_t s) {
  const int tc = plan->tc;
  dim3 grid((a.ncols + tc - 1) / tc, (a.nrows + TR - 1) / TR);
  dim3 block(tc, TR);
  size_t smem = fused_smem(plan->w, TR, plan->D, plan->L, tc);
  if (tc == 16) {
    if (plan->w == 8) k_fused<8, 16><<<grid, block, smem, s>>>(a, TR);
    else k_fused<16, 16><<<grid, block, smem, s>>>(a, TR);
  } else {
    if (plan->w == 8) k_fused<8, 32><<<grid, block, smem, s>>>(a, TR);
    else if (plan->w == 16) k_fused<16, 32><<<grid, block, smem, s>>>(a, TR);
    else k_fused<32, 32><<<grid, block, smem, s>>>(a, TR);
  }
  return cudaGetLastError();
}

int update_launch(UpdatePlan* plan, cudaStream_t s, uint32_t* a_limbs, int32_t* a_exp, uint8_t* a_cls,
                  int64_t a_count, const uint8_t* pbuf, const uint32_t* z_limbs, const int32_t* z_exp,
                  const uint8_t* z_cls, int nloc, int n, int i, int jl0, int collect_minors, int32_t* status,
                  int64_t* launches) {
  if (!plan->fused) return DS_INVALID;
  int rc = ensure_work(plan, nloc);
  if (rc != DS_OK) return rc;
  UpdateWork* wk = (UpdateWork*)plan->workspace;
  const int L = plan->L, p = plan->p, Db = plan->D;
  int nrows = nloc - jl0;
  int kstart = collect_minors ? 0 : i + 1;
  int ncols = n - kstart;
  if (nrows <= 0 || ncols <= 0) return DS_OK;
  const uint32_t* b_limbs = (const uint32_t*)pbuf;
  const int32_t* b_exp = (const int32_t*)(pbuf + (size_t)4 * L * n);
  const uint8_t* b_cls = (const uint8_t*)(pbuf + (size_t)4 * L * n + (size_t)4 * n);
  prep_launch(z_limbs + jl0, nloc, nrows, L, p, Db, wk->zdig, Db, 1, wk->zf, s);
  prep_launch(b_limbs, n, n, L, p, Db, wk->bdig, 1, n, wk->bf, s);
  UArgs a;
  base_args(plan, a, status);
  a.mode = 0;
  a.nrows = nrows;
  a.ncols = ncols;
  a.zdig = wk->zdig; a.zf = wk->zf; a.zexp = z_exp + jl0; a.zcls = z_cls + jl0;
  a.bdig = wk->bdig; a.bf = wk->bf; a.bexp = b_exp; a.bcls = b_cls; a.bstride = n;
  a.col_off = kstart; a.skip_col = i; a.o_same = 1; a.ocol_off = 0;
  a.o_limbs = a_limbs; a.o_exp = a_exp; a.o_cls = a_cls; a.o_count = a_count; a.ostride = n; a.orow0 = jl0;
  a.step = i;
  cudaError_t e = launch_fused(plan, a, plan->tr, s);
  *launches += 3;
  return e == cudaSuccess ? DS_OK : DS_CUDA;
}

// out[c] = RN(x * y_c) for c in [0, count): x one real scalar (SoA count xcount,
// element 0 at x_limbs), y_c elements of a real SoA row (plane stride ycount).
// Used for the det chain (elim.py:214) and the signed minors (elim.py:59).
int mul_row_launch(UpdatePlan* plan, cudaStream_t s, const uint32_t* x_limbs, int64_t xcount, const int32_t* x_exp,
                   const uint8_t* x_cls, const uint32_t* y_limbs, int64_t ycount, const int32_t* y_exp,
                   const uint8_t* y_cls, int count, uint32_t* o_limbs, int64_t o_count, int32_t* o_exp,
                   uint8_t* o_cls, int32_t* status, int64_t* launches, int step, double* wsx, double* wsy) {
  int rc = ensure_work(plan, 1);
  if (rc != DS_OK) return rc;
  if (count <= 0) return DS_OK;
  UpdateWork* wk = (UpdateWork*)plan->workspace;
  const int L = plan->L, p = plan->p, Db = plan->D;
  if (count > plan->n) return DS_INVALID;
  // workspaces: the det chain and the minors emission use separate buffers so
  // they can run on the side stream without racing each other
  double* xd = wsx ? wsx : wk->ddig;
  double* yd = wsy ? wsy : wk->edig;
  double* xf = xd + Db;  // topf slots after the digits
  double* yf = yd + (size_t)Db * count;
  prep_launch(x_limbs, xcount, 1, L, p, Db, xd, Db, 1, xf, s);
  prep_launch(y_limbs, ycount, count, L, p, Db, yd, 1, count, yf, s);
  UArgs a;
  base_args(plan, a, status);
  a.mode = 1;
  a.nrows = 1;
  a.ncols = count;
  a.zdig = xd; a.zf = xf; a.zexp = x_exp; a.zcls = x_cls;
  a.bdig = yd; a.bf = yf; a.bexp = y_exp; a.bcls = y_cls; a.bstride = count;
  a.step = step;
  a.col_off = 0; a.skip_col = -1; a.o_same = 1; a.ocol_off = 0;
  a.o_limbs = o_limbs; a.o_exp = o_exp; a.o_cls = o_cls; a.o_count = o_count; a.ostride = 0; a.orow0 = 0;
  const int wpb = 4;
  const int SW = 4;  // small column blocks: enough blocks to keep the 32 lanes busy
  int nbs = (a.cmax - a.c_lo) / SW + 1;
  size_t smem = split_smem(SW, Db, L, a.cmax, a.c_lo, wpb);
  k_mul_split<SW><<<(count + wpb - 1) / wpb, 32 * wpb, smem, s>>>(a, nbs);
  *launches += 3;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DS_OK : DS_CUDA;
}
