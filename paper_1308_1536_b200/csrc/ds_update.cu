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
#include <string>

#include "../../include/detseries_b200.h"
#include "ds_mp.cuh"
#include "ds_update.cuh"

namespace {

constexpr int TC = 32;        // columns per CTA (one warp row)
constexpr int GUARD = 4;      // guard digits of the short product
constexpr int FLUSH = 64;     // s-steps between carry flushes (64 * 2^46 < 2^53)
constexpr double R24 = 1.0 / 16777216.0;
constexpr double B24 = 16777216.0;

struct UArgs {
  int p, L, Db, zb, n, i, jl0, nrows, ncols, collect_minors;
  int c_lo, cmax, eps;
  uint32_t* a_limbs;
  int32_t* a_exp;
  uint8_t* a_cls;
  int64_t a_count;
  const double* zdig;  // [nloc][Db]
  const double* bdig;  // [Db][n]
  const double* zf;    // [nloc] leading 64 bits of z as a double in [1,2)
  const double* bf;    // [n]
  const int32_t* z_exp;
  const uint8_t* z_cls;
  const int32_t* b_exp;
  const uint8_t* b_cls;
  int32_t* status;
};

__device__ __forceinline__ int map_col(const UArgs& a, int c) {
  if (!a.collect_minors) return a.i + 1 + c;
  return c < a.i ? c : c + 1;
}

// ------------------------------------------------------------ prep kernels
// Balanced radix-2^24 digits of the p-bit integer mantissa m = M >> (32L-p),
// d_s in [-2^23, 2^23), m = sum d_s 2^(24 s), Db = ceil(p/24) + 1 digits.
__global__ void k_prep_digits(const uint32_t* limbs, int64_t count, int64_t first, int64_t num, int L, int p,
                              int Db, double* dig, int64_t es, int64_t ds, double* topf) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= num) return;
  int64_t idx = first + e;
  ds::CPtr M{limbs + idx, count};
  int zb = 32 * L - p;
  int ndig = (p + 23) / 24;
  int carry = 0;
  for (int s = 0; s < Db; s++) {
    int v = carry;
    if (s < ndig) {
      uint32_t u = ds::bits32(M, L, (int64_t)24 * s + zb) & 0xFFFFFFu;
      if (24 * s + 24 > p) u &= (1u << (p - 24 * s)) - 1u;
      v += (int)u;
    }
    carry = 0;
    if (v >= (1 << 23)) {
      v -= (1 << 24);
      carry = 1;
    }
    dig[idx * es + (int64_t)s * ds] = (double)v;
  }
  uint64_t top = ((uint64_t)M[L - 1] << 32) | M[L - 2];
  topf[idx] = (double)top * 0x1p-63;
}

// ------------------------------------------------------------ S window
// Exact aligned sum S = |X| -/+ |Y| of a and t on a window of L+2 limbs:
// limb 0 = guard (register), limbs 1..L = a's own slots (in place), limb L+1
// = carry (register).  X is the operand with the larger exponent, anchored at
// limbs 1..L; Y is shifted right by dq limbs + dr bits; Y bits below the
// window become the sticky bit (effective subtraction borrows 1 ulp-of-guard
// when sticky, the standard round/sticky trick).
struct SWin {
  uint32_t* A;
  int64_t st;
  int L;
  bool xa;      // X = a (Y = t) or X = t (Y = a)
  bool sub;     // effective subtraction
  bool yzero;   // Y == 0 (a == 0)
  int dq, dr;
  uint32_t prev;
  int q, w;
  uint32_t S0, SL1;
  uint32_t cb;
  bool sticky;
  uint32_t curA;

  __device__ __forceinline__ uint32_t aload(int l) const { return (l >= 0 && l < L) ? A[(int64_t)l * st] : 0u; }

  __device__ __forceinline__ void emit(uint32_t X, uint32_t Yb) {
    uint32_t s;
    if (sub) {
      uint64_t y = (uint64_t)Yb + cb + ((w == 0 && sticky) ? 1u : 0u);
      s = (uint32_t)((uint64_t)X - y);
      cb = ((uint64_t)X < y) ? 1u : 0u;
    } else {
      uint64_t t = (uint64_t)X + Yb + cb;
      s = (uint32_t)t;
      cb = (uint32_t)(t >> 32);
    }
    if (w == 0) S0 = s;
    else if (w == L + 1) SL1 = s;
    else A[(int64_t)(w - 1) * st] = s;
    w++;
  }

  __device__ __forceinline__ uint32_t abits(int wi) {
    // Y = a:  window limb wi <- a bits [32(wi-1+dq)+dr, +32)
    uint32_t nxt = aload(wi + dq);
    uint32_t v = dr ? ((curA >> dr) | (nxt << (32 - dr))) : curA;
    curA = nxt;
    return v;
  }

  __device__ void init(uint32_t* A_, int64_t st_, int L_, bool xa_, bool sub_, bool yzero_, int64_t shift) {
    A = A_; st = st_; L = L_; xa = xa_; sub = sub_; yzero = yzero_;
    if (shift > 32 * (int64_t)(L + 3)) shift = 32 * (int64_t)(L + 3);  // all of Y below the window
    dq = (int)(shift >> 5);
    dr = (int)(shift & 31);
    prev = 0; q = 0; w = 0; S0 = 0; SL1 = 0; cb = 0; sticky = false; curA = 0;
    if (!xa) {
      if (yzero) {
        emit(0u, 0u);
        return;
      }
      // sticky: a bits [0, 32(dq-1)+dr)
      int64_t below = 32 * (int64_t)(dq - 1) + dr;
      for (int l = 0; l < L && (int64_t)l * 32 < below; l++) {
        uint32_t v = aload(l);
        int64_t lim = below - 32 * (int64_t)l;
        if (lim < 32) v &= (1u << lim) - 1u;
        if (v) sticky = true;
      }
      curA = aload(dq - 1);
      emit(0u, abits(0));
    }
  }

  // next limb of t (T_0 .. T_{L-1} left-aligned mantissa, then T_L = overflow)
  __device__ __forceinline__ void push(uint32_t T) {
    if (xa) {
      int wq = q - dq;
      if (wq < 0) {
        if (q >= 1 && prev) sticky = true;
      } else {
        if (wq == 0 && dr > 0 && (prev & ((1u << dr) - 1u))) sticky = true;
        uint32_t Yb = dr ? ((prev >> dr) | (T << (32 - dr))) : prev;
        uint32_t X = (wq >= 1 && wq <= L) ? A[(int64_t)(wq - 1) * st] : 0u;
        emit(X, Yb);
      }
      prev = T;
      q++;
    } else {
      uint32_t Yb = yzero ? 0u : abits(w);
      emit(T, Yb);
    }
  }

  __device__ void finish() {
    if (xa)
      while (w <= L + 1) push(0u);
  }

  __device__ __forceinline__ uint32_t get(int wi) const {
    if (wi == 0) return S0;
    if (wi == L + 1) return SL1;
    if (wi < 0 || wi > L + 1) return 0u;
    return A[(int64_t)(wi - 1) * st];
  }
  __device__ __forceinline__ void set(int wi, uint32_t v) {
    if (wi == 0) S0 = v;
    else if (wi == L + 1) SL1 = v;
    else A[(int64_t)(wi - 1) * st] = v;
  }
};

// ------------------------------------------------------------ digit consumers
// Top-bit probe (exact dry product): is bit 2p-1 of P set?
struct DryTop {
  int bitpos;
  int top;
  __device__ __forceinline__ bool digit(int c, uint32_t v) {
    int pos = 24 * c;
    if (bitpos >= pos && bitpos < pos + 24) top = (v >> (bitpos - pos)) & 1u;
    return true;
  }
  __device__ __forceinline__ bool finish(double) { return true; }
};

// Rounds P = z*b to the p-bit t and streams t's limbs into the S window.
struct Emit {
  SWin* S;
  int r, zb, p, L, cmax;
  bool exact;
  int lo_chk, hi_chk;  // decision region (short product)
  bool allz, allo, sticky, decided;
  uint32_t rbit, tcarry;
  uint64_t buf;
  int nb, tl;
  bool excess;

  __device__ __forceinline__ bool digit(int c, uint32_t v) {
    if (c > cmax) {
      if (v) excess = true;
      return true;
    }
    int pos = 24 * c;
    if (!decided) {
      if (pos < r) {  // bits of this digit below r
        int nlow = r - pos < 24 ? r - pos : 24;
        uint32_t vl = v & ((1u << nlow) - 1u);
        int rb = r - 1 - pos;  // round bit position inside the digit
        if (rb >= 0 && rb < 24) rbit = (v >> rb) & 1u;
        if (exact) {
          uint32_t below = (rb >= 24) ? vl : (rb > 0 ? (vl & ((1u << rb) - 1u)) : 0u);
          if (below) sticky = true;
        } else {
          int lo = pos > lo_chk ? pos : lo_chk;
          int hi = (pos + 23) < hi_chk ? (pos + 23) : hi_chk;
          if (hi >= lo) {
            int len = hi - lo + 1;
            uint32_t m = (len >= 32) ? 0xffffffffu : ((1u << len) - 1u);
            uint32_t bits = (v >> (lo - pos)) & m;
            if (bits != 0) allz = false;
            if (bits != m) allo = false;
          }
        }
      }
      if (r >= pos && r < pos + 24) {  // digit holding t's LSB: decide
        uint32_t lsb = (v >> (r - pos)) & 1u;
        uint32_t inc;
        if (exact) {
          inc = rbit & ((sticky ? 1u : 0u) | lsb);
        } else {
          if (allz || allo) return false;  // undecided: caller reruns exact
          inc = rbit;
        }
        decided = true;
        tcarry = inc;
      }
    }
    if (pos + 24 > r) {  // bits >= r belong to the mantissa of t
      int sh = r > pos ? r - pos : 0;
      buf |= (uint64_t)(v >> sh) << nb;
      nb += 24 - sh;
      while (tl < L) {
        int need = tl == 0 ? 32 - zb : 32;
        if (nb < need) break;
        uint32_t limb;
        if (tl == 0) {
          uint64_t part = buf & ((need == 32) ? 0xffffffffull : ((1ull << need) - 1ull));
          uint64_t sum = (part << zb) + ((uint64_t)tcarry << zb);
          limb = (uint32_t)sum;
          tcarry = (uint32_t)(sum >> 32);
        } else {
          uint64_t sum = (buf & 0xffffffffull) + tcarry;
          limb = (uint32_t)sum;
          tcarry = (uint32_t)(sum >> 32);
        }
        buf >>= need;
        nb -= need;
        S->push(limb);
        tl++;
      }
      if (tl == L && nb > 0) {
        if (buf) excess = true;
        buf = 0;
        nb = 0;
      }
    }
    return true;
  }

  __device__ __forceinline__ bool finish(double carry) {
    if (carry != 0.0 || tl != L) excess = true;
    S->push(tcarry);  // overflow limb T_L (t rounded up to 2^p)
    S->finish();
    return true;
  }
};

// ------------------------------------------------------------ the product
// P = sum_c col_c 2^(24c), col_c = sum_{s+t=c} z_s b_t, for columns
// c >= c_start, streamed low -> high as nonnegative digits to `cons`.
template <int W, class C>
__device__ __forceinline__ bool product(const double* __restrict__ zrow, const double* __restrict__ bcol, int Db,
                                        int c_start, int cmax, C& cons) {
  double carry = 0.0;
  for (int c0 = c_start; c0 <= cmax; c0 += W) {
    double acc[W + 1];
    acc[0] = carry;
#pragma unroll
    for (int w = 1; w <= W; w++) acc[w] = 0.0;
    int s_lo = c0 - (Db - 1);
    if (s_lo < 0) s_lo = 0;
    int s_hi = c0 + W - 1;
    if (s_hi > Db - 1) s_hi = Db - 1;
    if (s_lo <= s_hi) {
      double ph[W];
#pragma unroll
      for (int w = 0; w < W; w++) ph[w] = bcol[(c0 + w - s_lo + 2 * W) * TC];
      int ngroups = (s_hi - s_lo + W) / W;
      int s = s_lo;
      for (int g = 0; g < ngroups; g++) {
#pragma unroll
        for (int u = 0; u < W; u++) {
          double zv = zrow[s + u];
#pragma unroll
          for (int w = 0; w < W; w++) acc[w] = fma(zv, ph[(w - u + W) % W], acc[w]);
          ph[(2 * W - 1 - u) % W] = bcol[(c0 - (s + u) - 1 + 2 * W) * TC];
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
#pragma unroll
    for (int w = 0; w < W; w++) {
      double q = floor(acc[w] * R24);
      acc[w] = fma(-q, B24, acc[w]);
      acc[w + 1] += q;
    }
#pragma unroll
    for (int w = 0; w < W; w++)
      if (!cons.digit(c0 + w, (uint32_t)(int)acc[w])) return false;
    carry = acc[W];
  }
  return cons.finish(carry);
}

// ------------------------------------------------------------ element
template <int W>
__device__ void update_element(const UArgs& a, const double* zrow, const double* bcol, int jl, int k) {
  const int L = a.L, p = a.p;
  int64_t idx = (int64_t)jl * a.n + k;
  uint8_t ca = a.a_cls[idx];
  uint8_t cz = a.z_cls[jl];
  uint8_t cb = a.b_cls[k];
  bool za = ca >= DS_CLS_PZERO;
  int sa = ca & 1, st = (cz & 1) ^ (cb & 1);
  if (cz >= DS_CLS_PZERO || cb >= DS_CLS_PZERO) {  // t = (-1)^st 0
    if (!za) return;                                // a - 0 = a
    a.a_cls[idx] = (sa && !st) ? DS_CLS_NZERO : DS_CLS_PZERO;
    return;
  }
  int32_t ea = a.a_exp[idx];
  double pr = a.zf[jl] * a.bf[k];
  int norm = pr >= 2.0 ? 1 : 0;
  bool confident = fabs(pr - 2.0) > 0x1p-42;
  int64_t ebase = (int64_t)a.z_exp[jl] + a.b_exp[k];
  if (!za && (int64_t)ea - (ebase - 1) >= (int64_t)p + 2 + 1) return;  // a dominates whatever the norm
  if (!confident) {
    DryTop dt;
    dt.bitpos = 2 * p - 1;
    dt.top = 0;
    product<W>(zrow, bcol, a.Db, 0, a.cmax, dt);
    norm = dt.top;
  }
  int64_t et = ebase - (norm ? 0 : 1);
  int64_t d = za ? -(int64_t)(1 << 30) : (int64_t)ea - et;
  if (!za && d >= (int64_t)p + 2) return;  // RN(a - t) = a
  bool xa = !za && d >= 0;
  bool sub = !za && (sa == st);  // a + (-t): magnitudes subtract iff signs of a and -t differ
  int neg = xa ? sa : (st ^ 1);
  int64_t E = xa ? ea : et;
  uint32_t* A = a.a_limbs + idx;
  int64_t stA = a.a_count;

  SWin S;
  Emit em;
  bool done = false;
  for (int attempt = 0; attempt < 2 && !done; attempt++) {
    bool exact = attempt == 1 || a.c_lo == 0;
    S.init(A, stA, L, xa, sub, za, xa ? d : (za ? 0 : -d));
    em.S = &S;
    em.r = norm ? p : p - 1;
    em.zb = a.zb; em.p = p; em.L = L; em.cmax = a.cmax;
    em.exact = exact;
    em.lo_chk = 24 * a.c_lo + a.eps;
    em.hi_chk = em.r - 2;
    em.allz = true; em.allo = true; em.sticky = false; em.decided = false;
    em.rbit = 0; em.tcarry = 0; em.buf = 0; em.nb = 0; em.tl = 0; em.excess = false;
    done = product<W>(zrow, bcol, a.Db, exact ? 0 : a.c_lo, a.cmax, em);
  }
  if (em.excess) atomicAdd(&a.status[4], 1);  // normalisation misprediction (must never happen)

  // ---- normalise, round to nearest-even, write in place
  if (S.sub && S.cb) {  // negative (only possible when exponents are equal)
    uint32_t c = 1;
    for (int wi = 0; wi <= L + 1; wi++) {
      uint64_t v = (uint64_t)(uint32_t)~S.get(wi) + c;
      S.set(wi, (uint32_t)v);
      c = (uint32_t)(v >> 32);
    }
    neg ^= 1;
  }
  int h = -1;
  for (int wi = L + 1; wi >= 0; wi--) {
    uint32_t v = S.get(wi);
    if (v) {
      h = 32 * wi + 31 - __clz(v);
      break;
    }
  }
  if (h < 0) {  // exact cancellation -> +0
    for (int l = 0; l < L; l++) A[(int64_t)l * stA] = 0u;
    a.a_exp[idx] = 0;
    a.a_cls[idx] = DS_CLS_PZERO;
    return;
  }
  int64_t e = E - 32 * (int64_t)L - 31 + h;
  int off = h - 32 * L + 1;
  if (off < 0) {  // massive cancellation: move the window up by whole limbs
    int qs = (-off + 31) / 32;
    for (int wi = L + 1; wi >= 0; wi--) S.set(wi, S.get(wi - qs));
    h += 32 * qs;
    off += 32 * qs;
  }
  int lsbw = h - p + 1;
  uint32_t rbit = 0;
  bool stk = S.sticky;
  if (lsbw - 1 >= 0) {
    int rb = lsbw - 1;
    rbit = (S.get(rb >> 5) >> (rb & 31)) & 1u;
    for (int wi = 0; wi < (rb >> 5) && !stk; wi++)
      if (S.get(wi)) stk = true;
    if (!stk && (rb & 31) && (S.get(rb >> 5) & ((1u << (rb & 31)) - 1u))) stk = true;
  }
  const int zb = a.zb, zl = zb >> 5;
  int base = off >> 5, rs = off & 31;
  uint32_t lo = S.get(base);
  // result LSB value (for ties-to-even)
  uint32_t carry = 0;
  {
    // compute inc: need the LSB of the truncated mantissa = window bit lsbw
    uint32_t lsb = (lsbw >= 0) ? ((S.get(lsbw >> 5) >> (lsbw & 31)) & 1u) : 0u;
    carry = rbit & ((stk ? 1u : 0u) | lsb);
  }
  for (int l = 0; l < L; l++) {
    uint32_t hi = S.get(base + l + 1);
    uint32_t v = rs ? ((lo >> rs) | (hi << (32 - rs))) : lo;
    lo = hi;
    if (l < zl) v = 0;
    else if (l == zl && (zb & 31)) v &= ~((1u << (zb & 31)) - 1u);
    if (l >= zl && carry) {
      uint32_t add = (l == zl) ? (1u << (zb & 31)) : 1u;
      uint32_t r = v + add;
      carry = r < v ? 1u : 0u;
      v = r;
    }
    A[(int64_t)l * stA] = v;
  }
  if (carry) {
    A[(int64_t)(L - 1) * stA] = 0x80000000u;
    e += 1;
  }
  if (e < DS_EMIN || e > DS_EMAX) atomicAdd(&a.status[2], 1);
  a.a_exp[idx] = (int32_t)e;
  a.a_cls[idx] = neg ? DS_CLS_NEG : DS_CLS_POS;
}

template <int W>
__global__ void __launch_bounds__(256) k_update_dfma(UArgs a, int TR) {
  extern __shared__ double sm[];
  if (a.status[0] >= 0) return;
  const int Db = a.Db;
  const int ZP = Db + W;
  const int BP = Db + 3 * W;
  double* zs = sm;
  double* bs = sm + TR * ZP;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int col0 = blockIdx.x * TC, row0 = blockIdx.y * TR;
  const int tid = ty * TC + tx, nth = TC * TR;
  for (int e = tid; e < TR * ZP; e += nth) {
    int r = e / ZP, s = e - r * ZP;
    int rr = row0 + r;
    zs[e] = (rr < a.nrows && s < Db) ? a.zdig[(int64_t)(a.jl0 + rr) * Db + s] : 0.0;
  }
  for (int e = tid; e < BP * TC; e += nth) {
    int tt = e / TC, c = e - tt * TC;
    int t = tt - 2 * W;
    int cc = col0 + c;
    double v = 0.0;
    if (cc < a.ncols && t >= 0 && t < Db) v = a.bdig[(int64_t)t * a.n + map_col(a, cc)];
    bs[e] = v;
  }
  __syncthreads();
  const int r = row0 + ty, cc = col0 + tx;
  if (r >= a.nrows || cc >= a.ncols) return;
  update_element<W>(a, zs + ty * ZP, bs + tx, a.jl0 + r, map_col(a, cc));
}

std::string g_err;

}  // namespace

// ---------------------------------------------------------------- host API
struct UpdateWork {
  double* zdig;
  double* bdig;
  double* zf;
  double* bf;
  int nloc;
};

static int smem_bytes(int W, int TR, int Db) { return 8 * (TR * (Db + W) + (Db + 3 * W) * TC); }

int update_plan_init(UpdatePlan* plan, int n, int p, int device) {
  plan->enabled = 0;
  plan->n = n;
  plan->p = p;
  plan->L = (p + 31) / 32;
  plan->D = (p + 23) / 24 + 1;
  plan->device = device;
  plan->workspace = nullptr;
  if (getenv("DS_DISABLE_DFMA")) return DS_OK;
  int W = plan->D <= 24 ? 8 : 16;
  int TR = 8;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  while (TR > 1 && smem_bytes(W, TR, plan->D) > maxsm) TR /= 2;
  if (smem_bytes(W, TR, plan->D) > maxsm) return DS_OK;  // too wide: general engine
  plan->w = W;
  plan->tr = TR;
  plan->tc = TC;
  plan->smem = smem_bytes(W, TR, plan->D);
  cudaDeviceGetAttribute(&plan->sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e1 = cudaFuncSetAttribute(k_update_dfma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  cudaError_t e2 = cudaFuncSetAttribute(k_update_dfma<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  if (e1 != cudaSuccess || e2 != cudaSuccess) return DS_CUDA;
  plan->enabled = 1;
  return DS_OK;
}

void update_plan_free(UpdatePlan* plan) {
  if (plan->workspace) {
    UpdateWork* w = (UpdateWork*)plan->workspace;
    cudaFree(w->zdig);
    cudaFree(w->bdig);
    cudaFree(w->zf);
    cudaFree(w->bf);
    delete w;
    plan->workspace = nullptr;
  }
}

static int ensure_work(UpdatePlan* plan, int nloc) {
  if (plan->workspace) return DS_OK;
  UpdateWork* w = new UpdateWork();
  w->nloc = nloc;
  size_t D = plan->D;
  if (cudaMalloc(&w->zdig, sizeof(double) * D * (size_t)(nloc > 0 ? nloc : 1)) != cudaSuccess ||
      cudaMalloc(&w->bdig, sizeof(double) * D * plan->n) != cudaSuccess ||
      cudaMalloc(&w->zf, sizeof(double) * (size_t)(nloc > 0 ? nloc : 1)) != cudaSuccess ||
      cudaMalloc(&w->bf, sizeof(double) * plan->n) != cudaSuccess) {
    delete w;
    return DS_OOM;
  }
  plan->workspace = w;
  return DS_OK;
}

int update_launch(UpdatePlan* plan, cudaStream_t s, uint32_t* a_limbs, int32_t* a_exp, uint8_t* a_cls,
                  int64_t a_count, const uint8_t* pbuf, const uint32_t* z_limbs, const int32_t* z_exp,
                  const uint8_t* z_cls, int nloc, int n, int i, int jl0, int collect_minors, int32_t* status,
                  int64_t* launches) {
  int rc = ensure_work(plan, nloc);
  if (rc != DS_OK) return rc;
  UpdateWork* wk = (UpdateWork*)plan->workspace;
  const int L = plan->L, p = plan->p, Db = plan->D;
  int nrows = nloc - jl0;
  int ncols = collect_minors ? n - 1 : n - 1 - i;
  if (nrows <= 0 || ncols <= 0) return DS_OK;
  const uint32_t* b_limbs = (const uint32_t*)pbuf;
  const int32_t* b_exp = (const int32_t*)(pbuf + (size_t)4 * L * n);
  const uint8_t* b_cls = (const uint8_t*)(pbuf + (size_t)4 * L * n + (size_t)4 * n);
  k_prep_digits<<<(nrows + 127) / 128, 128, 0, s>>>(z_limbs, nloc, jl0, nrows, L, p, Db, wk->zdig, Db, 1, wk->zf);
  k_prep_digits<<<(n + 127) / 128, 128, 0, s>>>(b_limbs, n, 0, n, L, p, Db, wk->bdig, 1, n, wk->bf);
  UArgs a;
  a.p = p; a.L = L; a.Db = Db; a.zb = 32 * L - p; a.n = n; a.i = i; a.jl0 = jl0; a.nrows = nrows;
  a.ncols = ncols; a.collect_minors = collect_minors;
  int clo = (p - 2) / 24 - GUARD;
  a.c_lo = clo > 0 ? clo : 0;
  a.cmax = (2 * p - 1) / 24;
  int lg = 0;
  while ((1 << lg) < Db) lg++;
  a.eps = 23 + lg;
  a.a_limbs = a_limbs; a.a_exp = a_exp; a.a_cls = a_cls; a.a_count = a_count;
  a.zdig = wk->zdig; a.bdig = wk->bdig; a.zf = wk->zf; a.bf = wk->bf;
  a.z_exp = z_exp; a.z_cls = z_cls; a.b_exp = b_exp; a.b_cls = b_cls; a.status = status;
  int TR = plan->tr;
  dim3 grid((ncols + TC - 1) / TC, (nrows + TR - 1) / TR);
  dim3 block(TC, TR);
  if (plan->w == 8)
    k_update_dfma<8><<<grid, block, plan->smem, s>>>(a, TR);
  else
    k_update_dfma<16><<<grid, block, plan->smem, s>>>(a, TR);
  *launches += 3;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DS_OK : DS_CUDA;
}
