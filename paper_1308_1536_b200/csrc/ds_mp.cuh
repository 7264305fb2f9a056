// ds_mp.cuh -- thread-level correctly-rounded multiprecision arithmetic on the
// ds SoA format (include/detseries_b200.h).
//
// These routines restate, for one scalar per thread, the round-to-nearest-even
// semantics of the MPFR/MPC operations the reference calls:
//   mpfr_mul / mpfr_sub / mpfr_add / mpfr_div  (elim.py:47, 50, 52, 59, 148, 214)
//   mpc_mul / mpc_sub / mpc_div               (same call sites on mpc values)
// Every result is the exact result rounded once at precision p (ties to even),
// with IEEE-754 signed-zero rules, which is what MPFR/MPC guarantee.  They are
// the general (slow-path) engine: k_mult (division), k_emit (det chain, minors),
// the complex update and the scalar conformance kernel use them directly; the
// hot real update (ds_update.cu) has its own fused DFMA engine and falls back to
// nothing but itself.
//
// Big integers are little-endian arrays of 32-bit limbs accessed through a
// stride (so per-thread scratch can be laid out [word][thread], coalesced).
#pragma once
#include <stdint.h>
#include "../../include/detseries_b200.h"

namespace ds {

struct Ptr {
  uint32_t* p;
  int64_t s;  // stride in words
  __device__ __forceinline__ uint32_t& operator[](int64_t k) const { return p[k * s]; }
  __device__ __forceinline__ Ptr off(int64_t k) const { return Ptr{p + k * s, s}; }
};

struct CPtr {
  const uint32_t* p;
  int64_t s;
  __device__ __forceinline__ uint32_t operator[](int64_t k) const { return p[k * s]; }
};

// A scalar view (one component): mantissa limbs (L, left-aligned, MSB set),
// exponent (MPFR convention) and class.
struct Val {
  CPtr m;
  int64_t e;
  uint8_t c;  // DS_CLS_*
};

static __device__ __forceinline__ bool is_zero_cls(uint8_t c) { return c >= DS_CLS_PZERO; }
static __device__ __forceinline__ int neg_of(uint8_t c) { return (c == DS_CLS_NEG || c == DS_CLS_NZERO) ? 1 : 0; }
static __device__ __forceinline__ uint8_t zero_cls(int neg) { return neg ? DS_CLS_NZERO : DS_CLS_PZERO; }
static __device__ __forceinline__ uint8_t nz_cls(int neg) { return neg ? DS_CLS_NEG : DS_CLS_POS; }

// bits [q, q+32) of a big integer S (n limbs); zero outside [0, 32n)
static __device__ __forceinline__ uint32_t bits32(CPtr S, int n, int64_t q) {
  int64_t lw = q >> 5;  // floor
  int sh = (int)(q & 31);
  uint32_t lo = (lw >= 0 && lw < n) ? S[lw] : 0u;
  uint32_t hi = (lw + 1 >= 0 && lw + 1 < n) ? S[lw + 1] : 0u;
  return sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
}

// position of the highest set bit of S, or -1 if S == 0
static __device__ __forceinline__ int64_t top_bit(CPtr S, int n) {
  for (int k = n - 1; k >= 0; k--) {
    uint32_t v = S[k];
    if (v) return (int64_t)k * 32 + 31 - __clz(v);
  }
  return -1;
}

// any bit of S in [0, q) set?
static __device__ __forceinline__ bool any_below(CPtr S, int n, int64_t q) {
  if (q <= 0) return false;
  int64_t full = q >> 5;
  for (int64_t k = 0; k < full && k < n; k++)
    if (S[k]) return true;
  int r = (int)(q & 31);
  if (r && full < n) return (S[full] & ((1u << r) - 1u)) != 0;
  return false;
}

struct RoundOut {
  int64_t e;   // MPFR exponent of the rounded value
  bool inexact;
};

// Round the exact nonnegative integer S (n limbs, S != 0) plus an optional
// sticky tail (true value in (S, S+1) units when sticky) to p bits, ties to
// even.  Writes the left-aligned L-limb mantissa to `out`.  `base` is the
// exponent of S's LSB: value = S * 2^base.  Returns the MPFR exponent.
static __device__ RoundOut round_big(Ptr out, int L, int p, CPtr S, int n, int64_t base, bool sticky_in) {
  int64_t hb = top_bit(S, n);
  int64_t lsb = hb - p + 1;  // bit position (in S) of the result's LSB
  bool rbit = false, sticky = sticky_in;
  if (lsb - 1 >= 0) {
    rbit = (bits32(S, n, lsb - 1) & 1u) != 0;
    if (!sticky) sticky = any_below(S, n, lsb - 1);
  }
  int64_t off = hb + 1 - 32 * (int64_t)L;  // M bit j <-> S bit j + off
  int zb = 32 * L - p;                        // zero bits at the bottom of M
  uint32_t carry = 0;
  bool lsbit = false;
  // build M and find the result LSB value
  for (int l = 0; l < L; l++) {
    uint32_t v = bits32(S, n, (int64_t)l * 32 + off);
    if (l == zb / 32) {
      uint32_t mask = ~((1u << (zb & 31)) - 1u);
      if ((zb & 31) == 0) mask = 0xffffffffu;
      v &= mask;
      lsbit = ((v >> (zb & 31)) & 1u) != 0;
    } else if (l < zb / 32) {
      v = 0;
    }
    out[l] = v;
  }
  bool inc = rbit && (sticky || lsbit);
  int64_t e = base + hb + 1;
  if (inc) {
    carry = 1;
    for (int l = zb / 32; l < L && carry; l++) {
      uint32_t add = (l == zb / 32) ? (1u << (zb & 31)) : 1u;
      uint32_t v = out[l];
      uint32_t r = v + add;
      carry = (r < v) ? 1u : 0u;
      out[l] = r;
    }
    if (carry) {  // mantissa overflowed to 2^p: becomes 0.1000.. with e+1
      out[L - 1] = 0x80000000u;
      e += 1;
    }
  }
  RoundOut ro;
  ro.e = e;
  ro.inexact = rbit || sticky;
  return ro;
}

// P (2L limbs) = A * B, full schoolbook with 64-bit accumulation
static __device__ void mul_full(Ptr P, CPtr A, CPtr B, int L) {
  for (int k = 0; k < 2 * L; k++) P[k] = 0;
  for (int i = 0; i < L; i++) {
    uint64_t carry = 0;
    uint64_t ai = A[i];
    if (ai == 0) continue;
    for (int j = 0; j < L; j++) {
      uint64_t t = ai * (uint64_t)B[j] + (uint64_t)P[i + j] + carry;
      P[i + j] = (uint32_t)t;
      carry = t >> 32;
    }
    P[i + L] = (uint32_t)carry;
  }
}

// store result: out mantissa already written; sets exp/cls with range check.
// returns false on exponent overflow/underflow.
static __device__ __forceinline__ bool range_ok(int64_t e) { return e >= DS_EMIN && e <= DS_EMAX; }

// ---------------------------------------------------------------- real mul
// r = RN(a * b).  tmp needs 2L words.
static __device__ bool mul_rn(Ptr rm, int32_t* re, uint8_t* rc, const Val& a, const Val& b, int L, int p,
                       Ptr tmp) {
  int neg = neg_of(a.c) ^ neg_of(b.c);
  if (is_zero_cls(a.c) || is_zero_cls(b.c)) {
    for (int l = 0; l < L; l++) rm[l] = 0;
    *re = 0;
    *rc = zero_cls(neg);
    return true;
  }
  mul_full(tmp, a.m, b.m, L);
  RoundOut ro = round_big(rm, L, p, CPtr{tmp.p, tmp.s}, 2 * L, a.e + b.e - 64 * (int64_t)L, false);
  *re = (int32_t)ro.e;
  *rc = nz_cls(neg);
  return range_ok(ro.e);
}

// compare |a| vs |b| for nonzero a, b: -1, 0, 1
static __device__ int cmp_abs(const Val& a, const Val& b, int L) {
  if (a.e != b.e) return a.e > b.e ? 1 : -1;
  for (int l = L - 1; l >= 0; l--) {
    uint32_t x = a.m[l], y = b.m[l];
    if (x != y) return x > y ? 1 : -1;
  }
  return 0;
}

static __device__ __forceinline__ void copy_val(Ptr rm, int32_t* re, uint8_t* rc, const Val& a, int L, int neg) {
  for (int l = 0; l < L; l++) rm[l] = a.m[l];
  *re = (int32_t)a.e;
  *rc = is_zero_cls(a.c) ? a.c : nz_cls(neg);
}

// r = RN(a + (-1)^sub_b * b).  tmp needs 2L + 3 words.
static __device__ bool add_rn(Ptr rm, int32_t* re, uint8_t* rc, const Val& a, const Val& b, bool negate_b,
                       int L, int p, Ptr tmp) {
  int na = neg_of(a.c), nb = neg_of(b.c) ^ (negate_b ? 1 : 0);
  bool za = is_zero_cls(a.c), zb = is_zero_cls(b.c);
  if (za && zb) {
    // IEEE: x + y of zeros is -0 only if both are -0 (RN)
    for (int l = 0; l < L; l++) rm[l] = 0;
    *re = 0;
    *rc = zero_cls(na && nb);
    return true;
  }
  if (zb) { copy_val(rm, re, rc, a, L, na); return true; }
  if (za) { copy_val(rm, re, rc, b, L, nb); return true; }
  bool eff_sub = (na != nb);
  int c = cmp_abs(a, b, L);
  if (eff_sub && c == 0) {  // exact cancellation -> +0 under RN
    for (int l = 0; l < L; l++) rm[l] = 0;
    *re = 0;
    *rc = DS_CLS_PZERO;
    return true;
  }
  const Val& X = (c >= 0) ? a : b;
  const Val& Y = (c >= 0) ? b : a;
  int nx = (c >= 0) ? na : nb;
  int64_t d = X.e - Y.e;  // >= 0
  if (d >= (int64_t)p + 2) {  // Y below a quarter ulp of X: RN(X +- Y) = X
    copy_val(rm, re, rc, X, L, nx);
    return true;
  }
  // S = MX * 2^d +- MY, in n = L + ceil(d/32) + 1 limbs
  int dl = (int)(d >> 5);
  int n = L + dl + 2;
  // X shifted left by d bits
  for (int k = 0; k < n; k++) {
    int64_t q = (int64_t)k * 32 - d;  // S bit 32k <- X bit q
    tmp[k] = bits32(X.m, L, q);
  }
  if (!eff_sub) {
    uint64_t carry = 0;
    for (int k = 0; k < n; k++) {
      uint64_t t = (uint64_t)tmp[k] + (k < L ? Y.m[k] : 0u) + carry;
      tmp[k] = (uint32_t)t;
      carry = t >> 32;
    }
  } else {
    int64_t borrow = 0;
    for (int k = 0; k < n; k++) {
      int64_t t = (int64_t)tmp[k] - (int64_t)(k < L ? Y.m[k] : 0u) - borrow;
      borrow = t < 0 ? 1 : 0;
      tmp[k] = (uint32_t)(t + (borrow << 32));
    }
  }

  RoundOut ro = round_big(rm, L, p, CPtr{tmp.p, tmp.s}, n, Y.e - 32 * (int64_t)L, false);
  *re = (int32_t)ro.e;
  *rc = nz_cls(nx);
  return range_ok(ro.e);
}

// Knuth algorithm D: Q = floor(U / V), R = U mod V.
// U: nu limbs (modified in place to hold the remainder in its low nv limbs),
// V: nv limbs with the MSB of V[nv-1] set (normalized), nu > nv.
// Q: nu - nv limbs.  Returns true if the remainder is nonzero.
static __device__ bool divrem_norm(Ptr Q, Ptr U, int nu, CPtr V, int nv) {
  uint64_t vtop = V[nv - 1];
  uint64_t vnext = nv >= 2 ? V[nv - 2] : 0;
  for (int j = nu - nv - 1; j >= 0; j--) {
    uint64_t num = ((uint64_t)U[j + nv] << 32) | U[j + nv - 1];
    uint64_t qhat = num / vtop;
    if (qhat > 0xffffffffull) qhat = 0xffffffffull;  // Knuth: min(num / v1, b - 1)
    uint64_t rhat = num - qhat * vtop;
    while (rhat < (1ull << 32) && qhat * vnext > ((rhat << 32) | (uint64_t)U[j + nv - 2])) {
      qhat -= 1;
      rhat += vtop;
    }
    // multiply-subtract
    int64_t borrow = 0;
    uint64_t carry = 0;
    for (int i = 0; i < nv; i++) {
      uint64_t pr = qhat * (uint64_t)V[i] + carry;
      carry = pr >> 32;
      int64_t t = (int64_t)U[i + j] - (int64_t)(uint32_t)pr - borrow;
      borrow = t < 0 ? 1 : 0;
      U[i + j] = (uint32_t)(t + (borrow << 32));
    }
    int64_t t = (int64_t)U[j + nv] - (int64_t)carry - borrow;
    borrow = t < 0 ? 1 : 0;
    U[j + nv] = (uint32_t)(t + (borrow << 32));
    if (borrow) {  // add back
      qhat -= 1;
      uint64_t c2 = 0;
      for (int i = 0; i < nv; i++) {
        uint64_t s2 = (uint64_t)U[i + j] + V[i] + c2;
        U[i + j] = (uint32_t)s2;
        c2 = s2 >> 32;
      }
      U[j + nv] = U[j + nv] + (uint32_t)c2;
    }
    Q[j] = (uint32_t)qhat;
  }
  for (int i = 0; i < nv; i++)
    if (U[i]) return true;
  return false;
}

// r = RN(a / b), b != 0.  tmp needs 3L + 8 words.
static __device__ bool div_rn(Ptr rm, int32_t* re, uint8_t* rc, const Val& a, const Val& b, int L, int p,
                       Ptr tmp) {
  int neg = neg_of(a.c) ^ neg_of(b.c);
  if (is_zero_cls(a.c)) {
    for (int l = 0; l < L; l++) rm[l] = 0;
    *re = 0;
    *rc = zero_cls(neg);
    return true;
  }
  // U = MA * 2^(32*kq) with kq limbs of extra quotient precision: quotient
  // MA*2^(32kq)/MB in (2^(32kq-1), 2^(32kq+1)), kq = ceil((p+2)/32)
  int kq = (p + 2 + 31) / 32;
  int nu = L + kq + 1;
  Ptr U = tmp;
  Ptr Q = tmp.off(nu);
  for (int k = 0; k < nu; k++) U[k] = (k >= kq && k < kq + L) ? a.m[k - kq] : 0u;
  bool rem = divrem_norm(Q, U, nu, b.m, L);
  int nq = nu - L;
  // value = Q * 2^(ea - eb - 32*kq)
  RoundOut ro = round_big(rm, L, p, CPtr{Q.p, Q.s}, nq, a.e - b.e - 32 * (int64_t)kq, rem);
  *re = (int32_t)ro.e;
  *rc = nz_cls(neg);
  return range_ok(ro.e);
}


// ------------------------------------------------------------- complex
// An exact term  (-1)^neg * M * 2^base  with M an n-limb integer (or zero).
struct XTerm {
  CPtr m;
  int n;
  int64_t base;
  int neg;
  bool zero;
};

// Result of an exact (windowed) sum.  pert = +1 / -1 when a term lay entirely
// below the window and was folded in as a magnitude perturbation (the true
// |value| is slightly larger / smaller than |S|), else 0.
struct XSum {
  int n;
  int64_t base;
  int neg;
  bool zero;
  int pert;
};

// S = X + (-1)^subY * Y exactly when the weight gap between the terms is at
// most `win_bits`; otherwise the smaller term becomes a perturbation.
// out needs nx + ny + win_bits/32 + 4 words.  Zero terms: IEEE zero-sum
// rules (x + y of signed zeros is -0 only if both are -0; exact nonzero
// cancellation gives +0).
static __device__ XSum exact_sum(Ptr out, XTerm X, XTerm Y, bool subY, int64_t win_bits) {
  XSum r;
  r.pert = 0;
  int sx = X.neg, sy = Y.neg ^ (subY ? 1 : 0);
  if (X.zero && Y.zero) {
    r.n = 0; r.base = 0; r.zero = true; r.neg = (sx && sy) ? 1 : 0;
    return r;
  }
  if (X.zero || Y.zero) {
    XTerm T = X.zero ? Y : X;
    int st = X.zero ? sy : sx;
    for (int k = 0; k < T.n; k++) out[k] = T.m[k];
    r.n = T.n; r.base = T.base; r.neg = st; r.zero = false;
    return r;
  }
  int64_t tx = X.base + top_bit(X.m, X.n), ty = Y.base + top_bit(Y.m, Y.n);
  if (tx < ty) {  // make X the term with the larger top weight
    XTerm T = X; X = Y; Y = T;
    int s = sx; sx = sy; sy = s;
    int64_t t = tx; tx = ty; ty = t;
  }
  if (tx - ty > win_bits) {  // Y far below X: perturbation only
    for (int k = 0; k < X.n; k++) out[k] = X.m[k];
    r.n = X.n; r.base = X.base; r.neg = sx; r.zero = false;
    r.pert = (sx == sy) ? 1 : -1;
    return r;
  }
  int64_t lo = X.base < Y.base ? X.base : Y.base;
  int64_t gx = X.base - lo, gy = Y.base - lo;
  int64_t bitsx = 32 * (int64_t)X.n + gx, bitsy = 32 * (int64_t)Y.n + gy;
  int n = (int)(((bitsx > bitsy ? bitsx : bitsy) + 31) / 32) + 1;
  if (sx == sy) {
    uint64_t carry = 0;
    for (int k = 0; k < n; k++) {
      uint64_t t = (uint64_t)bits32(X.m, X.n, 32 * (int64_t)k - gx) + bits32(Y.m, Y.n, 32 * (int64_t)k - gy) + carry;
      out[k] = (uint32_t)t;
      carry = t >> 32;
    }
    r.neg = sx;
  } else {
    int64_t borrow = 0;
    for (int k = 0; k < n; k++) {
      int64_t t = (int64_t)bits32(X.m, X.n, 32 * (int64_t)k - gx) - (int64_t)bits32(Y.m, Y.n, 32 * (int64_t)k - gy) - borrow;
      borrow = t < 0 ? 1 : 0;
      out[k] = (uint32_t)(t + (borrow << 32));
    }
    r.neg = sx;
    if (borrow) {  // negative: negate (two's complement)
      uint64_t c = 1;
      for (int k = 0; k < n; k++) {
        uint64_t t = (uint64_t)(uint32_t)~out[k] + c;
        out[k] = (uint32_t)t;
        c = t >> 32;
      }
      r.neg = sy;
    }
  }
  r.n = n; r.base = lo; r.zero = (top_bit(CPtr{out.p, out.s}, n) < 0);
  if (r.zero) r.neg = 0;  // exact cancellation -> +0
  return r;
}

// round an XSum to p bits (value = S * 2^base, perturbation-aware)
static __device__ bool round_xsum(Ptr rm, int32_t* re, uint8_t* rc, Ptr S, const XSum& x, int L, int p) {
  if (x.zero) {
    for (int l = 0; l < L; l++) rm[l] = 0;
    *re = 0;
    *rc = zero_cls(x.neg);
    return true;
  }
  bool sticky = false;
  if (x.pert != 0) {
    sticky = true;
    if (x.pert < 0) {  // |true| in (S - 1, S): use S - 1 with sticky
      for (int k = 0; k < x.n; k++) {
        uint32_t v = S[k];
        S[k] = v - 1u;
        if (v != 0) break;
      }
    }
  }
  RoundOut ro = round_big(rm, L, p, CPtr{S.p, S.s}, x.n, x.base, sticky);
  *re = (int32_t)ro.e;
  *rc = nz_cls(x.neg);
  return range_ok(ro.e);
}

static __device__ __forceinline__ XTerm prod_term(Ptr P, const Val& A, const Val& B, int L) {
  XTerm t;
  t.neg = neg_of(A.c) ^ neg_of(B.c);
  t.zero = is_zero_cls(A.c) || is_zero_cls(B.c);
  t.n = 2 * L;
  t.base = A.e + B.e - 64 * (int64_t)L;
  t.m = CPtr{P.p, P.s};
  if (!t.zero) mul_full(P, A.m, B.m, L);
  return t;
}

// r = RN(A*B -/+ C*D): one component of mpc_mul.  tmp: 8L + 8 words.
static __device__ bool cmul_part(Ptr rm, int32_t* re, uint8_t* rc, const Val& A, const Val& B, const Val& C,
                          const Val& D, bool sub, int L, int p, Ptr tmp) {
  XTerm x = prod_term(tmp, A, B, L);
  XTerm y = prod_term(tmp.off(2 * L), C, D, L);
  Ptr S = tmp.off(4 * L);
  // products have <= 2p bits: a term more than 2p+2 bits below the other's
  // top is below its LSB and only perturbs (exactness preserved by rounding)
  XSum s = exact_sum(S, x, y, sub, 2 * (int64_t)p + 4);
  return round_xsum(rm, re, rc, S, s, L, p);
}

// q = RN(N / D) for exact sums N (numerator) and D > 0.  Writes rm/re/rc.
// tmp: nN + nD + (p+2)/32 + 8 words (U, Q).
static __device__ bool div_xsum(Ptr rm, int32_t* re, uint8_t* rc, Ptr N, XSum xn, Ptr D, XSum xd, int L,
                         int p, Ptr tmp, unsigned int* warn) {
  if (xn.zero) {
    for (int l = 0; l < L; l++) rm[l] = 0;
    *re = 0;
    *rc = zero_cls(xn.neg ^ xd.neg);
    return true;
  }
  // trim D and normalize its top limb
  int nD = xd.n;
  while (nD > 0 && D[nD - 1] == 0) nD--;
  int s = __clz(D[nD - 1]);
  int64_t topN = top_bit(CPtr{N.p, N.s}, xn.n), topD = (int64_t)(nD - 1) * 32 + 31 - s;
  int64_t sh = (int64_t)p + 2 - (topN - topD);
  if (sh < 0) sh = 0;
  // U = N << (sh + s), one extra zero limb on top
  int64_t ubits = topN + 1 + sh + s;
  int nU = (int)((ubits + 31) / 32) + 1;
  if (nU <= nD) nU = nD + 1;
  Ptr U = tmp;
  Ptr Q = tmp.off(nU);
  for (int k = 0; k < nU; k++) U[k] = bits32(CPtr{N.p, N.s}, xn.n, 32 * (int64_t)k - (sh + s));
  // D <<= s in place (D is scratch owned by the caller)
  if (s) {
    for (int k = nD - 1; k >= 0; k--) {
      uint32_t hi = D[k] << s;
      uint32_t lo = k > 0 ? (D[k - 1] >> (32 - s)) : 0u;
      D[k] = hi | lo;
    }
  }
  bool rem = divrem_norm(Q, U, nU, CPtr{D.p, D.s}, nD);
  int nq = nU - nD;
  // perturbations: N larger (+1) -> q larger; D larger (+1) -> q smaller
  int pq = xn.pert;
  int pd = -xd.pert;
  int dir = pq != 0 ? pq : pd;
  if (pq != 0 && pd != 0 && pq != pd && warn) atomicAdd(warn, 1u);  // undecidable tie direction
  bool sticky = rem;
  if (!rem && dir != 0) {
    sticky = true;
    if (dir < 0) {
      for (int k = 0; k < nq; k++) {
        uint32_t v = Q[k];
        Q[k] = v - 1u;
        if (v != 0) break;
      }
    }
  } else if (dir != 0) {
    sticky = true;
  }
  RoundOut ro = round_big(rm, L, p, CPtr{Q.p, Q.s}, nq, xn.base - xd.base - sh, sticky);
  *re = (int32_t)ro.e;
  *rc = nz_cls(xn.neg ^ xd.neg);
  return range_ok(ro.e);
}

// window (in bits) inside which complex-division sums are kept exact
static __device__ __forceinline__ int64_t cdiv_window(int p) { return 4 * (int64_t)p + 64; }

// limbs of one exact-sum window in cdiv_part (terms of 2L limbs, gap <= win)
static __host__ __device__ __forceinline__ int cdiv_nwin(int L, int p) {
  return 4 * L + (int)((4 * (int64_t)p + 64) / 32) + 6;
}

// scratch words needed by cdiv_part: 4 products (8L) + N, D windows +
// U (<= nwin + L + 3) + Q (<= nwin + L)
static __host__ __device__ __forceinline__ int64_t cdiv_scratch_words(int L, int p) {
  return 8 * (int64_t)L + 4 * (int64_t)cdiv_nwin(L, p) + 2 * (int64_t)L + 64;
}

// One component of mpc_div:  re: (ar*br + ai*bi) / (br^2 + bi^2)
//                            im: (ai*br - ar*bi) / (br^2 + bi^2)
static __device__ bool cdiv_part(Ptr rm, int32_t* re, uint8_t* rc, const Val& ar, const Val& ai, const Val& br,
                          const Val& bi, bool imag, int L, int p, Ptr tmp, unsigned int* warn) {
  int64_t win = cdiv_window(p);
  int nwin = cdiv_nwin(L, p);
  Ptr P0 = tmp, P1 = tmp.off(2 * L), P2 = tmp.off(4 * L), P3 = tmp.off(6 * L);
  Ptr N = tmp.off(8 * L), D = N.off(nwin), rest = D.off(nwin);
  XTerm x, y;
  if (!imag) {
    x = prod_term(P0, ar, br, L);
    y = prod_term(P1, ai, bi, L);
  } else {
    x = prod_term(P0, ai, br, L);
    y = prod_term(P1, ar, bi, L);
  }
  XSum sn = exact_sum(N, x, y, imag, win);
  XTerm d1 = prod_term(P2, br, br, L);
  XTerm d2 = prod_term(P3, bi, bi, L);
  XSum sd = exact_sum(D, d1, d2, false, win);
  return div_xsum(rm, re, rc, N, sn, D, sd, L, p, rest, warn);
}

}  // namespace ds
