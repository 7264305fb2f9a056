// ds_stream.cuh -- the per-element rounding stream shared by the fused DFMA
// update (ds_update.cu) and the tensor-core update (ds_tc.cu):
//   product limbs (low -> high) -> Emit (round to the p-bit t, short-product
//   decision) -> SWin (exact aligned a -/+ t window with guard limb + sticky,
//   in shared memory) -> round_write (normalise, RN, coalesced store).
#pragma once
#include <stdint.h>
#include "../../include/detseries_b200.h"
#include "ds_carry.cuh"

#ifndef DS_VAR_TSKIP
#define DS_VAR_TSKIP 1
#endif

namespace dss {

// ------------------------------------------------------------ S window
// Exact aligned sum S = |X| -/+ |Y| of a and t on a window of L+2 limbs held
// in SHARED memory (limb w at S[w*nth]): limb 0 = guard, limbs 1..L = X's
// mantissa positions, limb L+1 = carry.  a's limbs were prefetched into
// limbs 1..L with cp.async while the product ran.  X is the operand with the
// larger exponent; Y is shifted right by dq limbs + dr bits; Y bits below the
// window become the sticky bit (effective subtraction borrows one guard ulp
// when sticky -- the standard round/sticky trick).
// shared-memory accesses by 32-bit shared address (LDS/STS; the window
// pointer would otherwise be generic after inlining through the structs)
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

struct SWin {
  uint32_t sa;  // shared address of window limb 0 of this thread
  uint32_t sb;  // byte stride between window limbs (4 * threads sharing the window array)
  int L;
  bool xa;     // X = a (Y = t) or X = t (Y = a)
  bool sub;    // effective subtraction
  bool yzero;  // Y == 0 (a == 0, or a pure product)
  int dq, dr;
  uint32_t prev;
  int q, w;
  uint32_t cb;
  bool sticky;
  uint32_t curA;
  // direct mode (single pass): the normalisation offset off = 32 obase + ors of
  // the result was predicted, so each window limb S_w is turned into the
  // truncated result limb l = w - obase - 1 (bits [off + 32 l, +32)) as soon as
  // it is produced and written in place to slot l + 1; S_0, S_1 (round/sticky
  // bits) and the last two S limbs (verification) are kept in registers
  bool single;
  int obase, ors;
  uint32_t sprev, sprev2, s0, s1;

  __device__ __forceinline__ void base(uint32_t* S, int nth) {
    sa = (uint32_t)__cvta_generic_to_shared(S);
    sb = 4u * (uint32_t)nth;
  }
  __device__ __forceinline__ uint32_t at(int wi) const { return sa + (uint32_t)wi * sb; }
  __device__ __forceinline__ uint32_t get(int wi) const {
    return (wi >= 0 && wi <= L + 1) ? lds32(at(wi)) : 0u;
  }
  __device__ __forceinline__ void set(int wi, uint32_t v) { sts32(at(wi), v); }
  // a limb l (0 <= l < L) lives in window slot l + 1 until overwritten
  __device__ __forceinline__ uint32_t aload(int l) const { return (l >= 0 && l < L) ? lds32(at(l + 1)) : 0u; }

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
    put(s);
  }

  __device__ __forceinline__ void put(uint32_t s) {
    if (single) {
      if (w == 0) s0 = s;
      if (w == 1) s1 = s;
      const int sl = w - obase;  // slot of result limb l = w - obase - 1 (0, L + 1: scratch)
      if (sl >= 0) set(sl, __funnelshift_r(sprev, s, ors));
      sprev2 = sprev;
      sprev = s;
    } else {
      set(w, s);
    }
    w++;
  }

  __device__ __forceinline__ uint32_t abits(int wi) {
    uint32_t nxt = aload(wi + dq);
    uint32_t v = dr ? ((curA >> dr) | (nxt << (32 - dr))) : curA;
    curA = nxt;
    return v;
  }

  // off >= 0: direct mode with the predicted normalisation offset (in-place windows only)
  __device__ void init(int L_, bool xa_, bool sub_, bool yzero_, int64_t shift, int off = -1) {
    L = L_; xa = xa_; sub = sub_; yzero = yzero_;
    if (shift > 32 * (int64_t)(L + 3)) shift = 32 * (int64_t)(L + 3);
    dq = (int)(shift >> 5);
    dr = (int)(shift & 31);
    prev = 0; q = 0; w = 0; cb = 0; sticky = false; curA = 0;
    single = off >= 0;
    obase = off >> 5;
    ors = off & 31;
    sprev = sprev2 = s0 = s1 = 0u;
    if (xa) {
      set(0, 0u);
      set(L + 1, 0u);
      return;
    }
    if (yzero) {
      emit(0u, 0u);
      return;
    }
    set(L + 1, 0u);  // a limb L (above a's top) reads as zero in the branch-free blocks
    int64_t below = 32 * (int64_t)(dq - 1) + dr;  // a bits [0, below) are under the window
    for (int l = 0; l < L && (int64_t)l * 32 < below; l++) {
      uint32_t v = aload(l);
      int64_t lim = below - 32 * (int64_t)l;
      if (lim < 32) v &= (1u << lim) - 1u;
      if (v) sticky = true;
    }
    curA = aload(dq - 1);
    emit(0u, abits(0));
  }

  __device__ __forceinline__ void push(uint32_t T) {
    if (xa) {
      int wq = q - dq;
      if (wq < 0) {
        if (q >= 1 && prev) sticky = true;
      } else {
        if (wq == 0 && dr > 0 && (prev & ((1u << dr) - 1u))) sticky = true;
        uint32_t Yb = dr ? ((prev >> dr) | (T << (32 - dr))) : prev;
        emit((wq >= 1 && wq <= L) ? lds32(at(wq)) : 0u, Yb);
      }
      prev = T;
      q++;
    } else {
      emit(T, yzero ? 0u : abits(w));
    }
  }

  __device__ void finish() {
    if (xa)
      while (w <= L + 1) push(0u);
  }

  // NL interior limbs of P -> T (funnel by orr, + carry) -> S window.
  // Preconditions (checked by the caller): T indices and window indices in
  // the interior, so no masking, sticky or range logic is needed.
  // One branch-free path for both operand orders (lanes of a warp differ in
  // xa / sub): X -/+ Y as X + (Y ^ m) + carry with PTX carry chains
  // (subtraction = add of the complement; the borrow is 1 - carry).
  // fz >= 0: this block starts at T_0 (q0 = 0): low fz = zb bits masked, the
  // round increment added at bit zb (as Emit::limb does for q = 0).
  // ALIGNED: t's limbs are whole P limbs (orr = 0, the tensor-core engine)
  template <int NL, bool ALIGNED = false>
  __device__ __forceinline__ void fast_block(uint32_t prevP, const uint32_t (&P)[NL], int orr, uint32_t& tcarry,
                                             int fz = -1) {
    uint32_t T[NL], Z[NL];
    uint32_t pp = prevP;
#pragma unroll
    for (int k = 0; k < NL; k++) {
      T[k] = ALIGNED ? pp : __funnelshift_r(pp, P[k], orr);  // orr = 0: funnel(lo, hi, 0) = lo
      Z[k] = 0u;
      pp = P[k];
    }
    uint32_t tc = tcarry;
    if (fz >= 0) {
      T[0] &= ~((1u << fz) - 1u);
      Z[0] = tcarry << fz;
      tc = 0u;
    }
    // the round increment propagates through t's limbs only while they are all ones:
    // past the first block this chain is idle for (almost) every lane
#if DS_VAR_TSKIP
    if (fz >= 0 || tc) {
      addc_n<NL>(T, T, Z, tc);
      tcarry = tc;
    }
#else
    addc_n<NL>(T, T, Z, tc);
    tcarry = tc;
#endif
    // X = a (slot w+k) or T;  Y stream = T (xa) or a limbs (slot w+k+dq+1)
    const uint32_t ad0 = at(w + (xa ? 0 : dq + 1));
    uint32_t Ld[NL];
#pragma unroll
    for (int k = 0; k < NL; k++) Ld[k] = lds32(ad0 + (uint32_t)k * sb);  // all loads first (ILP)
    const uint32_t m = sub ? 0xffffffffu : 0u;
    uint32_t yp = xa ? prev : curA;
    uint32_t X[NL], Y[NL];
#pragma unroll
    for (int k = 0; k < NL; k++) {
      uint32_t yh = xa ? T[k] : Ld[k];
      Y[k] = __funnelshift_r(yp, yh, dr) ^ m;
      yp = yh;
      X[k] = xa ? Ld[k] : T[k];
    }
    uint32_t cy = sub ? (cb ^ 1u) : cb;
    addc_n<NL>(X, X, Y, cy);
    cb = sub ? (cy ^ 1u) : cy;
    if (single && w <= 1) {  // keep S_0, S_1 for the rounding bits
#pragma unroll
      for (int k = 0; k < NL; k++) {
        if (w + k == 0) s0 = X[k];
        if (w + k == 1) s1 = X[k];
      }
    }
    // store S_w (two-pass) or the shifted result limb w - obase - 1 to slot
    // w - obase (direct mode).  Slots 0 and L + 1 are scratch by then (their
    // X / a reads happened earlier or in this block's loads), so the only write
    // to skip is slot -1 (first block, obase 1).
    const uint32_t adw = at(single ? w - obase : w);
    const bool skip0 = single && w < obase;
    const int rse = single ? ors : 32;  // clamped funnel: shift 32 gives S_w itself (two-pass lanes)
    uint32_t sp = sprev;
#pragma unroll
    for (int k = 0; k < NL; k++) {
      const uint32_t v = __funnelshift_rc(sp, X[k], rse);
      if (k > 0 || !skip0) sts32(adw + (uint32_t)k * sb, v);
      sp = X[k];
    }
    sprev2 = NL >= 2 ? X[NL - 2] : sprev;
    sprev = X[NL - 1];
    w += NL;
    if (xa) {
      prev = yp;
      q += NL;
    } else {
      curA = yp;
    }
  }
};

// ------------------------------------------------------------ limb consumers
// The product arrives low -> high as 32-bit limbs of P (blocks of W digits
// starting at a column c0 = 0 mod 4 are exactly 3W/4 whole limbs).
// Top-bit probe (exact dry product): is bit 2p-1 of P set?
struct DryTop {
  int bitpos;
  int top;
  __device__ __forceinline__ bool limb(int g, uint32_t v) {
    if ((bitpos >> 5) == g) top = (v >> (bitpos & 31)) & 1u;
    return true;
  }
  template <int NL, bool ALIGNED = false>
  __device__ __forceinline__ bool block(int g0, const uint32_t (&P)[NL]) {
#pragma unroll
    for (int k = 0; k < NL; k++) limb(g0 + k, P[k]);
    return true;
  }
  __device__ __forceinline__ bool finish(double) { return true; }
};

// Rounds P = z*b to the p-bit t (P bit r = t's LSB) and streams t's
// left-aligned limbs T_0..T_{L-1} (+ overflow limb T_L) into the S window.
// T_q = P bits [o + 32q, o + 32q + 32) = funnel(P_{g-1}, P_g, orr) with
// g = q + oq + 1, o = r - zb; low zb bits of T_0 masked, the round increment
// added at bit zb of T_0.  Blocks arrive as NL = 3W/4 whole limbs; blocks
// after the decision that lie in the interior of the T and S ranges take a
// branch-free path (funnel shifts + carry chains in shared memory).
struct Emit {
  SWin* S;
  int r, zb, p, L, o, oq, orr;
  bool exact;
  bool onesided;       // omitted low part E >= 0 (unsigned digits) instead of |E| < 2^eps
  int lo_chk, hi_chk;  // short-product decision region [lo_chk, hi_chk]
  bool allz, allo, sticky, decided, excess;
  uint32_t rbit, tcarry, prevP, prevT;
  int tl, gtop, gn;
  int glo, ghi;  // blocks starting at limb g0 in [glo, ghi] are interior (see block)

  // call after S->init; NL = limbs per block the producer delivers
  template <int NL>
  __device__ __forceinline__ void setup() {
    o = r - zb;
    oq = o >> 5;
    orr = o & 31;
    prevP = 0;
    prevT = 0;
    gn = 0;
    gtop = (r + p + 31) >> 5;
    // interior: T indices q0 = g0 - oq - 1 with [q0, q0+NL) inside [1, L), and
    // the S window slots inside [1, L]:  xa: q0 - dq >= 1, q0 - dq + NL <= L;
    // otherwise a limbs read up to q0 + dq + NL stay below L
    // q0 = 0 (T_0, masked + round increment) is interior when nothing of t falls
    // below the window: non-xa, or xa with dq = 0 (T_0 lands in the guard slot).
    // Non-xa reads a limbs up to slot q0 + dq + NL + 1 <= L + 1 (slot L + 1 = 0).
    int qlo = 0, qhi = L - NL;
    if (S->xa) {
      qlo = S->dq == 0 ? 0 : 1 + S->dq;
    } else if (S->yzero) {
      qhi = -1;  // no a limbs in the window (pure products, a = 0): generic path
    } else {
      qhi = L - NL - S->dq;
    }
    glo = qlo + oq + 1;
    ghi = qhi + oq + 1;
  }

  __device__ __forceinline__ bool decide_limb(int g, uint32_t v) {
    const int lo = 32 * g;
    if (lo < r) {
      int rb = r - 1 - lo;
      if (rb >= 0 && rb < 32) rbit = (v >> rb) & 1u;
      if (exact) {
        uint32_t below = rb >= 32 ? v : (rb > 0 ? (v & ((1u << rb) - 1u)) : 0u);
        if (below) sticky = true;
      } else {
        int a0 = lo > lo_chk ? lo : lo_chk;
        int a1 = (lo + 31) < hi_chk ? (lo + 31) : hi_chk;
        if (a1 >= a0) {
          int len = a1 - a0 + 1;
          uint32_t m = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
          uint32_t bits = (v >> (a0 - lo)) & m;
          allz &= bits == 0u;
          allo &= bits == m;
        }
      }
    }
    if (r >= lo && r < lo + 32) {  // limb holding t's LSB: decide
      uint32_t lsb = (v >> (r - lo)) & 1u;
      if (exact) {
        tcarry = rbit & ((sticky ? 1u : 0u) | lsb);
      } else {
        if (onesided ? (allo || (rbit && allz)) : (allz || allo)) return false;  // undecided
        tcarry = rbit;
      }
      decided = true;
    }
    return true;
  }

  // general path for one P limb
  __device__ __forceinline__ bool limb(int g, uint32_t v) {
    gn = g + 1;
    if (!decided && !decide_limb(g, v)) return false;
    int q = g - oq - 1;
    if (q >= 0 && q < L) {
      uint32_t t = __funnelshift_r(prevP, v, orr);
      uint32_t add = tcarry;
      if (q == 0) {
        if (zb) t &= ~((1u << zb) - 1u);
        add <<= zb;
      }
      uint32_t s = t + add;
      tcarry = (s < t) ? 1u : 0u;
      S->push(s);
      tl = q + 1;
    } else if (q >= L) {
      if (__funnelshift_r(prevP, v, orr)) excess = true;  // bits >= r + p must be zero
    }
    prevP = v;
    return true;
  }

  template <int NL, bool ALIGNED = false>
  __device__ __forceinline__ bool block(int g0, const uint32_t (&P)[NL]) {
    const int q0 = g0 - oq - 1;
    // interior fast path (bounds from setup<NL>)
    if (!(decided && g0 >= glo && g0 <= ghi)) {
#pragma unroll
      for (int k = 0; k < NL; k++)
        if (!limb(g0 + k, P[k])) return false;
      return true;
    }
    gn = g0 + NL;
    S->fast_block<NL, ALIGNED>(prevP, P, orr, tcarry, q0 == 0 ? zb : -1);
    prevP = P[NL - 1];
    tl = q0 + NL;
    return true;
  }

  __device__ __forceinline__ bool finish(double carry) {
    if (carry != 0.0) excess = true;
    for (int guard = 0; tl < L && guard < L + 4; guard++) limb(gn, 0u);
    if (tl != L) excess = true;
    S->push(tcarry);  // overflow limb T_L (t rounded up to 2^p)
    S->finish();
    return true;
  }
};


// Normalise the S window, round to nearest-even at p bits and write the
// left-aligned result limbs, exponent and class.  E is the exponent of the
// window's X operand.  INPLACE: result limb l goes to window slot l + 1 (the
// slots a's limbs were loaded into; a tile store writes them back), else to
// O[l*so] in global memory (coalesced across a warp).
// A negative window (X < Y: only possible when the exponents are equal) is
// negated on the fly: -S = ~S + 1, where the +1 only reaches the limbs up to
// the lowest nonzero one (z0); above it -S_w = ~S_w.
template <bool INPLACE>
__device__ __forceinline__ void round_out(SWin& S, int neg, int64_t E, int L, int p, int zb, uint32_t* O,
                                          int64_t so, int32_t* oexp, uint8_t* ocls, int32_t* status) {
  const uint32_t sb = S.sb;
  // ---- sign: a negative window is read as ~slot (mneg); the limbs up to the
  // lowest nonzero one z0 are fixed up so that ~slot = -S there too:
  // slot z0 <- S_z0 - 1 (= ~(-S_z0)), slots below <- ~0 (-S_w = 0)
  uint32_t mneg = 0u;
  if (S.sub && S.cb) {
    neg ^= 1;
    mneg = 0xffffffffu;
    int z0 = 0;
    while (z0 <= L + 1) {
      uint32_t v = lds32(S.at(z0));
      if (v) {
        sts32(S.at(z0), v - 1u);
        break;
      }
      sts32(S.at(z0), 0xffffffffu);
      z0++;
    }
  }
  auto get = [&](int w) -> uint32_t { return (w >= 0 && w <= L + 1) ? (lds32(S.at(w)) ^ mneg) : 0u; };
  int h = -1;
  for (int wi = L + 1; wi >= 0; wi--) {
    uint32_t v = get(wi);
    if (v) {
      h = 32 * wi + 31 - __clz(v);
      break;
    }
  }
  if (h < 0) {  // exact cancellation -> +0
    for (int l = 0; l < L; l++) {
      if (INPLACE) sts32(S.at(l + 1), 0u);
      else O[(int64_t)l * so] = 0u;
    }
    *oexp = 0;
    *ocls = DS_CLS_PZERO;
    return;
  }
  int64_t e = E - 32 * (int64_t)L - 31 + h;
  int off = h - 32 * L + 1;
  if (off < 0) {  // massive cancellation: move the window up by whole limbs
    if (mneg) {  // materialise |S| first (rare)
      for (int wi = 0; wi <= L + 1; wi++) sts32(S.at(wi), get(wi));
      mneg = 0u;
    }
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
    rbit = (get(rb >> 5) >> (rb & 31)) & 1u;
    for (int wi = 0; wi < (rb >> 5) && !stk; wi++)
      if (get(wi)) stk = true;
    if (!stk && (rb & 31) && (get(rb >> 5) & ((1u << (rb & 31)) - 1u))) stk = true;
  }
  uint32_t lsb = (lsbw >= 0) ? ((get(lsbw >> 5) >> (lsbw & 31)) & 1u) : 0u;
  uint32_t carry = rbit & ((stk ? 1u : 0u) | lsb);
  // 0 <= off <= 33 here, so base = off >> 5 is 0 or 1 and the window limbs
  // base + l + 1 (l < L) stay inside [0, L + 1]; in place, slot l + 1 is
  // written only after slots base + l, base + l + 1 were read
  const int base = off >> 5, rs = off & 31;
  uint32_t ad = S.at(base);
  uint32_t lo = lds32(ad) ^ mneg;
  ad += sb;
  uint32_t first;
  {
    uint32_t hi = lds32(ad) ^ mneg;
    ad += sb;
    uint32_t v = __funnelshift_r(lo, hi, rs);
    lo = hi;
    if (zb) v &= ~((1u << zb) - 1u);
    uint32_t add = carry << zb;
    uint32_t rr = v + add;
    carry = rr < v ? 1u : 0u;
    first = rr;
  }
  if (INPLACE) sts32(S.at(1), first);
  else O[0] = first;
  uint32_t* Op = O + so;
  uint32_t wa = S.at(2);
  int l = 1;
  for (; l + 4 <= L; l += 4) {
    uint32_t h4[4], v4[4];
    const uint32_t z4[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 4; k++) h4[k] = lds32(ad + (uint32_t)k * sb) ^ mneg;
    ad += 4 * sb;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      v4[k] = __funnelshift_r(lo, h4[k], rs);
      lo = h4[k];
    }
    addc4(v4, v4, z4, carry);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (INPLACE) {
        sts32(wa, v4[k]);
        wa += sb;
      } else {
        *Op = v4[k];
        Op += so;
      }
    }
  }
  for (; l < L; l++) {
    uint32_t hi = lds32(ad) ^ mneg;
    ad += sb;
    uint32_t v = __funnelshift_r(lo, hi, rs);
    lo = hi;
    uint32_t rr = v + carry;
    carry = rr < v ? 1u : 0u;
    if (INPLACE) {
      sts32(wa, rr);
      wa += sb;
    } else {
      *Op = rr;
      Op += so;
    }
  }
  if (carry) {
    if (INPLACE) sts32(S.at(L), 0x80000000u);
    else O[(int64_t)(L - 1) * so] = 0x80000000u;
    e += 1;
  }
  if (e < DS_EMIN || e > DS_EMAX) atomicAdd(&status[2], 1);
  *oexp = (int32_t)e;
  *ocls = neg ? DS_CLS_NEG : DS_CLS_POS;
}

// Direct mode finish: the truncated result limbs are already in slots 1..L.
// Verify the predicted normalisation (nonnegative window, MSB of the top limb
// set, nothing above it), round to nearest-even at p bits (round bit / sticky
// from S_0, S_1 and the low result limb, carry propagated while it lasts) and
// write exponent and class.  Returns false on a misprediction (the caller puts
// a back and hands the element to the exact fallback).
__device__ __forceinline__ bool round_direct(SWin& S, int neg, int64_t E, int L, int p, int zb, int32_t* oexp,
                                             uint8_t* ocls, int32_t* status) {
  const int off = 32 * S.obase + S.ors;
  if (S.sub && S.cb) return false;                       // negative window
  const uint32_t top = lds32(S.at(L));
  if (!(top >> 31)) return false;                         // normalised lower than predicted
  // bits at or above window bit off + 32 L: S_{obase+L} >> ors and, for obase 0, S_{L+1}
  const uint32_t s_hi = S.obase ? S.sprev : S.sprev2;     // S_{obase + L}
  if (S.ors ? (s_hi >> S.ors) : s_hi) return false;
  if (S.obase == 0 && S.sprev) return false;
  uint32_t out0 = lds32(S.at(1));
  // round bit = window bit off + zb - 1, sticky = the bits below it (+ S.sticky)
  uint32_t rbit;
  bool stk = S.sticky;
  if (zb >= 1) {
    rbit = (out0 >> (zb - 1)) & 1u;
    if (zb >= 2 && (out0 & ((1u << (zb - 1)) - 1u))) stk = true;
    // window bits [0, off): S_0 and the low off - 32 bits of S_1
    if (off >= 32) {
      if (S.s0 || (off > 32 && (S.s1 & ((off - 32 >= 32) ? 0xffffffffu : ((1u << (off - 32)) - 1u))))) stk = true;
    } else if (off > 0 && (S.s0 & ((1u << off) - 1u))) {
      stk = true;
    }
  } else {
    // zb = 0: round bit = window bit off - 1, sticky = window bits [0, off - 1)
    const int rb = off - 1;
    if (rb < 0) {
      rbit = 0u;
    } else if (rb < 32) {
      rbit = (S.s0 >> rb) & 1u;
      if (rb > 0 && (S.s0 & ((1u << rb) - 1u))) stk = true;
    } else {
      rbit = (S.s1 >> (rb - 32)) & 1u;
      if (S.s0 || (rb > 32 && (S.s1 & ((1u << (rb - 32)) - 1u)))) stk = true;
    }
  }
  const uint32_t lsb = (out0 >> zb) & 1u;
  uint32_t carry = rbit & ((stk ? 1u : 0u) | lsb);
  if (zb) out0 &= ~((1u << zb) - 1u);
  uint32_t r0 = out0 + (carry << zb);
  carry = r0 < out0 ? 1u : 0u;
  sts32(S.at(1), r0);
  for (int l = 1; l < L && carry; l++) {  // usually stops at once
    const uint32_t a2 = S.at(l + 1);
    const uint32_t v = lds32(a2) + 1u;
    sts32(a2, v);
    carry = v == 0u ? 1u : 0u;
  }
  int64_t e = E + off - 32;
  if (carry) {  // rounded up to 2^p
    sts32(S.at(L), 0x80000000u);
    e += 1;
  }
  if (e < DS_EMIN || e > DS_EMAX) atomicAdd(&status[2], 1);
  *oexp = (int32_t)e;
  *ocls = neg ? DS_CLS_NEG : DS_CLS_POS;
  return true;
}

__device__ __forceinline__ void round_write(SWin& S, int neg, int64_t E, int L, int p, int zb, uint32_t* O,
                                            int64_t so, int32_t* oexp, uint8_t* ocls, int32_t* status) {
  round_out<false>(S, neg, E, L, p, zb, O, so, oexp, ocls, status);
}

}  // namespace dss
