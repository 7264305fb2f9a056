// ds_cfinish.cuh -- warp-cooperative finish of the complex wide update
// (included by ds_tc.cu inside its anonymous namespace: uses TcArgs, TwArgs and
// finish_c_elem).
//
// The same integers and the same decisions as finish_c_elem, which restates
// mpc_mul's single rounding of zr br -/+ zi bi and then mpc_sub (elim.py:49-52 on
// mpc values), but one element per warp with its numbers in registers -- word i
// of a number in lane i mod 32, slot i / 32:
//   * carries cross lanes by carry lookahead on two ballots: with G (words that
//     carry out) and P (words that are all ones), the carries into the words are
//     (G + (G | P) + cin) ^ P;
//   * shifts by arbitrary bit counts read a per-warp shared-memory copy;
//   * top bits, all-ones / all-zeros ranges and sticky bits are warp votes.
// A block of 8 warps takes 8 consecutive elements: their product words and a's
// limbs arrive with block-wide asynchronous copies (cp.async; 8 elements x 4 words
// per warp instruction, whole 32-byte sectors) into one of two shared-memory stages
// -- the next group's copies run under this group's arithmetic -- and a's results
// leave the same way, so every global access is coalesced and nothing per element
// goes through global scratch.  Elements outside the fast shapes (both products of a component zero,
// a gap that makes one product a mere perturbation, sums or alignments wider than
// the registers, an a - t alignment past the registers) run finish_c_elem on lane
// 0, unchanged.  DS_CX_FINISH_THREAD=1 selects the thread-per-element kernel
// (A/B; tests/test_gpu_cfinish.py compares the two bit for bit); below ~1400 bits
// the thread kernel is the default (cf_k_for).

#ifndef DS_VAR_CF_STAGES
#define DS_VAR_CF_STAGES 1  // staging stages of k_cfw_finish: 1 measured faster than 2 (power N=1000 -2 %, 300 @8192 update -18 %; profiles/r02_cfinish_stages_ab.log)
#endif
#ifndef DS_VAR_CF_MINB
#define DS_VAR_CF_MINB 3    // k_cfw_finish blocks per SM the registers are capped for (K = 9: 2, measured
                            // -7 % update at 8192 bits; 3 stays best at 4096, profiles/r02_cfinish_stages_ab.log)
#endif
constexpr uint32_t CF_FULL = 0xffffffffu;
constexpr int CF_GE = 8;  // elements (warps) per block

// smallest m >= n with m == 4 (mod 32): the block loads write 8 elements x 4
// consecutive words per warp without bank conflicts
__host__ __device__ constexpr int cf_pad(int n) { return ((n + 27) & ~31) + 4; }

// bits [32 i + q0, 32 i + q0 + 32) of the n-word array s (shared memory), zero
// outside [0, 32 n): the warp-uniform offset q0 is split once into a word and a
// bit shift
struct CfShift {
  int wb;
  uint32_t sh;
};
__device__ __forceinline__ CfShift cf_shift(int64_t q0) { return CfShift{(int)(q0 >> 5), (uint32_t)(q0 & 31)}; }
__device__ __forceinline__ uint32_t cf_rd(const uint32_t* s, int n, int i, CfShift f) {
  const int w = i + f.wb;
  const uint32_t lo = (unsigned)w < (unsigned)n ? s[w] : 0u;
  const uint32_t hi = (unsigned)(w + 1) < (unsigned)n ? s[w + 1] : 0u;
  return __funnelshift_r(lo, hi, f.sh);
}
// a single bit q of the n-word array s
__device__ __forceinline__ uint32_t cf_bit(const uint32_t* s, int n, int64_t q) {
  const int64_t w = q >> 5;
  return (w >= 0 && w < n) ? (s[w] >> (q & 31)) & 1u : 0u;
}

// s = x + y + cin over K slots; returns the carry out of the top word
template <int K>
__device__ __forceinline__ uint32_t cf_add(uint32_t (&s)[K], const uint32_t (&x)[K], const uint32_t (&y)[K],
                                           uint32_t cin, int lane) {
#pragma unroll
  for (int j = 0; j < K; j++) {
    const uint32_t u = x[j] + y[j];
    const uint32_t G = __ballot_sync(CF_FULL, u < x[j]);
    const uint32_t P = __ballot_sync(CF_FULL, u == CF_FULL);
    const uint64_t t = (uint64_t)G + (uint64_t)(G | P) + cin;
    const uint32_t C = (uint32_t)t ^ P;  // bit t: carry into word 32 j + t
    cin = (uint32_t)(t >> 32);
    s[j] = u + ((C >> lane) & 1u);
  }
  return cin;
}

// highest set bit of the K-slot number, -1 if zero (warp-uniform)
template <int K>
__device__ __forceinline__ int64_t cf_top(const uint32_t (&s)[K]) {
#pragma unroll
  for (int j = K - 1; j >= 0; j--) {
    const uint32_t B = __ballot_sync(CF_FULL, s[j] != 0u);
    if (B) {
      const int hl = 31 - __clz(B);
      const uint32_t v = __shfl_sync(CF_FULL, s[j], hl);
      return ((int64_t)(32 * j + hl) << 5) + 31 - __clz(v);
    }
  }
  return -1;
}

// highest set bit of the n words at m (shared memory), -1 if zero (ds::top_bit);
// scanned from the top, 32 words per vote
__device__ __forceinline__ int64_t cf_top_sm(const uint32_t* m, int n, int lane) {
  for (int base = ((n - 1) >> 5) << 5; base >= 0; base -= 32) {
    const int i = base + lane;
    const uint32_t v = i < n ? m[i] : 0u;
    const uint32_t B = __ballot_sync(CF_FULL, v != 0u);
    if (B) {
      const int hl = 31 - __clz(B);
      const uint32_t x = __shfl_sync(CF_FULL, v, hl);
      return ((int64_t)(base + hl) << 5) + 31 - __clz(x);
    }
  }
  return -1;
}

// any bit of the n words at m (shared memory) below position q
__device__ __forceinline__ bool cf_any_sm(const uint32_t* m, int n, int64_t q, int lane) {
  const int64_t qw = q >> 5;
  const int full = (int)min((int64_t)n, max((int64_t)0, qw));
  bool any = false;
  for (int i = lane; i < full; i += 32) any = any || m[i] != 0u;
  if (lane == 0 && qw >= 0 && qw < n && (q & 31)) any = any || (m[qw] & ((1u << (q & 31)) - 1u)) != 0u;
  return __any_sync(CF_FULL, any);
}

// bits [lo, hi) (lo >= 0) of the K-slot number: all ones / none set (both true
// when the range is empty) -- bit_range of ds_tc.cu
template <int K>
__device__ __forceinline__ void cf_range(const uint32_t (&s)[K], int64_t lo, int64_t hi, int lane, bool* ones,
                                         bool* zeros) {
  constexpr int NB = 32 * 32 * K;
  const int l32 = (int)max((int64_t)0, min((int64_t)NB, lo)), h32 = (int)max((int64_t)0, min((int64_t)NB, hi));
  bool o = true, z = true;
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int b0 = (32 * j + lane) << 5;
    const int x0 = min(32, max(0, l32 - b0)), x1 = min(32, max(0, h32 - b0));
    if (x1 > x0) {
      const uint32_t m = (x1 == 32 ? CF_FULL : ((1u << x1) - 1u)) & ~((1u << x0) - 1u);
      const uint32_t v = s[j] & m;
      o = o && v == m;
      z = z && v == 0u;
    }
  }
  *ones = __all_sync(CF_FULL, o);
  *zeros = __all_sync(CF_FULL, z);
}

// any bit of the K-slot number below position q (ds::any_below)
template <int K>
__device__ __forceinline__ bool cf_any_below(const uint32_t (&s)[K], int64_t q, int lane) {
  constexpr int NB = 32 * 32 * K;
  const int q32 = (int)max((int64_t)0, min((int64_t)NB, q));
  bool any = false;
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int x1 = min(32, max(0, q32 - ((32 * j + lane) << 5)));
    if (x1 > 0) any = any || (s[j] & (x1 == 32 ? CF_FULL : ((1u << x1) - 1u))) != 0u;
  }
  return __any_sync(CF_FULL, any);
}

// ds::round_big of the K-slot number S (S != 0, top bit hb) to p bits, the true
// value lying in (S, S + 1) units when sticky_in: out[0..L) (shared memory) = the
// left-aligned mantissa.  Returns hb + 1, or
// hb + 2 when rounding carried out (the MPFR exponent minus S's base).  sb: this
// warp's 32 K-word staging area.
template <int K>
__device__ int64_t cf_round(const uint32_t (&S)[K], int64_t hb, int p, int L, uint32_t* sb, uint32_t* out,
                            int lane, bool sticky_in) {
  constexpr int n = 32 * K;
#pragma unroll
  for (int j = 0; j < K; j++) sb[32 * j + lane] = S[j];
  __syncwarp();
  const int64_t lsb = hb - p + 1;  // bit of S holding the result's LSB
  bool rbit = false, sticky = sticky_in;
  if (lsb - 1 >= 0) {
    rbit = cf_bit(sb, n, lsb - 1) != 0u;
    sticky = sticky || cf_any_below<K>(S, lsb - 1, lane);
  }
  const int64_t off = hb + 1 - 32 * (int64_t)L;  // mantissa bit j <-> S bit j + off
  const CfShift f = cf_shift(off);
  const int zb = 32 * L - p, zq = zb >> 5, zr = zb & 31;
  const uint32_t zmask = ~((1u << zr) - 1u);
  const bool lsbit = cf_bit(sb, n, lsb) != 0u;
  const bool inc = rbit && (sticky || lsbit);
  uint32_t M[K];
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int l = 32 * j + lane;
    uint32_t v = 0u;
    if (l < L && l >= zq) {
      v = cf_rd(sb, n, l, f);
      if (l == zq) v &= zmask;
    }
    M[j] = v;
  }
  int64_t e = hb + 1;
  if (inc) {
    uint32_t Y[K];
#pragma unroll
    for (int j = 0; j < K; j++) Y[j] = (32 * j + lane == zq) ? (1u << zr) : 0u;
    const uint32_t cout = cf_add<K>(M, M, Y, 0u, lane);
    bool top = false;  // the carry reached limb L
#pragma unroll
    for (int j = 0; j < K; j++) top = top || (32 * j + lane >= L && M[j] != 0u);
    if (__any_sync(CF_FULL, top) || cout) {  // mantissa overflowed to 2^p: 0.1000.. with e + 1
#pragma unroll
      for (int j = 0; j < K; j++) M[j] = (32 * j + lane == L - 1) ? 0x80000000u : 0u;
      e += 1;
    }
  }
  __syncwarp();  // every lane's staging reads are done before the caller reuses sb
#pragma unroll
  for (int j = 0; j < K; j++)
    if (32 * j + lane < L) out[32 * j + lane] = M[j];
  __syncwarp();
  return e;
}

struct CfTerm {
  const uint32_t* m;  // W words in shared memory
  int64_t base;
  int neg;
  bool zero;
  bool exact;         // no nonzero digit product below c_lo: the short product is the product
};

// T = RN(X +/- Y) -- ds::exact_sum, the error-bound test of finish_c_elem and
// ds::round_xsum.  Only the window of the sum above hi = the larger of the two
// bases is formed: below hi at most one term has bits, so they reach the window
// only as a borrow (when that term is subtracted) and as sticky bits, and every
// bit the decision and the rounding read lies above bnd > hi.  The window is at
// most W + 2 words whatever the gap between the terms (a term far below the other
// -- the perturbation case of exact_sum -- is just a borrow here; both formulations
// decide only when the rounding of the exact value is certain, so the results are
// the same bits).  Products whose omitted digit products are all zero (k_lowdig:
// low(z) + low(b) >= c_lo, e.g. a pivot row of small integers) carry no error: a
// sum of such terms is rounded directly.  Returns 0 (T written; a zero T has a zero class), 1 (undecided:
// fallback list).
template <int K>
__device__ int cf_xsum_round(const CfTerm& X, const CfTerm& Y, bool subY, int W, int eps, int p, int L,
                             uint32_t* sb, uint32_t* Tout, int32_t* te, uint8_t* tcl, bool* rng, int lane) {
  const int sx = X.neg, sy = Y.neg ^ (subY ? 1 : 0);
  if (X.zero && Y.zero) {  // IEEE: the sum of zeros is -0 only if both are -0
    *te = 0;
    *tcl = ds::zero_cls(sx && sy);
    *rng = true;
    return 0;
  }
  int64_t bnd = INT64_MIN;
  if (!X.zero && !X.exact) bnd = max(bnd, X.base + eps);
  if (!Y.zero && !Y.exact) bnd = max(bnd, Y.base + eps);
  const bool exact = bnd == INT64_MIN;  // the sum formed below is the exact value
  bnd += 1;  // both truncation errors together < 2^bnd
  const int64_t tx = X.zero ? INT64_MIN : X.base + cf_top_sm(X.m, W, lane);
  const int64_t ty = Y.zero ? INT64_MIN : Y.base + cf_top_sm(Y.m, W, lane);
  // A: the term with the larger top weight (or the only nonzero one)
  const bool swap = X.zero || (!Y.zero && tx < ty);
  const CfTerm& A = swap ? Y : X;
  const CfTerm& B = swap ? X : Y;
  const int sa = swap ? sy : sx, sbn = swap ? sx : sy;
  const bool single = X.zero || Y.zero;
  const int64_t hi = single ? A.base : max(A.base, B.base);
  // the term with bits below hi (if any) and whether it has any there
  const bool a_low = !single && A.base < hi, b_low = !single && B.base < hi;
  const bool low_nz = a_low ? cf_any_sm(A.m, W, hi - A.base, lane) : (b_low ? cf_any_sm(B.m, W, hi - B.base, lane)
                                                                             : false);
  uint32_t xa[K], yb[K], S[K];
  const CfShift fa = cf_shift(hi - A.base), fb = cf_shift(single ? 0 : hi - B.base);
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int i = 32 * j + lane;
    xa[j] = cf_rd(A.m, W, i, fa);
    yb[j] = single ? 0u : cf_rd(B.m, W, i, fb);
  }
  int neg = sa;
  if (single || sa == sbn) {
    cf_add<K>(S, xa, yb, 0u, lane);  // no carry from below hi: one term only there
  } else {
#pragma unroll
    for (int j = 0; j < K; j++) yb[j] = ~yb[j];
    if (!cf_add<K>(S, xa, yb, (b_low && low_nz) ? 0u : 1u, lane)) {  // |A| < |B|: B - A instead
#pragma unroll
      for (int j = 0; j < K; j++) {
        const uint32_t t = xa[j];
        xa[j] = ~yb[j];
        yb[j] = ~t;
      }
      cf_add<K>(S, xa, yb, (a_low && low_nz) ? 0u : 1u, lane);
      neg = sbn;
    }
  }
  const int64_t hS = cf_top<K>(S);
  if (hS < 0) return 1;  // the sum is below 2^hi: undecided (exact engine)
  const int64_t R = hi + hS - p + 1;  // weight of the result's LSB
  int64_t e;
  if (exact) {
    // exact products: round the exact sum (round bit in the window, sticky from the
    // window and the low term)
    if (R - 1 < hi) return 1;
    e = hi + cf_round<K>(S, hS, p, L, sb, Tout, lane, low_nz);
  } else {
    if (R - 1 <= bnd) return 1;
    bool ones, zeros;
    cf_range<K>(S, bnd - hi, R - 1 - hi, lane, &ones, &zeros);
    if (ones || zeros) return 1;
    // the bits checked above lie below the round bit and are not all zeros: sticky
    e = hi + cf_round<K>(S, hS, p, L, sb, Tout, lane, true);
  }
  *te = (int32_t)e;
  *tcl = ds::nz_cls(neg);
  *rng = ds::range_ok(e);
  return 0;
}

// compare |a| and |t| mantissas (L limbs each, shared memory) from the top
__device__ __forceinline__ int cf_cmp_sm(const uint32_t* Am, const uint32_t* Tm, int L, int lane) {
  for (int j = (L - 1) >> 5; j >= 0; j--) {
    const int l = 32 * j + lane;
    const uint32_t x = l < L ? Am[l] : 0u, y = l < L ? Tm[l] : 0u;
    const uint32_t B = __ballot_sync(CF_FULL, x != y);
    if (B) {
      const int hl = 31 - __clz(B);
      const uint32_t xs = __shfl_sync(CF_FULL, x, hl), ys = __shfl_sync(CF_FULL, y, hl);
      return xs > ys ? 1 : -1;
    }
  }
  return 0;
}

// a - t (ds::add_rn(a, t, negate_b)): what to do, decided before anything is written
struct CfSub {
  int mode;  // 1: +0, 2: a unchanged, 3: copy t with sign nx, 4: general, 5: zero with sign nx
  int nx;
  bool x_is_a, eff_sub;
  int w0;    // general: first word of X 2^d +/- Y kept in registers (the words below only borrow / stick)
  int64_t d, ey;
};

template <int K>
__device__ int cf_sub_plan(const uint32_t* Am, int64_t ea, uint8_t ca, const uint32_t* Tm, int64_t te, uint8_t tcl,
                           int L, int p, int lane, CfSub* s) {
  const int na = ds::neg_of(ca), nb = ds::neg_of(tcl) ^ 1;
  const bool za = ds::is_zero_cls(ca), zt = ds::is_zero_cls(tcl);
  if (zt) {  // a - 0: a, or a signed zero when a is zero too
    s->mode = za ? 5 : 2;
    s->nx = na && nb;
    return 0;
  }
  if (za) {  // the result is -t
    s->mode = 3;
    s->nx = nb;
    return 0;
  }
  const bool eff_sub = na != nb;
  const int c = ea != te ? (ea > te ? 1 : -1) : cf_cmp_sm(Am, Tm, L, lane);
  if (eff_sub && c == 0) {  // exact cancellation: +0 under RN
    s->mode = 1;
    return 0;
  }
  s->x_is_a = c >= 0;
  s->nx = c >= 0 ? na : nb;
  s->d = c >= 0 ? ea - te : te - ea;
  if (s->d >= (int64_t)p + 2) {  // the smaller operand is below a quarter ulp: RN = the larger
    s->mode = s->x_is_a ? 2 : 3;
    return 0;
  }
  // S = MX 2^d +/- MY has L + d/32 + 2 words; when that exceeds the registers keep
  // the words from two below X's lowest (the result's round bit is above them)
  const int n2 = L + (int)(s->d >> 5) + 2;
  s->w0 = n2 > 32 * K ? (int)max((int64_t)0, (s->d - 64) >> 5) : 0;
  if (n2 - s->w0 > 32 * K) return 2;
  s->mode = 4;
  s->eff_sub = eff_sub;
  s->ey = c >= 0 ? te : ea;
  return 0;
}

// apply a plan: Am / *ea / *ca updated; returns the exponent range check
template <int K>
__device__ bool cf_sub_apply(const CfSub& s, uint32_t* Am, int32_t* ea, uint8_t* ca, const uint32_t* Tm, int32_t te,
                             int L, int p, uint32_t* sb, int lane) {
  if (s.mode == 2) return true;
  if (s.mode != 4) {
    for (int l = lane; l < L; l += 32) Am[l] = s.mode == 3 ? Tm[l] : 0u;
    __syncwarp();
    *ea = s.mode == 3 ? te : 0;
    *ca = s.mode == 3 ? ds::nz_cls(s.nx) : (s.mode == 5 ? ds::zero_cls(s.nx) : (uint8_t)DS_CLS_PZERO);
    return true;
  }
  const uint32_t* X = s.x_is_a ? Am : Tm;
  const uint32_t* Y = s.x_is_a ? Tm : Am;
  // Y's words below w0 only borrow (subtraction) and stick: the true value is in
  // (S, S + 1) units of word w0 when any is nonzero
  const bool low_nz = s.w0 > 0 && cf_any_sm(Y, L, 32 * (int64_t)s.w0, lane);
  uint32_t xs[K], ys[K], S[K];
  const CfShift fd = cf_shift(32 * (int64_t)s.w0 - s.d);
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int i = 32 * j + lane, k = s.w0 + i;
    xs[j] = cf_rd(X, L, i, fd);  // MX 2^d
    ys[j] = k < L ? Y[k] : 0u;
  }
  if (s.eff_sub) {
#pragma unroll
    for (int j = 0; j < K; j++) ys[j] = ~ys[j];
    cf_add<K>(S, xs, ys, low_nz ? 0u : 1u, lane);  // MX 2^d > MY: no borrow out
  } else {
    cf_add<K>(S, xs, ys, 0u, lane);
  }
  __syncwarp();  // X / Y reads done: Am may be overwritten
  const int64_t hS = cf_top<K>(S);
  const int64_t e = s.ey - 32 * (int64_t)L + 32 * (int64_t)s.w0 + cf_round<K>(S, hS, p, L, sb, Am, lane, low_nz);
  *ea = (int32_t)e;
  *ca = ds::nz_cls(s.nx);
  return ds::range_ok(e);
}

// one element on one warp; returns true when a's staged limbs (Asu) changed
template <int K>
__device__ bool cf_element(const TcArgs& a, const TwArgs& w, int row_first, int ri, int cidx, const uint32_t* Tsu,
                           int64_t tstride, uint32_t* Asu, int64_t astride, uint32_t* wsb, int Lp, ds::Ptr Ssum,
                           ds::Ptr Tre, ds::Ptr Tim, ds::Ptr tmp, int lane) {
  const int L = a.L, p = a.p, W = w.W;
  const int k = a.kstart + cidx;
  const int zr = row_first + ri;
  const int jl = a.jl0 + zr;
  const int64_t idx = (int64_t)jl * a.n + k;
  int64_t ze[2], be[2];
  uint8_t zc[2], bc[2];
#pragma unroll
  for (int c = 0; c < 2; c++) {
    ze[c] = a.zexp[(int64_t)c * a.zstride + zr];
    zc[c] = a.zcls[(int64_t)c * a.zstride + zr];
    be[c] = a.bexp[(int64_t)c * a.n + k];
    bc[c] = a.bcls[(int64_t)c * a.n + k];
  }
  auto term = [&](int c1, int c2) -> CfTerm {
    CfTerm t;
    t.m = Tsu + (2 * c1 + c2) * tstride;
    t.base = ze[c1] + be[c2] - 64 * (int64_t)L + 32 * (int64_t)w.qlo;
    t.neg = (zc[c1] & 1) ^ (bc[c2] & 1);
    t.zero = zc[c1] >= DS_CLS_PZERO || bc[c2] >= DS_CLS_PZERO;
    t.exact = a.zlow[(int64_t)c1 * a.zstride + zr] + a.blow[(int64_t)c2 * a.n + k] >= w.c_lo;
    return t;
  };
  uint32_t* sb = wsb;
  uint32_t* Tb[2] = {wsb + 32 * K, wsb + 32 * K + Lp};
  int32_t te[2];
  uint8_t tcl[2];
  bool rng[2];
  int r = 0;
  for (int c = 0; c < 2 && r == 0; c++)
    r = c == 0 ? cf_xsum_round<K>(term(0, 0), term(1, 1), true, W, w.eps, p, L, sb, Tb[0], &te[0], &tcl[0], &rng[0],
                                  lane)
               : cf_xsum_round<K>(term(0, 1), term(1, 0), false, W, w.eps, p, L, sb, Tb[1], &te[1], &tcl[1],
                                  &rng[1], lane);
  int32_t ea[2];
  uint8_t ca[2];
  CfSub sp[2];
  for (int c = 0; c < 2 && r == 0; c++) {
    const int64_t mo = (int64_t)c * a.a_count + idx;
    ea[c] = a.a_exp[mo];
    ca[c] = a.a_cls[mo];
    r = cf_sub_plan<K>(Asu + c * astride, ea[c], ca[c], Tb[c], te[c], tcl[c], L, p, lane, &sp[c]);
  }
  if (r == 1) {
    if (lane == 0) {
      int slot = atomicAdd(a.fb_count, 1);
      if (slot < a.fb_cap) a.fb_list[slot] = make_int2(jl, k);
      else atomicAdd(&a.status[5], 1);
    }
    return false;
  }
  if (r == 2) {  // the thread engine on lane 0, over the staged limbs
    bool ok = false;
    if (lane == 0) {
      const ds::Ptr am[2] = {ds::Ptr{Asu, 1}, ds::Ptr{Asu + astride, 1}};
      ok = finish_c_elem(a, w, ri, cidx, row_first, Ssum, Tre, Tim, tmp, am);
    }
    return __shfl_sync(CF_FULL, ok ? 1 : 0, 0) != 0;
  }
  bool range = rng[0] && rng[1];
  for (int c = 0; c < 2; c++) {
    range = cf_sub_apply<K>(sp[c], Asu + c * astride, &ea[c], &ca[c], Tb[c], te[c], L, p, sb, lane) && range;
    if (lane == 0) {
      const int64_t mo = (int64_t)c * a.a_count + idx;
      a.a_exp[mo] = ea[c];
      a.a_cls[mo] = ca[c];
    }
  }
  if (!range && lane == 0) atomicAdd(&a.status[2], 1);
  return true;
}

// the element of group g0's slot u: row in the chunk, column index, a's index; false
// when the element is outside the launch or not updated
__device__ __forceinline__ bool cf_elem_at(const TcArgs& a, int row_first, int64_t total, int64_t e, int* ri,
                                           int* cidx, int64_t* idx) {
  if (e >= total) return false;
  *ri = (int)(e / a.ncols);
  *cidx = (int)(e - (int64_t)*ri * a.ncols);
  const int k = a.kstart + *cidx;
  *idx = (int64_t)(a.jl0 + row_first + *ri) * a.n + k;
  return !(k < a.kmin || k == a.skip_col || k >= a.n);
}

__device__ __forceinline__ void cf_cp4(uint32_t* sdst, const uint32_t* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}

template <int K>
__global__ void __launch_bounds__(256, K >= 9 ? 2 : DS_VAR_CF_MINB) k_cfw_finish(TcArgs a, TwArgs w, int row_first, uint32_t* scratch,
                                                       int64_t sstride) {
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  extern __shared__ __align__(16) uint32_t cfs[];
  __shared__ int s_dirty[2][CF_GE];
  const int L = a.L, W = w.W, Wp = cf_pad(W), Lp = cf_pad(L);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // two stages of [4][CF_GE][Wp] product words + [2][CF_GE][Lp] a limbs, then per warp
  // staging | T_re | T_im
  const int stage_words = 4 * CF_GE * Wp + 2 * CF_GE * Lp;
  uint32_t* wsb = cfs + DS_VAR_CF_STAGES * stage_words + warp * (32 * K + 2 * Lp);
  const int64_t total = (int64_t)w.nrows * a.ncols;
  const int64_t region = w.pstride * (int64_t)W;
  const int64_t gstep = (int64_t)gridDim.x * CF_GE;
  // legacy-path scratch of this warp (the layout of k_tcw_finish_c, slot = warp)
  uint32_t* srow = scratch + (int64_t)blockIdx.x * CF_GE + warp;
  const ds::Ptr Ssum{srow, sstride}, Tre{srow + (4 * (int64_t)L + 16) * sstride, sstride},
      Tim{srow + (5 * (int64_t)L + 16) * sstride, sstride}, tmp{srow + (6 * (int64_t)L + 16) * sstride, sstride};
  const int u = tid & 7, q0 = tid >> 3;  // block copies: element u, words q0 + 32 m
  // asynchronous copies of group g's words into stage st (cp.async: no registers, the
  // next group's copies run under this group's arithmetic)
  auto load = [&](int64_t g, int st) {
    int ri, cidx;
    int64_t idx;
    if (!cf_elem_at(a, row_first, total, g + u, &ri, &cidx, &idx)) return;
    uint32_t* Ts = cfs + st * stage_words;
    uint32_t* As = Ts + 4 * CF_GE * Wp;
    const uint32_t* src = w.tprod + (int64_t)ri * w.ncp + cidx + (int64_t)q0 * w.pstride;
    const int64_t step = 32 * w.pstride;
#pragma unroll
    for (int r = 0; r < 4; r++) {
      uint32_t* dst = Ts + (r * CF_GE + u) * Wp;
      const uint32_t* sp = src + r * region;
      for (int q = q0; q < W; q += 32, sp += step) cf_cp4(dst + q, sp);
    }
    const int64_t astep = 32 * a.a_count;
#pragma unroll
    for (int c = 0; c < 2; c++) {
      uint32_t* dst = As + (c * CF_GE + u) * Lp;
      const uint32_t* sp = a.a_limbs + (int64_t)c * L * a.a_count + idx + (int64_t)q0 * a.a_count;
      for (int l = q0; l < L; l += 32, sp += astep) cf_cp4(dst + l, sp);
    }
  };
  int64_t g0 = (int64_t)blockIdx.x * CF_GE;
#if DS_VAR_CF_STAGES == 2
  load(g0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
#endif
  for (int it = 0; g0 < total; g0 += gstep, it++) {
#if DS_VAR_CF_STAGES == 2
    const int st = it & 1;
    __syncthreads();  // every thread is done with stage st ^ 1 (group it - 1's stores)
    if (g0 + gstep < total) load(g0 + gstep, st ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // this group's copies have landed
#else
    const int st = 0;
    __syncthreads();  // every thread is done with the stage (the previous group's stores)
    load(g0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#endif
    __syncthreads();
    uint32_t* Ts = cfs + st * stage_words;
    uint32_t* As = Ts + 4 * CF_GE * Wp;
    {
      int ri, cidx;
      int64_t idx;
      bool dirty = false;
      if (cf_elem_at(a, row_first, total, g0 + warp, &ri, &cidx, &idx))
        dirty = cf_element<K>(a, w, row_first, ri, cidx, Ts + warp * Wp, (int64_t)CF_GE * Wp, As + warp * Lp,
                              (int64_t)CF_GE * Lp, wsb, Lp, Ssum, Tre, Tim, tmp, lane);
      if (lane == 0) s_dirty[st][warp] = dirty ? 1 : 0;
    }
    __syncthreads();
    {
      int ri, cidx;
      int64_t idx;
      if (s_dirty[st][u] && cf_elem_at(a, row_first, total, g0 + u, &ri, &cidx, &idx)) {
#pragma unroll
        for (int c = 0; c < 2; c++) {
          uint32_t* dp = a.a_limbs + (int64_t)c * L * a.a_count + idx + (int64_t)q0 * a.a_count;
          const uint32_t* src = As + (c * CF_GE + u) * Lp;
          const int64_t astep = 32 * a.a_count;
          for (int l = q0; l < L; l += 32, dp += astep) *dp = src[l];
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// words per lane for the finish of W-word products (0: the thread kernel).  Measured
// (N=1000 @1024, 800 @2000, 600 @3000, 500 @4096, 300 @8192 complex, update time, warp
// vs thread finish): 2.21 vs 1.26 s, 1.39 vs 1.43, 0.74 vs 1.09, 0.49 vs 0.97, 0.30 vs
// 0.70 -- so the K = 2 shapes (p up to ~1400 bits) keep the thread kernel unless
// force_warp (DS_CX_FINISH_WARP=1, tests).
inline int cf_k_for(int W, bool force_warp) {
  const int need = W + 17;  // >= 16 words of alignment room
  if (need <= 64) return force_warp ? 2 : 0;
  return need <= 96 ? 3 : need <= 160 ? 5 : need <= 288 ? 9 : 0;
}

inline size_t cf_smem(int K, int W, int L) {
  return sizeof(uint32_t) * (DS_VAR_CF_STAGES * ((size_t)4 * CF_GE * cf_pad(W) + (size_t)2 * CF_GE * cf_pad(L)) +
                             (size_t)CF_GE * (32 * K + 2 * cf_pad(L)));
}
