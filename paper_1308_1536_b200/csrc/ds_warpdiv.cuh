// ds_warpdiv.cuh -- warp-cooperative correctly rounded real division
//     q = RN_p(a / b)        (mpfr_div, elim.py:47 and elim.py:148)
//
// One warp per quotient.  Knuth algorithm D on 32-bit limbs held in shared
// memory: each lane owns K = ceil(L/32) consecutive limbs of the divisor (in
// registers) and of the running remainder window; the per-digit
// multiply-subtract runs lane-locally, and the 1-bit carries/borrows between
// lanes are resolved with a ballot carry-lookahead:
//     carry into lane i = bit i of ((G|P) + G + cin) ^ P
// (G = lanes that generate, P = lanes that propagate).  The quotient gets
// kq = ceil((p+2)/32) limbs, the remainder gives the sticky bit, and the
// rounding to p bits (ties to even) is lane-parallel too.  Cost per quotient
// ~ (L+2) digits x O(K) lane ops, vs O(L^2) serial for one thread.
#pragma once
#include <stdint.h>
#include "../../include/detseries_b200.h"
#include "ds_carry.cuh"

namespace dsw {

constexpr unsigned FULL = 0xffffffffu;

// 1-bit carry lookahead across lanes for a lane-local "add with carry-in"
// where lane value g (generate) / p (propagate) are known.  Returns the carry
// into this lane and updates cio (carry into the chunk -> carry out of the
// `nvalid` lowest lanes).
__device__ __forceinline__ uint32_t cla(bool g, bool p, uint32_t& cio, int nvalid) {
  const int lane = threadIdx.x & 31;
  unsigned G = __ballot_sync(FULL, g);
  unsigned P = __ballot_sync(FULL, p);
  uint64_t S = (uint64_t)(G | P) + G + cio;
  uint64_t C = S ^ (uint64_t)P;
  cio = (uint32_t)((C >> nvalid) & 1u);
  return (uint32_t)((C >> lane) & 1u);
}

// Knuth D: Q = floor(U / V), remainder left in U[0..n).  U has nu limbs (top
// limb zero), V has n limbs with the MSB of V[n-1] set; the lane-blocked copy
// vb[] (lane t holds V[t*K .. t*K+K)) lives in registers.  Q gets nu-n limbs.
// Returns true when the remainder is nonzero.
// padded U index (one pad word per 32): conflict-free lane blocks
__host__ __device__ __forceinline__ int upad(int i) { return i + (i >> 5); }
// words of a padded U of nu limbs
__host__ __device__ __forceinline__ int upad_words(int nu) { return nu + (nu >> 5) + 1; }

template <int K>
__device__ bool wdivrem(uint32_t* Q, uint32_t* U, int nu, const uint32_t* V, const uint32_t (&vb)[K], int n) {
  const int lane = threadIdx.x & 31;
  // U is stored padded (one word after every 32, upad) so that the lanes'
  // K-limb blocks fall in distinct banks
#define UP(i) U[upad(i)]
  const uint64_t vtop = V[n - 1];
  const uint64_t vnext = V[n - 2];
  const double vinv = 1.0 / (double)vtop;  // vtop >= 2^31: the estimate below is within 1 of num / vtop
  for (int j = nu - n - 1; j >= 0; j--) {
    uint64_t num = ((uint64_t)UP(j + n) << 32) | UP(j + n - 1);
    // qhat = min(floor(num / vtop), 2^32 - 1): double estimate + exact correction
    uint64_t qhat = (uint64_t)((double)num * vinv);
    if (qhat > 0x1ffffffffull) qhat = 0x1ffffffffull;
    int64_t rr = (int64_t)(num - qhat * vtop);
    while (rr < 0) {
      qhat -= 1;
      rr += (int64_t)vtop;
    }
    while (rr >= (int64_t)vtop) {
      qhat += 1;
      rr -= (int64_t)vtop;
    }
    if (qhat > 0xffffffffull) qhat = 0xffffffffull;
    uint64_t rhat = num - qhat * vtop;
    while (rhat < (1ull << 32) && qhat * vnext > ((rhat << 32) | (uint64_t)UP(j + n - 2))) {
      qhat -= 1;
      rhat += vtop;
    }
    // lane-local product block qhat * V_blk: K limbs + 32-bit carry out h
    uint32_t pb[K];
    uint64_t h = 0;
#pragma unroll
    for (int u = 0; u < K; u++) {
      uint64_t t = qhat * (uint64_t)vb[u] + h;
      pb[u] = (uint32_t)t;
      h = t >> 32;
    }
    // add the previous lane's carry word at the bottom of this block (carry chain)
    uint32_t hin = __shfl_up_sync(FULL, (uint32_t)h, 1);
    if (lane == 0) hin = 0;
    uint32_t zk[K], mk[K];
#pragma unroll
    for (int u = 0; u < K; u++) zk[u] = 0u;
    zk[0] = hin;
    uint32_t ov = 0;
    dss::addc_n<K>(pb, pb, zk, ov);
    uint32_t andv = pb[0];
#pragma unroll
    for (int u = 1; u < K; u++) andv &= pb[u];
    const bool allones = andv == 0xffffffffu;
    // carries of the block additions between lanes (product is < 2^(32(n+1)))
    uint32_t cio = 0;
    uint32_t c = cla(ov != 0, allones && ov == 0, cio, 32);
#pragma unroll
    for (int u = 0; u < K; u++) zk[u] = 0u;
    dss::addc_n<K>(pb, pb, zk, c);  // + carry-in from the lane below
    // product top limb: last lane's carry word + carry out of the lane chain
    uint32_t htop = __shfl_sync(FULL, (uint32_t)h, 31) + cio;
    // subtract the block from U[j + lane*K ..]: U + ~pb + 1 (carry chain; borrow = 1 - carry)
    const int ub0 = j + lane * K;
    uint32_t ub[K];
#pragma unroll
    for (int u = 0; u < K; u++) {
      ub[u] = UP(ub0 + u);
      mk[u] = ~pb[u];
    }
    uint32_t cy = 1u;
    dss::addc_n<K>(ub, ub, mk, cy);
    const uint32_t bo = cy ^ 1u;  // lane-local borrow
    uint32_t orv = ub[0];
#pragma unroll
    for (int u = 1; u < K; u++) orv |= ub[u];
    const bool allzero = orv == 0u;
    uint32_t bio = 0;
    uint32_t b = cla(bo != 0, allzero && bo == 0, bio, 32);
    // borrow-in from the lane below: ub - b = ub + (b ? ~0 : 0) over the K limbs
#pragma unroll
    for (int u = 0; u < K; u++) mk[u] = b ? 0xffffffffu : 0u;
    uint32_t c0 = 0u;
    dss::addc_n<K>(ub, ub, mk, c0);
#pragma unroll
    for (int u = 0; u < K; u++) UP(ub0 + u) = ub[u];
    __syncwarp();
    // top limb U[j + 32K] (= U[j+n] when n == 32K; the zero-padded tail of V
    // makes the blocks cover n limbs exactly when n < 32K as well)
    int top = j + 32 * K;
    uint64_t ytop = (uint64_t)htop + bio;
    uint32_t utop = UP(top);
    bool neg = (uint64_t)utop < ytop;
    __syncwarp();
    if (lane == 0) UP(top) = (uint32_t)((uint64_t)utop - ytop);
    __syncwarp();
    if (neg) {  // add V back (rare): U[j .. j+32K] += V
      qhat -= 1;
      uint32_t a2[K];
      uint32_t co = 0;
#pragma unroll
      for (int u = 0; u < K; u++) {
        uint64_t t = (uint64_t)UP(ub0 + u) + vb[u] + co;
        a2[u] = (uint32_t)t;
        co = (uint32_t)(t >> 32);
      }
      bool ao = true;
#pragma unroll
      for (int u = 0; u < K; u++) ao &= (a2[u] == 0xffffffffu);
      uint32_t cio2 = 0;
      uint32_t c2 = cla(co != 0, ao && co == 0, cio2, 32);
      if (c2) {
#pragma unroll
        for (int u = 0; u < K; u++) {
          a2[u] += 1u;
          if (a2[u] != 0) break;
        }
      }
#pragma unroll
      for (int u = 0; u < K; u++) UP(ub0 + u) = a2[u];
      __syncwarp();
      if (lane == 0) UP(top) += cio2;
      __syncwarp();
    }
    if (lane == 0) Q[j] = (uint32_t)qhat;
    __syncwarp();
  }
  bool nz = false;
  for (int i = lane; i < n; i += 32) nz |= UP(i) != 0;
#undef UP
  return __any_sync(FULL, nz);
}

// Round the nq-limb integer Q (+ sticky) to p bits, write the left-aligned
// L-limb mantissa to out[l * os] (lane-parallel); returns the MPFR exponent
// given value = Q * 2^base.
__device__ int64_t wround(const uint32_t* Q, int nq, bool sticky_in, int64_t base, int L, int p, uint32_t* out,
                          int64_t os) {
  const int lane = threadIdx.x & 31;
  // top bit
  int hb = -1;
  for (int k0 = ((nq - 1) / 32) * 32; k0 >= 0 && hb < 0; k0 -= 32) {
    int k = k0 + lane;
    uint32_t v = k < nq ? Q[k] : 0u;
    unsigned m = __ballot_sync(FULL, v != 0);
    if (m) {
      int hl = 31 - __clz(m);
      uint32_t tv = __shfl_sync(FULL, v, hl);
      hb = (k0 + hl) * 32 + 31 - __clz(tv);
    }
  }
  int64_t lsb = hb - p + 1;
  auto bit = [&](int64_t b) -> uint32_t {
    if (b < 0 || b >= 32 * (int64_t)nq) return 0u;
    return (Q[b >> 5] >> (b & 31)) & 1u;
  };
  uint32_t rbit = lsb >= 1 ? bit(lsb - 1) : 0u;
  // sticky: any bit below lsb - 1
  bool st = false;
  int64_t below = lsb - 1;
  for (int k = lane; (int64_t)k * 32 < below; k += 32) {
    uint32_t v = Q[k];
    int64_t lim = below - 32 * (int64_t)k;
    if (lim < 32) v &= (1u << lim) - 1u;
    st |= v != 0;
  }
  bool sticky = sticky_in || __any_sync(FULL, st);
  uint32_t lsbit = bit(lsb);
  uint32_t inc = rbit & ((sticky ? 1u : 0u) | lsbit);
  int64_t off = hb + 1 - 32 * (int64_t)L;
  int zb = 32 * L - p, zl = zb >> 5;
  int64_t e = base + hb + 1;
  // lane-parallel extraction + increment carry (CLA over 32-limb chunks)
  uint32_t cio = inc;
  for (int l0 = 0; l0 < L; l0 += 32) {
    int l = l0 + lane;
    uint32_t v = 0;
    if (l < L) {
      int64_t q = (int64_t)l * 32 + off;
      int64_t lw = q >> 5;
      int sh = (int)(q & 31);
      uint32_t lo = (lw >= 0 && lw < nq) ? Q[lw] : 0u;
      uint32_t hi = (lw + 1 >= 0 && lw + 1 < nq) ? Q[lw + 1] : 0u;
      v = sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
      if (l < zl) v = 0;
      else if (l == zl && (zb & 31)) v &= ~((1u << (zb & 31)) - 1u);
    }
    // add cio at bit zb of limb zl (only the chunk holding zl; below it, carry passes through zeros)
    bool active = l < L && l >= zl;
    uint32_t add_here = (l == zl) ? (1u << (zb & 31)) : 1u;
    // generate/propagate for "v + add_here*carry_in": g only possible at limb zl path
    bool g = false, pr = false;
    if (active) {
      if (l == zl) {
        uint64_t t = (uint64_t)v + add_here;
        pr = (t >> 32) != 0;  // overflows iff a carry arrives here
      } else {
        pr = v == 0xffffffffu;
      }
    }
    int nvalid = (L - l0) < 32 ? (L - l0) : 32;
    uint32_t cin = cla(g, pr, cio, nvalid);
    // inactive lanes below zl pass carries through: model them as propagate
    if (active && cin) v += add_here;
    if (l < L) out[(int64_t)l * os] = v;
  }
  if (cio) {  // overflow to 2^p
    if (lane == 0) out[(int64_t)(L - 1) * os] = 0x80000000u;
    e += 1;
  }
  return e;
}

}  // namespace dsw
