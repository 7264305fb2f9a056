// ds_cwarp.cuh -- warp-cooperative complex multiply and divide, one component
// per warp, correctly rounded exactly like mpc_mul / mpc_div (the thread-level
// cmul_part / cdiv_part of ds_mp.cuh, same integers, same rounding):
//   re(a*b) = RN(ar*br - ai*bi),  im(a*b) = RN(ar*bi + ai*br)
//   re(a/b) = RN((ar*br + ai*bi) / (br^2 + bi^2)),
//   im(a/b) = RN((ai*br - ar*bi) / (br^2 + bi^2))
// The O(L^2) parts run across the 32 lanes: the exact products (lane t owns
// the digit columns c = t mod 32, then a carry pass) and the long division
// (dsw::wdivrem, Knuth D on lane-blocked divisor limbs).  The O(L) parts --
// exact windowed sums, perturbations, rounding -- are the thread-level code of
// ds_mp.cuh on lane 0.  Everything lives in the warp's shared-memory region.
// Used by the complex step (elim.py:47 division, 56-61 signed minors, 148
// normalisation, 213-215 det chain, on mpc values).
#pragma once
#include <stdint.h>
#include "ds_mp.cuh"
#include "ds_warpdiv.cuh"

namespace dscw {

using ds::CPtr;
using ds::Ptr;
using ds::Val;
using ds::XSum;
using ds::XTerm;

constexpr unsigned FULL = 0xffffffffu;

// largest divisor block (limbs per lane) of the warp division; wider exact
// denominators (huge exponent gaps, or p > ~8000 bits) take the lane-0 path
constexpr int KMAX = 40;

// U of the warp division: nU <= nD + L + 4 limbs, zero-filled up to nU + 32 K
__host__ __device__ inline int64_t u_words(int L, int p) {
  return dsw::upad_words(ds::cdiv_nwin(L, p) + L + 8 + 32 * KMAX);
}

// shared-memory words of one warp's region at L limbs / p bits
__host__ __device__ inline int64_t warp_words(int L, int p) {
  const int64_t nwin = ds::cdiv_nwin(L, p);
  return 4 * (int64_t)L              // staged operands ar, ai, br, bi
         + 8 * (int64_t)L             // products P0..P3 (2L each)
         + 6 * (int64_t)L + 8         // column sums of one product (lo, mid, hi)
         + 2 * nwin                   // exact sums N, D
         + u_words(L, p)              // U (padded, zero tail for the lane blocks) -- also lane-0 fallback scratch
         + nwin + 4                   // V (normalised divisor)
         + nwin + 4;                  // Q
}

// region layout
struct Region {
  uint32_t *op, *P, *col, *N, *D, *U, *V, *Q;
  __device__ Region(uint32_t* base, int L, int p) {
    const int64_t nwin = ds::cdiv_nwin(L, p);
    op = base;
    P = op + 4 * L;
    col = P + 8 * L;
    N = col + 6 * L + 8;
    D = N + nwin;
    U = D + nwin;
    V = U + u_words(L, p);
    Q = V + nwin + 4;
  }
};

// copy a value's limbs into shared memory (all lanes), returning a Val over them
__device__ __forceinline__ Val stage(const Val& v, uint32_t* dst, int L) {
  const int lane = threadIdx.x & 31;
  for (int l = lane; l < L; l += 32) dst[l] = v.m[l];
  Val o;
  o.m = CPtr{dst, 1};
  o.e = v.e;
  o.c = v.c;
  return o;
}

// P (2L limbs) = A * B exactly.  Lane t sums the digit columns c = t, t+32, ...
// (up to L 64-bit products each, kept as lo64 + overflow count), then lane 0
// propagates the carries through the 2L columns.  Caller syncs before reading P.
__device__ void wmul_full(uint32_t* P, const uint32_t* A, const uint32_t* B, int L, uint32_t* col) {
  const int lane = threadIdx.x & 31;
  for (int c = lane; c < 2 * L - 1; c += 32) {
    const int i0 = c - L + 1 > 0 ? c - L + 1 : 0;
    const int i1 = c < L - 1 ? c : L - 1;
    uint64_t lo = 0;
    uint32_t hi = 0;
    for (int i = i0; i <= i1; i++) {
      const uint64_t t = (uint64_t)A[i] * B[c - i];
      lo += t;
      hi += lo < t ? 1u : 0u;
    }
    col[3 * c] = (uint32_t)lo;
    col[3 * c + 1] = (uint32_t)(lo >> 32);
    col[3 * c + 2] = hi;
  }
  __syncwarp();
  if (lane == 0) {
    // P = sum_c (lo_c + hi_c 2^64) 2^(32c): limb c collects the low word of column c,
    // the high word of column c-1 and the overflow count of column c-2, plus carry
    uint64_t carry = 0;
    for (int c = 0; c < 2 * L; c++) {
      uint64_t t = carry;
      if (c < 2 * L - 1) t += col[3 * c];
      if (c >= 1 && c - 1 < 2 * L - 1) t += col[3 * (c - 1) + 1];
      if (c >= 2 && c - 2 < 2 * L - 1) t += col[3 * (c - 2) + 2];
      P[c] = (uint32_t)t;
      carry = t >> 32;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ XTerm wprod_term(uint32_t* P, const Val& A, const Val& B, int L, uint32_t* col) {
  XTerm t;
  t.neg = ds::neg_of(A.c) ^ ds::neg_of(B.c);
  t.zero = ds::is_zero_cls(A.c) || ds::is_zero_cls(B.c);
  t.n = 2 * L;
  t.base = A.e + B.e - 64 * (int64_t)L;
  t.m = CPtr{P, 1};
  if (!t.zero) wmul_full(P, A.m.p, B.m.p, L, col);  // operands staged (stride 1)
  return t;
}

// one component of mpc_mul: r = RN(A*B -/+ C*D); lane 0 writes the result.
// Returns the range check on lane 0 (true on the other lanes).
__device__ bool wcmul_part(Ptr rm, int32_t* re, uint8_t* rc, const Val& A, const Val& B, const Val& C, const Val& D,
                           bool sub, int L, int p, const Region& R) {
  const int lane = threadIdx.x & 31;
  XTerm x = wprod_term(R.P, A, B, L, R.col);
  XTerm y = wprod_term(R.P + 2 * L, C, D, L, R.col);
  bool ok = true;
  if (lane == 0) {
    Ptr S{R.N, 1};
    XSum s = ds::exact_sum(S, x, y, sub, 2 * (int64_t)p + 4);
    ok = ds::round_xsum(rm, re, rc, S, s, L, p);
  }
  __syncwarp();
  return ok;
}

// RN(N / D) for exact sums (the division of ds::div_xsum with the long division
// on the warp); K = divisor limbs per lane
template <int K>
__device__ bool wdiv_body(Ptr rm, int32_t* re, uint8_t* rc, const XSum& xn, const XSum& xd, int nD, int L, int p,
                          const Region& R, unsigned int* warn) {
  const int lane = threadIdx.x & 31;
  const CPtr Nc{R.N, 1};
  const int s = __clz(R.D[nD - 1]);
  const int64_t topN = ds::top_bit(Nc, xn.n), topD = (int64_t)(nD - 1) * 32 + 31 - s;
  int64_t sh = (int64_t)p + 2 - (topN - topD);
  if (sh < 0) sh = 0;
  const int64_t ubits = topN + 1 + sh + s;
  int nU = (int)((ubits + 31) / 32) + 1;
  if (nU <= nD) nU = nD + 1;
  // U = N << (sh + s) (padded layout of the warp division; zero tail for the lane
  // blocks, which cover 32 K limbs of V), V = D << s
  for (int k = lane; k < nU + 32 * K; k += 32)
    R.U[dsw::upad(k)] = k < nU ? ds::bits32(Nc, xn.n, 32 * (int64_t)k - (sh + s)) : 0u;
  for (int k = lane; k < nD; k += 32) {
    const uint32_t hi = R.D[k] << s;
    const uint32_t lo = (s && k > 0) ? (R.D[k - 1] >> (32 - s)) : 0u;
    R.V[k] = hi | lo;
  }
  __syncwarp();
  uint32_t vb[K];
#pragma unroll
  for (int u = 0; u < K; u++) {
    const int idx = lane * K + u;
    vb[u] = idx < nD ? R.V[idx] : 0u;
  }
  const bool rem = dsw::wdivrem<K>(R.Q, R.U, nU, R.V, vb, nD);
  bool ok = true;
  if (lane == 0) {
    const int nq = nU - nD;
    Ptr Q{R.Q, 1};
    const int pq = xn.pert, pd = -xd.pert;
    const int dir = pq != 0 ? pq : pd;
    if (pq != 0 && pd != 0 && pq != pd && warn) atomicAdd(warn, 1u);
    bool sticky = rem;
    if (!rem && dir != 0) {
      sticky = true;
      if (dir < 0) {
        for (int k = 0; k < nq; k++) {
          const uint32_t v = Q[k];
          Q[k] = v - 1u;
          if (v != 0) break;
        }
      }
    } else if (dir != 0) {
      sticky = true;
    }
    ds::RoundOut ro = ds::round_big(rm, L, p, CPtr{Q.p, Q.s}, nq, xn.base - xd.base - sh, sticky);
    *re = (int32_t)ro.e;
    *rc = ds::nz_cls(xn.neg ^ xd.neg);
    ok = ds::range_ok(ro.e);
  }
  __syncwarp();
  return ok;
}

// one component of mpc_div (ds::cdiv_part on the warp)
__device__ bool wcdiv_part(Ptr rm, int32_t* re, uint8_t* rc, const Val& ar, const Val& ai, const Val& br,
                           const Val& bi, bool imag, int L, int p, const Region& R, unsigned int* warn) {
  const int lane = threadIdx.x & 31;
  const int64_t win = ds::cdiv_window(p);
  XTerm x, y;
  if (!imag) {
    x = wprod_term(R.P, ar, br, L, R.col);
    y = wprod_term(R.P + 2 * L, ai, bi, L, R.col);
  } else {
    x = wprod_term(R.P, ai, br, L, R.col);
    y = wprod_term(R.P + 2 * L, ar, bi, L, R.col);
  }
  XTerm d1 = wprod_term(R.P + 4 * L, br, br, L, R.col);
  XTerm d2 = wprod_term(R.P + 6 * L, bi, bi, L, R.col);
  // exact sums on lane 0, shared through the region
  __shared__ XSum xs_n[32], xs_d[32];  // one slot per warp of the block
  const int w = threadIdx.x >> 5;
  if (lane == 0) {
    xs_n[w] = ds::exact_sum(Ptr{R.N, 1}, x, y, imag, win);
    xs_d[w] = ds::exact_sum(Ptr{R.D, 1}, d1, d2, false, win);
  }
  __syncwarp();
  const XSum xn = xs_n[w], xd = xs_d[w];
  if (xn.zero) {
    if (lane == 0) {
      for (int l = 0; l < L; l++) rm[l] = 0;
      *re = 0;
      *rc = ds::zero_cls(xn.neg ^ xd.neg);
    }
    __syncwarp();
    return true;
  }
  int nD = xd.n;
  while (nD > 0 && R.D[nD - 1] == 0) nD--;
  const int K = (nD + 31) / 32;
  if (K <= 4) return wdiv_body<4>(rm, re, rc, xn, xd, nD, L, p, R, warn);
  if (K <= 8) return wdiv_body<8>(rm, re, rc, xn, xd, nD, L, p, R, warn);
  if (K <= 12) return wdiv_body<12>(rm, re, rc, xn, xd, nD, L, p, R, warn);
  if (K <= 16) return wdiv_body<16>(rm, re, rc, xn, xd, nD, L, p, R, warn);
  if (K <= 24) return wdiv_body<24>(rm, re, rc, xn, xd, nD, L, p, R, warn);
  if (K <= KMAX) return wdiv_body<KMAX>(rm, re, rc, xn, xd, nD, L, p, R, warn);
  // very wide denominator (exponent gap near the window): the thread-level division
  bool ok = true;
  if (lane == 0) ok = ds::div_xsum(rm, re, rc, Ptr{R.N, 1}, xn, Ptr{R.D, 1}, xd, L, p, Ptr{R.U, 1}, warn);
  __syncwarp();
  return ok;
}

}  // namespace dscw
