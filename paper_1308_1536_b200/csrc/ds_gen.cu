// ds_gen.cu -- device-side input builder: the
// random_uniform family of genmat.synth_matrix (reference genmat.py:242-246,
// x = 2U - 1 with U a p-bit uniform, i.e. mpfr_random -> 2*U - 1 rounded at
// p, which is exact) generated straight into this rank's rows in HBM, so a
// config-5 matrix (N = 10,000 at 33,220 bits, ~416 GB) never exists on the
// host.
//
// Counter-based generator ("ds-splitmix", documented in DESIGN.md): the p-bit
// integer k = U * 2^p of element (row, col) is the left-aligned 32L-bit value
// K whose 32-bit limbs are
//     R_{2q} | R_{2q+1} << 32 = mix64(key + (idx * npairs + q + 1) * G),
//     idx = row * n + col,  npairs = ceil(L / 2),  G = 0x9E3779B97F4A7C15,
//     key = mix64(seed ^ 0x243F6A8885A308D3),
// mix64 = the SplitMix64 finaliser, with the low zb = 32L - p bits of R_0
// cleared.  x = 2U - 1 = (k - 2^(p-1)) 2^(1-p) exactly: its sign is the
// complement of K's top bit, |x| = M 2^(1 - 32L) with M = K - 2^(32L-1)
// (top bit set) or 2^(32L-1) - K (top bit clear), normalised by a left shift
// of clz(M) bits (exponent 1 - clz(M)).  Every element is a pure function of
// (seed, row, col, p): any rank, any row order and the host twin
// (synth.counter_uniform_soa, numpy) produce the same bits.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/detseries_b200.h"

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct GenArgs {
  uint32_t* limbs;
  int32_t* exp;
  uint8_t* cls;
  int64_t count;  // plane stride (elements)
  int n, L, p, rank, world, nloc;
  uint64_t key;
};

__device__ __forceinline__ uint32_t rlimb(const GenArgs& g, uint64_t idx, int l, int zb) {
  const uint64_t npairs = (uint64_t)((g.L + 1) >> 1);
  const uint64_t v = mix64(g.key + (idx * npairs + (uint64_t)(l >> 1) + 1ull) * 0x9E3779B97F4A7C15ull);
  uint32_t r = (l & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
  if (l == 0 && zb) r &= ~((1u << zb) - 1u);
  return r;
}

// one thread per owned element; threads of a warp = consecutive columns, so
// every limb-plane store is one coalesced 128-byte transaction
__global__ void k_gen_uniform(GenArgs g) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)g.nloc * g.n) return;
  const int jl = (int)(t / g.n), col = (int)(t % g.n);
  const uint64_t row = (uint64_t)g.rank + (uint64_t)jl * g.world;
  const uint64_t idx = row * (uint64_t)g.n + col;
  const int L = g.L, zb = 32 * L - g.p;
  const uint32_t rtop = rlimb(g, idx, L - 1, zb);
  const bool pos = rtop >> 31;  // K >= 2^(32L-1)  <=>  x >= 0
  // first nonzero limb of K (the +1 of the two's complement stops there)
  int f = 0;
  while (f < L && rlimb(g, idx, f, zb) == 0u) f++;
  auto mlimb = [&](int l) -> uint32_t {
    uint32_t r = rlimb(g, idx, l, zb);
    uint32_t m = pos ? r : (l < f ? 0u : (l == f ? 0u - r : ~r));
    if (l == L - 1) m &= 0x7fffffffu;
    return m;
  };
  uint32_t* out = g.limbs + t;
  if (!pos && f == L) {  // K = 0: x = -1 exactly
    for (int l = 0; l < L - 1; l++) out[(int64_t)l * g.count] = 0u;
    out[(int64_t)(L - 1) * g.count] = 0x80000000u;
    g.exp[t] = 1;
    g.cls[t] = DS_CLS_NEG;
    return;
  }
  // leading one of M
  int top = L - 1;
  uint32_t mt = mlimb(top);
  while (mt == 0u && top > 0) mt = mlimb(--top);
  if (mt == 0u) {  // K = 2^(32L-1): x = +0
    for (int l = 0; l < L; l++) out[(int64_t)l * g.count] = 0u;
    g.exp[t] = 0;
    g.cls[t] = DS_CLS_PZERO;
    return;
  }
  const int lz = 32 * (L - 1 - top) + __clz(mt);
  const int lq = lz >> 5, lr = lz & 31;
  // O_l = bits [32 l, 32 l + 32) of M << lz = funnel(M_{l-lq-1}, M_{l-lq}, lr)
  uint32_t lo = 0u;
  for (int l = 0; l < L; l++) {
    const int s = l - lq;
    const uint32_t hi = s >= 0 ? mlimb(s) : 0u;
    out[(int64_t)l * g.count] = lr ? __funnelshift_l(lo, hi, lr) : hi;
    lo = hi;
  }
  g.exp[t] = 1 - lz;
  g.cls[t] = pos ? DS_CLS_POS : DS_CLS_NEG;
}

}  // namespace

static uint64_t gen_key(uint64_t seed) { return mix64(seed ^ 0x243F6A8885A308D3ull); }

// C linkage: declared inside ds_engine.cu's extern "C" block
extern "C" int gen_uniform_launch(cudaStream_t s, uint32_t* limbs, int32_t* ex, uint8_t* cl, int64_t count, int n, int L, int p,
                       int rank, int world, int nloc, uint64_t seed) {
  GenArgs g{limbs, ex, cl, count, n, L, p, rank, world, nloc, gen_key(seed)};
  const int64_t total = (int64_t)nloc * n;
  if (total == 0) return 0;
  const int block = 256;
  k_gen_uniform<<<(unsigned)((total + block - 1) / block), block, 0, s>>>(g);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
