// ds_tc.cu -- the update a_jk <- RN(a_jk - RN(z_j * b_k)) (elim.py:49-52) with
// the mantissa products on the 5th-generation tensor cores.
//
// z_j * b_k = sum_c col_c 2^(8c),  col_c = sum_s B_k[s] Z_j[c - s]  over the
// unsigned 8-bit digits (bytes) of the left-aligned mantissas.  For 128
// consecutive columns k of the pivot row and one row j this is one int8 GEMM
//     D[k][c] = sum_s B[k][s] * T_j[s][c],   T_j[s][c] = Z_j[c - s]  (Toeplitz)
// computed by tcgen05.mma.cta_group::1.kind::i8 (u8 x u8 -> s32) into TMEM:
// M = 128 columns k (TMEM lanes), N = tn output digit columns per tile (96 at
// 4096 bits), K = 32 digits per instruction.  Only digit columns c >= c_lo are
// formed (short product: the omitted part E is >= 0 and < D8*2^8 units of
// 2^(8 c_lo)); the rounding of z*b is decided from the computed columns unless
// the bits under the round bit are all ones (or a possible tie), in which case
// the element is handed to the exact general engine through a fallback list
// (probability ~2^-40 on non-exact data).
//
// A operand (pivot-row digits) in TMEM, B operand = per-row Toeplitz bank in
// shared memory addressed by descriptor offsets, a's limbs moved by TMA tiles
// (128 columns x L planes) into per-group windows, rounded in place and stored
// back with one bulk tensor store.  Roles, pipelining and barriers: see the
// comment above k_update_tc and DESIGN.md section 5.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/detseries_b200.h"
#include "ds_mp.cuh"
#include "ds_stream.cuh"
#include "ds_tc.cuh"

// implementation variants (A/B measured on the B200)
#ifndef DS_VAR_MMAWARP
#define DS_VAR_MMAWARP 1
#endif
#ifndef DS_VAR_MULSHIFT
#define DS_VAR_MULSHIFT 0
#endif

#ifndef DS_TCW_FINISH_MINB
#define DS_TCW_FINISH_MINB 3  // k_tcw_finish blocks per SM the registers are capped for
#endif

namespace {

using namespace dss;

constexpr int TM = 128;      // columns per CTA (TMEM lanes)
constexpr int KS = 32;       // digits per MMA K step
// NG epilogue groups of 4 warps (rows ri = grp mod NG) and NG producer
// pipelines of 2 warps; NG = 4 up to ~2048 bits, 2 up to 4096 bits, 1 where two groups' windows do
// not fit in shared memory (8192 bits)
constexpr int NPIPE = 64;    // producer threads per pipeline
template <int NG>
struct Cfg {
  static constexpr int NEPI = 128 * NG;
  static constexpr int NTHREADS = NEPI + NG * NPIPE;
};
constexpr int RBR = 16;      // rows per CTA (the lookahead tile uses RBR_LA)
#ifndef DS_VAR_PREF
#define DS_VAR_PREF 1  // rows (of the group) ahead that the a-tile L2 prefetch targets
#endif
#ifndef DS_VAR_RBR_LA
#define DS_VAR_RBR_LA 8  // lookahead-tile rows per CTA: 8 measured -0.8 % update at N=2000 @4096, -1.5 % at N=1000 (profiles/r02_lookahead_rbr_ab.log)
#endif
constexpr int RBR_LA = DS_VAR_RBR_LA;

struct TcArgs {
  int p, L, zb, D8p, nks, ntiles, c_lo, eps;
  int tn;                  // output digit columns per MMA tile (N)
  int br;                  // Toeplitz bank rows: ntiles * tn + 32 (nks - 1)
  int tma_ok;              // a planes reachable by the tile tensor map
  int no_direct;           // DS_TC_NO_DIRECT: always the two-pass rounding
  int nrows, ncols, kstart, skip_col, n;
  int kmin;                // first column to update (kstart = kmin rounded down to 4: aligned tiles)
  int tile0, tskip;        // column tile of blockIdx.x 0; tile index skipped (-1: none)
  int rbr;                 // rows per CTA
  int jl0;
  int64_t zstride;         // component stride of the z meta (complex: nloc)
  const uint8_t* zbytes;   // [nrows][D8p]
  const uint8_t* bbytes;   // [n][D8p]
  const double* zf;        // [nrows]
  const double* bf;        // [n]
  const int32_t* zexp;     // z meta, offset by jl0
  const uint8_t* zcls;
  const int32_t* bexp;     // pivot row meta
  const uint8_t* bcls;
  uint32_t* a_limbs;
  int32_t* a_exp;
  uint8_t* a_cls;
  int64_t a_count;
  int32_t* status;
  int step;
  int* fb_count;           // fallback list
  int2* fb_list;
  int fb_cap;
  const int* zlow;         // complex warp finish: lowest nonzero digit of z [c][row] and b [c][col]
  const int* blow;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware until
// the phase completes instead of spinning through issue slots
#ifndef DS_VAR_WAITHINT
#define DS_VAR_WAITHINT 1000000  // try_wait suspend-time hint (ns); 0: no hint
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
#if DS_VAR_WAITHINT
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(DS_VAR_WAITHINT));
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(b)),
      "r"(parity));
#endif
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void cp16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp4(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.commit_group;");
  asm volatile("cp.async.wait_group 0;");
}
// ---- TMA (bulk tensor) tile copies of the a planes: box = 128 columns x L planes
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(
                   smem_u32(b)),
               "r"(bytes));
}
__device__ __forceinline__ void tma_load_2d(void* sdst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(sdst)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* ssrc) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"((uint64_t)map),
               "r"(x), "r"(y), "r"(smem_u32(ssrc))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"((uint64_t)map), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count));
}

// ---------------------------------------------------------------- prep
// bytes of the left-aligned mantissa (= the 32-bit limbs, little-endian),
// zero padded to D8p; one thread per (element, limb)
__global__ void k_tc_bytes(const uint32_t* src, int64_t count, int num, int L, int D8p, uint8_t* dst, double* topf) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int W = D8p / 4;
  if (t >= (int64_t)num * W) return;
  int e = (int)(t / W), l = (int)(t % W);
  uint32_t v = l < L ? src[(int64_t)l * count + e] : 0u;
  ((uint32_t*)(dst + (int64_t)e * D8p))[l] = v;
  if (l == 0) {
    uint64_t top = ((uint64_t)src[(int64_t)(L - 1) * count + e] << 32) | src[(int64_t)(L - 2) * count + e];
    topf[e] = (double)top * 0x1p-63;
  }
}

// index of the lowest nonzero digit (byte of the limbs) of each element, 1 << 28 for
// zero: a short product z b omits no nonzero digit product exactly when
// low(z) + low(b) >= c_lo (ds_cfinish.cuh treats such products as exact)
__global__ void k_lowdig(const uint32_t* src, int64_t count, int num, int L, int* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= num) return;
  int low = 1 << 28;
  for (int l = 0; l < L; l++) {
    const uint32_t v = src[(int64_t)l * count + e];
    if (v) {
      low = 4 * l + (__ffs(v) - 1) / 8;
      break;
    }
  }
  out[e] = low;
}

// ---------------------------------------------------------------- main
__device__ __forceinline__ void bar_pipe(int id, int count) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(count));
}

// Roles (384 threads; one CTA = 128 consecutive columns k x RBR rows j):
//   warps 0-7   epilogue, two groups (warps 0-3: even rows, 4-7: odd rows);
//               thread = column k = TMEM lane 32 (warp % 4) + lane, so a
//               warp touches 32 consecutive a_jk of one row (coalesced).
//   warps 8-9   pipeline 0 (even rows), warps 10-11 pipeline 1 (odd rows):
//               per row, the Toeplitz bank of z_j's digits in the canonical
//               K-major layout -- bank row r <-> m = m_min + r holds bytes
//               k = 0..31 = Z[m - k] -- so the B tile of (tile t, K step ks)
//               is bank rows [t*tn + 32 (nks-1-ks), +tn): a descriptor offset
//               (8-row aligned), no per-MMA copies.  Lane 0 of warps 8 / 10
//               issues the pipeline's MMAs.
// TMEM: accumulators [0, 4 tn) = (group, double buffer) x tn columns; the
// pivot-row digits (MMA A operand, lane = column k, 4 digits per 32-bit
// column) at [4 tn, 4 tn + 8 nks).
// register cap 144 (launch bound 448 threads): 384 x 144 leaves ~10K registers per SM for a
// side-stream block (minors emission, det chain) to co-run in the epilogue's idle issue slots
// NG = 2 is bounded as if 448 threads: the 128-register cap measured faster than ~158
template <int NG>
__global__ void __launch_bounds__(NG == 2 ? 448 : Cfg<NG>::NTHREADS, 1) k_update_tc(TcArgs a, const __grid_constant__ CUtensorMap amap) {
  constexpr int NEPI = Cfg<NG>::NEPI;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_bank_empty[NG];
  __shared__ __align__(8) uint64_t bar_tfull[NG][2];
  __shared__ __align__(8) uint64_t bar_tempty[NG][2];
  __shared__ __align__(8) uint64_t bar_tile[NG];  // a-tile loads (TMA), one per epilogue group
  __shared__ uint32_t tmem_base_sh;
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nks = a.nks, ntiles = a.ntiles, L = a.L, TN = a.tn, BR = a.br;
  const int m_min = a.c_lo - KS * (nks - 1);
  const int zbase = (m_min - 32) & ~3;  // zw[v] = Z[zbase + v]
  const int ZWL = ((BR + 64) + 15) & ~15;
  uint8_t* bank0 = smem;                               // NG banks of BR * 32 bytes
  uint32_t* Swin = (uint32_t*)(smem + NG * BR * KS);   // per group: [L + 2 slots][TM columns]
  uint8_t* zw0 = (uint8_t*)(Swin + (L + 2) * NEPI);     // NG x ZWL bytes
  const int tile = (int)blockIdx.x + a.tile0 + ((a.tskip >= 0 && (int)blockIdx.x >= a.tskip) ? 1 : 0);
  const int kbase = a.kstart + tile * TM;
  const int row0 = blockIdx.y * a.rbr;
  const int nrow_cta = min(a.rbr, a.nrows - row0);
  const uint32_t ACOL = 2 * NG * TN;

  if (tid == 0) {
    for (int g = 0; g < NG; g++) {
      mbar_init(&bar_bank_empty[g], 1);
      mbar_init(&bar_tile[g], 1);
      for (int b = 0; b < 2; b++) {
        mbar_init(&bar_tfull[g][b], 1);
        mbar_init(&bar_tempty[g][b], 4);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  // pivot-row digits of the CTA's columns -> TMEM (group-0 threads, lane = column)
  if (tid < TM) {
    const int k = kbase + tid;
    const uint4* src = (const uint4*)(a.bbytes + (int64_t)(k < a.n ? k : 0) * a.D8p);
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + ACOL;
    for (int c = 0; c < a.D8p / 4; c += 8) {
      uint4 u0 = make_uint4(0, 0, 0, 0), u1 = u0;
      if (k < a.n) {
        u0 = src[c / 4];
        u1 = src[c / 4 + 1];
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + c), "r"(u0.x),
                   "r"(u0.y), "r"(u0.z), "r"(u0.w), "r"(u1.x), "r"(u1.y), "r"(u1.z), "r"(u1.w));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  if (tid >= NEPI) {
    // =================================================== pipelines: banks + MMAs
    const int pp = (tid - NEPI) / NPIPE;  // row parity
    const int ptid = (tid - NEPI) % NPIPE;
    uint8_t* bank = bank0 + pp * BR * KS;
    uint8_t* zw = zw0 + pp * ZWL;
    const uint32_t bank_sa = smem_u32(bank);
    int q = 0;  // row counter of this pipeline
    for (int ri = pp; ri < nrow_cta; ri += NG, q++) {
      if (q >= 1) mbar_wait(&bar_bank_empty[pp], (q - 1) & 1);  // MMAs of row ri-2 completed
      const uint8_t* zrow = a.zbytes + (int64_t)(row0 + ri) * a.D8p;
      for (int v = ptid; v < ZWL / 4; v += NPIPE) {
        int t = zbase + 4 * v;
        ((uint32_t*)zw)[v] = (t >= 0 && t < a.D8p) ? *(const uint32_t*)(zrow + t) : 0u;
      }
      bar_pipe(1 + pp, NPIPE);
      // chunk (r, h): bytes k = 16h .. 16h+15 of bank row r = reversed Z[u .. u+16),
      // u = m_min + r - 16h - 15
      for (int c = ptid; c < 2 * BR; c += NPIPE) {
        const int h = c >= BR ? 1 : 0, r = c - h * BR;
        const int off = m_min + r - 16 * h - 15 - zbase;
        const uint32_t* wp = (const uint32_t*)zw + (off >> 2);
        const int sh = 8 * (off & 3);
        uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2], w3 = wp[3], w4 = wp[4];
        uint32_t x0 = __funnelshift_r(w0, w1, sh), x1 = __funnelshift_r(w1, w2, sh);
        uint32_t x2 = __funnelshift_r(w2, w3, sh), x3 = __funnelshift_r(w3, w4, sh);
        *(uint4*)(bank + h * BR * 16 + (r >> 3) * 128 + (r & 7) * 16) =
            make_uint4(__byte_perm(x3, 0, 0x0123), __byte_perm(x2, 0, 0x0123), __byte_perm(x1, 0, 0x0123),
                       __byte_perm(x0, 0, 0x0123));
      }
      asm volatile("fence.proxy.async.shared::cta;");
      bar_pipe(1 + pp, NPIPE);
#if DS_VAR_MMAWARP
      if (ptid < 32) {
        // the whole issuer warp runs the loop (warp-uniform descriptors live in
        // uniform registers, no per-MMA register->uniform moves); lane 0 issues
        const uint64_t bd_hi = umma_desc(0u, (uint32_t)BR * 16u, 128);  // LBO / SBO / version fields
        const uint32_t idesc = idesc_i8(TM, TN);
        for (int t = 0; t < ntiles; t++) {
          const int gt = q * ntiles + t;  // tile counter of this group
          const int buf = gt & 1;
          if (gt >= 2) mbar_wait(&bar_tempty[pp][buf], ((gt >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const int c0 = a.c_lo + t * TN;
          int s_lo = c0 - (a.D8p - 1);
          if (s_lo < 0) s_lo = 0;
          int s_hi = c0 + TN - 1;
          if (s_hi > a.D8p - 1) s_hi = a.D8p - 1;
          const int ks0 = s_lo / KS, ks1 = s_hi / KS;
          const uint32_t dcol = tmem + (uint32_t)((2 * pp + buf) * TN);
          // B tile of K step ks: bank rows from t*TN + 32 (nks - 1 - ks) (a multiple of 8):
          // the descriptor's 16-byte address field steps down by 32 per K step
          uint64_t bd = bd_hi | (uint64_t)(((bank_sa + (uint32_t)((t * TN + KS * (nks - 1 - ks0)) >> 3) * 128u) >> 4) &
                                           0x3FFFu);
          uint32_t acol = tmem + ACOL + 8 * ks0;
          for (int ks = ks0; ks <= ks1; ks++) {
            if (lane == 0)
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dcol),
                  "r"(acol), "l"(bd), "r"(idesc), "r"((uint32_t)(ks - ks0)));
            bd -= 32;
            acol += 8;
          }
          if (lane == 0) umma_commit(&bar_tfull[pp][buf]);
        }
        if (lane == 0) umma_commit(&bar_bank_empty[pp]);
      }
#else
      const bool issuer = ptid == 0;
      if (issuer) {
        for (int t = 0; t < ntiles; t++) {
          const int gt = q * ntiles + t;  // tile counter of this group
          const int buf = gt & 1;
          if (gt >= 2) mbar_wait(&bar_tempty[pp][buf], ((gt >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const int c0 = a.c_lo + t * TN;
          int s_lo = c0 - (a.D8p - 1);
          if (s_lo < 0) s_lo = 0;
          int s_hi = c0 + TN - 1;
          if (s_hi > a.D8p - 1) s_hi = a.D8p - 1;
          const int ks0 = s_lo / KS, ks1 = s_hi / KS;
          const uint32_t dcol = tmem + (uint32_t)((2 * pp + buf) * TN);
          for (int ks = ks0; ks <= ks1; ks++) {
            const int r0 = t * TN + KS * (nks - 1 - ks);  // multiple of 8
            uint64_t bd = umma_desc(bank_sa + (uint32_t)(r0 >> 3) * 128u, (uint32_t)BR * 16u, 128);
            uint32_t acc = ks > ks0 ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dcol),
                "r"(tmem + ACOL + 8 * ks), "l"(bd), "r"(idesc_i8(TM, TN)), "r"(acc));
          }
          umma_commit(&bar_tfull[pp][buf]);
        }
        umma_commit(&bar_bank_empty[pp]);
      }
#endif
      __syncwarp();
    }
  } else {
    // =================================================== epilogue
    const int grp = warp >> 2, qw = warp & 3;
    const int r = qw * 32 + lane;  // TMEM lane = column within the CTA
    const int k = kbase + r;
    const bool col_ok = k < a.n && k >= a.kmin && k != a.skip_col;
    uint32_t* region = Swin + grp * (L + 2) * TM;  // the group's windows: slot w of column r at [w * TM + r]
    uint32_t* Sw = region + r;
    // full 128-column tiles move a's limbs with one TMA load / store per row
    // (box = 128 columns x L planes into slots 1..L); edge tiles per thread
    const bool tile_io = a.tma_ok && kbase + TM <= a.n && (a.n & 3) == 0;  // box start 16-byte aligned
    // per-column pivot-row scalars are loop invariant; the per-row scalars (a's class
    // and exponent, z's class, exponent and fp64 top) are loaded one row ahead so
    // their HBM latency overlaps the previous row's epilogue
    const uint8_t cb = col_ok ? a.bcls[k] : (uint8_t)DS_CLS_PZERO;
    const double bfk = col_ok ? a.bf[k] : 0.0;
    const int32_t bexk = col_ok ? a.bexp[k] : 0;
    uint8_t nx_ca = 0, nx_cz = 0;
    int32_t nx_ea = 0, nx_zexp = 0;
    double nx_zf = 0.0;
    if (col_ok && grp < nrow_cta) {
      const int zr = row0 + grp;
      const int64_t idx = (int64_t)(a.jl0 + zr) * a.n + k;
      nx_ca = a.a_cls[idx];
      nx_ea = a.a_exp[idx];
      nx_cz = a.zcls[zr];
      nx_zf = a.zf[zr];
      nx_zexp = a.zexp[zr];
    }
    int q = 0;
    for (int ri = grp; ri < nrow_cta; ri += NG, q++) {
      const int zr = row0 + ri;  // row index relative to jl0
      const int jl = a.jl0 + zr;
      const int64_t idx = (int64_t)jl * a.n + k;
      const int tx = (int)((int64_t)jl * a.n + kbase);
      const uint8_t cur_ca = nx_ca, cur_cz = nx_cz;
      const int32_t cur_ea = nx_ea, cur_zexp = nx_zexp;
      const double cur_zf = nx_zf;
      if (col_ok && ri + NG < nrow_cta) {
        const int zn = zr + NG;
        const int64_t idn = idx + (int64_t)NG * a.n;
        nx_ca = a.a_cls[idn];
        nx_ea = a.a_exp[idn];
        nx_cz = a.zcls[zn];
        nx_zf = a.zf[zn];
        nx_zexp = a.zexp[zn];
      }
      if (tile_io) {
        if (r == 0) {
          bulk_wait_read0();  // this group's previous tile store has read the window
          mbar_expect_tx(&bar_tile[grp], (uint32_t)(TM * L * 4));
          tma_load_2d(region + TM, &amap, tx, 0, &bar_tile[grp]);
          if (ri + DS_VAR_PREF * NG < nrow_cta)  // the group's next tile into L2 while this row runs
            tma_prefetch_2d(&amap, (int)((int64_t)(jl + DS_VAR_PREF * NG) * a.n + kbase), 0);
        }
      }
      // ---- element setup (mirrors ds_update.cu fused_element)
      bool process = false, fallback = false;
      int neg = 0, norm = 0;
      int64_t E = 0, d = 0;
      bool xa = false, sub = false, za = false;
      if (col_ok) {
        const uint8_t cz = cur_cz, ca = cur_ca;
        za = ca >= DS_CLS_PZERO;
        int sa = ca & 1, st = (cz & 1) ^ (cb & 1);
        if (cz >= DS_CLS_PZERO || cb >= DS_CLS_PZERO) {
          if (za) a.a_cls[idx] = (sa && !st) ? DS_CLS_NZERO : DS_CLS_PZERO;
        } else {
          int32_t ea = za ? 0 : cur_ea;
          double pr = cur_zf * bfk;
          norm = pr >= 2.0 ? 1 : 0;
          bool confident = fabs(pr - 2.0) > 0x1p-42;
          int64_t ebase = (int64_t)cur_zexp + bexk;
          if (!za && (int64_t)ea - (ebase - 1) >= (int64_t)a.p + 3) {
            // a dominates whatever the normalisation: unchanged
          } else if (!confident) {
            fallback = true;
          } else {
            int64_t et = ebase - (norm ? 0 : 1);
            d = za ? -(int64_t)(1 << 30) : (int64_t)ea - et;
            if (za || d < (int64_t)a.p + 2) {
              xa = !za && d >= 0;
              sub = !za && (sa == st);
              neg = xa ? sa : (st ^ 1);
              E = xa ? ea : et;
              process = true;
            }
          }
        }
      }
      // a's limbs in the window (slots 1..L): coalesced across the warp
      if (tile_io) {
        mbar_wait(&bar_tile[grp], q & 1);
      } else {
        if (process && !za) {
          const uint32_t* A = a.a_limbs + idx;
#pragma unroll 4
          for (int l = 0; l < L; l++) cp4(Sw + (l + 1) * TM, A + (int64_t)l * a.a_count);
        }
        cp_wait_all();
      }
      SWin S;
      S.base(Sw, TM);
      Emit em;
      // direct (single-pass) rounding: predict the result's normalisation from the
      // leading bits -- a's top 64 bits (exact, from the window) and t's fp64
      // estimate (relative error < 2^-50) -- when it is certain with a 2^-40 margin
      // (cancellation of at most ~20 bits); an exactly predicted negative window
      // (equal exponents, |t| > |a|) swaps the operand roles.  Others: two-pass.
      int off_pred = -1;
      if (process && !za && tile_io && !a.no_direct) {
        const uint64_t atop = ((uint64_t)Sw[L * TM] << 32) | Sw[(L - 1) * TM];
        const double am = (double)atop * 0x1p-63;  // [1, 2)
        const double prv = cur_zf * bfk;
        const double tm = norm ? prv * 0.5 : prv;  // [1, 2)
        const int64_t sh = xa ? d : -d;
        const double yv = sh < 200 ? ldexp(xa ? tm : am, -(int)sh) : 0.0;
        double sd = sub ? (xa ? am : tm) - yv : (xa ? am : tm) + yv;
        if (sd < 0.0) {  // only xa, d == 0, sub: t - a with the roles swapped
          sd = -sd;
          xa = false;
          neg = (int)(((cur_cz & 1) ^ (cb & 1)) ^ 1);
          E = (int64_t)cur_zexp + bexk - (norm ? 0 : 1);
        }
        if (sd > 0x1p-20) {
          int e2;
          const double fr = frexp(sd, &e2);  // sd = fr 2^e2, fr in [0.5, 1)
          const int off = 32 + (e2 - 1);
          if (fr - 0.5 > 0x1p-41 && 1.0 - fr > 0x1p-41 && off >= 0 && off <= 33) off_pred = off;
        }
      }
      if (process) {
        S.init(L, xa, sub, za, xa ? d : (za ? 0 : -d), off_pred);
        em.S = &S;
        // every lane's P' is shifted to the normalised position (non-normalised
        // products x 2, nsh = 1): t's LSB at r' = p + 2 zb for all lanes, so T limbs
        // are whole P' limbs and all lanes of a warp share block boundaries
        em.r = a.p + 2 * a.zb;
        em.zb = a.zb;
        em.p = a.p;
        em.L = L;
        em.exact = false;
        em.onesided = true;
        em.lo_chk = 8 * a.c_lo + a.eps + 1;  // the omitted part doubles with the shift
        em.hi_chk = em.r - 2;
        em.allz = true; em.allo = true; em.sticky = false; em.decided = false;
        em.rbit = 0; em.tcarry = 0; em.tl = 0; em.excess = false;
        em.setup<8>();
      }
      bool ok = true;
      uint32_t carry = 0;
      // non-normalised products are doubled (P' = P 2^nsh) inside the column
      // combination: the digit weights 2^(8j) become 2^(8j + nsh), so P' limbs come
      // straight out of the carry chain (no funnel shift per limb)
#if DS_VAR_MULSHIFT
      const uint32_t nsh = norm ? 0u : 1u;
      const uint32_t m0 = 1u << nsh, m1 = 256u << nsh, m2 = 65536u << nsh, m3 = 16777216u << nsh;
#else
      const int nsh = norm ? 0 : 1;
      uint32_t praw = 0u;  // previous unshifted P limb
      constexpr uint32_t m0 = 1u, m1 = 256u, m2 = 65536u, m3 = 16777216u;
#endif
      for (int t = 0; t < ntiles; t++) {
        const int gt = q * ntiles + t;
        const int buf = gt & 1;
        mbar_wait(&bar_tfull[grp][buf], (gt >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t taddr = tmem + ((uint32_t)(qw * 32) << 16) + (uint32_t)((2 * grp + buf) * TN);
        // digit columns >= 8L are zero (P < 2^(64L)): stop at the chunk holding column 8L - 1
        const int cend = min(TN, 8 * L - (a.c_lo + t * TN));
#pragma unroll 1
        for (int cb = 0; cb < cend; cb += 32) {
          uint32_t v[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
              : "r"(taddr + cb));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          if (process && ok) {
            // limb g = w_g + (high word of w_(g-1)) + carry, w_g = sum_j v[4g+j] 2^(8j) < 2^50:
            // three independent wide multiply-adds per limb, then one add.cc/addc chain
            uint32_t lo[8], hi[8], P[8];
#pragma unroll
            for (int g = 0; g < 8; g++) {
              uint64_t w = (uint64_t)v[4 * g + 3] * m3;  // IMAD.WIDE chain, no zero-extension moves
              w += (uint64_t)v[4 * g + 2] * m2;
              w += (uint64_t)v[4 * g + 1] * m1;
              w += (uint64_t)v[4 * g] * m0;  // < 2^51
              lo[g] = (uint32_t)w;
              hi[g] = (uint32_t)(w >> 32);
            }
            asm("add.cc.u32 %0, %9, %8;\n\t"
              "addc.cc.u32 %1, %10, %17;\n\t"
              "addc.cc.u32 %2, %11, %18;\n\t"
              "addc.cc.u32 %3, %12, %19;\n\t"
              "addc.cc.u32 %4, %13, %20;\n\t"
              "addc.cc.u32 %5, %14, %21;\n\t"
              "addc.cc.u32 %6, %15, %22;\n\t"
              "addc.cc.u32 %7, %16, %23;\n\t"
              "addc.u32 %8, %24, 0;"
                : "=r"(P[0]), "=r"(P[1]), "=r"(P[2]), "=r"(P[3]), "=r"(P[4]), "=r"(P[5]), "=r"(P[6]), "=r"(P[7]), "+r"(carry)
                : "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7]));
#if !DS_VAR_MULSHIFT
#pragma unroll
            for (int g = 0; g < 8; g++) {
              const uint32_t raw = P[g];
              P[g] = __funnelshift_l(praw, raw, nsh);
              praw = raw;
            }
#endif

            const int g0 = (a.c_lo + t * TN + cb) >> 2;
            ok = em.block<8, true>(g0, P);  // r' - zb = 32 L: aligned limbs
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_tempty[grp][buf]);
      }
      if (process && ok) {
#if DS_VAR_MULSHIFT
        em.finish(carry ? 1.0 : 0.0);  // anything above the top limb of P'
#else
        em.finish((carry || (nsh && (praw >> 31))) ? 1.0 : 0.0);  // the bit shifted out of the top limb
#endif
        if (em.excess) ok = false;
      }
      if (process && !ok) fallback = true;
      if (process && ok && S.single) {
        if (!round_direct(S, neg, E, L, a.p, a.zb, a.a_exp + idx, a.a_cls + idx, a.status)) {
          fallback = true;
          atomicAdd(&a.status[7], 1);  // direct-mode misprediction (counted; exact fallback)
        }
      } else if (process && ok) {
        if (tile_io)
          round_out<true>(S, neg, E, L, a.p, a.zb, nullptr, 0, a.a_exp + idx, a.a_cls + idx, a.status);
        else
          round_write(S, neg, E, L, a.p, a.zb, a.a_limbs + idx, a.a_count, a.a_exp + idx, a.a_cls + idx, a.status);
      }
      if (fallback) {
        if (tile_io && process) {  // the window was written: the tile store must put a back unchanged
          const uint32_t* A = a.a_limbs + idx;
          for (int l = 0; l < L; l++) Sw[(l + 1) * TM] = A[(int64_t)l * a.a_count];
        }
        int slot = atomicAdd(a.fb_count, 1);
        if (slot < a.fb_cap) a.fb_list[slot] = make_int2(jl, k);
        else atomicAdd(&a.status[5], 1);
      }
      if (tile_io) {  // all 128 results of the row in the window -> one tile store
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_pipe(1 + NG + grp, TM);
        if (r == 0) tma_store_2d(&amap, tx, 0, region + TM);
      }
    }
    if (tile_io && r == 0) bulk_wait0();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// exact general-engine update of the listed elements (undecided short
// products / uncertain normalisation): mul_rn then add_rn (ds_mp.cuh)
__global__ void k_tc_fallback(TcArgs a, const uint32_t* z_limbs, int64_t z_count, const uint32_t* b_limbs,
                              uint32_t* scratch, int64_t sthreads) {
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  int cnt = *a.fb_count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && cnt > 0) atomicAdd(&a.status[6], cnt);
  if (cnt > a.fb_cap) cnt = a.fb_cap;
  const int L = a.L;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
    int2 e = a.fb_list[q];
    int jl = e.x, k = e.y;
    int64_t idx = (int64_t)jl * a.n + k;
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    ds::Ptr tmp{scratch + tid, sthreads};
    ds::Ptr tv = tmp, work = tmp.off(2 * (int64_t)L + 4), res = work.off(2 * (int64_t)L + 4);
    ds::Val z{ds::CPtr{z_limbs + jl, z_count}, a.zexp[jl - a.jl0], a.zcls[jl - a.jl0]};
    ds::Val b{ds::CPtr{b_limbs + k, a.n}, a.bexp[k], a.bcls[k]};
    int32_t te;
    uint8_t tc;
    ds::mul_rn(tv, &te, &tc, z, b, L, a.p, work);
    ds::Val t{ds::CPtr{tv.p, tv.s}, te, tc};
    ds::Val av{ds::CPtr{a.a_limbs + idx, a.a_count}, a.a_exp[idx], a.a_cls[idx]};
    int32_t re;
    uint8_t rc;
    if (!ds::add_rn(res, &re, &rc, av, t, true, L, a.p, work)) atomicAdd(&a.status[2], 1);
    for (int l = 0; l < L; l++) a.a_limbs[(int64_t)l * a.a_count + idx] = res[l];
    a.a_exp[idx] = re;
    a.a_cls[idx] = rc;
  }
}

// ================================================================ wide precision
// Above ~8192 bits the pivot-row digits no longer fit in TMEM and the per-column
// windows of a no longer fit in shared memory, so the update splits in two:
//   k_prod_tcw   the short products P_jk = z_j * b_k (digit columns c >= c_lo)
//                on the tensor cores, A = pivot-row digits streamed by TMA per
//                K chunk, B = the row's Toeplitz bank built per chunk; the
//                epilogue carries the digit sums into 32-bit limbs and stores
//                limbs q >= c_lo / 4 of every product (plane-major, coalesced)
//   k_tcw_finish one thread per element: decides RN(P) at p bits from the
//                stored limbs (undecidable -> the exact fallback list), then
//                a <- RN(a - RN(P)) with the general engine's add_rn
// Work per element: O(L^2) digit MACs on the tensor pipe vs O(L) in the finish.
constexpr int TW_EPI = 128;                 // epilogue threads (TMEM lanes = columns)
constexpr int TW_PROD = 128;                // bank / TMA producer threads
constexpr int TW_THREADS = TW_EPI + TW_PROD + 32;  // + one MMA issuer warp
constexpr int TW_ZLO = -128;                // zw[x] = Z[TW_ZLO + x]

struct TwArgs {
  int p, L, D8p, nks, c_lo, qlo, W, eps;
  int tn, ntiles, kc, nst, brc;  // MMA N, tiles, K steps per stage, stages, bank rows per stage
  int nrows, rbr, kstart, ncp, zwb;
  const uint8_t* zbytes;  // the chunk's rows [nrows][D8p]
  const uint8_t* apack;   // k_tcw_pack image of the pivot-row digits
  uint32_t* tprod;        // [W][nrows][ncp]
  int64_t pstride;        // nrows * ncp
  int32_t* status;
  int step;
};

__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// pivot-row digits packed in the MMA A operand's shared-memory image: for column
// tile ct (128 columns from kstart) and K step ks, 2 halves x 128 rows x 16 B
// (digits 32 ks + 16 h .. +16 of column kstart + 128 ct + r), so one stage of A
// is one contiguous bulk copy.  One thread per 16-byte piece (4 limbs).
__global__ void k_tcw_pack(const uint32_t* b_limbs, int n, int L, int nks, int kstart, int ntile, uint8_t* apack) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)ntile * nks * 2 * TM) return;
  const int r = (int)(t % TM);
  const int64_t rest = t / TM;  // (ct * nks + ks) * 2 + h
  const int h = (int)(rest & 1);
  const int ks = (int)((rest >> 1) % nks);
  const int ct = (int)((rest >> 1) / nks);
  const int col = kstart + ct * TM + r;
  const int l0 = 8 * ks + 4 * h;
  uint32_t v[4];
#pragma unroll
  for (int u = 0; u < 4; u++) v[u] = (col < n && l0 + u < L) ? b_limbs[(int64_t)(l0 + u) * n + col] : 0u;
  *(uint4*)(apack + rest * 2048 + (int64_t)r * 16) = make_uint4(v[0], v[1], v[2], v[3]);
}

__device__ __forceinline__ void tld32(uint32_t (&v)[32], uint32_t addr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr));
}

__global__ void __launch_bounds__(TW_THREADS, 1) k_prod_tcw(TwArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_full[8];
  __shared__ __align__(8) uint64_t bar_empty[8];
  __shared__ __align__(8) uint64_t bar_tfull[2];
  __shared__ __align__(8) uint64_t bar_tempty[2];
  __shared__ uint32_t tmem_base_sh;
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int TN = a.tn, KC = a.kc, NST = a.nst, BRC = a.brc, D8p = a.D8p;
  const uint32_t ABYTES = (uint32_t)KC * 4096u;               // A chunk: KC steps x (2 halves x 128 rows x 16 B)
  const uint32_t SBYTES = ABYTES + (uint32_t)BRC * 32u;       // + bank: 2 halves x BRC rows x 16 B
  uint8_t* zw = smem + (size_t)NST * SBYTES;
  const int kbase = a.kstart + (int)blockIdx.x * TM;
  const int row0 = (int)blockIdx.y * a.rbr;
  const int nrow_cta = min(a.rbr, a.nrows - row0);
  if (tid == 0) {
    for (int s = 0; s < NST; s++) {
      mbar_init(&bar_full[s], TW_PROD);
      mbar_init(&bar_empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&bar_tfull[b], 1);
      mbar_init(&bar_tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  if (tid >= TW_EPI && tid < TW_EPI + TW_PROD) {
    // =================================================== producers
    const int ptid = tid - TW_EPI;
    int sc = 0;  // stage counter
    for (int ri = 0; ri < nrow_cta; ri++) {
      bar_pipe(1, TW_PROD);  // every producer is done with the previous row's zw
      const uint8_t* zrow = a.zbytes + (int64_t)(row0 + ri) * D8p;
      for (int v = ptid; v < a.zwb / 4; v += TW_PROD) {
        const int t = TW_ZLO + 4 * v;
        ((uint32_t*)zw)[v] = (t >= 0 && t < D8p) ? *(const uint32_t*)(zrow + t) : 0u;
      }
      bar_pipe(1, TW_PROD);
      for (int t = 0; t < a.ntiles; t++) {
        const int c0 = a.c_lo + t * TN;
        const int s_lo = max(0, c0 - (D8p - 1)), s_hi = min(D8p - 1, c0 + TN - 1);
        const int ks0 = s_lo / KS, ks1 = s_hi / KS;
        for (int ka = ks0; ka <= ks1; ka += KC, sc++) {
          const int kb = min(ks1, ka + KC - 1);
          const int st = sc % NST;
          if (sc >= NST) mbar_wait(&bar_empty[st], ((sc / NST) - 1) & 1);
          uint8_t* A = smem + (size_t)st * SBYTES;
          uint8_t* bank = A + ABYTES;
          if (ptid == 0) {
            const uint32_t bytes = (uint32_t)(kb - ka + 1) * 4096u;
            mbar_expect(&bar_full[st], bytes);
            bulk_load(A, a.apack + ((int64_t)blockIdx.x * a.nks + ka) * 4096, bytes, &bar_full[st]);
          }
          // bank row r <-> m = c0 - 32 kb + r: half h holds Z[m - 16h - j], j = 0..15
          const int bru = TN + KS * (kb - ka);
          const int mb = c0 - KS * kb;
          for (int c = ptid; c < 2 * bru; c += TW_PROD) {
            const int h = c >= bru ? 1 : 0, r = c - h * bru;
            const int off = mb + r - 16 * h - 15 - TW_ZLO;
            const uint32_t* wp = (const uint32_t*)zw + (off >> 2);
            const int sh = 8 * (off & 3);
            uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2], w3 = wp[3], w4 = wp[4];
            uint32_t x0 = __funnelshift_r(w0, w1, sh), x1 = __funnelshift_r(w1, w2, sh);
            uint32_t x2 = __funnelshift_r(w2, w3, sh), x3 = __funnelshift_r(w3, w4, sh);
            *(uint4*)(bank + h * BRC * 16 + (r >> 3) * 128 + (r & 7) * 16) =
                make_uint4(__byte_perm(x3, 0, 0x0123), __byte_perm(x2, 0, 0x0123), __byte_perm(x1, 0, 0x0123),
                           __byte_perm(x0, 0, 0x0123));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&bar_full[st]);
        }
      }
    }
  } else if (tid >= TW_EPI + TW_PROD) {
    // =================================================== MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_i8(TM, TN);
      int sc = 0, gt = 0;
      for (int ri = 0; ri < nrow_cta; ri++) {
        for (int t = 0; t < a.ntiles; t++, gt++) {
          const int buf = gt & 1;
          if (gt >= 2) mbar_wait(&bar_tempty[buf], ((gt >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t dcol = tmem + (uint32_t)(buf * TN);
          const int c0 = a.c_lo + t * TN;
          const int s_lo = max(0, c0 - (D8p - 1)), s_hi = min(D8p - 1, c0 + TN - 1);
          const int ks0 = s_lo / KS, ks1 = s_hi / KS;
          for (int ka = ks0; ka <= ks1; ka += KC, sc++) {
            const int kb = min(ks1, ka + KC - 1);
            const int st = sc % NST;
            mbar_wait(&bar_full[st], (sc / NST) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t A = smem_u32(smem + (size_t)st * SBYTES);
            const uint32_t B = A + ABYTES;
            for (int ks = ka; ks <= kb; ks++) {
              const uint64_t ad = umma_desc(A + (uint32_t)(ks - ka) * 4096u, 2048u, 128u);
              const uint64_t bd = umma_desc(B + (uint32_t)(kb - ks) * 512u, (uint32_t)BRC * 16u, 128u);
              const uint32_t acc = ks > ks0 ? 1u : 0u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dcol),
                  "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
            umma_commit(&bar_empty[st]);
          }
          umma_commit(&bar_tfull[buf]);
        }
      }
    }
    __syncwarp();
  } else {
    // =================================================== epilogue: digit sums -> limbs
    const int r = tid;  // column within the tile = TMEM lane
    const int col = (int)blockIdx.x * TM + r;
    int gt = 0;
    for (int ri = 0; ri < nrow_cta; ri++) {
      uint32_t* out = a.tprod + (int64_t)(row0 + ri) * a.ncp + col;
      uint32_t carry = 0;
      for (int t = 0; t < a.ntiles; t++, gt++) {
        const int buf = gt & 1;
        mbar_wait(&bar_tfull[buf], (gt >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(buf * TN);
        const int c0 = a.c_lo + t * TN;
        const int cend = min(TN, 2 * D8p - c0);
        // limb q = w_q + hi(w_(q-1)) + carry, w_q = sum_j v[4q+j] 2^(8j) < 2^54: independent
        // wide multiply-adds, one add.cc chain per 8 limbs; the next 32 columns are
        // loaded from TMEM while this chunk is converted and stored
        auto conv = [&](const uint32_t(&v)[32], int cb) {
          uint32_t lo[8], hi[8], P[8];
#pragma unroll
          for (int g = 0; g < 8; g++) {
            uint64_t w = (uint64_t)v[4 * g + 3] * 16777216u;
            w += (uint64_t)v[4 * g + 2] * 65536u;
            w += (uint64_t)v[4 * g + 1] * 256u;
            w += (uint64_t)v[4 * g] * 1u;
            lo[g] = (uint32_t)w;
            hi[g] = (uint32_t)(w >> 32);
          }
          asm("add.cc.u32 %0, %9, %8;\n\t"
              "addc.cc.u32 %1, %10, %17;\n\t"
              "addc.cc.u32 %2, %11, %18;\n\t"
              "addc.cc.u32 %3, %12, %19;\n\t"
              "addc.cc.u32 %4, %13, %20;\n\t"
              "addc.cc.u32 %5, %14, %21;\n\t"
              "addc.cc.u32 %6, %15, %22;\n\t"
              "addc.cc.u32 %7, %16, %23;\n\t"
              "addc.u32 %8, %24, 0;"
              : "=r"(P[0]), "=r"(P[1]), "=r"(P[2]), "=r"(P[3]), "=r"(P[4]), "=r"(P[5]), "=r"(P[6]), "=r"(P[7]),
                "+r"(carry)
              : "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]),
                "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7]));
          const int q0 = (c0 + cb) >> 2;
          uint32_t* op = out + (int64_t)(q0 - a.qlo) * a.pstride;
          if (q0 + 8 <= 2 * a.L) {
#pragma unroll
            for (int g = 0; g < 8; g++) {
              *op = P[g];
              op += a.pstride;
            }
          } else {
#pragma unroll
            for (int g = 0; g < 8; g++) {
              if (q0 + g < 2 * a.L) *op = P[g];
              op += a.pstride;
            }
          }
        };
        uint32_t va[32], vb[32];
        tld32(va, taddr);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll 1
        for (int cb = 0; cb < cend; cb += 64) {
          const bool m1 = cb + 32 < cend, m2 = cb + 64 < cend;
          if (m1) tld32(vb, taddr + cb + 32);
          conv(va, cb);
          if (m1) {
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            if (m2) tld32(va, taddr + cb + 64);
            conv(vb, cb + 32);
            if (m2) asm volatile("tcgen05.wait::ld.sync.aligned;");
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_tempty[buf]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// bits [lo, hi) of S all ones / all zeros (hi > lo)
__device__ __forceinline__ void bit_range(ds::CPtr S, int n, int64_t lo, int64_t hi, bool* ones, bool* zeros) {
  bool o = true, z = true;
  for (int64_t pos = lo; pos < hi; pos += 32) {
    const int nb = (int)min((int64_t)32, hi - pos);
    const uint32_t mask = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
    const uint32_t v = ds::bits32(S, n, pos) & mask;
    if (v != mask) o = false;
    if (v != 0) z = false;
  }
  *ones = o;
  *zeros = z;
}

// bits32(src, n, 32 k + off) for k = 0, 1, 2, ... with one load per limb
struct BitStream {
  ds::CPtr s;
  int n, sh;
  int64_t lw;
  uint32_t lo;
  __device__ __forceinline__ uint32_t get(int64_t i) const { return (i >= 0 && i < n) ? s[i] : 0u; }
  __device__ __forceinline__ void init(ds::CPtr src, int nl, int64_t off) {
    s = src;
    n = nl;
    lw = off >> 5;
    sh = (int)(off & 31);
    lo = get(lw);
  }
  __device__ __forceinline__ uint32_t next() {
    const uint32_t hi = get(lw + 1);
    const uint32_t r = __funnelshift_r(lo, hi, sh);
    lo = hi;
    lw++;
    return r;
  }
};

// the limbs T[0], T[1], ... of T = RN(P) (left-aligned L limbs): P's bits from
// S bit offT up, the low zb bits cleared, + inc at bit zb with carry
struct TGen {
  BitStream b;
  int k, zl, zs;
  uint32_t carry, inc;
  __device__ __forceinline__ void init(ds::CPtr S, int W, int64_t offT, int zb, uint32_t incr) {
    b.init(S, W, offT);
    k = 0;
    zl = zb >> 5;
    zs = zb & 31;
    carry = 0;
    inc = incr;
  }
  __device__ __forceinline__ uint32_t next() {
    uint32_t v = b.next();
    uint64_t t;
    if (k < zl) {
      t = 0;
    } else if (k == zl) {
      v &= ~((1u << zs) - 1u);
      t = (uint64_t)v + ((uint64_t)inc << zs);
    } else {
      t = (uint64_t)v + carry;
    }
    carry = (uint32_t)(t >> 32);
    k++;
    return (uint32_t)t;
  }
};

// a_jk <- RN(a_jk - RN(P_jk)) for the chunk's elements.  Fast path: T = RN(P)
// is generated limb by limb from the stored product limbs and summed with a in
// one pass into scratch ([word][thread], L + d/32 + 2 words), then rounded into
// a's limbs.  Equal exponents with top limbs within one (the order of |a| and
// |T| unknown before the carry): T materialised and the general add_rn.
// Undecidable RN(P), or T rounding up to 2^p: the exact fallback list.
__global__ void __launch_bounds__(256, DS_TCW_FINISH_MINB) k_tcw_finish(TcArgs a, TwArgs w, int row_first, uint32_t* scratch,
                                                    int64_t sthreads) {
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  const int L = a.L, p = a.p, zb = 32 * L - p;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)w.nrows * a.ncols;
  // per-thread scratch row (contiguous, 32-byte aligned): the S2 limbs are written
  // as whole sectors and re-read at per-element offsets from L1
  const int RW = (3 * L + 24 + 7) & ~7;
  (void)sthreads;
  uint32_t* row = scratch + tid * (int64_t)RW;
  ds::Ptr tmp{row, 1};
  for (int64_t e = tid; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int ri = (int)(e / a.ncols), cidx = (int)(e % a.ncols);
    const int k = a.kstart + cidx;
    if (k < a.kmin || k == a.skip_col || k >= a.n) continue;
    const int zr = row_first + ri;  // relative to jl0
    const int jl = a.jl0 + zr;
    const int64_t idx = (int64_t)jl * a.n + k;
    const uint8_t cz = a.zcls[zr], cb = a.bcls[k], ca = a.a_cls[idx];
    const int st = (cz & 1) ^ (cb & 1);
    if (cz >= DS_CLS_PZERO || cb >= DS_CLS_PZERO) {  // a - (+-0)
      if (ca >= DS_CLS_PZERO) a.a_cls[idx] = ((ca & 1) && !st) ? DS_CLS_NZERO : DS_CLS_PZERO;
      continue;
    }
    const ds::CPtr S{w.tprod + (int64_t)ri * w.ncp + cidx, w.pstride};
    const int W = w.W;
    const uint32_t stop = S[W - 1];
    const int64_t hb = 32 * (int64_t)(W - 1) + 31 - __clz(stop);  // P >= 2^(64L-2): top limb nonzero
    const int64_t lsb = hb - p + 1;
    bool amb = lsb - 1 <= w.eps;
    uint32_t g = 0;
    if (!amb) {
      bool ones, zeros, lo_ones, lz;
      bit_range(S, W, w.eps, lsb - 1, &ones, &zeros);
      g = ds::bits32(S, W, lsb - 1) & 1u;
      bit_range(S, W, 0, w.eps, &lo_ones, &lz);
      amb = ones || (g && zeros && lz);
    }
    const int64_t offT = hb + 1 - 32 * (int64_t)L;
    // rounding T up overflows to 2^p only if its p kept bits are all ones (rare): exact engine
    if (!amb && g) {
      bool ones = true;  // scanned from the top: almost always decided by the first word
      for (int64_t pos = hb + 1; pos > lsb && ones; pos -= 32) {
        const int nb = (int)min((int64_t)32, pos - lsb);
        const uint32_t v = ds::bits32(S, W, pos - nb) | (nb == 32 ? 0u : ~((1u << nb) - 1u));
        ones = v == 0xffffffffu;
      }
      amb = ones;
    }
    if (amb) {
      int slot = atomicAdd(a.fb_count, 1);
      if (slot < a.fb_cap) a.fb_list[slot] = make_int2(jl, k);
      else atomicAdd(&a.status[5], 1);
      continue;
    }
    const int64_t eT = (int64_t)a.zexp[zr] + a.bexp[k] - 64 * (int64_t)L + 32 * (int64_t)w.qlo + hb + 1;
    const int nT = st ^ 1;  // sign of -T
    const ds::Ptr out{a.a_limbs + idx, a.a_count};
    TGen tg;
    tg.init(S, W, offT, zb, g);
    if (ca >= DS_CLS_PZERO) {  // 0 - T = -T exactly
      for (int l = 0; l < L; l++) out[l] = tg.next();
      a.a_exp[idx] = (int32_t)eT;
      a.a_cls[idx] = ds::nz_cls(nT);
      if (!ds::range_ok(eT)) atomicAdd(&a.status[2], 1);
      continue;
    }
    const int na = ca & 1;
    const int64_t ea = a.a_exp[idx];
    const ds::CPtr am{a.a_limbs + idx, a.a_count};
    int xa;  // 1: |a| > |T|, 0: |T| > |a|, -1: undecided here
    if (ea != eT) {
      xa = ea > eT ? 1 : 0;
    } else {
      const uint32_t at = am[L - 1], tt = ds::bits32(S, W, 32 * (int64_t)(L - 1) + offT);
      xa = (at > tt && at - tt >= 2u) ? 1 : ((tt > at && tt - at >= 2u) ? 0 : -1);
    }
    if (xa < 0) {
      // general path: T into scratch, add_rn (needs 2L + 4 more words)
      ds::Ptr T = tmp;
      for (int l = 0; l < L; l++) T[l] = tg.next();
      ds::Val t{ds::CPtr{T.p, T.s}, eT, (uint8_t)(st ? DS_CLS_NEG : DS_CLS_POS)};
      ds::Val av{am, ea, ca};
      int32_t re;
      uint8_t rc;
      if (!ds::add_rn(out, &re, &rc, av, t, true, L, p, tmp.off(L))) atomicAdd(&a.status[2], 1);
      a.a_exp[idx] = re;
      a.a_cls[idx] = rc;
      continue;
    }
    const int64_t d = xa ? ea - eT : eT - ea;
    if (d >= (int64_t)p + 2) {  // RN(X +- Y) = X
      if (!xa) {
        for (int l = 0; l < L; l++) out[l] = tg.next();
        a.a_exp[idx] = (int32_t)eT;
        a.a_cls[idx] = ds::nz_cls(nT);
        if (!ds::range_ok(eT)) atomicAdd(&a.status[2], 1);
      }
      continue;
    }
    const bool sub = na != nT;
    const int n2 = L + (int)(d >> 5) + 2;
    constexpr int FB = 8;  // limbs per batch (16 measured the same)
    // S2 = X 2^d +- Y (X the larger operand) into scratch, 8 limbs per batch so
    // each thread keeps ~16 independent loads in flight
    const int64_t lwT = offT >> 5;  // T(i) = low-masked funnel(S[lwT + i], S[lwT + i + 1], shT) + carry
    const int shT = (int)(offT & 31);
    const int zl = zb >> 5, zs = zb & 31;
    uint32_t tcar = 0;
    auto tval = [&](int64_t i, uint32_t raw) -> uint32_t {
      if (i < zl || i >= L) return 0u;  // (i < 0 included)
      uint64_t t;
      if (i == zl) t = (uint64_t)(raw & ~((1u << zs) - 1u)) + ((uint64_t)g << zs);
      else t = (uint64_t)raw + tcar;
      tcar = (uint32_t)(t >> 32);
      return (uint32_t)t;
    };
    auto sget = [&](int64_t i) -> uint32_t { return (i >= 0 && i < W) ? S[i] : 0u; };
    auto aget = [&](int64_t i) -> uint32_t { return (i >= 0 && i < L) ? am[i] : 0u; };
    const int64_t lwX = (-d) >> 5;  // X2[q] = funnel(X(q + lwX), X(q + lwX + 1), shX)
    const int shX = (int)((-d) & 31);
    uint32_t cb2 = 0;
    uint32_t tprev = 0;  // X = T: T(q0 + lwX) carried between batches
    if (!xa) tprev = tval(lwX, __funnelshift_r(sget(lwT + lwX), sget(lwT + lwX + 1), shT));
    // X - Y as X + ~Y + 1: one branch-free carry chain for both signs
    const uint32_t ym = sub ? 0xffffffffu : 0u;
    cb2 = sub ? 1u : 0u;
    for (int q0 = 0; q0 < n2; q0 += FB) {
      const int64_t ti0 = xa ? q0 : q0 + lwX + 1;  // first new T index of the batch
      const int64_t ai0 = xa ? q0 + lwX : q0;      // first a index of the batch
      uint32_t sv[FB + 1], av[FB + 1], tv[FB], s2[FB];
      if (lwT + ti0 >= 0 && lwT + ti0 + FB < W && ti0 > zl && ti0 + FB <= L && ai0 >= 0 && ai0 + FB < L) {
        // interior batch: no bounds, no low mask
#pragma unroll
        for (int u = 0; u < FB + 1; u++) sv[u] = S[lwT + ti0 + u];
#pragma unroll
        for (int u = 0; u < FB + 1; u++) av[u] = am[ai0 + u];
#pragma unroll
        for (int u = 0; u < FB; u++) {
          const uint64_t t = (uint64_t)__funnelshift_r(sv[u], sv[u + 1], shT) + tcar;
          tcar = (uint32_t)(t >> 32);
          tv[u] = (uint32_t)t;
        }
      } else {
#pragma unroll
        for (int u = 0; u < FB + 1; u++) sv[u] = sget(lwT + ti0 + u);
#pragma unroll
        for (int u = 0; u < FB + 1; u++) av[u] = aget(ai0 + u);
#pragma unroll
        for (int u = 0; u < FB; u++) tv[u] = tval(ti0 + u, __funnelshift_r(sv[u], sv[u + 1], shT));
      }
#pragma unroll
      for (int u = 0; u < FB; u++) {
        const uint32_t lo = xa ? av[u] : (u == 0 ? tprev : tv[u - 1]);
        const uint32_t hi = xa ? av[u + 1] : tv[u];
        const uint32_t x = __funnelshift_r(lo, hi, shX);
        const uint32_t y = (xa ? tv[u] : av[u]) ^ ym;
        const uint64_t t = (uint64_t)x + y + cb2;
        cb2 = (uint32_t)(t >> 32);
        s2[u] = (uint32_t)t;
      }
      tprev = tv[FB - 1];
#pragma unroll
      for (int u = 0; u < FB; u += 4) *(uint4*)(row + q0 + u) = make_uint4(s2[u], s2[u + 1], s2[u + 2], s2[u + 3]);
    }
    // round S2 (n2 limbs, nonzero) to p bits into a's limbs
    const ds::CPtr S2{tmp.p, tmp.s};
    int64_t hb2 = -1;
    for (int q = n2 - 1; q >= 0; q--) {
      const uint32_t v = S2[q];
      if (v) {
        hb2 = 32 * (int64_t)q + 31 - __clz(v);
        break;
      }
    }
    const int64_t lsb2 = hb2 - p + 1;
    uint32_t inc = 0;
    if (lsb2 >= 1 && ((ds::bits32(S2, n2, lsb2 - 1) & 1u) != 0)) {
      const bool sticky = ds::any_below(S2, n2, lsb2 - 1);
      const bool lsbit = (ds::bits32(S2, n2, lsb2) & 1u) != 0;
      inc = (sticky || lsbit) ? 1u : 0u;
    }
    const int64_t off2 = hb2 + 1 - 32 * (int64_t)L;
    const int64_t lw2 = off2 >> 5;
    const int sh2 = (int)(off2 & 31);
    uint32_t rc2 = 0;
    for (int l0 = 0; l0 < L; l0 += FB) {
      uint32_t v[FB + 1];
      if (lw2 + l0 >= 0 && lw2 + l0 + FB < n2 && l0 > zl && l0 + FB <= L) {  // interior batch
#pragma unroll
        for (int u = 0; u < FB + 1; u++) v[u] = S2[lw2 + l0 + u];
#pragma unroll
        for (int u = 0; u < FB; u++) {
          const uint64_t t = (uint64_t)__funnelshift_r(v[u], v[u + 1], sh2) + rc2;
          rc2 = (uint32_t)(t >> 32);
          out[l0 + u] = (uint32_t)t;
        }
        continue;
      }
#pragma unroll
      for (int u = 0; u < FB + 1; u++) {
        const int64_t q = lw2 + l0 + u;
        v[u] = (q >= 0 && q < n2) ? S2[q] : 0u;
      }
#pragma unroll
      for (int u = 0; u < FB; u++) {
        const int l = l0 + u;
        if (l < L) {
          const uint32_t raw = __funnelshift_r(v[u], v[u + 1], sh2);
          uint64_t t;
          if (l < zl) t = 0;
          else if (l == zl) t = (uint64_t)(raw & ~((1u << zs) - 1u)) + ((uint64_t)inc << zs);
          else t = (uint64_t)raw + rc2;
          rc2 = (uint32_t)(t >> 32);
          out[l] = (uint32_t)t;
        }
      }
    }
    int64_t e2 = (xa ? eT : ea) - 32 * (int64_t)L + hb2 + 1;
    if (rc2) {  // the mantissa rounded up to 2^p
      out[L - 1] = 0x80000000u;
      e2 += 1;
    }
    a.a_exp[idx] = (int32_t)e2;
    a.a_cls[idx] = ds::nz_cls(xa ? na : nT);
    if (!ds::range_ok(e2)) atomicAdd(&a.status[2], 1);
  }
}

// ---------------------------------------------------------------- complex
// a <- RN(a - RN(z b)) per component on the wide engine (elim.py:49-52 on mpc).
//
// One element (row ri of the chunk, column index cidx) of the complex finish; a's
// limbs of component c are read and written through am[c] (global planes, or a
// shared-memory staging copy).  Returns false when the element went to the
// fallback list (a unchanged).
__device__ bool finish_c_elem(const TcArgs& a, const TwArgs& w, int ri, int cidx, int row_first, ds::Ptr Ssum,
                              ds::Ptr Tre, ds::Ptr Tim, ds::Ptr tmp, const ds::Ptr* am) {
  const int L = a.L, p = a.p;
  const int k = a.kstart + cidx;
  const int zr = row_first + ri;  // relative to jl0
  const int jl = a.jl0 + zr;
  const int64_t idx = (int64_t)jl * a.n + k;
  const int64_t region = w.pstride * (int64_t)w.W;  // words per product region (c1, c2)
  int64_t ze[2], be[2];
  uint8_t zc[2], bc[2];
  for (int c = 0; c < 2; c++) {
    ze[c] = a.zexp[(int64_t)c * a.zstride + zr];
    zc[c] = a.zcls[(int64_t)c * a.zstride + zr];
    be[c] = a.bexp[(int64_t)c * a.n + k];
    bc[c] = a.bcls[(int64_t)c * a.n + k];
  }
  auto term = [&](int c1, int c2) -> ds::XTerm {
    ds::XTerm t;
    t.m = ds::CPtr{w.tprod + (2 * c1 + c2) * region + (int64_t)ri * w.ncp + cidx, w.pstride};
    t.n = w.W;
    t.base = ze[c1] + be[c2] - 64 * (int64_t)L + 32 * (int64_t)w.qlo;
    t.neg = (zc[c1] & 1) ^ (bc[c2] & 1);
    t.zero = zc[c1] >= DS_CLS_PZERO || bc[c2] >= DS_CLS_PZERO;
    return t;
  };
  bool ok = true;
  int32_t te[2];
  uint8_t tcl[2];
  for (int c = 0; c < 2 && ok; c++) {
    const ds::XTerm X = c == 0 ? term(0, 0) : term(0, 1);
    const ds::XTerm Y = c == 0 ? term(1, 1) : term(1, 0);
    const ds::XSum x = ds::exact_sum(Ssum, X, Y, c == 0, 2 * (int64_t)p + 64);
    if (x.zero) {
      ok = X.zero && Y.zero;  // a truncated nonzero sum that cancels: undecided
    } else {
      const int64_t H = x.base + ds::top_bit(ds::CPtr{Ssum.p, Ssum.s}, x.n);
      const int64_t R = H - p + 1;  // weight of the result's LSB
      int64_t bnd = INT64_MIN;
      int64_t tmin = INT64_MAX;
      if (!X.zero) {
        bnd = max(bnd, X.base + w.eps);
        tmin = min(tmin, X.base + ds::top_bit(X.m, X.n));
      }
      if (!Y.zero) {
        bnd = max(bnd, Y.base + w.eps);
        tmin = min(tmin, Y.base + ds::top_bit(Y.m, Y.n));
      }
      bnd += 1;                                // both errors together < 2^bnd
      if (x.pert) bnd = max(bnd, tmin + 2);    // the far term only perturbs
      if (R - 1 <= bnd) {
        ok = false;
      } else {
        bool ones, zeros;
        bit_range(ds::CPtr{Ssum.p, Ssum.s}, x.n, max((int64_t)0, bnd - x.base), R - 1 - x.base, &ones, &zeros);
        ok = !ones && !zeros;
      }
    }
    if (ok) {
      const ds::Ptr T = c == 0 ? Tre : Tim;
      if (!ds::round_xsum(T, &te[c], &tcl[c], Ssum, x, L, p)) atomicAdd(&a.status[2], 1);
    }
  }
  if (!ok) {
    int slot = atomicAdd(a.fb_count, 1);
    if (slot < a.fb_cap) a.fb_list[slot] = make_int2(jl, k);
    else atomicAdd(&a.status[5], 1);
    return false;
  }
  for (int c = 0; c < 2; c++) {
    const int64_t mo = (int64_t)c * a.a_count + idx;
    ds::Val av{ds::CPtr{am[c].p, am[c].s}, a.a_exp[mo], a.a_cls[mo]};
    ds::Val tv{ds::CPtr{(c == 0 ? Tre : Tim).p, (c == 0 ? Tre : Tim).s}, te[c], tcl[c]};
    int32_t re;
    uint8_t rc;
    if (!ds::add_rn(am[c], &re, &rc, av, tv, true, L, p, tmp)) atomicAdd(&a.status[2], 1);
    a.a_exp[mo] = re;
    a.a_cls[mo] = rc;
  }
  return true;
}

// Re = RN(zr br - zi bi), Im = RN(zr bi + zi br), each the exact formula rounded
// once (mpc_mul), then a_c <- RN(a_c - t_c) (mpc_sub).  The four products come
// from k_prod_tcw as truncated limbs (each short by < 2^eps units of its limb
// q_lo); their exact aligned sum (ds::exact_sum) is rounded when the bits
// between the combined error bound and the round bit are neither all zeros nor
// all ones, so no rounding boundary lies within the error; else the element
// takes the exact complex fallback.  Scratch row per thread: sum | T_re | T_im |
// add_rn.  Thread per element (DS_CX_FINISH_THREAD=1; the default is the
// warp-cooperative k_cfw_finish below).
__global__ void __launch_bounds__(256) k_tcw_finish_c(TcArgs a, TwArgs w, int row_first, uint32_t* scratch) {
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  const int L = a.L;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)w.nrows * a.ncols;
  // per-thread scratch interleaved across the grid (word k of thread t at k * T + t):
  // the generic limb loops below touch the same word index in every lane, so each
  // warp access is one coalesced line instead of 32 (and the rows stay in L2)
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  uint32_t* row = scratch + tid;
  const ds::Ptr Ssum{row, T}, Tre{row + (4 * (int64_t)L + 16) * T, T}, Tim{row + (5 * (int64_t)L + 16) * T, T},
      tmp{row + (6 * (int64_t)L + 16) * T, T};
  for (int64_t e = tid; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int ri = (int)(e / a.ncols), cidx = (int)(e % a.ncols);
    const int k = a.kstart + cidx;
    if (k < a.kmin || k == a.skip_col || k >= a.n) continue;
    const int64_t idx = (int64_t)(a.jl0 + row_first + ri) * a.n + k;
    const ds::Ptr am[2] = {ds::Ptr{a.a_limbs + idx, a.a_count}, ds::Ptr{a.a_limbs + (int64_t)L * a.a_count + idx,
                                                                       a.a_count}};
    finish_c_elem(a, w, ri, cidx, row_first, Ssum, Tre, Tim, tmp, am);
  }
}

#include "ds_cfinish.cuh"

// exact complex update of the listed elements: cmul_part x 2 then add_rn x 2
__global__ void k_tc_fallback_c(TcArgs a, const uint32_t* z_limbs, int64_t z_count, const uint32_t* b_limbs,
                                uint32_t* scratch, int64_t sthreads) {
  if (a.status[0] >= 0 && a.status[0] <= a.step) return;
  int cnt = *a.fb_count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && cnt > 0) atomicAdd(&a.status[6], cnt);
  if (cnt > a.fb_cap) cnt = a.fb_cap;
  const int L = a.L;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
    int2 e = a.fb_list[q];
    const int jl = e.x, k = e.y;
    const int zr = jl - a.jl0;
    const int64_t idx = (int64_t)jl * a.n + k;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    ds::Ptr base{scratch + tid, sthreads};
    ds::Ptr tre = base, tim = base.off(L), work = base.off(2 * (int64_t)L);
    ds::Val zv[2], bv[2], av[2];
    for (int c = 0; c < 2; c++) {
      zv[c] = ds::Val{ds::CPtr{z_limbs + (int64_t)c * L * z_count + jl, z_count}, a.zexp[(int64_t)c * a.zstride + zr],
                      a.zcls[(int64_t)c * a.zstride + zr]};
      bv[c] = ds::Val{ds::CPtr{b_limbs + (int64_t)c * L * a.n + k, a.n}, a.bexp[(int64_t)c * a.n + k],
                      a.bcls[(int64_t)c * a.n + k]};
      const int64_t mo = (int64_t)c * a.a_count + idx;
      av[c] = ds::Val{ds::CPtr{a.a_limbs + (int64_t)c * L * a.a_count + idx, a.a_count}, a.a_exp[mo], a.a_cls[mo]};
    }
    int32_t te[2];
    uint8_t tc[2];
    ds::cmul_part(tre, &te[0], &tc[0], zv[0], bv[0], zv[1], bv[1], true, L, a.p, work);
    ds::cmul_part(tim, &te[1], &tc[1], zv[0], bv[1], zv[1], bv[0], false, L, a.p, work);
    for (int c = 0; c < 2; c++) {
      ds::Val t{ds::CPtr{(c == 0 ? tre : tim).p, sthreads}, te[c], tc[c]};
      const int64_t mo = (int64_t)c * a.a_count + idx;
      int32_t re;
      uint8_t rc;
      if (!ds::add_rn(ds::Ptr{a.a_limbs + (int64_t)c * L * a.a_count + idx, a.a_count}, &re, &rc, av[c], t, true, L,
                      a.p, work))
        atomicAdd(&a.status[2], 1);
      a.a_exp[mo] = re;
      a.a_cls[mo] = rc;
    }
  }
}

size_t tc_smem(int L, int br, int ng) {
  const size_t zwl = ((br + 64) + 15) & ~15;
  return ng * ((size_t)br * KS + 4 * (size_t)(L + 2) * TM + zwl);
}

}  // namespace

// ---------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

static void launch_update(int ng, dim3 grid, size_t smem, cudaStream_t s, const TcArgs& a, const CUtensorMap& m) {
  if (ng == 4)
    k_update_tc<4><<<grid, Cfg<4>::NTHREADS, smem, s>>>(a, m);
  else if (ng == 3)
    k_update_tc<3><<<grid, Cfg<3>::NTHREADS, smem, s>>>(a, m);
  else if (ng == 2)
    k_update_tc<2><<<grid, Cfg<2>::NTHREADS, smem, s>>>(a, m);
  else
    k_update_tc<1><<<grid, Cfg<1>::NTHREADS, smem, s>>>(a, m);
}

#define CK_TC(x)                                   \
  do {                                             \
    if ((x) != cudaSuccess) return DS_CUDA;        \
  } while (0)

struct TcWork {
  uint8_t* zbytes;
  uint8_t* bbytes;
  double* zf;
  double* bf;
  int* fb_count;
  int2* fb_list;
  uint32_t* scratch;
  int64_t sthreads;
  int fb_cap;
  CUtensorMap amap;        // a planes: dims {a_count, L}, box {128, L}
  uint32_t* tprod;         // wide: product limbs [W][rows][ncp]
  uint32_t* tscratch;      // wide: finish-kernel scratch [3L + 8][tthreads]
  int64_t tthreads;
  int* zlow;               // complex warp finish: k_lowdig of z [2][nloc] and of the pivot row [2][n]
  int* blow;
  const void* amap_base;
  int64_t amap_count;
  int amap_ok;
};

static EncodeTiledFn encode_tiled();

// wide-precision plan: product kernel tiles, stages and the row chunk bounded by
// the product-limb buffer
// fallback-list entries per launch: every element one update launch can touch
// (nrows x ncols <= nloc x n), so inputs with many undecidable short products
// degrade to the exact path instead of overflowing; capped at 2^25 entries
// (256 MB per list) -- beyond it the overflow is counted in status[5] and
// reported as an error
static int fb_capacity(int nloc, int n) {
  const int64_t want = (int64_t)(nloc > 0 ? nloc : 1) * n;
  return (int)(want < (1 << 16) ? (1 << 16) : (want > (1 << 25) ? (1 << 25) : want));
}

static int tcw_plan_init(TcPlan* plan, int n, int nloc, int p, int device, int maxsm) {
  (void)device;
  const int L = plan->L, D8p = plan->D8p, zb = 32 * L - p;
  // short product: E < 2^eps units of limb q_lo; >= 32 decision bits between
  // 2^eps and the round bit (at >= 64 L - p - 2 in P)
  int clo = ((32 * L + zb - 34 - plan->eps) / 8) & ~3;
  if (clo < 0) clo = 0;
  int tn = 256;
  if (2 * D8p - clo < tn) tn = (2 * D8p - clo + 31) & ~31;
  if (clo + tn <= D8p || clo - D8p + 1 - 31 - TW_ZLO < 0) return DS_OK;  // zw window assumptions
  int kc = 16, nst = 2;  // tools/tcw_sweep.sh: -13 % product time at 32768 bits vs 8 x 3
  if (const char* e = getenv("DS_TCW_KC")) kc = atoi(e);
  if (const char* e = getenv("DS_TCW_NST")) nst = atoi(e);
  if (nst > 8) nst = 8;
  const int zwb = (D8p + tn + 256 + 15) & ~15;
  size_t sm = 0;
  for (;;) {
    sm = (size_t)nst * ((size_t)kc * 4096 + (size_t)(tn + KS * (kc - 1)) * 32) + zwb + 1024;
    if ((int)sm <= maxsm - 2048) break;
    if (nst > 2) nst--;
    else if (kc > 2) kc /= 2;
    else return DS_OK;
  }
  plan->wide = 1;
  plan->c_lo = clo;
  plan->tn = tn;
  plan->ntiles = (2 * D8p - clo + tn - 1) / tn;
  plan->w_kc = kc;
  plan->w_nst = nst;
  plan->w_brc = tn + KS * (kc - 1);
  plan->w_qlo = clo / 4;
  plan->w_W = 2 * L - clo / 4;
  plan->w_zwb = zwb;
  plan->w_rbr = 2;
  if (const char* e = getenv("DS_TCW_RBR")) plan->w_rbr = atoi(e) > 0 ? atoi(e) : 1;
  plan->smem = sm;
  if (cudaFuncSetAttribute(k_prod_tcw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return DS_CUDA;
  const int64_t ncp = (int64_t)((n + TM - 1) / TM) * TM;
  size_t budget = (size_t)2 << 30;
  if (const char* e = getenv("DS_TCW_BUDGET_MB")) budget = (size_t)atol(e) << 20;
  const int nc = plan->ncomp > 1 ? 2 : 1;
  int64_t rows = (int64_t)(budget / ((size_t)ncp * plan->w_W * 4 * nc * nc));
  if (rows < 1) rows = 1;
  if (rows > nloc) rows = nloc > 0 ? nloc : 1;
  plan->w_rows = (int)rows;
  TcWork* w = new TcWork();
  memset(w, 0, sizeof(*w));
  plan->work = w;
  w->fb_cap = fb_capacity(nloc, n);
  w->sthreads = 64 * 128;
  {  // finish-kernel threads: 6 blocks of 256 per SM (measured: -4 % update at 16384 bits vs 3, equal at
     // 33220 bits and for complex; DS_TCW_FINISH_BLOCKS overrides, A/B)
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    int bps = 6;
    if (const char* e = getenv("DS_TCW_FINISH_BLOCKS")) bps = atoi(e) > 0 ? atoi(e) : 6;
    w->tthreads = (int64_t)sms * bps * 256;
  }
  bool ok = cudaMalloc(&w->zbytes, (size_t)D8p * (nloc > 0 ? nloc : 1) * nc) == cudaSuccess &&
            cudaMalloc(&w->bbytes, (size_t)D8p * ncp * nc) == cudaSuccess &&  // k_tcw_pack image(s)
            cudaMalloc(&w->zf, sizeof(double) * (nloc > 0 ? nloc : 1)) == cudaSuccess &&
            cudaMalloc(&w->bf, sizeof(double) * n) == cudaSuccess &&
            cudaMalloc(&w->fb_count, 2 * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&w->fb_list, 2 * sizeof(int2) * w->fb_cap) == cudaSuccess &&
            cudaMalloc(&w->scratch, 2 * sizeof(uint32_t) * w->sthreads * (14 * (size_t)L + 96)) == cudaSuccess &&
            cudaMalloc(&w->tprod, sizeof(uint32_t) * (size_t)rows * ncp * plan->w_W * nc * nc) == cudaSuccess &&
            cudaMalloc(&w->tscratch, sizeof(uint32_t) * (size_t)w->tthreads *
                                         (nc == 2 ? ((8 * (size_t)L + 32 + 7) & ~(size_t)7)
                                                  : ((3 * (size_t)L + 24 + 7) & ~(size_t)7))) == cudaSuccess;
  if (!ok) return DS_OOM;
  plan->enabled = 1;
  return DS_OK;
}

int tc_plan_init(TcPlan* plan, int n, int nloc, int p, int device) {
  memset(plan, 0, sizeof(*plan));
  if (getenv("DS_DISABLE_TC")) return DS_OK;
  plan->p = p;
  plan->L = (p + 31) / 32;
  plan->D8p = ((4 * plan->L + KS - 1) / KS) * KS;
  plan->nks = plan->D8p / KS;
  int zb = 32 * plan->L - p;
  int lg = 0;
  while ((1 << lg) < plan->D8p) lg++;
  plan->eps = 9 + lg;
  // t's LSB in P' is at r' >= p - 1 + 2 zb; keep >= 32 decision bits above eps
  int rmin = p - 1 + 2 * zb;
  int clo = (rmin - 2 - 32 - plan->eps) / 8;
  clo &= ~3;
  if (clo < 0) clo = 0;
  // align the 8-limb epilogue blocks so one starts at limb L + 1, the first T
  // limb of normalised products (T_q = P' bits from r' - zb = 32 L + 32 q): then
  // every T block of those lanes is an interior (branch-free) block
  {
    int g = clo / 4;
    int d = ((g - (plan->L + 1)) % 8 + 8) % 8;
    g -= d;
    clo = g > 0 ? 4 * g : 0;
  }
  plan->c_lo = clo;
  // TMEM: 2 NG accumulator buffers of tn columns + 8 nks columns of A <= 512;
  // two epilogue groups if their windows fit in shared memory, else one
  // measured crossover (N=1000, all minors, device time): with two epilogue groups the
  // FP64-digit engine won at 256 and 512 bits (profiles/r02_smallp_engines.log); with
  // four (profiles/r02_engine_crossover_4groups.log) it still wins at 256 bits (0.103 vs
  // 0.113 s) and the tensor cores win from 512 bits (0.123 vs 0.129 s; 640: 0.155 vs
  // 0.183 s); DS_TC_MIN_BITS overrides
  int min_bits = 512;
  if (const char* e = getenv("DS_TC_MIN_BITS")) min_bits = atoi(e);
  if (min_bits < 256) min_bits = 256;
  if (p < min_bits) return DS_OK;  // not applicable: other engines
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  size_t smem = 0;
  int ng = 0;
  // more epilogue groups (more rows in flight per SM) where TMEM and shared memory
  // allow, i.e. up to ~2048 bits: three groups measured -4..-8 % device time at N=1000
  // @768 / 1024 / 2048 and N=2000 @1024 (profiles/r02_three_groups_ab.log), four a
  // further -10 % update time at 768 / 1024 bits (profiles/r02_four_groups_ab.log).
  // DS_TC_GROUPS_MAX caps the count (A/B).
  int g0 = 4;
  if (const char* e = getenv("DS_TC_GROUPS_MAX")) g0 = atoi(e) >= 1 && atoi(e) <= 4 ? atoi(e) : 4;
  for (int g = g0; g >= 1 && !ng; g--) {
    if (g == 2 && getenv("DS_TC_ONE_GROUP")) continue;
    int tn = ((512 - 8 * plan->nks) / (2 * g)) & ~31;  // multiple of the 32-column epilogue chunk
    if (tn > 256) tn = 256;
    if (tn < 32) continue;
    int ntiles = (2 * plan->D8p - clo + tn - 1) / tn;
    int br = ntiles * tn + KS * (plan->nks - 1);
    size_t sm = tc_smem(plan->L, br, g) + 1024;
    if ((int)sm > maxsm - 2048) continue;
    ng = g;
    plan->tn = tn;
    plan->ntiles = ntiles;
    plan->br = br;
    smem = sm;
  }
  if (!ng || getenv("DS_TC_WIDE")) return tcw_plan_init(plan, n, nloc, p, device, maxsm);
  plan->ng = ng;
  cudaError_t ea = ng == 4 ? cudaFuncSetAttribute(k_update_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                   : ng == 3 ? cudaFuncSetAttribute(k_update_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                   : ng == 2 ? cudaFuncSetAttribute(k_update_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(k_update_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (ea != cudaSuccess) return DS_CUDA;
  plan->smem = smem;
  TcWork* w = new TcWork();
  memset(w, 0, sizeof(*w));
  w->fb_cap = fb_capacity(nloc, n);
  w->sthreads = 64 * 128;
  bool ok = cudaMalloc(&w->zbytes, (size_t)plan->D8p * (nloc > 0 ? nloc : 1)) == cudaSuccess &&
            cudaMalloc(&w->bbytes, (size_t)plan->D8p * n) == cudaSuccess &&
            cudaMalloc(&w->zf, sizeof(double) * (nloc > 0 ? nloc : 1)) == cudaSuccess &&
            cudaMalloc(&w->bf, sizeof(double) * n) == cudaSuccess &&
            cudaMalloc(&w->fb_count, 2 * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&w->fb_list, 2 * sizeof(int2) * w->fb_cap) == cudaSuccess &&
            cudaMalloc(&w->scratch, 2 * sizeof(uint32_t) * w->sthreads * (14 * (size_t)plan->L + 96)) == cudaSuccess;
  plan->work = w;
  if (!ok) return DS_OOM;
  plan->enabled = 1;
  return DS_OK;
}

// complex elements: the wide engine with the four component products
int tc_plan_init_c(TcPlan* plan, int n, int nloc, int p, int device) {
  memset(plan, 0, sizeof(*plan));
  if (getenv("DS_DISABLE_TC") || getenv("DS_DISABLE_TC_COMPLEX") || p < 256) return DS_OK;
  plan->p = p;
  plan->L = (p + 31) / 32;
  plan->D8p = ((4 * plan->L + KS - 1) / KS) * KS;
  plan->nks = plan->D8p / KS;
  int lg = 0;
  while ((1 << lg) < plan->D8p) lg++;
  plan->eps = 9 + lg;
  plan->ncomp = 2;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int rc = tcw_plan_init(plan, n, nloc, p, device, maxsm);
  if (rc != DS_OK || !plan->wide) return rc;
  // the warp-cooperative finish (ds_cfinish.cuh) unless DS_CX_FINISH_THREAD=1
  const char* ft = getenv("DS_CX_FINISH_THREAD");
  const char* fw = getenv("DS_CX_FINISH_WARP");
  const int K = (ft && atoi(ft)) ? 0 : cf_k_for(plan->w_W, fw && atoi(fw));
  if (K) {
    const size_t sm = cf_smem(K, plan->w_W, plan->L);
    cudaError_t e = cudaSuccess;
    switch (K) {
      case 2: e = cudaFuncSetAttribute(k_cfw_finish<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); break;
      case 3: e = cudaFuncSetAttribute(k_cfw_finish<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); break;
      case 5: e = cudaFuncSetAttribute(k_cfw_finish<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); break;
      default: e = cudaFuncSetAttribute(k_cfw_finish<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); break;
    }
    TcWork* w = (TcWork*)plan->work;
    if (e == cudaSuccess && (int)sm <= maxsm &&
        cudaMalloc(&w->zlow, sizeof(int) * 2 * (size_t)(nloc > 0 ? nloc : 1)) == cudaSuccess &&
        cudaMalloc(&w->blow, sizeof(int) * 2 * (size_t)n) == cudaSuccess) {
      plan->cf_k = K;
      plan->cf_smem = sm;
    } else {
      cudaGetLastError();
    }
  }
  return DS_OK;
}

void tc_plan_free(TcPlan* plan) {
  TcWork* w = (TcWork*)plan->work;
  if (!w) return;
  void* ptrs[] = {w->zbytes, w->bbytes, w->zf, w->bf, w->fb_count, w->fb_list, w->scratch, w->tprod, w->tscratch,
                  w->zlow, w->blow};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete w;
  plan->work = nullptr;
}

// Rows per CTA of the main update launch (one CTA per SM).  At a fixed 16 the
// grid runs in ceil(CTAs / SMs) waves, so late steps (few rows) lose part of a
// wave to quantisation.  pick_rbr (opt-in, DS_TC_RBR_ADAPT=1) picks the rbr in
// {16,12,8,6,4} minimising waves x (rbr + per-CTA setup).  Measured on B200: it
// lowers the summed update-kernel time (N=1000 @8192: 0.85 -> 0.79 s) but not the
// elimination (0.88 -> 0.90 s; N=2000 @4096: 2.10 -> 2.17 s): the lookahead tile
// on its own stream then finds no free SM.  So the default stays 16 for one rank;
// a row-cyclic shard (nloc < n) adapts: rank 0 of 8 at N=2000 @4096, update time
// 0.427 -> 0.337 s, of 4: 0.649 -> 0.577 s (tools/shard_projection.py,
// profiles/r02_shard_projection_rbr.json).  DS_TC_RBR=r fixes r.
static int pick_rbr(int ntiles, int nrows, int ng, bool sharded) {
  static int sms = 0, fixed = -1, adapt_all = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    const char* e = getenv("DS_TC_RBR");
    fixed = e ? atoi(e) : 0;
    adapt_all = getenv("DS_TC_RBR_ADAPT") ? 1 : 0;
  }
  if (fixed > 0) return fixed < 64 ? fixed : 64;  // A/B above the default 16 too
  (void)ng;
  if (!adapt_all && !sharded) return RBR;
  if (ntiles < 1) ntiles = 1;
  const int cand[5] = {16, 12, 8, 6, 4};
  int best = RBR;
  double best_cost = 1e300;
  for (int c : cand) {
    const long ctas = (long)ntiles * ((nrows + c - 1) / c);
    const long waves = (ctas + sms - 1) / sms;
    const double cost = (double)waves * (c + 0.5);  // +0.5 row: TMEM A load, barriers, TMA descriptors
    if (cost < best_cost * 0.98) { best_cost = cost; best = c; }
  }
  return best;
}

int tc_update_launch(TcPlan* plan, cudaStream_t s, uint32_t* a_limbs, int32_t* a_exp, uint8_t* a_cls,
                     int64_t a_count, const uint8_t* pbuf, const uint32_t* z_limbs, const int32_t* z_exp,
                     const uint8_t* z_cls, int nloc, int n, int i, int jl0, int collect_minors, int32_t* status,
                     int64_t* launches, cudaStream_t la, cudaEvent_t ev_prep, cudaEvent_t ev_a, int la_col,
                     int* la_used) {
  if (la_used) *la_used = 0;
  TcWork* w = (TcWork*)plan->work;
  const int L = plan->L;
  const int nrows = nloc - jl0;
  const int kmin = collect_minors ? 0 : i + 1;
  const int kstart = kmin & ~3;  // column tiles start 16-byte aligned (tile tensor map)
  const int ncols = n - kstart;
  if (nrows <= 0 || ncols <= 0) return DS_OK;
  const int nc = plan->ncomp == 2 ? 2 : 1;  // complex: pivot buffer [c][l][k], exp [c][k], cls [c][k]
  const uint32_t* b_limbs = (const uint32_t*)pbuf;
  const int32_t* b_exp = (const int32_t*)(pbuf + (size_t)4 * nc * L * n);
  const uint8_t* b_cls = (const uint8_t*)(pbuf + (size_t)4 * nc * L * n + (size_t)4 * nc * n);
  const int W4 = plan->D8p / 4;
  for (int c = 0; c < nc; c++)
    k_tc_bytes<<<(unsigned)(((int64_t)nrows * W4 + 255) / 256), 256, 0, s>>>(
        z_limbs + (int64_t)c * L * nloc + jl0, nloc, nrows, L, plan->D8p, w->zbytes + (size_t)c * nloc * plan->D8p,
        w->zf);
  if (!plan->wide)
    k_tc_bytes<<<(unsigned)(((int64_t)n * W4 + 255) / 256), 256, 0, s>>>(b_limbs, n, n, L, plan->D8p, w->bbytes, w->bf);
  // fallback lists: [0] the main launch, [1] the lookahead tile (its fallbacks must
  // be applied before the next step's multipliers read column i + 1)
  cudaMemsetAsync(w->fb_count, 0, 2 * sizeof(int), s);
  TcArgs a;
  a.p = plan->p; a.L = L; a.zb = 32 * L - plan->p; a.D8p = plan->D8p; a.nks = plan->nks; a.ntiles = plan->ntiles;
  a.c_lo = plan->c_lo; a.eps = plan->eps;
  a.nrows = nrows; a.ncols = ncols; a.kstart = kstart; a.kmin = kmin; a.skip_col = i; a.n = n; a.jl0 = jl0;
  a.zbytes = w->zbytes; a.bbytes = w->bbytes; a.zf = w->zf; a.bf = w->bf;
  a.zexp = z_exp + jl0; a.zcls = z_cls + jl0; a.bexp = b_exp; a.bcls = b_cls; a.zstride = nloc;
  a.a_limbs = a_limbs; a.a_exp = a_exp; a.a_cls = a_cls; a.a_count = a_count;
  a.status = status; a.step = i;
  a.fb_count = w->fb_count; a.fb_list = w->fb_list; a.fb_cap = w->fb_cap;
  a.tn = plan->tn;
  a.br = plan->br;
  if (plan->wide) {
    // wide precision: product limbs per row chunk, then the finish kernel
    a.tile0 = 0;
    a.tskip = -1;
    const int ntile = (ncols + TM - 1) / TM;
    const int ncp = ntile * TM;
    const int64_t npieces = (int64_t)ntile * plan->nks * 2 * TM;
    const size_t img = (size_t)plan->D8p * (((n + TM - 1) / TM) * TM);  // pack image per component
    for (int c = 0; c < nc; c++)
      k_tcw_pack<<<(unsigned)((npieces + 255) / 256), 256, 0, s>>>(b_limbs + (int64_t)c * L * n, n, L, plan->nks,
                                                                   kstart, ntile, w->bbytes + c * img);
    a.zlow = w->zlow;
    a.blow = w->blow;
    if (nc == 2 && plan->cf_k) {
      for (int c = 0; c < 2; c++) {
        k_lowdig<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(z_limbs + (int64_t)c * L * nloc + jl0, nloc, nrows,
                                                                  L, w->zlow + (size_t)c * nloc);
        k_lowdig<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(b_limbs + (int64_t)c * L * n, n, n, L,
                                                              w->blow + (size_t)c * n);
      }
      *launches += 4;
    }
    for (int r0 = 0; r0 < nrows; r0 += plan->w_rows) {
      const int rc = nrows - r0 < plan->w_rows ? nrows - r0 : plan->w_rows;
      TwArgs tw;
      tw.p = plan->p; tw.L = L; tw.D8p = plan->D8p; tw.nks = plan->nks; tw.c_lo = plan->c_lo;
      tw.qlo = plan->w_qlo; tw.W = plan->w_W; tw.eps = plan->eps;
      tw.tn = plan->tn; tw.ntiles = plan->ntiles; tw.kc = plan->w_kc; tw.nst = plan->w_nst; tw.brc = plan->w_brc;
      tw.nrows = rc; tw.rbr = plan->w_rbr; tw.kstart = kstart; tw.ncp = ncp; tw.zwb = plan->w_zwb;
      tw.zbytes = w->zbytes + (size_t)r0 * plan->D8p;
      tw.apack = w->bbytes;
      tw.tprod = w->tprod;
      tw.pstride = (int64_t)rc * ncp;
      tw.status = status; tw.step = i;
      if (nc == 1) {
        k_prod_tcw<<<dim3(ntile, (rc + tw.rbr - 1) / tw.rbr), TW_THREADS, plan->smem, s>>>(tw);
        k_tcw_finish<<<(unsigned)(w->tthreads / 256), 256, 0, s>>>(a, tw, r0, w->tscratch, w->tthreads);
        *launches += 2;
      } else {
        // the four component products (c1, c2) = z_c1 * b_c2 into regions 2 c1 + c2
        for (int c1 = 0; c1 < 2; c1++)
          for (int c2 = 0; c2 < 2; c2++) {
            TwArgs tc = tw;
            tc.zbytes = w->zbytes + ((size_t)c1 * nloc + r0) * plan->D8p;
            tc.apack = w->bbytes + c2 * img;
            tc.tprod = w->tprod + (size_t)(2 * c1 + c2) * tw.pstride * tw.W;
            k_prod_tcw<<<dim3(ntile, (rc + tw.rbr - 1) / tw.rbr), TW_THREADS, plan->smem, s>>>(tc);
          }
        const unsigned fb = (unsigned)(w->tthreads / 256);
        switch (plan->cf_k) {
          case 2: k_cfw_finish<2><<<fb, 256, plan->cf_smem, s>>>(a, tw, r0, w->tscratch, w->tthreads); break;
          case 3: k_cfw_finish<3><<<fb, 256, plan->cf_smem, s>>>(a, tw, r0, w->tscratch, w->tthreads); break;
          case 5: k_cfw_finish<5><<<fb, 256, plan->cf_smem, s>>>(a, tw, r0, w->tscratch, w->tthreads); break;
          case 9: k_cfw_finish<9><<<fb, 256, plan->cf_smem, s>>>(a, tw, r0, w->tscratch, w->tthreads); break;
          default: k_tcw_finish_c<<<fb, 256, 0, s>>>(a, tw, r0, w->tscratch);
        }
        *launches += 5;
      }
    }
    if (nc == 1)
      k_tc_fallback<<<64, 128, 0, s>>>(a, z_limbs, nloc, b_limbs, w->scratch, w->sthreads);
    else
      k_tc_fallback_c<<<64, 128, 0, s>>>(a, z_limbs, nloc, b_limbs, w->scratch, w->sthreads);
    *launches += 3;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DS_OK : DS_CUDA;
  }
  if (w->amap_base != (const void*)a_limbs || w->amap_count != a_count) {
    w->amap_base = a_limbs;
    w->amap_count = a_count;
    w->amap_ok = 0;
    EncodeTiledFn enc = encode_tiled();
    if (enc && !getenv("DS_TC_NO_TMA") && (a_count * 4) % 16 == 0 && L <= 256 && a_count < (1ll << 31)) {
      cuuint64_t dims[2] = {(cuuint64_t)a_count, (cuuint64_t)L};
      cuuint64_t strides[1] = {(cuuint64_t)a_count * 4};
      cuuint32_t box[2] = {(cuuint32_t)TM, (cuuint32_t)L};
      cuuint32_t estr[2] = {1, 1};
      CUresult cr = enc(&w->amap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)a_limbs, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      w->amap_ok = cr == CUDA_SUCCESS ? 1 : 0;
    }
  }
  a.tma_ok = w->amap_ok;
  a.no_direct = getenv("DS_TC_NO_DIRECT") ? 1 : 0;
  const int ntile = (ncols + TM - 1) / TM;
  a.rbr = pick_rbr(ntile - (la_col >= 0 && ntile >= 2 ? 1 : 0), nrows, plan->ng, nloc < n);
  const int nrg = (nrows + a.rbr - 1) / a.rbr;
  const int ts = la_col >= 0 ? (la_col - kstart) / TM : -1;  // tile holding the lookahead column
  if (ts >= 0 && ts < ntile && ntile >= 2 && la) {
    // A: that tile on the lookahead stream (the caller chains the next multipliers
    // after it); B: the other tiles on the main stream; fallback after both
    CK_TC(cudaEventRecord(ev_prep, s));
    CK_TC(cudaStreamWaitEvent(la, ev_prep, 0));
    TcArgs aa = a;
    aa.tile0 = ts;
    aa.tskip = -1;
    aa.rbr = RBR_LA;  // short CTAs: the next step's multipliers wait on this tile only
    aa.fb_count = w->fb_count + 1;
    aa.fb_list = w->fb_list + w->fb_cap;
    launch_update(plan->ng, dim3(1, (nrows + RBR_LA - 1) / RBR_LA), plan->smem, la, aa, w->amap);
    k_tc_fallback<<<64, 128, 0, la>>>(aa, z_limbs, nloc, b_limbs, w->scratch + w->sthreads * (14 * (size_t)L + 96),
                                     w->sthreads);
    *launches += 1;
    CK_TC(cudaEventRecord(ev_a, la));
    TcArgs ab = a;
    ab.tile0 = 0;
    ab.tskip = ts;
    launch_update(plan->ng, dim3(ntile - 1, nrg), plan->smem, s, ab, w->amap);
    CK_TC(cudaStreamWaitEvent(s, ev_a, 0));
    *launches += 1;
    *la_used = 1;
  } else {
    a.tile0 = 0;
    a.tskip = -1;
    launch_update(plan->ng, dim3(ntile, nrg), plan->smem, s, a, w->amap);
  }
  k_tc_fallback<<<64, 128, 0, s>>>(a, z_limbs, nloc, b_limbs, w->scratch, w->sthreads);
  *launches += 4;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DS_OK : DS_CUDA;
}
