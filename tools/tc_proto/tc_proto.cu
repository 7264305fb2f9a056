// tc_proto.cu -- prototype: multiprecision digit convolutions on the 5th-gen
// tensor cores (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM).
//
// For 128 rows z_j (D8 unsigned 8-bit digits each) and one column b (D8
// digits), computes the column sums   C[j][c] = sum_s z_j[s] * b[c - s]
// for c in [c0, c0 + 256) as one GEMM:  A = Z (M=128 rows x K=D8, K-major),
// B = Toeplitz(b) (K=D8 x N=256, K-major rows n: B[n][s] = b[c0 + n - s]),
// materialised per K-step in shared memory in the canonical no-swizzle
// K-major layout (8-row x 16-byte core matrices).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int M = 128, N = 256, KS = 32;  // MMA shape, K bytes per instruction

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__host__ __device__ constexpr uint32_t instr_desc_i8(int m, int n) {
  // c_format S32 (2) bits[4,6); a/b format u8 (0); K-major both; n_dim N>>3 bits[17,23); m_dim M>>4 bits[24,29)
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// canonical K-major no-swizzle offset of element (row r, k byte kk) within one
// K-step tile of R rows x 32 bytes: [k-half][row-group][row-in-group][16 B]
__device__ __forceinline__ uint32_t kmaj_off(int r, int kk, int R) {
  return (uint32_t)((kk >> 4) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (kk & 15));
}

__global__ void __launch_bounds__(128) k_conv(const uint8_t* Z, const uint8_t* b, int D8, int c0, int32_t* out,
                                              int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int nks = D8 / KS;
  uint8_t* As = sm;                       // nks * (M * 32) bytes
  uint8_t* Bs = As + nks * M * KS;        // nks * (N * 32) bytes
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // stage A
  for (int e = tid; e < M * D8; e += blockDim.x) {
    int r = e / D8, s = e % D8;
    int ks = s / KS, kk = s % KS;
    As[ks * M * KS + kmaj_off(r, kk, M)] = Z[r * D8 + s];
  }
  // build Toeplitz B tiles
  for (int e = tid; e < N * D8; e += blockDim.x) {
    int n = e / D8, s = e % D8;
    int ks = s / KS, kk = s % KS;
    int t = c0 + n - s;
    Bs[ks * N * KS + kmaj_off(n, kk, N)] = (t >= 0 && t < D8) ? b[t] : 0;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(1));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy (MMA)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = instr_desc_i8(M, N);
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; rep++) {
    if (tid == 0) {
      for (int ks = 0; ks < nks; ks++) {
        uint32_t a_addr = (uint32_t)__cvta_generic_to_shared(As + ks * M * KS);
        uint32_t b_addr = (uint32_t)__cvta_generic_to_shared(Bs + ks * N * KS);
        // LBO = distance between the two 16-byte K halves; SBO = between 8-row groups
        uint64_t adesc = smem_desc(a_addr, M * 16, 128);
        uint64_t bdesc = smem_desc(b_addr, N * 16, 128);
        uint32_t acc = ks > 0 ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&mbar)));
    }
    // wait for the MMAs
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)),
        "r"(phase));
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  // epilogue: warp w reads lanes 32w..32w+31, 16 columns at a time
  for (int cb = 0; cb < N; cb += 16) {
    uint32_t v[16];
    uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int row = warp * 32 + lane;
    for (int q = 0; q < 16; q++) out[row * N + cb + q] = (int32_t)v[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}


// Variant: A (Z digits) in TENSOR MEMORY (written by tcgen05.st, lane = row,
// K bytes packed 4 per 32-bit column), B from shared memory.
__global__ void __launch_bounds__(128) k_conv_ta(const uint8_t* Z, const uint8_t* b, int D8, int c0, int32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int nks = D8 / KS;
  uint8_t* Bs = sm;  // nks * (N * 32) bytes
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < N * D8; e += blockDim.x) {
    int n = e / D8, s = e % D8;
    int ks = s / KS, kk = s % KS;
    int t = c0 + n - s;
    Bs[ks * N * KS + kmaj_off(n, kk, N)] = (t >= 0 && t < D8) ? b[t] : 0;
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(1));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t abase = tmem + 256;  // A in columns [256, 256 + D8/4)
  // row r = tid writes its D8 bytes as D8/4 words, 8 columns per st
  for (int c = 0; c < D8 / 4; c += 8) {
    uint32_t w[8];
    for (int q = 0; q < 8; q++) {
      const uint8_t* zp = Z + tid * D8 + 4 * (c + q);
      w[q] = zp[0] | (zp[1] << 8) | (zp[2] << 16) | ((uint32_t)zp[3] << 24);
    }
    uint32_t ta = abase + ((uint32_t)(warp * 32) << 16) + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(w[0]), "r"(w[1]),
                 "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = instr_desc_i8(M, N);
  if (tid == 0) {
    for (int ks = 0; ks < nks; ks++) {
      uint32_t b_addr = (uint32_t)__cvta_generic_to_shared(Bs + ks * N * KS);
      uint64_t bdesc = smem_desc(b_addr, N * 16, 128);
      uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
          "r"(abase + ks * 8), "l"(bdesc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&mbar)));
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int cb = 0; cb < N; cb += 16) {
    uint32_t v[16];
    uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int row = warp * 32 + lane;
    for (int q = 0; q < 16; q++) out[row * N + cb + q] = (int32_t)v[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main(int argc, char** argv) {
  const int D8 = argc > 1 ? atoi(argv[1]) : 512;
  const int c0 = argc > 2 ? atoi(argv[2]) : D8 - 16;
  std::vector<uint8_t> Z(M * D8), b(D8);
  srand(7);
  for (auto& x : Z) x = rand() & 255;
  for (auto& x : b) x = rand() & 255;
  uint8_t *dZ, *db;
  int32_t* dout;
  CK(cudaMalloc(&dZ, Z.size()));
  CK(cudaMalloc(&db, b.size()));
  CK(cudaMalloc(&dout, sizeof(int32_t) * M * N));
  CK(cudaMemcpy(dZ, Z.data(), Z.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice));
  size_t smem = (size_t)(D8 / KS) * (M + N) * KS;
  CK(cudaFuncSetAttribute(k_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_conv<<<1, 128, smem>>>(dZ, db, D8, c0, dout, 1);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> out(M * N);
  CK(cudaMemcpy(out.data(), dout, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int r = 0; r < M; r++)
    for (int n = 0; n < N; n++) {
      int c = c0 + n;
      long ref = 0;
      for (int s = 0; s < D8; s++) {
        int t = c - s;
        if (t >= 0 && t < D8) ref += (long)Z[r * D8 + s] * b[t];
      }
      if (ref != out[r * N + n]) {
        if (bad < 5) printf("mismatch r=%d n=%d got %d want %ld\n", r, n, out[r * N + n], ref);
        bad++;
      }
    }
  printf("D8=%d c0=%d mismatches=%ld\n", D8, c0, bad);
  {
    size_t smem2 = (size_t)(D8 / KS) * N * KS;
    CK(cudaFuncSetAttribute(k_conv_ta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    CK(cudaMemset(dout, 0, sizeof(int32_t) * M * N));
    k_conv_ta<<<1, 128, smem2>>>(dZ, db, D8, c0, dout);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> out2(M * N);
    CK(cudaMemcpy(out2.data(), dout, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost));
    long bad2 = 0;
    for (int i = 0; i < M * N; i++) if (out2[i] != out[i]) { if (bad2 < 5) printf("TA mismatch %d: %d vs %d\n", i, out2[i], out[i]); bad2++; }
    printf("A-in-TMEM variant: mismatches vs smem-A result=%ld\n", bad2);
    bad += bad2;
  }
  // timing: many reps of the MMA chain in one CTA per SM
  int reps = 200;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaEventRecord(e0);
  k_conv<<<sms, 128, smem>>>(dZ, db, D8, c0, dout, reps);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double macs = (double)sms * reps * (D8 / KS) * (double)M * N * KS;
  printf("timing: %d CTAs x %d reps: %.3f ms, %.3e int8 MAC/s (incl. staging)\n", sms, reps, ms, macs / (ms * 1e-3));
  return bad ? 1 : 0;
}
