// Pipe-throughput microbenchmark for the limb-product inner loop candidates
// (decides the limb radix of k_update). Each kernel runs many independent
// chains per thread; reported as lane-ops per SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

// (1) 32-bit radix carry chain: mad.lo.cc / madc.hi.cc pairs, 8 products per row
__global__ void k_madcc(uint32_t* out, uint32_t seed, long long* clk) {
  uint32_t a = seed + threadIdx.x, acc[10];
  uint32_t w[8];
  for (int i = 0; i < 10; i++) acc[i] = i;
  for (int i = 0; i < 8; i++) w[i] = seed * (i + 3) + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    asm volatile(
      "mad.lo.cc.u32 %0, %10, %11, %0;\n\t"
      "madc.lo.cc.u32 %1, %10, %12, %1;\n\t"
      "madc.lo.cc.u32 %2, %10, %13, %2;\n\t"
      "madc.lo.cc.u32 %3, %10, %14, %3;\n\t"
      "madc.lo.cc.u32 %4, %10, %15, %4;\n\t"
      "madc.lo.cc.u32 %5, %10, %16, %5;\n\t"
      "madc.lo.cc.u32 %6, %10, %17, %6;\n\t"
      "madc.lo.cc.u32 %7, %10, %18, %7;\n\t"
      "addc.u32 %8, %8, 0;\n\t"
      "mad.hi.cc.u32 %1, %10, %11, %1;\n\t"
      "madc.hi.cc.u32 %2, %10, %12, %2;\n\t"
      "madc.hi.cc.u32 %3, %10, %13, %3;\n\t"
      "madc.hi.cc.u32 %4, %10, %14, %4;\n\t"
      "madc.hi.cc.u32 %5, %10, %15, %5;\n\t"
      "madc.hi.cc.u32 %6, %10, %16, %6;\n\t"
      "madc.hi.cc.u32 %7, %10, %17, %7;\n\t"
      "madc.hi.cc.u32 %8, %10, %18, %8;\n\t"
      "addc.u32 %9, %9, 0;\n\t"
      : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]),
        "+r"(acc[5]), "+r"(acc[6]), "+r"(acc[7]), "+r"(acc[8]), "+r"(acc[9])
      : "r"(a), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    a += acc[9];
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 10; i++) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// (2) 64-bit accumulate: mad.wide.u32 into independent 64-bit accumulators
__global__ void k_madwide(uint32_t* out, uint32_t seed, long long* clk) {
  uint32_t a = seed + threadIdx.x;
  uint64_t acc[8];
  uint32_t w[8];
  for (int i = 0; i < 8; i++) { acc[i] = i; w[i] = seed * (i + 3) + threadIdx.x; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] += (uint64_t)a * w[i];
    a += (uint32_t)acc[3];
  }
  long long t1 = clock64();
  uint64_t s = 0;
  for (int i = 0; i < 8; i++) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(s ^ (s >> 32));
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// (3) plain 32-bit IMAD (mul.lo + add)
__global__ void k_imad(uint32_t* out, uint32_t seed, long long* clk) {
  uint32_t a = seed + threadIdx.x;
  uint32_t acc[8], w[8];
  for (int i = 0; i < 8; i++) { acc[i] = i; w[i] = seed * (i + 3) + threadIdx.x; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = acc[i] + a * w[i];
    a += acc[3];
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// (4) DFMA
__global__ void k_dfma(uint32_t* out, uint32_t seed, long long* clk) {
  double a = 1.0 + 1e-9 * (seed + threadIdx.x);
  double acc[8], w[8];
  for (int i = 0; i < 8; i++) { acc[i] = i; w[i] = 1.0 + 1e-7 * i; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = fma(a, w[i], acc[i]);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// (5) mul.hi.u32 + mul.lo.u32 separately (2 IMAD per product) into 3-word sums
__global__ void k_lohi(uint32_t* out, uint32_t seed, long long* clk) {
  uint32_t a = seed + threadIdx.x;
  uint32_t lo[8], hi[8], w[8];
  for (int i = 0; i < 8; i++) { lo[i] = hi[i] = i; w[i] = seed * (i + 3) + threadIdx.x; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) { lo[i] += a * w[i]; hi[i] += __umulhi(a, w[i]); }
    a += lo[3];
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s ^= lo[i] ^ hi[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(uint32_t*, uint32_t, long long*);

static void run(const char* name, kfn k, double ops_per_iter_per_thread, int blocks, int threads) {
  uint32_t* out; long long* clk;
  cudaMalloc(&out, sizeof(uint32_t) * blocks * threads);
  cudaMalloc(&clk, sizeof(long long) * blocks);
  k<<<blocks, threads>>>(out, 1, clk);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, 2, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, clk, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < blocks; i++) if (h[i] > mx) mx = h[i];
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double total = ops_per_iter_per_thread * ITERS * (double)blocks * threads;
  double per_sm_clk = total / sms / mx;  // approx: blocks evenly spread, one wave
  printf("%-10s blocks=%d thr=%d  %.3f ms  %.3e ops/s  ~%.1f ops/clk/SM (clk-based, max block %.0f cyc)\n",
         name, blocks, threads, ms, total / (ms * 1e-3), per_sm_clk, mx);
  cudaFree(out); cudaFree(clk); delete[] h;
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clockRate=%d kHz\n", sms, clk);
  for (int occ : {4, 8}) {
    int blocks = sms * occ, threads = 256;
    run("madcc", k_madcc, 8, blocks, threads);     // 8 limb products / iter
    run("madwide", k_madwide, 8, blocks, threads); // 8 wide products / iter
    run("imad", k_imad, 8, blocks, threads);
    run("lohi", k_lohi, 8, blocks, threads);       // 8 products (16 IMAD) / iter
    run("dfma", k_dfma, 8, blocks, threads);
  }
  return 0;
}
