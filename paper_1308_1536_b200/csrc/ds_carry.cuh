// ds_carry.cuh -- multi-limb add-with-carry chains (PTX add.cc / addc) shared by
// the rounding stream (ds_stream.cuh) and the warp division (ds_warpdiv.cuh).
#pragma once
#include <stdint.h>

#ifndef DS_VAR_ADDC8
#define DS_VAR_ADDC8 1
#endif

namespace dss {

// s = x + y + cy over N limbs (low -> high) with the PTX carry chain;
// cy (0/1) in, carry out.  Chains of 4 and 2 limbs, the carry handed over in
// a register between them.
__device__ __forceinline__ void addc4(uint32_t* s, const uint32_t* x, const uint32_t* y, uint32_t& cy) {
  asm("{\n\t.reg .u32 t;\n\t"
      "add.cc.u32 t, %4, 0xffffffff;\n\t"
      "addc.cc.u32 %0, %5, %9;\n\t"
      "addc.cc.u32 %1, %6, %10;\n\t"
      "addc.cc.u32 %2, %7, %11;\n\t"
      "addc.cc.u32 %3, %8, %12;\n\t"
      "addc.u32 %4, 0, 0;\n\t}"
      : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "+r"(cy)
      : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
}
__device__ __forceinline__ void addc2(uint32_t* s, const uint32_t* x, const uint32_t* y, uint32_t& cy) {
  asm("{\n\t.reg .u32 t;\n\t"
      "add.cc.u32 t, %2, 0xffffffff;\n\t"
      "addc.cc.u32 %0, %3, %5;\n\t"
      "addc.cc.u32 %1, %4, %6;\n\t"
      "addc.u32 %2, 0, 0;\n\t}"
      : "=r"(s[0]), "=r"(s[1]), "+r"(cy)
      : "r"(x[0]), "r"(x[1]), "r"(y[0]), "r"(y[1]));
}
__device__ __forceinline__ void addc1(uint32_t* s, const uint32_t* x, const uint32_t* y, uint32_t& cy) {
  asm("{\n\t.reg .u32 t;\n\t"
      "add.cc.u32 t, %1, 0xffffffff;\n\t"
      "addc.cc.u32 %0, %2, %3;\n\t"
      "addc.u32 %1, 0, 0;\n\t}"
      : "=r"(s[0]), "+r"(cy)
      : "r"(x[0]), "r"(y[0]));
}
// one 8-limb chain (10 instructions instead of two 4-limb chains' 12)
__device__ __forceinline__ void addc8(uint32_t* s, const uint32_t* x, const uint32_t* y, uint32_t& cy) {
  asm("{\n\t.reg .u32 t;\n\t"
      "add.cc.u32 t, %8, 0xffffffff;\n\t"
      "addc.cc.u32 %0, %9, %17;\n\t"
      "addc.cc.u32 %1, %10, %18;\n\t"
      "addc.cc.u32 %2, %11, %19;\n\t"
      "addc.cc.u32 %3, %12, %20;\n\t"
      "addc.cc.u32 %4, %13, %21;\n\t"
      "addc.cc.u32 %5, %14, %22;\n\t"
      "addc.cc.u32 %6, %15, %23;\n\t"
      "addc.cc.u32 %7, %16, %24;\n\t"
      "addc.u32 %8, 0, 0;\n\t}"
      : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7]), "+r"(cy)
      : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]), "r"(y[0]), "r"(y[1]),
        "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]));
}

template <int N>
__device__ __forceinline__ void addc_n(uint32_t (&s)[N], const uint32_t (&x)[N], const uint32_t (&y)[N], uint32_t& cy) {
  int k0 = 0;
#if DS_VAR_ADDC8
#pragma unroll
  for (; k0 + 8 <= N; k0 += 8) addc8(s + k0, x + k0, y + k0, cy);
#endif
#pragma unroll
  for (int k = k0; k + 4 <= N; k += 4) addc4(s + k, x + k, y + k, cy);
  if (N & 2) addc2(s + (N & ~3), x + (N & ~3), y + (N & ~3), cy);
  if (N & 1) addc1(s + (N - 1), x + (N - 1), y + (N - 1), cy);
}

}  // namespace dss
