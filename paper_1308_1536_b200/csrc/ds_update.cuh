// ds_update.cuh -- interface of the fused real update engine (ds_update.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

struct UpdatePlan {
  int enabled;        // the DFMA kernels are usable (row products k_mul_split)
  int fused;          // ... and the fused update k_fused fits one CTA
  int n, p, L, D;     // precision, 32-bit limbs, 24-bit digits
  int device, sms;
  int tr, tc, w;       // tile rows/cols, register block
  size_t smem;
  void* workspace;
};

int update_plan_init(UpdatePlan* plan, int n, int p, int device);
void update_plan_free(UpdatePlan* plan);
int update_launch(UpdatePlan* plan, cudaStream_t s, uint32_t* a_limbs, int32_t* a_exp, uint8_t* a_cls,
                  int64_t a_count, const uint8_t* pbuf, const uint32_t* z_limbs, const int32_t* z_exp,
                  const uint8_t* z_cls, int nloc, int n, int i, int jl0, int collect_minors, int32_t* status,
                  int64_t* launches);
int mul_row_launch(UpdatePlan* plan, cudaStream_t s, const uint32_t* x_limbs, int64_t xcount, const int32_t* x_exp,
                   const uint8_t* x_cls, const uint32_t* y_limbs, int64_t ycount, const int32_t* y_exp,
                   const uint8_t* y_cls, int count, uint32_t* o_limbs, int64_t o_count, int32_t* o_exp,
                   uint8_t* o_cls, int32_t* status, int64_t* launches, int step, double* wsx, double* wsy);
size_t mul_ws_doubles(const UpdatePlan* plan, int count);
