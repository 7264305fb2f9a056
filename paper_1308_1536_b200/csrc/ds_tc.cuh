// ds_tc.cuh -- interface of the tensor-core (tcgen05 kind::i8) real update (ds_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

struct TcPlan {
  int enabled;
  int p, L, D8p, nks;  // precision, 32-bit limbs, 8-bit digits (padded to the MMA K), K steps
  int c_lo, ntiles, eps;
  int tn, br;          // MMA N per tile, Toeplitz bank rows
  int ng;              // epilogue groups / producer pipelines per CTA (1 or 2)
  size_t smem;
  // wide precision (pivot-row digits beyond TMEM): product kernel + finish kernel
  int wide;
  int ncomp;           // 2: complex elements (wide engine, four component products)
  int w_kc, w_nst, w_brc, w_qlo, w_W, w_zwb, w_rows, w_rbr;
  int cf_k;            // complex: words per lane of the warp finish (0: thread-per-element finish)
  size_t cf_smem;
  void* work;
};

int tc_plan_init(TcPlan* plan, int n, int nloc, int p, int device);
int tc_plan_init_c(TcPlan* plan, int n, int nloc, int p, int device);
void tc_plan_free(TcPlan* plan);
int tc_update_launch(TcPlan* plan, cudaStream_t s, uint32_t* a_limbs, int32_t* a_exp, uint8_t* a_cls,
                     int64_t a_count, const uint8_t* pbuf, const uint32_t* z_limbs, const int32_t* z_exp,
                     const uint8_t* z_cls, int nloc, int n, int i, int jl0, int collect_minors, int32_t* status,
                     int64_t* launches, cudaStream_t la = nullptr, cudaEvent_t ev_prep = nullptr,
                     cudaEvent_t ev_a = nullptr, int la_col = -1, int* la_used = nullptr);
