// ds_update.cu -- fused real update engine (placeholder until the DFMA kernel).
#include "ds_update.cuh"
#include "../../include/detseries_b200.h"

int update_plan_init(UpdatePlan* plan, int n, int p, int device) {
  plan->enabled = 0;
  plan->n = n; plan->p = p; plan->device = device;
  plan->workspace = nullptr;
  return DS_OK;
}
void update_plan_free(UpdatePlan* plan) { (void)plan; }
int update_launch(UpdatePlan*, cudaStream_t, uint32_t*, int32_t*, uint8_t*, int64_t, const uint8_t*,
                  const uint32_t*, const int32_t*, const uint8_t*, int, int, int, int, int, int32_t*, int64_t*) {
  return DS_INVALID;
}
