// fs_step_incr.cu — instantiations of k_step_incr (incremental counts) and k_gather_merge
// (a separate translation unit so the step-kernel variants compile in parallel)
#include "fs_step.cuh"

namespace fs {

StepFn pick_stream(bool mixed, bool mat) {
  if (mixed) return mat ? k_step_incr<int8_t, __half, true, 512> : k_step_incr<int8_t, __half, false, 512>;
  return mat ? k_step_incr<int32_t, float, true, 512> : k_step_incr<int32_t, float, false, 512>;
}


MergeFn pick_merge(bool inf_bf16, int mode, int& block) {
  if (mode == 1) { block = 1024; return inf_bf16 ? k_gather_merge<__nv_bfloat16, 1, 1024> : k_gather_merge<float, 1, 1024>; }
  block = 512;
  if (mode == 2) return inf_bf16 ? k_gather_merge<__nv_bfloat16, 2, 512> : k_gather_merge<float, 2, 512>;
  return inf_bf16 ? k_gather_merge<__nv_bfloat16, 0, 512> : k_gather_merge<float, 0, 512>;
}


}  // namespace fs
