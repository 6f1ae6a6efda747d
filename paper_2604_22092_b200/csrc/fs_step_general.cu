// fs_step_general.cu — instantiations of the general step kernel k_step
// (a separate translation unit so the step-kernel variants compile in parallel)
#include "fs_step.cuh"

namespace fs {

// ---------------------------------------------------------------------------
// kernel selection
// ---------------------------------------------------------------------------

template <typename ST, typename AT, typename IT, bool MAT>
StepFn pick_step2(int gather, int strat, int& block) {
  switch (gather) {
    case G_COUNT_SMEM:
      block = 1024;
      if (strat == S_HYBRID) return k_step<ST, AT, IT, G_COUNT_SMEM, S_HYBRID, MAT, 1024>;
      return strat == S_WARP ? k_step<ST, AT, IT, G_COUNT_SMEM, S_WARP, MAT, 1024>
                             : k_step<ST, AT, IT, G_COUNT_SMEM, S_THREAD, MAT, 1024>;
    case G_COUNT_GLOBAL:
      block = 512;
      if (strat == S_HYBRID) return k_step<ST, AT, IT, G_COUNT_GLOBAL, S_HYBRID, MAT, 512>;
      return strat == S_WARP ? k_step<ST, AT, IT, G_COUNT_GLOBAL, S_WARP, MAT, 512>
                             : k_step<ST, AT, IT, G_COUNT_GLOBAL, S_THREAD, MAT, 512>;
    case G_INCR:
      block = 512;
      return k_step<ST, AT, IT, G_INCR, S_THREAD, MAT, 512>;
    case G_F32:
      block = 512;
      return strat == S_WARP ? k_step<ST, AT, IT, G_F32, S_WARP, MAT, 512>
                             : k_step<ST, AT, IT, G_F32, S_THREAD, MAT, 512>;
    case G_F32M_SMEM:  // the mask in shared memory: one CTA per SM
      block = 1024;
      return strat == S_HYBRID ? k_step<ST, AT, IT, G_F32M_SMEM, S_HYBRID, MAT, 1024>
                               : k_step<ST, AT, IT, G_F32M_SMEM, S_THREAD, MAT, 1024>;
    case G_F32M_GLOBAL:
      block = 512;
      return strat == S_HYBRID ? k_step<ST, AT, IT, G_F32M_GLOBAL, S_HYBRID, MAT, 512>
                               : k_step<ST, AT, IT, G_F32M_GLOBAL, S_THREAD, MAT, 512>;
    default:
      block = 512;
      return k_step<ST, AT, IT, G_PRE, S_THREAD, MAT, 512>;
  }
}

StepFn pick_step(bool mixed, int gather, int strat, bool mat, int& block) {
  if (mixed)
    return mat ? pick_step2<int8_t, __half, __nv_bfloat16, true>(gather, strat, block)
               : pick_step2<int8_t, __half, __nv_bfloat16, false>(gather, strat, block);
  return mat ? pick_step2<int32_t, float, float, true>(gather, strat, block)
             : pick_step2<int32_t, float, float, false>(gather, strat, block);
}


}  // namespace fs
