// fs_step_incr.cu — instantiations of k_step_incr (incremental counts) and k_gather_merge
// (a separate translation unit so the step-kernel variants compile in parallel)
#include "fs_step.cuh"

namespace fs {

template <bool MEMO, bool HUBS, bool UNI>
StepFn pick_stream3(bool mixed, bool mat) {
  if (mixed) return mat ? k_step_incr<int8_t, __half, true, MEMO, HUBS, UNI, 512> : k_step_incr<int8_t, __half, false, MEMO, HUBS, UNI, 512>;
  return mat ? k_step_incr<int32_t, float, true, MEMO, HUBS, UNI, 512> : k_step_incr<int32_t, float, false, MEMO, HUBS, UNI, 512>;
}

template <bool MEMO, bool HUBS>
StepFn pick_stream2(bool mixed, bool mat, bool uni) {
  return uni ? pick_stream3<MEMO, HUBS, true>(mixed, mat) : pick_stream3<MEMO, HUBS, false>(mixed, mat);
}

// MEMO: the age-cohort hazard memo's shared table; HUBS: warp-cooperative
// pushes for rows over 32 edges (compiled out for bounded-degree graphs);
// UNI: S ages kept as one uniform scalar, quiet tiles skipped
// node-partitioned engines (PART): multi-rank pushes (direct peer atomics or
// the staged bulk exchange)
template <bool MEMO, bool HUBS, bool UNI>
StepFn pick_part3(bool mixed, bool mat) {
  if (mixed)
    return mat ? k_step_incr<int8_t, __half, true, MEMO, HUBS, UNI, 512, true>
               : k_step_incr<int8_t, __half, false, MEMO, HUBS, UNI, 512, true>;
  return mat ? k_step_incr<int32_t, float, true, MEMO, HUBS, UNI, 512, true>
             : k_step_incr<int32_t, float, false, MEMO, HUBS, UNI, 512, true>;
}

template <bool MEMO, bool HUBS>
StepFn pick_part(bool mixed, bool mat, bool uni) {
  return uni ? pick_part3<MEMO, HUBS, true>(mixed, mat) : pick_part3<MEMO, HUBS, false>(mixed, mat);
}

StepFn pick_stream(bool mixed, bool mat, bool memo, bool hubs, bool uni, bool part) {
  if (part) {
    if (memo) return hubs ? pick_part<true, true>(mixed, mat, uni) : pick_part<true, false>(mixed, mat, uni);
    return hubs ? pick_part<false, true>(mixed, mat, uni) : pick_part<false, false>(mixed, mat, uni);
  }
  if (memo) return hubs ? pick_stream2<true, true>(mixed, mat, uni) : pick_stream2<true, false>(mixed, mat, uni);
  return hubs ? pick_stream2<false, true>(mixed, mat, uni) : pick_stream2<false, false>(mixed, mat, uni);
}


MergeFn pick_merge(bool inf_bf16, int mode, int& block) {
  if (mode == 1) { block = 1024; return inf_bf16 ? k_gather_merge<__nv_bfloat16, 1, 1024> : k_gather_merge<float, 1, 1024>; }
  block = 512;
  if (mode == 2) return inf_bf16 ? k_gather_merge<__nv_bfloat16, 2, 512> : k_gather_merge<float, 2, 512>;
  return inf_bf16 ? k_gather_merge<__nv_bfloat16, 0, 512> : k_gather_merge<float, 0, 512>;
}


}  // namespace fs
