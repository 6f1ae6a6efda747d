// fs_step_tma.cu — instantiations of k_step_tma (mask gather, TMA column streaming)
// (a separate translation unit so the step-kernel variants compile in parallel)
#include "fs_step.cuh"

namespace fs {


template <typename ST, typename AT, bool SM, bool MAT, int B>
TmaFn pick_tma3(bool ptab_mul) {
  return ptab_mul ? k_step_tma<ST, AT, SM, MAT, true, B> : k_step_tma<ST, AT, SM, MAT, false, B>;
}
template <typename ST, typename AT, int B>
TmaFn pick_tma2(bool smem_mask, bool mat, bool ptab_mul) {
  if (smem_mask) return mat ? pick_tma3<ST, AT, true, true, B>(ptab_mul) : pick_tma3<ST, AT, true, false, B>(ptab_mul);
  return mat ? pick_tma3<ST, AT, false, true, B>(ptab_mul) : pick_tma3<ST, AT, false, false, B>(ptab_mul);
}
TmaFn pick_tma(bool mixed, bool smem_mask, bool mat, bool ptab_mul, int block) {
  if (block == 768)
    return mixed ? pick_tma2<int8_t, __half, 768>(smem_mask, mat, ptab_mul) : pick_tma2<int32_t, float, 768>(smem_mask, mat, ptab_mul);
  return mixed ? pick_tma2<int8_t, __half, 512>(smem_mask, mat, ptab_mul) : pick_tma2<int32_t, float, 512>(smem_mask, mat, ptab_mul);
}


}  // namespace fs
