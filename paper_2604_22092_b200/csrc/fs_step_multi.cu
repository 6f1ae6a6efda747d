// fs_step_multi.cu — instantiations of k_step_incr_multi, the ensemble launch
// of the incremental-count step (one grid steps every member engine; see
// fs_ensemble in fs_engine.cu).  Ensembles never materialise pressure / rates.
#include "fs_step.cuh"

namespace fs {

template <bool MEMO, bool HUBS, bool UNI>
MultiFn pick_multi3(bool mixed) {
  if (mixed) return k_step_incr_multi<int8_t, __half, false, MEMO, HUBS, UNI, 512>;
  return k_step_incr_multi<int32_t, float, false, MEMO, HUBS, UNI, 512>;
}

template <bool MEMO, bool HUBS>
MultiFn pick_multi2(bool mixed, bool uni) {
  return uni ? pick_multi3<MEMO, HUBS, true>(mixed) : pick_multi3<MEMO, HUBS, false>(mixed);
}

MultiFn pick_stream_multi(bool mixed, bool mat, bool memo, bool hubs, bool uni) {
  if (mat) return nullptr;
  if (memo) return hubs ? pick_multi2<true, true>(mixed, uni) : pick_multi2<true, false>(mixed, uni);
  return hubs ? pick_multi2<false, true>(mixed, uni) : pick_multi2<false, false>(mixed, uni);
}

template <bool HUBS, bool UNI>
PersistFn pick_persist2(bool mixed) {
  if (mixed) return k_step_incr_persist<int8_t, __half, HUBS, UNI, 512>;
  return k_step_incr_persist<int32_t, float, HUBS, UNI, 512>;
}

PersistFn pick_stream_persist(bool mixed, bool hubs, bool uni) {
  if (hubs) return uni ? pick_persist2<true, true>(mixed) : pick_persist2<true, false>(mixed);
  return uni ? pick_persist2<false, true>(mixed) : pick_persist2<false, false>(mixed);
}

}  // namespace fs
