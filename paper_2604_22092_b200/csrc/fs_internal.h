// fs_internal.h — helpers shared by the translation units of the library.
#pragma once
#include <string>

namespace fs {
extern thread_local std::string g_last_error;
int set_error(int code, const char* fmt, ...);
}  // namespace fs

#include <cstdint>
#include <cuda_runtime.h>
namespace fs {
// fs_comm.cpp: the per-step exchange of a node-partitioned run:
// all-reduce-sum of the step's 16 count deltas, all-reduce-max of its max-rate
// bits, in-place all-gather of the next-step infectious mask (seg_words per
// rank), as one NCCL group on `st`.
// fs_setup.cu: hub list of the fused edge-merge step (in-degree > wide,
// heaviest first) into out[], its length into *num_out
int fs_hub_list(const int64_t* row_offsets, int64_t n, int wide, int32_t* out, int64_t* num_out, void* stream);
int fs_exchange_step(void* comm, unsigned long long* d16, unsigned* max_bits, uint32_t* mask, int64_t seg_words,
                     int rank, cudaStream_t st);
}  // namespace fs
