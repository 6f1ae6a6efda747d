// fs_comm.cpp — NCCL plumbing of the node-partitioned engine.
//
// One communicator per rank (one process per GPU).  The unique id is made by
// rank 0 and travels over any host channel (the Python layer uses
// torch.distributed's object broadcast); the engine then issues one NCCL
// group per step on its own stream, inside the batch CUDA graph.
#include <nccl.h>
#include <cstring>
#include "../../include/flashspread.h"
#include "fs_internal.h"

#define FS_NCCL(call)                                                                              \
  do {                                                                                             \
    ncclResult_t r__ = (call);                                                                     \
    if (r__ != ncclSuccess) return fs::set_error(FS_ECUDA, "%s failed: %s", #call, ncclGetErrorString(r__)); \
  } while (0)

namespace fs {

int fs_exchange_step(void* comm, unsigned long long* d16, unsigned* max_bits, uint32_t* mask, int64_t seg_words,
                     int rank, cudaStream_t st) {
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  FS_NCCL(ncclGroupStart());
  FS_NCCL(ncclAllReduce(d16, d16, FS_MAX_COMPARTMENTS, ncclUint64, ncclSum, c, st));
  FS_NCCL(ncclAllReduce(max_bits, max_bits, 1, ncclUint32, ncclMax, c, st));  // rates >= 0: bits order as values
  if (mask) FS_NCCL(ncclAllGather(mask + (int64_t)rank * seg_words, mask, (size_t)seg_words, ncclUint32, c, st));
  FS_NCCL(ncclGroupEnd());
  return 0;
}

}  // namespace fs

extern "C" {

int fs_comm_unique_id(uint8_t* out, int32_t len) {
  if (!out || len < (int32_t)sizeof(ncclUniqueId)) return fs::set_error(FS_EINVAL, "unique id buffer needs %zu bytes", sizeof(ncclUniqueId));
  ncclUniqueId id;
  FS_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof id);
  return (int)sizeof id;
}

int fs_comm_init(int32_t world, int32_t rank, const uint8_t* id_bytes, int32_t device, void** out) {
  if (!id_bytes || !out || world < 1 || rank < 0 || rank >= world) return fs::set_error(FS_EINVAL, "bad communicator arguments");
  if (cudaSetDevice(device) != cudaSuccess) return fs::set_error(FS_ECUDA, "cudaSetDevice(%d)", device);
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof id);
  ncclComm_t c = nullptr;
  FS_NCCL(ncclCommInitRank(&c, world, id, rank));
  *out = c;
  return 0;
}

int fs_comm_time_exchange(void* comm, int32_t rank, int64_t seg_words, int32_t iters, void* stream, float* us) {
  if (!comm || iters < 1 || !us) return fs::set_error(FS_EINVAL, "bad exchange timing arguments");
  cudaStream_t st = (cudaStream_t)stream;
  void* buf = nullptr;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int world = 1;
  FS_NCCL(ncclCommCount(c, &world));
  const size_t bytes = 256 + (size_t)seg_words * (size_t)world * 4;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return fs::set_error(FS_ECUDA, "exchange timing buffer");
  cudaMemset(buf, 0, bytes);
  auto* d16 = static_cast<unsigned long long*>(buf);
  auto* mx = reinterpret_cast<unsigned*>(d16 + FS_MAX_COMPARTMENTS);
  uint32_t* mask = seg_words > 0 ? reinterpret_cast<uint32_t*>(static_cast<char*>(buf) + 256) : nullptr;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int rc = fs::fs_exchange_step(comm, d16, mx, mask, seg_words, rank, st);  // warm-up
  cudaEventRecord(a, st);
  for (int i = 0; i < iters && !rc; ++i) rc = fs::fs_exchange_step(comm, d16, mx, mask, seg_words, rank, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, a, b);
  *us = ms * 1e3f / (float)iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  return rc;
}

void fs_comm_destroy(void* comm) {
  if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
}

}  // extern "C"
