// fs_hostio.cpp — host side of getting a reference CsrGraph onto the device
// (the e2e path: run_renewal on a fresh host graph).  Two jobs the Python
// layer did in numpy / with page-locking before:
//
//  * fs_h2d_staged: host -> device copy of a large pageable array through a
//    small pool of page-locked staging slots owned by the library: the host
//    threads (OpenMP) copy chunk k into a slot while the copy engine moves
//    chunk k-1, so neither the array is page-locked (cudaHostRegister of
//    fresh pages cost ~0.4 ms per MB on the B200 hosts) nor a pageable copy
//    is serialised behind the driver's own staging.
//  * fs_host_csr_scan: the per-graph host scans of _build_plan — maximum
//    in-degree (R/graph.py:194-201 degree_stats) and whether every weight is
//    equal (the uniform-weight scalar, R/graph.py:230) — in parallel.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/flashspread.h"
#include "fs_internal.h"

namespace fs {
namespace {

constexpr int kSlots = 3;
constexpr size_t kSlotBytes = (size_t)8 << 20;

struct Staging {
  std::mutex mu;
  void* slot[kSlots] = {};
  cudaEvent_t done[kSlots] = {};
  int device = -1;
};
Staging g_stage;

int ensure_staging() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_stage.slot[0] && g_stage.device == dev) return 0;
  for (int i = 0; i < kSlots; ++i) {
    if (cudaHostAlloc(&g_stage.slot[i], kSlotBytes, cudaHostAllocDefault) != cudaSuccess)
      return set_error(FS_ECUDA, "cudaHostAlloc of the staging pool failed");
    if (cudaEventCreateWithFlags(&g_stage.done[i], cudaEventDisableTiming) != cudaSuccess)
      return set_error(FS_ECUDA, "staging event");
  }
  g_stage.device = dev;
  return 0;
}

void par_copy(void* dst, const void* src, size_t bytes) {
  const int nt = std::max(1, std::min(omp_get_max_threads(), (int)(bytes >> 20)));
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int t = 0; t < nt; ++t) {
    const size_t a = bytes * (size_t)t / (size_t)nt, b = bytes * (size_t)(t + 1) / (size_t)nt;
    std::memcpy((char*)dst + a, (const char*)src + a, b - a);
  }
}

}  // namespace
}  // namespace fs

using namespace fs;

extern "C" {

int fs_h2d_staged(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return set_error(FS_EINVAL, "bad staged copy arguments");
  if (bytes == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lock(g_stage.mu);
  int rc = ensure_staging();
  if (rc) return rc;
  int k = 0;
  for (int64_t off = 0; off < bytes; off += (int64_t)kSlotBytes, k = (k + 1) % kSlots) {
    const size_t len = (size_t)std::min<int64_t>((int64_t)kSlotBytes, bytes - off);
    if (cudaEventSynchronize(g_stage.done[k]) != cudaSuccess) return set_error(FS_ECUDA, "staging wait");
    par_copy(g_stage.slot[k], (const char*)src + off, len);
    if (cudaMemcpyAsync((char*)dst + off, g_stage.slot[k], len, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return set_error(FS_ECUDA, "staged H2D copy failed");
    if (cudaEventRecord(g_stage.done[k], st) != cudaSuccess) return set_error(FS_ECUDA, "staging event record");
  }
  // the slots are reused by the next call only after their events; the
  // caller's stream orders the copies before its kernels
  return 0;
}

int fs_host_csr_scan(const int64_t* row_offsets, int64_t n, const float* weights, int64_t num_edges, int64_t* d_max,
                     int32_t* uniform, float* w0) {
  if (n < 0 || num_edges < 0 || !d_max || !uniform || !w0 || (n > 0 && !row_offsets) || (num_edges > 0 && !weights))
    return set_error(FS_EINVAL, "bad csr scan arguments");
  int64_t dm = 0;
#pragma omp parallel for reduction(max : dm) schedule(static)
  for (int64_t i = 0; i < n; ++i) dm = std::max(dm, row_offsets[i + 1] - row_offsets[i]);
  *d_max = dm;
  if (num_edges == 0) {
    *uniform = 1;
    *w0 = 1.0f;
    return 0;
  }
  uint32_t ref;
  std::memcpy(&ref, weights, 4);
  const uint32_t* wb = reinterpret_cast<const uint32_t*>(weights);
  int bad = 0;
  // bitwise equality, as numpy's (w == w[0]).all() for every non-NaN value
#pragma omp parallel for reduction(| : bad) schedule(static)
  for (int64_t i = 0; i < num_edges; ++i) bad |= (wb[i] != ref) ? 1 : 0;
  float f;
  std::memcpy(&f, &ref, 4);
  // +0.0 / -0.0 compare equal in numpy: treat a mixed-sign-zero array as uniform 0
  if (bad && f == 0.0f) {
    bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
    for (int64_t i = 0; i < num_edges; ++i) bad |= (weights[i] != 0.0f) ? 1 : 0;
  }
  *uniform = (bad || f != f) ? 0 : 1;
  *w0 = f;
  return 0;
}

}  // extern "C"
