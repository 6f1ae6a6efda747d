// fs_ops.cu — device utilities behind the reference's host-side helpers:
// counter-based uniforms (rng.py:60-67), erfcx / hazard evaluation
// (hazards.py:108-146) and the active-set refresh (renewal.py:426-432).
#include <cuda_runtime.h>
#include <algorithm>
#include "fs_device.cuh"
#include "fs_internal.h"

namespace fs {

__global__ void k_uniform(uint64_t seed, uint64_t step, const uint64_t* __restrict__ streams, int64_t n, int rng,
                          double* __restrict__ out) {
  const uint64_t key = splitmix_step_key(seed, step);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t s = streams ? streams[i] : (uint64_t)i;
    out[i] = rng == FS_RNG_SPLITMIX ? splitmix_uniform(key, s) : philox_uniform(seed, step, s);
  }
}

__global__ void k_hazard(fs_compartment c, const double* __restrict__ tau, int64_t n, int prec, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = tau[i];
    double h;
    if (prec == FS_HAZ_F64) {
      switch (c.hazard) {
        case FS_HZ_EXPONENTIAL: h = c.p0; break;
        case FS_HZ_LOGNORMAL: h = hazard_lognormal_f64(t, c.p0, c.p1); break;
        case FS_HZ_WEIBULL: h = hazard_weibull_f64(t, c.p0, c.p1); break;
        case FS_HZ_ERLANG: h = hazard_erlang_f64(t, (int)c.p0, c.p1); break;
        default: h = 0.0;
      }
    } else {
      h = (double)nodal_rate(c.hazard, c.p0, c.p1, (float)t, FS_HAZ_F32);
    }
    out[i] = h;
  }
}

__global__ void k_erfcx(const double* __restrict__ z, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = erfcx_piecewise(z[i]);
}

// ordered stream compaction of non-terminal node ids, three passes:
// per-block counts -> exclusive scan of the counts -> ordered writes
constexpr int kRefreshItems = 4096;  // nodes per block

template <typename ST>
__global__ void __launch_bounds__(256) k_active_count(const ST* __restrict__ st, int64_t n, uint32_t term_bits,
                                                      int64_t* __restrict__ block_counts) {
  const int64_t base = (int64_t)blockIdx.x * kRefreshItems;
  int c = 0;
  for (int k = threadIdx.x; k < kRefreshItems; k += blockDim.x) {
    const int64_t i = base + k;
    if (i < n && !((term_bits >> (int)st[i]) & 1u)) ++c;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int s[8];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < 8; ++w) t += s[w];
    block_counts[blockIdx.x] = t;
  }
}

__global__ void k_exclusive_scan(int64_t* __restrict__ v, int64_t m, int64_t* __restrict__ total) {
  // single-thread scan: m = N / 4096 entries (244k at N=1e9), run once per refresh
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t acc = 0;
    for (int64_t i = 0; i < m; ++i) { int64_t x = v[i]; v[i] = acc; acc += x; }
    *total = acc;
  }
}

template <typename ST>
__global__ void __launch_bounds__(256) k_active_write(const ST* __restrict__ st, int64_t n, uint32_t term_bits,
                                                      const int64_t* __restrict__ block_offsets, int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_w[8];
  __shared__ int64_t s_base;
  if (threadIdx.x == 0) s_base = block_offsets[blockIdx.x];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRefreshItems;
  for (int k0 = 0; k0 < kRefreshItems; k0 += 256) {
    const int64_t i = base + k0 + threadIdx.x;
    const bool act = i < n && !((term_bits >> (int)st[i]) & 1u);
    const unsigned b = __ballot_sync(0xffffffffu, act);
    if (lane == 0) s_w[warp] = __popc(b);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < 8; ++w) { if (w < warp) before += s_w[w]; total += s_w[w]; }
    if (act) out[s_base + before + __popc(b & ((1u << lane) - 1u))] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
}

}  // namespace fs

using namespace fs;

#define FS_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t err__ = (call);                                                               \
    if (err__ != cudaSuccess)                                                                 \
      return set_error(FS_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(err__), \
                       __FILE__, __LINE__);                                                   \
  } while (0)

static int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
}

extern "C" int fs_uniform_fill(uint64_t seed, uint64_t step, const uint64_t* streams, int64_t n, int32_t rng,
                               double* out, void* stream) {
  if (n < 0 || (n > 0 && !out)) return set_error(FS_EINVAL, "bad uniform_fill arguments");
  if (rng != FS_RNG_SPLITMIX && rng != FS_RNG_PHILOX) return set_error(FS_EINVAL, "unknown rng %d", rng);
  if (n == 0) return 0;
  k_uniform<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(seed, step, streams, n, rng, out);
  FS_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int fs_hazard_eval(const fs_compartment* c, const double* tau, int64_t n, double* out, int32_t precision,
                              void* stream) {
  if (!c || n < 0 || (n > 0 && (!tau || !out))) return set_error(FS_EINVAL, "bad hazard_eval arguments");
  if (n == 0) return 0;
  k_hazard<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(*c, tau, n, precision, out);
  FS_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int fs_erfcx_eval(const double* z, int64_t n, double* out, void* stream) {
  if (n < 0 || (n > 0 && (!z || !out))) return set_error(FS_EINVAL, "bad erfcx_eval arguments");
  if (n == 0) return 0;
  k_erfcx<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(z, n, out);
  FS_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int fs_refresh_active(const void* states, int32_t states_dtype, int64_t n, const uint8_t* terminal,
                                 int32_t num_compartments, int32_t* out_ids, int64_t capacity, int64_t* num_active,
                                 void* stream) {
  if (!states || !terminal || !out_ids || !num_active || n < 0) return set_error(FS_EINVAL, "bad refresh_active arguments");
  if (capacity < n) return set_error(FS_EINVAL, "capacity %lld < N %lld", (long long)capacity, (long long)n);
  if (num_compartments < 1 || num_compartments > FS_MAX_COMPARTMENTS) return set_error(FS_EINVAL, "bad num_compartments");
  if (states_dtype != FS_I32 && states_dtype != FS_I8) return set_error(FS_EINVAL, "states dtype must be i32 or i8");
  uint32_t term_bits = 0;
  for (int i = 0; i < num_compartments; ++i) if (terminal[i]) term_bits |= 1u << i;
  cudaStream_t st = (cudaStream_t)stream;
  FS_CUDA(cudaMemsetAsync(out_ids, 0, capacity * sizeof(int32_t), st));
  if (n == 0) { *num_active = 0; return 0; }
  const int64_t nb = (n + kRefreshItems - 1) / kRefreshItems;
  int64_t* buf = nullptr;
  FS_CUDA(cudaMallocAsync((void**)&buf, (nb + 1) * sizeof(int64_t), st));
  if (states_dtype == FS_I32) k_active_count<int32_t><<<(int)nb, 256, 0, st>>>((const int32_t*)states, n, term_bits, buf);
  else k_active_count<int8_t><<<(int)nb, 256, 0, st>>>((const int8_t*)states, n, term_bits, buf);
  k_exclusive_scan<<<1, 1, 0, st>>>(buf, nb, buf + nb);
  if (states_dtype == FS_I32) k_active_write<int32_t><<<(int)nb, 256, 0, st>>>((const int32_t*)states, n, term_bits, buf, out_ids);
  else k_active_write<int8_t><<<(int)nb, 256, 0, st>>>((const int8_t*)states, n, term_bits, buf, out_ids);
  FS_CUDA(cudaMemcpyAsync(num_active, buf + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaFreeAsync(buf, st));
  FS_CUDA(cudaStreamSynchronize(st));
  FS_CUDA(cudaGetLastError());
  return 0;
}
