// fs_setup.cu — run setup on the device, so no PyTorch compute runs in
// init_renewal_state / _build_plan:
//
//  * seed selection — the reference's _pick_seed_nodes (R/renewal.py:162-169):
//    the `count` nodes with the smallest u = uniform_array(derive_seed(seed,
//    0x5EEDC0DE), 0, id).  u = (x >> 11) 2^-53 orders like the 53-bit key
//    x >> 11, so the choice is a radix select of the count-th smallest
//    (key, id) pair P: 16-bit digits from the top, one histogram pass each
//    (the keys are recomputed, never stored), until the candidates that share
//    the selected digits fit one CTA, which sorts them.  Every node with
//    (key, id) <= P is a seed.  Ties (equal 53-bit keys, p ~ N^2 2^-54) are
//    broken by the smaller id; numpy's argpartition leaves them unspecified.
//  * the symmetry check of the incoming CSR (is it its own transpose, i.e.
//    an undirected graph as every reference generator builds, R/graph.py:
//    221-231): for every edge j -> i, the multiplicity of j in row i equals
//    that of i in row j — two binary searches in sorted rows per edge.
//  * the int32 copy of the row offsets.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "fs_device.cuh"
#include "fs_internal.h"

namespace fs {
namespace {

constexpr int kDigitBits = 12;  // 4096 bins: a shared-memory histogram
constexpr int kBins = 1 << kDigitBits;
constexpr int kSortCap = 2048;  // candidates one CTA sorts in shared memory (32 KB)

__device__ __forceinline__ uint64_t seed_key(uint64_t step_key, uint64_t id) {
  return avalanche(step_key ^ (id * kStreamMult)) >> 11;  // 53 bits, same order as u
}

// histogram of the key bits [shift, shift_hi) over the nodes whose bits
// above shift_hi equal `prefix`
__global__ void k_seed_hist(int64_t n, uint64_t step_key, int shift_hi, uint64_t prefix, int shift, uint32_t dmask,
                            unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = seed_key(step_key, (uint64_t)i);
    if ((k >> shift_hi) != prefix) continue;
    atomicAdd(&h[(k >> shift) & dmask], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, (unsigned long long)h[i]);
}

// the nodes whose key bits above `shift` equal `prefix` (<= kSortCap of them)
__global__ void k_seed_collect(int64_t n, uint64_t step_key, int shift, uint64_t prefix,
                               unsigned long long* __restrict__ keys, long long* __restrict__ ids,
                               unsigned int* __restrict__ num) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = seed_key(step_key, (uint64_t)i);
    if ((k >> shift) != prefix) continue;
    const unsigned at = atomicAdd(num, 1u);
    if (at < (unsigned)kSortCap) {
      keys[at] = k;
      ids[at] = i;
    }
  }
}

// one CTA: sort the candidates by (key, id) and publish the r-th (1-based)
__global__ void k_seed_pivot(const unsigned long long* __restrict__ keys, const long long* __restrict__ ids,
                             const unsigned int* __restrict__ num, long long r, unsigned long long* __restrict__ pivot) {
  __shared__ unsigned long long sk[kSortCap];
  __shared__ long long si[kSortCap];
  const int m = (int)min(*num, (unsigned)kSortCap);
  int p2 = 1;
  while (p2 < m) p2 <<= 1;
  for (int i = threadIdx.x; i < p2; i += blockDim.x) {
    sk[i] = i < m ? keys[i] : ~0ull;
    si[i] = i < m ? ids[i] : (long long)0x7FFFFFFFFFFFFFFFLL;
  }
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < p2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = sk[i] > sk[j] || (sk[i] == sk[j] && si[i] > si[j]);
          if (gt == up) {
            const unsigned long long tk = sk[i];
            sk[i] = sk[j];
            sk[j] = tk;
            const long long ti = si[i];
            si[i] = si[j];
            si[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    pivot[0] = sk[r - 1];
    pivot[1] = (unsigned long long)si[r - 1];
  }
}

template <typename ST, typename IT>
__global__ void k_seed_mark(int64_t n, uint64_t step_key, const unsigned long long* __restrict__ pivot, ST* states,
                            int comp, IT* inf, float inf_val, uint8_t* __restrict__ flags) {
  const uint64_t pk = pivot[0];
  const int64_t pi = (int64_t)pivot[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = seed_key(step_key, (uint64_t)i);
    const bool sel = k < pk || (k == pk && i <= pi);
    if (flags) flags[i] = sel ? 1 : 0;
    if (!sel) continue;
    if (states) states[i] = (ST)comp;
    if (inf) inf[i] = from_f32<IT>(inf_val);
  }
}

// symmetric iff every edge's multiplicity matches its reverse's.  Edge e
// (row i, [a, b)) is checked when it is the first of its run of equal
// columns: the run's length against the length of i's run in row j.
template <typename RO>
__device__ __forceinline__ bool edge_symmetric(const RO* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
                                               int64_t i, int64_t a, int64_t b, int64_t e) {
  const int32_t j = col[e];
  if (e > a && col[e - 1] == j) return true;  // counted with the first of its run
  if (j < 0 || j >= n) return false;
  int64_t mult = 1;
  while (e + mult < b && col[e + mult] == j) ++mult;
  // equal range of i in row j (sorted by source)
  int64_t lo = ro[j], hi = ro[j + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] < i) lo = mid + 1; else hi = mid;
  }
  int64_t lo2 = lo, hi2 = ro[j + 1];
  while (lo2 < hi2) {
    const int64_t mid = (lo2 + hi2) >> 1;
    if (col[mid] <= i) lo2 = mid + 1; else hi2 = mid;
  }
  return lo2 - lo == mult;
}

// a warp takes 32 rows: a lane checks a short row (<= 32 edges) alone; the
// long rows (scale-free hubs) are checked by the whole warp, 32 edges at a
// time, so one hub does not serialise the check
template <typename RO>
__global__ void k_symmetric(const RO* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
                            int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp_g * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    int64_t a = 0, b = 0;
    if (i < n) {
      a = ro[i];
      b = ro[i + 1];
    }
    const bool wide = b - a > 32;
    bool ok = true;
    if (!wide)
      for (int64_t e = a; e < b && ok; ++e) ok = edge_symmetric(ro, col, n, i, a, b, e);
    unsigned rest = __ballot_sync(0xffffffffu, wide);
    while (rest) {
      const int src = __ffs(rest) - 1;
      rest &= rest - 1;
      const int64_t r = base + src;
      const int64_t ra = __shfl_sync(0xffffffffu, a, src), rb = __shfl_sync(0xffffffffu, b, src);
      for (int64_t e = ra + lane; e < rb && ok; e += 32) ok = edge_symmetric(ro, col, n, r, ra, rb, e);
    }
    if (!ok) atomicExch(bad, 1);
  }
}

// row offsets must be non-decreasing and sorted within rows for the check
template <typename RO>
__global__ void k_rows_sorted(const RO* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
                              int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = ro[i] + 1; e < ro[i + 1]; ++e)
      if (col[e - 1] > col[e]) { atomicExch(bad, 1); return; }
}

template <typename T>
__global__ void k_fill_pattern(T* __restrict__ p, int64_t n, T v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_narrow(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

// many trials of a small graph at once (ensembles): one CTA per trial sorts
// all N <= kSmallSeedN (key, id) pairs in shared memory and marks the first
// `count` — the same selection as the radix path, without host round trips
constexpr int kSmallSeedN = 4096;
template <typename ST, typename IT>
__global__ void __launch_bounds__(1024) k_seed_small(int64_t n, const uint64_t* __restrict__ pick_keys, int64_t count,
                                                     ST* __restrict__ states, int64_t stride, int comp,
                                                     IT* __restrict__ inf, float inf_val) {
  __shared__ unsigned long long sk[kSmallSeedN];
  __shared__ unsigned short si[kSmallSeedN];
  const int t = blockIdx.x;
  const uint64_t step_key = splitmix_step_key(pick_keys[t], 0);
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  for (int i = threadIdx.x; i < p2; i += blockDim.x) {
    sk[i] = i < n ? (unsigned long long)seed_key(step_key, (uint64_t)i) : ~0ull;
    si[i] = (unsigned short)(i < n ? i : 0xFFFF);
  }
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride2 = size >> 1; stride2 > 0; stride2 >>= 1) {
      for (int i = threadIdx.x; i < p2; i += blockDim.x) {
        const int j = i ^ stride2;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = sk[i] > sk[j] || (sk[i] == sk[j] && si[i] > si[j]);
          if (gt == up) {
            const unsigned long long tk = sk[i];
            sk[i] = sk[j];
            sk[j] = tk;
            const unsigned short ti = si[i];
            si[i] = si[j];
            si[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const int id = si[i];
    states[(int64_t)t * stride + id] = (ST)comp;
    if (inf) inf[(int64_t)t * stride + id] = from_f32<IT>(inf_val);
  }
}

int grid_of(int64_t n, int block = 256) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + block - 1) / block, (int64_t)sms * 8));
}

}  // namespace
}  // namespace fs

using namespace fs;

#define FS_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t err__ = (call);                                                               \
    if (err__ != cudaSuccess)                                                                 \
      return set_error(FS_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(err__), \
                       __FILE__, __LINE__);                                                   \
  } while (0)

extern "C" {

int fs_seed_select(int64_t n, uint64_t seed_key_in, int64_t count, void* states, int32_t states_dtype,
                   int32_t compartment, void* inf, int32_t inf_dtype, float inf_value, uint8_t* flags,
                   void* stream) {
  if (n < 0 || count < 0 || count > n) return set_error(FS_EINVAL, "seed count %lld outside [0, N=%lld]", (long long)count, (long long)n);
  if (states && states_dtype != FS_I32 && states_dtype != FS_I8) return set_error(FS_EINVAL, "states dtype must be i32 or i8");
  if (inf && inf_dtype != FS_F32 && inf_dtype != FS_BF16) return set_error(FS_EINVAL, "infectivity dtype must be f32 or bf16");
  if (count == 0) {
    if (flags && n) FS_CUDA(cudaMemsetAsync(flags, 0, (size_t)n, (cudaStream_t)stream));
    return 0;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t step_key = splitmix_step_key(seed_key_in, 0);  // uniform_array(seed, step 0, ids)
  unsigned long long* hist = nullptr;
  unsigned long long* keys = nullptr;
  long long* ids = nullptr;
  unsigned int* num = nullptr;
  unsigned long long* pivot = nullptr;
  FS_CUDA(cudaMallocAsync(&hist, sizeof(unsigned long long) * kBins, st));
  FS_CUDA(cudaMallocAsync(&keys, sizeof(unsigned long long) * kSortCap, st));
  FS_CUDA(cudaMallocAsync(&ids, sizeof(long long) * kSortCap, st));
  FS_CUDA(cudaMallocAsync(&num, sizeof(unsigned int), st));
  FS_CUDA(cudaMallocAsync(&pivot, sizeof(unsigned long long) * 2, st));
  std::vector<unsigned long long> h(kBins);
  uint64_t prefix = 0;  // the key bits above shift_hi fixed so far
  int shift_hi = 53;
  long long r = count;  // rank still to find among the nodes sharing `prefix`
  int rc = 0;
  for (;;) {
    const int w = std::min(kDigitBits, shift_hi);
    const int sh = shift_hi - w;
    FS_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * kBins, st));
    k_seed_hist<<<grid_of(n, 512), 512, 0, st>>>(n, step_key, shift_hi, prefix, sh, (1u << w) - 1u, hist);
    FS_CUDA(cudaGetLastError());
    FS_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(unsigned long long) * kBins, cudaMemcpyDeviceToHost, st));
    FS_CUDA(cudaStreamSynchronize(st));
    long long below = 0;
    int bin = 0;
    for (; bin < (1 << w) - 1; ++bin) {
      if (below + (long long)h[bin] >= r) break;
      below += (long long)h[bin];
    }
    r -= below;
    prefix = (prefix << w) | (uint64_t)bin;
    shift_hi = sh;
    if ((long long)h[bin] <= kSortCap || sh == 0) break;
  }
  FS_CUDA(cudaMemsetAsync(num, 0, sizeof(unsigned int), st));
  k_seed_collect<<<grid_of(n, 512), 512, 0, st>>>(n, step_key, shift_hi, prefix, keys, ids, num);
  k_seed_pivot<<<1, 1024, 0, st>>>(keys, ids, num, r, pivot);
  FS_CUDA(cudaGetLastError());
  const int g = grid_of(n);
  if (states_dtype == FS_I8) {
    if (inf_dtype == FS_BF16)
      k_seed_mark<int8_t, __nv_bfloat16><<<g, 256, 0, st>>>(n, step_key, pivot, (int8_t*)states, compartment,
                                                           (__nv_bfloat16*)inf, inf_value, flags);
    else
      k_seed_mark<int8_t, float><<<g, 256, 0, st>>>(n, step_key, pivot, (int8_t*)states, compartment, (float*)inf,
                                                   inf_value, flags);
  } else {
    if (inf_dtype == FS_BF16)
      k_seed_mark<int32_t, __nv_bfloat16><<<g, 256, 0, st>>>(n, step_key, pivot, (int32_t*)states, compartment,
                                                            (__nv_bfloat16*)inf, inf_value, flags);
    else
      k_seed_mark<int32_t, float><<<g, 256, 0, st>>>(n, step_key, pivot, (int32_t*)states, compartment,
                                                    (float*)inf, inf_value, flags);
  }
  FS_CUDA(cudaGetLastError());
  for (void* q : {(void*)hist, (void*)keys, (void*)ids, (void*)num, (void*)pivot}) cudaFreeAsync(q, st);
  return rc;
}

int fs_seed_select_batch(int64_t n, int32_t trials, const uint64_t* pick_keys, int64_t count, void* states,
                         int64_t stride, int32_t states_dtype, int32_t compartment, void* inf, int32_t inf_dtype,
                         float inf_value, void* stream) {
  if (n < 1 || n > kSmallSeedN) return set_error(FS_EINVAL, "batched seed selection needs 1 <= N <= %d", kSmallSeedN);
  if (trials < 1 || !pick_keys || !states) return set_error(FS_EINVAL, "bad batched seed-selection arguments");
  if (count < 0 || count > n) return set_error(FS_EINVAL, "seed count %lld outside [0, N=%lld]", (long long)count, (long long)n);
  if (states_dtype != FS_I32 && states_dtype != FS_I8) return set_error(FS_EINVAL, "states dtype must be i32 or i8");
  if (inf && inf_dtype != FS_F32 && inf_dtype != FS_BF16) return set_error(FS_EINVAL, "infectivity dtype must be f32 or bf16");
  if (count == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t* dk = nullptr;
  FS_CUDA(cudaMallocAsync(&dk, sizeof(uint64_t) * trials, st));
  FS_CUDA(cudaMemcpyAsync(dk, pick_keys, sizeof(uint64_t) * trials, cudaMemcpyHostToDevice, st));
#define SEED_SMALL(ST_, IT_) \
  k_seed_small<ST_, IT_><<<trials, 1024, 0, st>>>(n, dk, count, (ST_*)states, stride, compartment, (IT_*)inf, inf_value)
  if (states_dtype == FS_I8) {
    if (inf_dtype == FS_BF16) SEED_SMALL(int8_t, __nv_bfloat16);
    else SEED_SMALL(int8_t, float);
  } else {
    if (inf_dtype == FS_BF16) SEED_SMALL(int32_t, __nv_bfloat16);
    else SEED_SMALL(int32_t, float);
  }
#undef SEED_SMALL
  FS_CUDA(cudaGetLastError());
  cudaFreeAsync(dk, st);
  return 0;
}

int fs_flags_to_ids(const uint8_t* flags, int64_t n, int64_t* out_ids, int64_t* num_out, void* stream) {
  if (n < 0 || (n > 0 && (!flags || !out_ids || !num_out))) return set_error(FS_EINVAL, "bad flags_to_ids arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) { *num_out = 0; return 0; }
  long long* d_num = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::CountingInputIterator<long long> it(0);
  cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flags, (long long*)out_ids, d_num, n, st);
  FS_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, st));
  FS_CUDA(cudaMallocAsync(&d_num, sizeof(long long), st));
  cub::DeviceSelect::Flagged(tmp, tmp_bytes, it, flags, (long long*)out_ids, d_num, n, st);
  long long hn = 0;
  FS_CUDA(cudaMemcpyAsync(&hn, d_num, sizeof hn, cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(d_num, st);
  *num_out = hn;
  return 0;
}

int fs_check_symmetric(const int64_t* row_offsets, const int32_t* row_offsets32, const int32_t* col, int64_t n,
                       int64_t num_edges, int32_t* symmetric, void* stream) {
  if (n < 0 || !symmetric || (n > 0 && !row_offsets && !row_offsets32)) return set_error(FS_EINVAL, "bad symmetry-check arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (num_edges == 0 || n == 0) { *symmetric = 1; return 0; }
  int* bad = nullptr;
  FS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  FS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const int g = grid_of(n);
  if (row_offsets32) {
    k_rows_sorted<int32_t><<<g, 256, 0, st>>>(row_offsets32, col, n, bad);
    k_symmetric<int32_t><<<g, 256, 0, st>>>(row_offsets32, col, n, bad);
  } else {
    k_rows_sorted<int64_t><<<g, 256, 0, st>>>(row_offsets, col, n, bad);
    k_symmetric<int64_t><<<g, 256, 0, st>>>(row_offsets, col, n, bad);
  }
  FS_CUDA(cudaGetLastError());
  int hb = 0;
  FS_CUDA(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(bad, st);
  *symmetric = hb ? 0 : 1;
  return 0;
}

int fs_fill(void* ptr, int64_t n, int32_t elem_bytes, uint64_t pattern, void* stream) {
  if (n < 0 || (n > 0 && !ptr)) return set_error(FS_EINVAL, "bad fill arguments");
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  switch (elem_bytes) {
    case 1: FS_CUDA(cudaMemsetAsync(ptr, (int)(pattern & 0xFF), (size_t)n, st)); return 0;
    case 2: k_fill_pattern<uint16_t><<<grid_of(n), 256, 0, st>>>((uint16_t*)ptr, n, (uint16_t)pattern); break;
    case 4: k_fill_pattern<uint32_t><<<grid_of(n), 256, 0, st>>>((uint32_t*)ptr, n, (uint32_t)pattern); break;
    case 8: k_fill_pattern<uint64_t><<<grid_of(n), 256, 0, st>>>((uint64_t*)ptr, n, pattern); break;
    default: return set_error(FS_EINVAL, "fill element size must be 1, 2, 4 or 8");
  }
  FS_CUDA(cudaGetLastError());
  return 0;
}

int fs_narrow_offsets(const int64_t* row_offsets, int64_t len, int32_t* out, void* stream) {
  if (len < 0 || (len > 0 && (!row_offsets || !out))) return set_error(FS_EINVAL, "bad narrow_offsets arguments");
  if (len == 0) return 0;
  k_narrow<<<grid_of(len), 256, 0, (cudaStream_t)stream>>>(row_offsets, len, out);
  FS_CUDA(cudaGetLastError());
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// hub list of the fused edge-merge step (fs_engine.cu build_hub_list): the
// nodes with more than `wide` in-edges, sorted by in-degree, heaviest first
// (ties by node id), so the step's round-robin pre-pass hands the longest
// folds out first
// ---------------------------------------------------------------------------
namespace fs {
namespace {
__global__ void k_hub_flags(const int64_t* __restrict__ ro, int64_t n, int64_t wide, uint8_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (ro[i + 1] - ro[i]) > wide ? 1 : 0;
}
__global__ void k_hub_degrees(const int64_t* __restrict__ ro, const int32_t* __restrict__ ids, const long long* num,
                              int32_t* __restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < *num; i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = (int32_t)(ro[ids[i] + 1] - ro[ids[i]]);
}
}  // namespace

int fs_hub_list(const int64_t* row_offsets, int64_t n, int wide, int32_t* out, int64_t* num_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *num_out = 0;
  if (n <= 0) return 0;
  uint8_t* flags = nullptr;
  int32_t *ids = nullptr, *deg = nullptr, *deg2 = nullptr;
  long long* d_num = nullptr;
  void* tmp = nullptr;
  size_t tb1 = 0, tb2 = 0;
  FS_CUDA(cudaMallocAsync(&flags, n, st));
  FS_CUDA(cudaMallocAsync(&ids, sizeof(int32_t) * n, st));
  FS_CUDA(cudaMallocAsync(&d_num, sizeof(long long), st));
  const int g = grid_of(n);
  k_hub_flags<<<g, 256, 0, st>>>(row_offsets, n, wide, flags);
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tb1, it, flags, ids, d_num, (int)n, st);
  FS_CUDA(cudaMallocAsync(&tmp, tb1 + 16, st));
  cub::DeviceSelect::Flagged(tmp, tb1, it, flags, ids, d_num, (int)n, st);
  long long hn = 0;
  FS_CUDA(cudaMemcpyAsync(&hn, d_num, sizeof hn, cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(tmp, st);
  tmp = nullptr;
  int rc = 0;
  if (hn > 0) {
    FS_CUDA(cudaMallocAsync(&deg, sizeof(int32_t) * hn, st));
    FS_CUDA(cudaMallocAsync(&deg2, sizeof(int32_t) * hn, st));
    k_hub_degrees<<<grid_of(hn), 256, 0, st>>>(row_offsets, ids, d_num, deg);
    cub::DoubleBuffer<int32_t> keys(deg, deg2), vals(ids, out);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb2, keys, vals, (int)hn, 0, 32, st);
    FS_CUDA(cudaMallocAsync(&tmp, tb2 + 16, st));
    cub::DeviceRadixSort::SortPairsDescending(tmp, tb2, keys, vals, (int)hn, 0, 32, st);
    if (vals.Current() != out) FS_CUDA(cudaMemcpyAsync(out, vals.Current(), sizeof(int32_t) * hn, cudaMemcpyDeviceToDevice, st));
    FS_CUDA(cudaGetLastError());
  }
  FS_CUDA(cudaStreamSynchronize(st));
  for (void* q : {(void*)flags, (void*)ids, (void*)deg, (void*)deg2, (void*)d_num, tmp})
    if (q) cudaFreeAsync(q, st);
  *num_out = hn;
  return rc;
}
}  // namespace fs
