// fs_graphgen.cu — device generator of random uniform-degree graphs for the
// N = 1e8 / 1e9 configurations.
//
// The reference's gen_fixed_degree (R/graph.py:289-328) is a CPU
// configuration model: shuffle N*d stubs, pair them, repair self-loops and
// multi-edges by random swaps, lexsort into CSR.  At N = 1e8 it needs ~100 GB
// of host RAM and ~25 min, at 1e9 ~1 TB, and it is sequential
// in its repair loop.  This generator builds a random d-regular graph that
// needs no memory beyond the CSR itself and no communication between
// partitions, so every rank of a node-partitioned run generates exactly its
// own rows:
//
//   d even: the union of d/2 random Hamiltonian cycles.  Cycle c visits the
//           nodes in the order sigma_c(0), sigma_c(1), ..., sigma_c(N-1),
//           where sigma_c is a keyed pseudo-random bijection of [0, N) (a
//           balanced Feistel network on 2h bits with cycle walking).  Node i
//           sits at position p = sigma_c^-1(i); its neighbours in the cycle
//           are sigma_c(p - 1) and sigma_c(p + 1) (mod N).
//   d odd:  one more random perfect matching (N even, as N*d must be):
//           partner = sigma_m(p xor 1).
//
// No self-loops can occur (N >= 3 for a cycle, p xor 1 != p).  Two cycles
// may share an edge; such a multi-edge is seen identically by both of its
// endpoints, which both drop the copy, so the graph stays simple and
// symmetric.  The expected number of dropped edges is about d^2/4 in total,
// independent of N (each pair of cycles shares ~2 edges in expectation), so
// all but O(d^2) nodes have degree exactly d.  Slices are sorted by source id
// like the reference's (R/graph.py:141); weights are the uniform 1.0 of every
// reference generator (R/graph.py:230) and are not materialised.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>
#include <algorithm>
#include "fs_device.cuh"
#include "fs_internal.h"

namespace fs {

constexpr int kGenMaxDegree = 64;
constexpr int kFeistelRounds = 6;

struct Feistel {
  int h;            // half width in bits; domain [0, 4^h)
  uint64_t mask;    // (1 << h) - 1
  uint64_t n;       // permuted range [0, n)
  uint64_t key[kFeistelRounds];
};

__host__ __device__ __forceinline__ uint64_t feistel_f(const Feistel& f, int r, uint64_t x) {
  return avalanche(x ^ f.key[r]) & f.mask;
}
__host__ __device__ __forceinline__ uint64_t feistel_fwd_once(const Feistel& f, uint64_t x) {
  uint64_t L = x >> f.h, R = x & f.mask;
#pragma unroll
  for (int r = 0; r < kFeistelRounds; ++r) {
    const uint64_t t = L ^ feistel_f(f, r, R);
    L = R;
    R = t;
  }
  return (L << f.h) | R;
}
__host__ __device__ __forceinline__ uint64_t feistel_inv_once(const Feistel& f, uint64_t y) {
  uint64_t L = y >> f.h, R = y & f.mask;
#pragma unroll
  for (int r = kFeistelRounds - 1; r >= 0; --r) {
    const uint64_t t = R ^ feistel_f(f, r, L);
    R = L;
    L = t;
  }
  return (L << f.h) | R;
}
// cycle walking keeps the bijection inside [0, n)
__host__ __device__ __forceinline__ uint64_t perm_fwd(const Feistel& f, uint64_t x) {
  do { x = feistel_fwd_once(f, x); } while (x >= f.n);
  return x;
}
__host__ __device__ __forceinline__ uint64_t perm_inv(const Feistel& f, uint64_t y) {
  do { y = feistel_inv_once(f, y); } while (y >= f.n);
  return y;
}

struct RegularSpec {
  uint64_t n;
  int k;
  int cycles;       // k / 2
  int matching;     // k odd
  Feistel perm[kGenMaxDegree / 2 + 1];
};

// the k neighbour ids of node i, sorted, duplicates (shared cycle edges)
// removed; returns the distinct count
__device__ __forceinline__ int regular_neighbours(const RegularSpec& s, uint64_t i, uint32_t* nb) {
  int m = 0;
  for (int c = 0; c < s.cycles; ++c) {
    const Feistel& f = s.perm[c];
    const uint64_t p = perm_inv(f, i);
    nb[m++] = (uint32_t)perm_fwd(f, p == 0 ? s.n - 1 : p - 1);
    nb[m++] = (uint32_t)perm_fwd(f, p + 1 == s.n ? 0 : p + 1);
  }
  if (s.matching) {
    const Feistel& f = s.perm[s.cycles];
    nb[m++] = (uint32_t)perm_fwd(f, perm_inv(f, i) ^ 1ull);
  }
  for (int a = 1; a < m; ++a) {  // insertion sort (m <= 64)
    const uint32_t v = nb[a];
    int b = a - 1;
    while (b >= 0 && nb[b] > v) { nb[b + 1] = nb[b]; --b; }
    nb[b + 1] = v;
  }
  // a value present twice is a multi-edge: drop every copy of it after the
  // first (both endpoints see the same multiplicity, so symmetry holds)
  int d = 0;
  for (int a = 0; a < m; ++a)
    if (d == 0 || nb[d - 1] != nb[a]) nb[d++] = nb[a];
  return d;
}

__global__ void __launch_bounds__(256) k_regular_degree(const RegularSpec s, uint64_t lo, uint64_t rows,
                                                        int64_t* __restrict__ deg_out) {
  uint32_t nb[kGenMaxDegree];
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x)
    deg_out[r + 1] = regular_neighbours(s, lo + r, nb);
  if (blockIdx.x == 0 && threadIdx.x == 0) deg_out[0] = 0;
}

__global__ void __launch_bounds__(256) k_regular_fill(const RegularSpec s, uint64_t lo, uint64_t rows,
                                                      const int64_t* __restrict__ ro, int32_t* __restrict__ col) {
  uint32_t nb[kGenMaxDegree];
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
    const int d = regular_neighbours(s, lo + r, nb);
    int32_t* out = col + ro[r];
    for (int a = 0; a < d; ++a) out[a] = (int32_t)nb[a];
  }
}

static RegularSpec make_regular_spec(uint64_t n, int k, uint64_t seed) {
  RegularSpec s{};
  s.n = n;
  s.k = k;
  s.cycles = k / 2;
  s.matching = k & 1;
  int bits = 1;
  while (bits < 64 && (1ull << bits) < n) ++bits;
  const int h = std::max(1, (bits + 1) / 2);
  for (int c = 0; c < s.cycles + s.matching; ++c) {
    Feistel& f = s.perm[c];
    f.h = h;
    f.mask = (1ull << h) - 1ull;
    f.n = n;
    for (int r = 0; r < kFeistelRounds; ++r)
      f.key[r] = avalanche(avalanche(seed ^ (0x6EA9ull * kStepMult)) ^ ((uint64_t)(c * kFeistelRounds + r + 1) * kStreamMult));
  }
  return s;
}

}  // namespace fs

using namespace fs;

extern "C" int fs_gen_regular(int64_t n, int32_t k, uint64_t seed, int64_t row_lo, int64_t row_hi,
                              int64_t* row_offsets, int32_t* col, int64_t col_capacity, int64_t* num_edges,
                              void* stream) {
  if (n < 2 || n > 2147483647LL) return set_error(FS_EINVAL, "fs_gen_regular: need 2 <= N <= 2^31-1 (got %lld)", (long long)n);
  if (k < 0 || k >= n || k > kGenMaxDegree) return set_error(FS_EINVAL, "fs_gen_regular: degree %d infeasible for N=%lld (max %d)", k, (long long)n, kGenMaxDegree);
  if ((n * (int64_t)k) % 2 != 0) return set_error(FS_EINVAL, "fs_gen_regular: N * d must be even");
  if (k >= 2 && n < 3) return set_error(FS_EINVAL, "fs_gen_regular: cycles need N >= 3");
  if (row_lo < 0 || row_hi < row_lo || row_hi > n) return set_error(FS_EINVAL, "fs_gen_regular: bad row range");
  if (!row_offsets || !num_edges) return set_error(FS_EINVAL, "fs_gen_regular: null output");
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t rows = (uint64_t)(row_hi - row_lo);
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = std::max(1, fs_device_sm_count(dev));
  const RegularSpec s = make_regular_spec((uint64_t)n, k, seed);
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((rows + 255) / 256, (uint64_t)sms * 16));
  k_regular_degree<<<grid, 256, 0, st>>>(s, (uint64_t)row_lo, rows, row_offsets);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(FS_ECUDA, "k_regular_degree: %s", cudaGetErrorString(err));
  // inclusive scan of deg[1..rows] in place -> row offsets
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, row_offsets + 1, row_offsets + 1, (int64_t)rows, st);
  void* tmp = nullptr;
  if (rows > 0) {
    if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) return set_error(FS_ENOMEM, "scan scratch");
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, row_offsets + 1, row_offsets + 1, (int64_t)rows, st);
    cudaFreeAsync(tmp, st);
  }
  int64_t e = 0;
  if (cudaMemcpyAsync(&e, row_offsets + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return set_error(FS_ECUDA, "fs_gen_regular: edge count readback");
  *num_edges = e;
  if (!col) return 0;  // sizing call
  if (e > col_capacity) return set_error(FS_EINVAL, "fs_gen_regular: %lld edges exceed col capacity %lld", (long long)e, (long long)col_capacity);
  k_regular_fill<<<grid, 256, 0, st>>>(s, (uint64_t)row_lo, rows, row_offsets, col);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(FS_ECUDA, "k_regular_fill: %s", cudaGetErrorString(err));
  return 0;
}

// host restatement of one neighbour list (for the CPU tests of the
// generator's construction, no device needed)
extern "C" int fs_gen_regular_row_host(int64_t n, int32_t k, uint64_t seed, int64_t node, int32_t* out) {
  if (n < 2 || k < 0 || k >= n || k > kGenMaxDegree || node < 0 || node >= n || !out)
    return set_error(FS_EINVAL, "fs_gen_regular_row_host: bad arguments");
  const RegularSpec s = make_regular_spec((uint64_t)n, k, seed);
  uint64_t nb[kGenMaxDegree];
  int m = 0;
  for (int c = 0; c < s.cycles; ++c) {
    const Feistel& f = s.perm[c];
    const uint64_t p = perm_inv(f, (uint64_t)node);
    nb[m++] = perm_fwd(f, p == 0 ? s.n - 1 : p - 1);
    nb[m++] = perm_fwd(f, p + 1 == s.n ? 0 : p + 1);
  }
  if (s.matching) nb[m++] = perm_fwd(s.perm[s.cycles], perm_inv(s.perm[s.cycles], (uint64_t)node) ^ 1ull);
  std::sort(nb, nb + m);
  int d = 0;
  for (int a = 0; a < m; ++a)
    if (d == 0 || nb[d - 1] != nb[a]) nb[d++] = nb[a];
  for (int a = 0; a < d; ++a) out[a] = (int32_t)nb[a];
  return d;
}
