// fs_gen_random.cu — device generators for the reference's other two random
// graph models: Barabási–Albert preferential
// attachment (R/graph.py:331-365, the C3 graph) and G(N, p)
// (R/graph.py:252-286).  Both write rows [row_lo, row_hi) of the symmetric
// incoming CSR with global column ids, slices sorted by source, like
// fs_gen_regular; weights are the uniform 1.0 and not materialised.
//
// Barabási–Albert.  The reference grows an endpoint list R: the m-clique's
// endpoints, then for every new node v the pairs (v, t_k) of its m distinct
// targets, each t_k drawn as R[uniform position < |R| at v's arrival] with
// rejection of repeats.  |R| at v's arrival is a closed form, base(v) =
// c0 + 2m(v - m), and position p of R is either a source entry (known: the
// block's owner), a clique entry (node p / (m-1)), or the k-th target of an
// earlier node — so every target is a function of counter-based draws and
// of EARLIER targets only (the communication-free formulation of Sanders &
// Schulz / Funke et al.).  k_ba_resolve sweeps all (v, k) slots; a slot whose
// draw lands on a still-unresolved earlier slot waits for the next sweep.
// The dependency chains point strictly backwards and stop with probability
// >= 1/2 per hop, so a few dozen sweeps resolve 1e9 nodes.  Slot values are
// written once (-1 -> value), so concurrent readers see either "pending" or
// the final value and the result is independent of scheduling.  Targets sit
// in R in draw order rather than sorted (R/graph.py:358); positions are
// drawn uniformly, so the attachment process is the reference's.
//
// G(N, p).  The reference walks the N(N-1)/2 pair indices with geometric
// gaps (log u / log(1-p)).  Here the pair range is cut into chunks, each
// walked by one thread with its own counter-based stream: a Bernoulli(p)
// process restarted at chunk boundaries is the same process (memoryless
// gaps), so the union is exactly G(N, p).  Chunks are walked twice (count,
// then fill), so no edge list is stored.  Pair indices decode to (i < j) as
// in R/graph.py:234-249.
//
// CSR assembly: per-row counts (atomics over the implicit edge set), CUB
// scan, atomic-cursor fill, CUB segmented sort of each row, in row blocks of
// < 2^31 entries.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <algorithm>
#include <cmath>
#include <vector>
#include "fs_device.cuh"
#include "fs_internal.h"

namespace fs {

constexpr int kBaMaxM = 64;

__device__ __forceinline__ uint64_t draw64(uint64_t key, uint64_t a, uint64_t b) {
  return avalanche(avalanche(key ^ (a * kStepMult)) ^ (b * kStreamMult));
}

struct BaSpec {
  int64_t n;
  int m;
  int64_t c0;  // clique entries of R (+1 for m == 1: R[0] = 0, R/graph.py:350-351)
  uint64_t key;
};

__host__ __device__ __forceinline__ int64_t ba_base(const BaSpec& s, int64_t v) { return s.c0 + 2 * (int64_t)s.m * (v - s.m); }

// resolve R[pos]; -1 when it is a slot that is not resolved yet
__device__ __forceinline__ int32_t ba_entry(const BaSpec& s, const int32_t* tgt, int64_t pos) {
  if (pos < s.c0) return s.m == 1 ? 0 : (int32_t)(pos / (s.m - 1));
  const int64_t off = pos - s.c0;
  const int64_t w = s.m + off / (2 * s.m);
  const int r = (int)(off % (2 * s.m));
  if ((r & 1) == 0) return (int32_t)w;
  return *(volatile const int32_t*)&tgt[(w - s.m) * s.m + (r >> 1)];
}

__global__ void __launch_bounds__(256) k_ba_resolve(const BaSpec s, int32_t* __restrict__ tgt, int* pending) {
  int left = 0;
  const int64_t nodes = s.n - s.m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nodes; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = s.m + i;
    int32_t* my = tgt + i * s.m;
    const uint64_t base = (uint64_t)ba_base(s, v);
    for (int k = 0; k < s.m; ++k) {
      if (my[k] >= 0) continue;
      int32_t got = -1;
      for (uint64_t a = 0;; ++a) {  // draw order; earlier rejections re-resolve to the same values
        const uint64_t u = draw64(s.key, (uint64_t)v, (uint64_t)k * 0x100000000ull + a);
        const int32_t c = ba_entry(s, tgt, (int64_t)__umul64hi(u, base));
        if (c < 0) break;  // waits on an earlier slot
        bool dup = false;
        for (int j = 0; j < k; ++j) dup |= my[j] == c;
        if (!dup) { got = c; break; }
      }
      if (got < 0) { left = 1; break; }
      *(volatile int32_t*)&my[k] = got;
    }
  }
  if (__syncthreads_or(left) && threadIdx.x == 0) atomicOr(pending, 1);
}

// visit every undirected edge {a, b} of the BA graph touching rows [lo, hi)
template <bool FILL>
__global__ void __launch_bounds__(256) k_ba_rows(const BaSpec s, const int32_t* __restrict__ tgt, int64_t lo, int64_t hi,
                                                 unsigned long long* __restrict__ cursor, int32_t* __restrict__ col) {
  auto emit = [&](int64_t row, int64_t other) {
    if (row < lo || row >= hi) return;
    const unsigned long long at = atomicAdd(&cursor[row - lo], 1ull);
    if (FILL) col[at] = (int32_t)other;
  };
  const int64_t m = s.m;
  const int64_t total = (s.n - m) * m + m * (m - 1) / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a, b;
    if (e < (s.n - m) * m) {
      a = m + e / m;
      b = tgt[e];
    } else {  // clique pair index -> (u < w)
      int64_t q = e - (s.n - m) * m, u = 0;
      while (q >= m - 1 - u) { q -= m - 1 - u; ++u; }
      a = u;
      b = u + 1 + q;
    }
    emit(a, b);
    emit(b, a);
  }
}

struct ErSpec {
  int64_t n;
  unsigned long long pairs;  // N(N-1)/2
  unsigned long long chunk;  // pair indices per chunk
  unsigned long long chunks;
  double log1mp;
  int complete;              // p >= 1
  uint64_t key;
};

__device__ __forceinline__ void er_decode(int64_t n, unsigned long long k, int64_t& i, int64_t& j) {
  // R/graph.py:234-249
  const double b = 2.0 * (double)n - 1.0;
  int64_t r = (int64_t)floor((b - sqrt(b * b - 8.0 * (double)k)) / 2.0);
  r = r < 0 ? 0 : (r > n - 2 ? n - 2 : r);
  auto row_start = [n](int64_t ii) { return (unsigned long long)(ii * (2 * n - ii - 1) / 2); };
  for (int t = 0; t < 2; ++t) {
    if (row_start(r) > k) --r;
    if (row_start(r + 1) <= k) ++r;
  }
  i = r;
  j = (int64_t)(k - row_start(r)) + r + 1;
}

template <bool FILL>
__global__ void __launch_bounds__(256) k_er_rows(const ErSpec s, int64_t lo, int64_t hi,
                                                 unsigned long long* __restrict__ cursor, int32_t* __restrict__ col) {
  auto emit = [&](int64_t row, int64_t other) {
    if (row < lo || row >= hi) return;
    const unsigned long long at = atomicAdd(&cursor[row - lo], 1ull);
    if (FILL) col[at] = (int32_t)other;
  };
  for (unsigned long long c = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; c < s.chunks;
       c += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long start = c * s.chunk;
    const unsigned long long end = min(start + s.chunk, s.pairs);
    unsigned long long pos = start;
    for (uint64_t a = 0;; ++a) {
      if (!s.complete) {
        // u in (0, 1]: gap = floor(log u / log(1-p)) + 1 >= 1
        const double u = (double)((draw64(s.key, c, a) >> 11) + 1) * 0x1.0p-53;
        const double g = floor(log(u) / s.log1mp);
        if (!(g < (double)(end - pos))) break;
        pos += (unsigned long long)g;
      }
      if (pos >= end) break;
      int64_t i, j;
      er_decode(s.n, pos, i, j);
      emit(i, j);
      emit(j, i);
      ++pos;
    }
  }
}

__global__ void k_offsets_init(int64_t* ro, const unsigned long long* cnt, int64_t rows) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= rows; r += (int64_t)gridDim.x * blockDim.x)
    ro[r] = r == 0 ? 0 : (int64_t)cnt[r - 1];
}
__global__ void k_cursor_init(unsigned long long* cur, const int64_t* ro, int64_t rows) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    cur[r] = (unsigned long long)ro[r];
}

// counts -> offsets (inclusive scan), cursor reset, fill, per-row sort
template <class Visit>
static int assemble_rows(int64_t rows, int64_t* row_offsets, int32_t* col, int64_t col_capacity, int64_t* num_edges,
                         cudaStream_t st, int grid, Visit visit) {
  unsigned long long* cnt = nullptr;
  if (cudaMallocAsync(&cnt, (size_t)std::max<int64_t>(rows, 1) * sizeof(unsigned long long), st) != cudaSuccess)
    return set_error(FS_ENOMEM, "graph generator: row counters");
  cudaMemsetAsync(cnt, 0, (size_t)rows * sizeof(unsigned long long), st);
  visit(false, cnt, (int32_t*)nullptr);
  size_t tmp_bytes = 0;
  void* tmp = nullptr;
  int rc = 0;
  if (rows > 0) {
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt, cnt, rows, st);
    if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) rc = set_error(FS_ENOMEM, "graph generator: scan scratch");
    if (!rc) cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, cnt, cnt, rows, st);
    cudaFreeAsync(tmp, st);
  }
  if (!rc) k_offsets_init<<<grid, 256, 0, st>>>(row_offsets, cnt, rows);
  int64_t e = 0;
  if (!rc && (cudaMemcpyAsync(&e, row_offsets + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess))
    rc = set_error(FS_ECUDA, "graph generator: edge count readback");
  *num_edges = e;
  if (!rc && col) {
    if (e > col_capacity) {
      rc = set_error(FS_EINVAL, "graph generator: %lld edges exceed col capacity %lld", (long long)e,
                     (long long)col_capacity);
    } else {
      k_cursor_init<<<grid, 256, 0, st>>>(cnt, row_offsets, rows);
      visit(true, cnt, col);
      // sort each row: row blocks of < 2^31 entries (CUB's int item counts)
      int32_t* alt = nullptr;
      std::vector<int64_t> ro_h((size_t)rows + 1);
      if (cudaMemcpyAsync(ro_h.data(), row_offsets, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st) !=
              cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
        rc = set_error(FS_ECUDA, "graph generator: offsets readback");
      const int64_t kBlock = (int64_t)1 << 30;
      if (!rc && e > 0 && cudaMallocAsync(&alt, (size_t)std::min<int64_t>(e, kBlock + 1) * 4 + 16, st) != cudaSuccess)
        rc = set_error(FS_ENOMEM, "graph generator: sort buffer");
      for (int64_t r0 = 0; !rc && r0 < rows;) {
        int64_t r1 = r0 + 1;
        {  // largest r1 with ro[r1] - ro[r0] <= kBlock (a single larger row is impossible: N < 2^31)
          int64_t lo_ = r0 + 1, hi_ = rows;
          while (lo_ < hi_) {
            const int64_t mid = (lo_ + hi_ + 1) / 2;
            if (ro_h[mid] - ro_h[r0] <= kBlock) lo_ = mid; else hi_ = mid - 1;
          }
          r1 = lo_;
        }
        const int64_t items = ro_h[r1] - ro_h[r0];
        if (items > 1) {
          cub::DoubleBuffer<int32_t> keys(col + ro_h[r0], alt);
          // segment offsets relative to the block: shift by ro[r0]
          int64_t* seg = nullptr;
          if (cudaMallocAsync(&seg, (size_t)(r1 - r0 + 1) * sizeof(int64_t), st) != cudaSuccess) {
            rc = set_error(FS_ENOMEM, "graph generator: segment offsets");
            break;
          }
          std::vector<int64_t> segh((size_t)(r1 - r0 + 1));
          for (int64_t r = r0; r <= r1; ++r) segh[(size_t)(r - r0)] = ro_h[(size_t)r] - ro_h[(size_t)r0];
          cudaMemcpyAsync(seg, segh.data(), segh.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st);
          size_t sb = 0;
          cub::DeviceSegmentedSort::SortKeys(nullptr, sb, keys, (int)items, (int)(r1 - r0), seg, seg + 1, st);
          void* stmp = nullptr;
          if (cudaMallocAsync(&stmp, sb, st) != cudaSuccess) {
            rc = set_error(FS_ENOMEM, "graph generator: sort scratch");
          } else {
            cub::DeviceSegmentedSort::SortKeys(stmp, sb, keys, (int)items, (int)(r1 - r0), seg, seg + 1, st);
            if (keys.Current() != col + ro_h[r0])
              cudaMemcpyAsync(col + ro_h[r0], keys.Current(), (size_t)items * 4, cudaMemcpyDeviceToDevice, st);
            cudaFreeAsync(stmp, st);
          }
          cudaStreamSynchronize(st);  // segh lives on the host stack frame
          cudaFreeAsync(seg, st);
        }
        r0 = r1;
      }
      if (alt) cudaFreeAsync(alt, st);
    }
  }
  cudaFreeAsync(cnt, st);
  if (!rc) {
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) rc = set_error(FS_ECUDA, "graph generator: %s", cudaGetErrorString(err));
  }
  return rc;
}

static int gen_grid(int64_t work) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = std::max(1, fs_device_sm_count(dev));
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)sms * 16));
}

}  // namespace fs

using namespace fs;

extern "C" int fs_gen_barabasi_albert(int64_t n, int32_t m, uint64_t seed, int64_t row_lo, int64_t row_hi,
                                      int64_t* row_offsets, int32_t* col, int64_t col_capacity, int64_t* num_edges,
                                      void* stream) {
  if (n < 2 || n > 2147483647LL) return set_error(FS_EINVAL, "fs_gen_barabasi_albert: need 2 <= N <= 2^31-1");
  if (m < 1 || m >= n || m > kBaMaxM)
    return set_error(FS_EINVAL, "fs_gen_barabasi_albert: need 1 <= m < N, m <= %d (got m=%d)", kBaMaxM, m);
  if (row_lo < 0 || row_hi < row_lo || row_hi > n) return set_error(FS_EINVAL, "fs_gen_barabasi_albert: bad row range");
  if (!row_offsets || !num_edges) return set_error(FS_EINVAL, "fs_gen_barabasi_albert: null output");
  cudaStream_t st = (cudaStream_t)stream;
  BaSpec s{n, m, (int64_t)m * (m - 1) + (m == 1 ? 1 : 0), avalanche(seed ^ 0xBA5EBA11ull)};
  const int64_t slots = (n - m) * (int64_t)m;
  int32_t* tgt = nullptr;
  int* pending = nullptr;
  if (cudaMallocAsync(&tgt, (size_t)std::max<int64_t>(slots, 1) * 4, st) != cudaSuccess ||
      cudaMallocAsync(&pending, sizeof(int), st) != cudaSuccess)
    return set_error(FS_ENOMEM, "fs_gen_barabasi_albert: slot table");
  cudaMemsetAsync(tgt, 0xFF, (size_t)slots * 4, st);
  const int grid = gen_grid(n - m);
  int rc = 0;
  for (int sweep = 0; sweep < 100000; ++sweep) {
    int h = 0;
    cudaMemsetAsync(pending, 0, sizeof(int), st);
    k_ba_resolve<<<grid, 256, 0, st>>>(s, tgt, pending);
    if (cudaMemcpyAsync(&h, pending, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = set_error(FS_ECUDA, "k_ba_resolve: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (!h) break;
  }
  if (!rc) {
    const int64_t edges_und = slots + (int64_t)m * (m - 1) / 2;
    const int eg = gen_grid(edges_und);
    rc = assemble_rows(row_hi - row_lo, row_offsets, col, col_capacity, num_edges, st, gen_grid(row_hi - row_lo + 1),
                       [&](bool fill, unsigned long long* cur, int32_t* c) {
                         if (fill) k_ba_rows<true><<<eg, 256, 0, st>>>(s, tgt, row_lo, row_hi, cur, c);
                         else k_ba_rows<false><<<eg, 256, 0, st>>>(s, tgt, row_lo, row_hi, cur, c);
                       });
  }
  cudaFreeAsync(tgt, st);
  cudaFreeAsync(pending, st);
  cudaStreamSynchronize(st);
  return rc;
}

extern "C" int fs_gen_erdos_renyi(int64_t n, double d_avg, uint64_t seed, int64_t row_lo, int64_t row_hi,
                                  int64_t* row_offsets, int32_t* col, int64_t col_capacity, int64_t* num_edges,
                                  void* stream) {
  if (n < 2 || n > 2147483647LL) return set_error(FS_EINVAL, "fs_gen_erdos_renyi: need 2 <= N <= 2^31-1");
  if (!(d_avg >= 0.0)) return set_error(FS_EINVAL, "fs_gen_erdos_renyi: d_avg must be >= 0");
  if (row_lo < 0 || row_hi < row_lo || row_hi > n) return set_error(FS_EINVAL, "fs_gen_erdos_renyi: bad row range");
  if (!row_offsets || !num_edges) return set_error(FS_EINVAL, "fs_gen_erdos_renyi: null output");
  cudaStream_t st = (cudaStream_t)stream;
  const double p = std::min(d_avg / (double)(n - 1), 1.0);  // R/graph.py:264
  ErSpec s{};
  s.n = n;
  s.pairs = (unsigned long long)n * (unsigned long long)(n - 1) / 2ull;
  s.complete = p >= 1.0;
  s.log1mp = std::log1p(-p);
  s.key = avalanche(seed ^ 0xE5D05E11ull);
  // ~1024 expected edges per chunk (or the whole range when p == 0)
  const double per = p > 0.0 ? std::max(1.0, std::floor(1024.0 / p)) : (double)s.pairs;
  s.chunk = (unsigned long long)std::min<double>(per, (double)s.pairs);
  if (s.chunk == 0) s.chunk = 1;
  s.chunks = p > 0.0 ? (s.pairs + s.chunk - 1) / s.chunk : 0;
  const int eg = gen_grid((int64_t)std::min<unsigned long long>(s.chunks, 1ull << 40));
  return assemble_rows(row_hi - row_lo, row_offsets, col, col_capacity, num_edges, st, gen_grid(row_hi - row_lo + 1),
                       [&](bool fill, unsigned long long* cur, int32_t* c) {
                         if (s.chunks == 0) return;
                         if (fill) k_er_rows<true><<<eg, 256, 0, st>>>(s, row_lo, row_hi, cur, c);
                         else k_er_rows<false><<<eg, 256, 0, st>>>(s, row_lo, row_hi, cur, c);
                       });
}
