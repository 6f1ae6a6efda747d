// fs_analysis.cu — device-side trajectory records and ensemble analysis
// (SURVEY.md §8f row 4): the consumers of the engine's per-step
// (clock, counts) log.
//
//   fs_traj_records        make_record (R/trajectory.py:31-61) for a batch of
//                          trials: last-value interpolation of each trial's
//                          log onto the uniform grid, fractions = f64(count)
//                          / f64(N), peak_I / its grid time / final_R.
//                          Stored grid-major ([t][g][c]): the reference's
//                          fractions are `counts[idx].T / N`, a Fortran-
//                          order (C, G) array, and numpy's reductions over
//                          it (np.mean in fidelity's l2) follow that order.
//   fs_ensemble_mean       A.mean(axis=0) over runs (R/analysis.py:137-138):
//                          numpy reduces the outer axis row by row, so the
//                          sum is sequential in run order, then / runs.
//   fs_column_quantiles    np.quantile(..., axis=0), method "linear"
//                          (quantile_band R/analysis.py:141-148,
//                          _percentile_ci :160-162): per column a shared
//                          memory bitonic sort of a total-order key, then
//                          numpy's _lerp with the host-computed indices.
//   fs_bootstrap_metrics   the resampling loop of `fidelity`
//                          (R/analysis.py:192-256): per resample r the
//                          weighted means (w = multinomial count / n) of
//                          both ensembles, and from them l_inf, l2,
//                          err_peak_i, err_final_r, plus w·per_run_peak and
//                          w·per_run_final.  One CTA per 8 resamples; the
//                          ensembles (runs x C x G f64) stay L2 resident.
//   fs_run_deviation       |max_g A[i, I, g] - ref_peak| and
//                          |A[i, R, G-1] - ref_final| per run.
//
// All of it is f64 with every product and sum individually rounded
// (-fmad=false).  The records, means, quantile interpolation and per-run
// deviations are bit-identical to numpy; the bootstrap means are a
// matrix product that numpy hands to BLAS (blocked, FMA), so those agree
// to rounding (tests/test_analysis.py states the tolerance).
#include <cuda_runtime.h>
#include <cstdint>
#include <cmath>
#include "fs_internal.h"
#include "../../include/flashspread.h"

namespace fs {

constexpr int kAnaThreads = 256;
constexpr int kBootRB = 8;        // resamples per CTA
constexpr int kMaxQuant = 8;
constexpr int kMaxSort = 16384;   // 128 KB of keys

struct QuantSpec {
  int nq;
  long long prev[kMaxQuant], next[kMaxQuant];
  double gamma[kMaxQuant], one_minus[kMaxQuant];
};

__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  // numpy argmax: first maximum; a NaN is the maximum (first NaN wins)
  const bool nan1 = v != v, nan2 = v2 != v2;
  if (nan1) { if (nan2 && i2 < i) i = i2; return; }
  if (nan2 || v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__global__ void __launch_bounds__(kAnaThreads) k_traj_records(
    const double* __restrict__ times, const int64_t* __restrict__ counts, const int64_t* __restrict__ lens,
    int64_t max_steps, int ncomp, const double* __restrict__ grid, int G, double nn,
    int i_idx, int r_idx, double* __restrict__ frac, double* __restrict__ summary) {
  const int64_t t = blockIdx.x;
  const int64_t len = lens[t];
  const double* tt = times + t * max_steps;
  const int64_t* cc = counts + t * max_steps * ncomp;
  double* ff = frac + t * (int64_t)ncomp * G;
  double best = -INFINITY;
  int best_i = G;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const double x = grid[g];
    // searchsorted(times, x, side="right") - 1, clipped to [0, len-1]
    int64_t lo = 0, hi = len;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (tt[mid] <= x) lo = mid + 1; else hi = mid;
    }
    int64_t at = lo - 1;
    at = at < 0 ? 0 : (at > len - 1 ? len - 1 : at);
    for (int c = 0; c < ncomp; ++c) {
      const double v = __ddiv_rn((double)cc[at * ncomp + c], nn);
      ff[(int64_t)g * ncomp + c] = v;
      if (c == i_idx) argmax_merge(best, best_i, v, g);
    }
  }
  if (i_idx < 0 && r_idx < 0) return;
  __shared__ double sv[kAnaThreads / 32];
  __shared__ int si[kAnaThreads / 32];
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, best_i, o);
    argmax_merge(best, best_i, v2, i2);
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = best_i; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)blockDim.x / 32; ++w) argmax_merge(best, best_i, sv[w], si[w]);
    if (i_idx >= 0) {
      summary[t * 3 + 0] = best;
      summary[t * 3 + 1] = grid[best_i];
    }
    if (r_idx >= 0) summary[t * 3 + 2] = ff[(int64_t)(G - 1) * ncomp + r_idx];
  }
}

__global__ void __launch_bounds__(kAnaThreads) k_col_mean(const double* __restrict__ x, int64_t runs, int64_t cols,
                                                          double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double s = x[j];
  for (int64_t i = 1; i < runs; ++i) s = __dadd_rn(s, x[i * cols + j]);
  out[j] = __ddiv_rn(s, (double)runs);
}

// total order on doubles (NaN above +inf, as numpy's sort places it)
__device__ __forceinline__ unsigned long long dkey(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  if (v != v) return 0xFFFFFFFFFFFFFFFEull;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
  if (k == 0xFFFFFFFFFFFFFFFEull) return __longlong_as_double(0x7FF8000000000000ll);
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

__global__ void __launch_bounds__(1024) k_col_quantiles(const double* __restrict__ x, int64_t n, int64_t row_stride,
                                                        int64_t col_stride, int pow2, QuantSpec q,
                                                        double* __restrict__ out, int64_t ncols) {
  extern __shared__ unsigned long long keys[];
  const int64_t col = blockIdx.x;
  const double* xc = x + col * col_stride;
  for (int i = threadIdx.x; i < pow2; i += blockDim.x)
    keys[i] = i < n ? dkey(xc[(int64_t)i * row_stride]) : 0xFFFFFFFFFFFFFFFFull;
  __syncthreads();
  for (int k = 2; k <= pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < pow2; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const unsigned long long a = keys[i], b = keys[p];
          const bool up = (i & k) == 0;
          if ((a > b) == up) { keys[i] = b; keys[p] = a; }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x < q.nq) {
    const int s = threadIdx.x;
    const long long pi = q.prev[s] < 0 ? n - 1 : q.prev[s];
    const long long ni = q.next[s] < 0 ? n - 1 : q.next[s];
    const double a = dval(keys[pi]), b = dval(keys[ni]);
    const double d = __dsub_rn(b, a);
    double r = q.gamma[s] >= 0.5 ? __dsub_rn(b, __dmul_rn(d, q.one_minus[s]))
                                 : __dadd_rn(a, __dmul_rn(d, q.gamma[s]));
    const double last = dval(keys[n - 1]);
    if (last != last) r = last;  // slices holding a NaN give NaN
    out[(int64_t)s * ncols + col] = r;
  }
}

__global__ void k_boot_weights(const int64_t* __restrict__ cnt, int64_t total, double n, double* __restrict__ w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = __ddiv_rn((double)cnt[i], n);
}

struct BootParams {
  const double *a, *b, *wa, *wb, *prp, *prf;
  int64_t na, nb, resamples, K;
  int G, i_idx, r_idx;
  double* samples;  // [6][resamples]
};

__device__ __forceinline__ double block_reduce(double v, bool is_max, double* sh) {
  for (int o = 16; o; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : __dadd_rn(v, u);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : (is_max ? -INFINITY : 0.0);
    for (int o = 16; o; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmax(v, u) : __dadd_rn(v, u);
    }
  }
  return v;
}

__global__ void __launch_bounds__(kAnaThreads) k_boot_metrics(BootParams p) {
  const int64_t r0 = (int64_t)blockIdx.x * kBootRB;
  const int nr = (int)(p.resamples - r0 < kBootRB ? p.resamples - r0 : kBootRB);
  double lmax[kBootRB], ssq[kBootRB], pa[kBootRB], pb[kBootRB];
#pragma unroll
  for (int s = 0; s < kBootRB; ++s) { lmax[s] = 0.0; ssq[s] = 0.0; pa[s] = -INFINITY; pb[s] = -INFINITY; }
  __shared__ double fin[2][kBootRB];
  __shared__ double red[kAnaThreads / 32];
  const int64_t i_lo = (int64_t)p.i_idx * p.G, i_hi = i_lo + p.G;
  const int64_t r_last = (int64_t)p.r_idx * p.G + p.G - 1;
  for (int64_t j = threadIdx.x; j < p.K; j += blockDim.x) {
    double ma[kBootRB], mb[kBootRB];
#pragma unroll
    for (int s = 0; s < kBootRB; ++s) { ma[s] = 0.0; mb[s] = 0.0; }
    for (int64_t i = 0; i < p.na; ++i) {
      const double v = p.a[i * p.K + j];
#pragma unroll
      for (int s = 0; s < kBootRB; ++s)
        if (s < nr) ma[s] = __dadd_rn(ma[s], __dmul_rn(p.wa[(r0 + s) * p.na + i], v));
    }
    for (int64_t i = 0; i < p.nb; ++i) {
      const double v = p.b[i * p.K + j];
#pragma unroll
      for (int s = 0; s < kBootRB; ++s)
        if (s < nr) mb[s] = __dadd_rn(mb[s], __dmul_rn(p.wb[(r0 + s) * p.nb + i], v));
    }
    const bool in_i = p.i_idx >= 0 && j >= i_lo && j < i_hi;
#pragma unroll
    for (int s = 0; s < kBootRB; ++s) {
      const double d = __dsub_rn(ma[s], mb[s]);
      lmax[s] = fmax(lmax[s], fabs(d));
      ssq[s] = __dadd_rn(ssq[s], __dmul_rn(d, d));
      if (in_i) { pa[s] = fmax(pa[s], ma[s]); pb[s] = fmax(pb[s], mb[s]); }
      if (p.r_idx >= 0 && j == r_last) { fin[0][s] = ma[s]; fin[1][s] = mb[s]; }
    }
  }
#pragma unroll
  for (int s = 0; s < kBootRB; ++s) {
    if (s >= nr) break;
    const double l = block_reduce(lmax[s], true, red);
    const double q = block_reduce(ssq[s], false, red);
    const double xa = block_reduce(pa[s], true, red);
    const double xb = block_reduce(pb[s], true, red);
    if (threadIdx.x == 0) {
      const int64_t r = r0 + s;
      p.samples[0 * p.resamples + r] = l;
      p.samples[1 * p.resamples + r] = sqrt(__ddiv_rn(q, (double)p.K));
      if (p.i_idx >= 0) p.samples[2 * p.resamples + r] = fabs(__dsub_rn(xa, xb));
    }
  }
  __syncthreads();
  // w · per-run deviations: warp s handles resample s
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < nr) {
    const int64_t r = r0 + w;
    double sp = 0.0, sf = 0.0;
    for (int64_t i = lane; i < p.na; i += 32) {
      const double wi = p.wa[r * p.na + i];
      if (p.prp) sp = __dadd_rn(sp, __dmul_rn(wi, p.prp[i]));
      if (p.prf) sf = __dadd_rn(sf, __dmul_rn(wi, p.prf[i]));
    }
    for (int o = 16; o; o >>= 1) {
      sp = __dadd_rn(sp, __shfl_xor_sync(0xffffffffu, sp, o));
      sf = __dadd_rn(sf, __shfl_xor_sync(0xffffffffu, sf, o));
    }
    if (lane == 0) {
      if (p.r_idx >= 0) p.samples[3 * p.resamples + r] = fabs(__dsub_rn(fin[0][w], fin[1][w]));
      if (p.prp) p.samples[4 * p.resamples + r] = sp;
      if (p.prf) p.samples[5 * p.resamples + r] = sf;
    }
  }
}

__global__ void __launch_bounds__(128) k_run_deviation(const double* __restrict__ a, int64_t runs, int64_t K, int G,
                                                       int i_idx, int r_idx, double ref_peak, double ref_final,
                                                       double* __restrict__ peak_dev, double* __restrict__ final_dev) {
  const int64_t i = blockIdx.x;
  const double* row = a + i * K;
  __shared__ double red[4];
  if (i_idx >= 0) {
    double m = -INFINITY;
    bool nan = false;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
      const double v = row[(int64_t)i_idx * G + g];
      nan |= v != v;
      m = fmax(m, v);
    }
    nan = __syncthreads_or(nan);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)blockDim.x / 32; ++w) m = fmax(m, red[w]);
      if (nan) m = __longlong_as_double(0x7FF8000000000000ll);  // numpy max propagates NaN
      peak_dev[i] = fabs(__dsub_rn(m, ref_peak));
    }
  }
  if (r_idx >= 0 && threadIdx.x == 0) final_dev[i] = fabs(__dsub_rn(row[(int64_t)r_idx * G + G - 1], ref_final));
}

static int launch_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(FS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace fs

using namespace fs;

extern "C" int fs_traj_records(const double* times, const int64_t* counts, const int64_t* lens, int64_t trials,
                               int64_t max_steps, int32_t ncomp, const double* grid, int32_t grid_points,
                               int64_t num_nodes, int32_t i_idx, int32_t r_idx, double* fractions, double* summary,
                               void* stream) {
  if (trials < 0 || max_steps < 1 || ncomp < 1 || grid_points < 1 || num_nodes < 1)
    return set_error(FS_EINVAL, "fs_traj_records: bad sizes");
  if (i_idx >= ncomp || r_idx >= ncomp) return set_error(FS_EINVAL, "fs_traj_records: compartment index");
  if (trials == 0) return 0;
  if (!times || !counts || !lens || !grid || !fractions || ((i_idx >= 0 || r_idx >= 0) && !summary))
    return set_error(FS_EINVAL, "fs_traj_records: null pointer");
  k_traj_records<<<(unsigned)trials, kAnaThreads, 0, (cudaStream_t)stream>>>(
      times, counts, lens, max_steps, ncomp, grid, grid_points, (double)num_nodes, i_idx, r_idx, fractions,
      summary);
  return launch_check("k_traj_records");
}

extern "C" int fs_ensemble_mean(const double* x, int64_t runs, int64_t cols, double* out, void* stream) {
  if (runs < 1 || cols < 0) return set_error(FS_EINVAL, "fs_ensemble_mean: empty ensemble");
  if (cols == 0) return 0;
  if (!x || !out) return set_error(FS_EINVAL, "fs_ensemble_mean: null pointer");
  k_col_mean<<<(unsigned)((cols + kAnaThreads - 1) / kAnaThreads), kAnaThreads, 0, (cudaStream_t)stream>>>(
      x, runs, cols, out);
  return launch_check("k_col_mean");
}

extern "C" int fs_column_quantiles(const double* x, int64_t n, int64_t ncols, int64_t row_stride, int64_t col_stride,
                                   int32_t nq, const int64_t* prev, const int64_t* next, const double* gamma,
                                   double* out, void* stream) {
  if (n < 1 || n > kMaxSort) return set_error(FS_EINVAL, "fs_column_quantiles: need 1 <= n <= %d (got %lld)",
                                              kMaxSort, (long long)n);
  if (nq < 1 || nq > kMaxQuant) return set_error(FS_EINVAL, "fs_column_quantiles: 1..%d quantiles", kMaxQuant);
  if (ncols == 0) return 0;
  if (!x || !out || !prev || !next || !gamma) return set_error(FS_EINVAL, "fs_column_quantiles: null pointer");
  QuantSpec q{};
  q.nq = nq;
  for (int s = 0; s < nq; ++s) {
    if (prev[s] < -1 || prev[s] >= n || next[s] < -1 || next[s] >= n)
      return set_error(FS_EINVAL, "fs_column_quantiles: index out of range");
    q.prev[s] = prev[s];
    q.next[s] = next[s];
    q.gamma[s] = gamma[s];
    q.one_minus[s] = 1.0 - gamma[s];
  }
  int pow2 = 1;
  while (pow2 < n) pow2 <<= 1;
  const size_t smem = (size_t)pow2 * sizeof(unsigned long long);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(k_col_quantiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return set_error(FS_ECUDA, "fs_column_quantiles: shared memory opt-in");
  const int threads = pow2 >= 1024 ? 1024 : (pow2 < 32 ? 32 : pow2);
  k_col_quantiles<<<(unsigned)ncols, threads, smem, (cudaStream_t)stream>>>(x, n, row_stride, col_stride, pow2, q, out,
                                                                            ncols);
  return launch_check("k_col_quantiles");
}

extern "C" int fs_bootstrap_metrics(const double* a, int64_t na, const double* b, int64_t nb, int32_t ncomp,
                                    int32_t grid_points, const int64_t* counts_a, const int64_t* counts_b,
                                    int64_t resamples, int32_t i_idx, int32_t r_idx, const double* per_run_peak,
                                    const double* per_run_final, double* weights_scratch, double* samples,
                                    void* stream) {
  if (na < 1 || nb < 1 || ncomp < 1 || grid_points < 1 || resamples < 1)
    return set_error(FS_EINVAL, "fs_bootstrap_metrics: bad sizes");
  if (i_idx >= ncomp || r_idx >= ncomp) return set_error(FS_EINVAL, "fs_bootstrap_metrics: compartment index");
  if (!a || !b || !counts_a || !counts_b || !weights_scratch || !samples)
    return set_error(FS_EINVAL, "fs_bootstrap_metrics: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  double* wa = weights_scratch;
  double* wb = weights_scratch + resamples * na;
  k_boot_weights<<<296, 256, 0, st>>>(counts_a, resamples * na, (double)na, wa);
  k_boot_weights<<<296, 256, 0, st>>>(counts_b, resamples * nb, (double)nb, wb);
  if (int rc = launch_check("k_boot_weights")) return rc;
  BootParams p{a, b, wa, wb, i_idx >= 0 ? per_run_peak : nullptr, r_idx >= 0 ? per_run_final : nullptr,
               na, nb, resamples, (int64_t)ncomp * grid_points, grid_points, i_idx, r_idx, samples};
  k_boot_metrics<<<(unsigned)((resamples + kBootRB - 1) / kBootRB), kAnaThreads, 0, st>>>(p);
  return launch_check("k_boot_metrics");
}

extern "C" int fs_run_deviation(const double* a, int64_t runs, int32_t ncomp, int32_t grid_points, int32_t i_idx,
                                int32_t r_idx, double ref_peak, double ref_final, double* peak_dev, double* final_dev,
                                void* stream) {
  if (runs < 1 || ncomp < 1 || grid_points < 1) return set_error(FS_EINVAL, "fs_run_deviation: bad sizes");
  if (i_idx >= ncomp || r_idx >= ncomp) return set_error(FS_EINVAL, "fs_run_deviation: compartment index");
  if (!a || (i_idx >= 0 && !peak_dev) || (r_idx >= 0 && !final_dev))
    return set_error(FS_EINVAL, "fs_run_deviation: null pointer");
  k_run_deviation<<<(unsigned)runs, 128, 0, (cudaStream_t)stream>>>(a, runs, (int64_t)ncomp * grid_points,
                                                                     grid_points, i_idx, r_idx, ref_peak, ref_final,
                                                                     peak_dev, final_dev);
  return launch_check("k_run_deviation");
}
