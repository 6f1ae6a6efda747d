// fs_markov.cu — the Markovian tau-leaping engine (R/markov.py) on sm_100a:
// SURVEY.md §8f row 3, the paper's companion engine.
//
// One reference markov_step (R/markov.py:143-181) is two launches, captured
// in a CUDA graph per batch:
//   k_mk_sum     fold the previous step's pushes into the per-node
//                infectious in-neighbour counts, rate = beta * count * w (S)
//                or the exponential holding rate, f64 rates[N], max by u64
//                atomicMax (rates >= 0: bits order like values), and their
//                sum in numpy's pairwise order (leaves of <= 128 with 8
//                interleaved accumulators, then the tree), bit-identical to
//                the reference's state.rates.sum(); the last CTA sets
//                tau = min(theta N / total, p_max / max, tau_max)
//                (R/markov.py:149-154) and the clock;
//   k_mk_fire    u < -expm1(-rate * tau) on the reference's uniforms, state
//                transitions, count deltas (last-CTA fold into the scalars
//                and the per-step log) and +-1 pushes along the outgoing CSR
//                for every node whose infectious status changed — the
//                reference's Inertial mode (R/markov.py:122-140), exact since
//                counts are integers, so Control / Inertial switching
//                (R/markov.py:168-176) never changes a bit.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstring>
#include <vector>
#include "fs_device.cuh"
#include "fs_internal.h"

namespace fs {

constexpr uint32_t kMkBias = 0x8000u;  // pending delta d stored as d + 0x8000
constexpr int kMkLeafBlock = 32;       // leaves summed per CTA of k_mk_leaves (<= 32 * 128 rates)
constexpr int kMkLvl = 8;              // max height of a block-local subtree (32 leaves: 6)

struct MkScalars {
  double clock;
  double tau;            // tau of the step in flight
  int64_t step;
  unsigned long long max_bits;  // max rate (f64 bits) of the current rates
  int64_t counts[FS_MAX_COMPARTMENTS];
  unsigned long long delta[FS_MAX_COMPARTMENTS];  // this step's count deltas (two's complement)
  unsigned int ticket;      // k_mk_fire's last-CTA election
  unsigned int sum_ticket;  // k_mk_sum's
};

struct MkParams {
  int64_t n;
  const int64_t* ro;        // incoming CSR (count init)
  const int32_t* col;
  const int64_t* out_ro;    // outgoing CSR (pushes)
  const int32_t* out_col;
  int32_t* states;
  double* rates;
  uint16_t* cnt;
  uint32_t* pend[2];
  MkScalars* S;
  double* leaf_val;         // [nleaf + ninternal]
  const int64_t* leaf_lo;
  const int32_t* leaf_len;
  int64_t nleaf;
  const int32_t* tree_l;    // internal nodes ordered by level
  const int32_t* tree_r;
  const int32_t* tree_out;  // value slot of each internal node
  const int32_t* level_end; // prefix ends of each level in the internal list
  int nlevels;
  int root;
  // block-local part of the tree: leaf blocks of kMkLeafBlock leaves; the
  // internal nodes whose leaves all fall in one block, per block and level
  const int32_t* loc_l;
  const int32_t* loc_r;
  const int32_t* loc_out;
  const int32_t* blk_lvl;   // [nblocks][kMkLvl + 1] prefix offsets into loc_*, by level 1..kMkLvl
  int nblocks;
  double* log_clock;
  double* log_tau;
  int64_t* log_counts;
  int64_t log_cap;
  // model
  int M, edge_from, infectious;
  int succ[FS_MAX_COMPARTMENTS];
  double nodal_rate[FS_MAX_COMPARTMENTS];  // exponential rate, 0 when none
  int has_nodal[FS_MAX_COMPARTMENTS];
  double beta, w;
  double theta, p_max, tau_max;
  uint64_t seed;
};

__device__ __forceinline__ double mk_rate(const MkParams& p, int s, uint32_t c) {
  if (s == p.edge_from) return __dmul_rn(p.beta, __dmul_rn((double)c, p.w));  // beta * influence
  return p.has_nodal[s] ? p.nodal_rate[s] : 0.0;
}

__global__ void __launch_bounds__(256) k_mk_rates(const MkParams p) {
  const int par = (int)(p.S->step & 1);
  uint16_t* pend = reinterpret_cast<uint16_t*>(p.pend[par]);
  unsigned long long mx = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = p.cnt[i];
    const uint32_t d = pend[i];
    if (d != kMkBias) {
      c = c + d - kMkBias;
      p.cnt[i] = (uint16_t)c;
      pend[i] = (uint16_t)kMkBias;
    }
    const double r = mk_rate(p, p.states[i], c);
    p.rates[i] = r;
    const unsigned long long b = (unsigned long long)__double_as_longlong(r);
    mx = b > mx ? b : mx;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = v > mx ? v : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&p.S->max_bits, mx);
}

// One launch for the rates and their pairwise sum.  CTA b owns the block
// of kMkLeafBlock consecutive leaves of numpy's pairwise summation, i.e. a
// contiguous run of <= 4096 nodes: it folds their pending pushes, computes
// their f64 rates (written out for k_mk_fire, staged in shared memory),
// sums each leaf with 8 threads — one per interleaved accumulator, exactly
// numpy's order — and folds the internal nodes local to the block; the last
// CTA to finish folds the cross-block top of the tree level by level and
// sets tau = min(theta N / total, p_max / max, tau_max) and the clock.
__global__ void __launch_bounds__(256) k_mk_sum(const MkParams p) {
  __shared__ double a[kMkLeafBlock * 128];
  __shared__ double racc[kMkLeafBlock][8];
  __shared__ bool last;
  const int b = blockIdx.x, t = threadIdx.x;
  MkScalars* S = p.S;
  const int64_t L0 = (int64_t)b * kMkLeafBlock, L1 = min(L0 + kMkLeafBlock, p.nleaf);
  const int64_t lo = p.leaf_lo[L0];
  const int64_t hi = p.leaf_lo[L1 - 1] + p.leaf_len[L1 - 1];
  uint16_t* pend = reinterpret_cast<uint16_t*>(p.pend[(int)(S->step & 1)]);
  unsigned long long mx = 0ull;
  for (int64_t i = t; i < hi - lo; i += blockDim.x) {
    const int64_t v = lo + i;
    uint32_t c = p.cnt[v];
    const uint32_t d = pend[v];
    if (d != kMkBias) {
      c = c + d - kMkBias;
      p.cnt[v] = (uint16_t)c;
      pend[v] = (uint16_t)kMkBias;
    }
    const double r = mk_rate(p, p.states[v], c);
    p.rates[v] = r;
    a[i] = r;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(r);
    mx = bits > mx ? bits : mx;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = w > mx ? w : mx;
  }
  if ((t & 31) == 0 && mx) atomicMax(&S->max_bits, mx);
  __syncthreads();
  const int li = t >> 3, j = t & 7;
  const int64_t leaf = L0 + li;
  int n = 0, off = 0;
  if (leaf < L1) {
    n = p.leaf_len[leaf];
    off = (int)(p.leaf_lo[leaf] - lo);
    if (n >= 8) {  // accumulator j: a[j], a[j+8], ... up to n - n % 8
      double r = a[off + j];
      for (int i = 8; i < n - (n % 8); i += 8) r = __dadd_rn(r, a[off + i + j]);
      racc[li][j] = r;
    }
  }
  __syncthreads();
  if (leaf < L1 && j == 0) {
    double res;
    if (n < 8) {
      res = 0.0;
      for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[off + i]);
    } else {
      const double* r = racc[li];
      res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (int i = n - (n % 8); i < n; ++i) res = __dadd_rn(res, a[off + i]);
    }
    p.leaf_val[leaf] = res;
  }
  __syncthreads();
  const int32_t* lv = p.blk_lvl + (size_t)b * (kMkLvl + 1);
  for (int h = 0; h < kMkLvl; ++h) {
    for (int i = lv[h] + t; i < lv[h + 1]; i += blockDim.x)
      p.leaf_val[p.loc_out[i]] = __dadd_rn(p.leaf_val[p.loc_l[i]], p.leaf_val[p.loc_r[i]]);
    __syncthreads();
  }
  // the last CTA folds the top of the tree
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(&S->sum_ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  int start = 0;
  for (int lvl = 0; lvl < p.nlevels; ++lvl) {
    const int end = p.level_end[lvl];
    for (int i = start + t; i < end; i += blockDim.x)
      p.leaf_val[p.tree_out[i]] = __dadd_rn(__ldcg(&p.leaf_val[p.tree_l[i]]), __ldcg(&p.leaf_val[p.tree_r[i]]));
    __threadfence_block();
    __syncthreads();
    start = end;
  }
  if (t == 0) {
    const double total = p.n ? __ldcg(&p.leaf_val[p.root]) : 0.0;
    const double m = __longlong_as_double((long long)atomicAdd(&S->max_bits, 0ull));
    double tau;
    if (total <= 0.0 || m <= 0.0) {
      tau = p.tau_max;
    } else {
      // min(theta * N / total, p_max / max_rate, tau_max), left to right
      tau = __ddiv_rn(__dmul_rn(p.theta, (double)p.n), total);
      const double c2 = __ddiv_rn(p.p_max, m);
      if (c2 < tau) tau = c2;
      if (p.tau_max < tau) tau = p.tau_max;
    }
    S->tau = tau;
    S->clock = __dadd_rn(S->clock, tau);
    const int64_t slot = S->step % p.log_cap;
    p.log_clock[slot] = S->clock;
    p.log_tau[slot] = tau;
    S->max_bits = 0ull;  // next step maxes afresh
    S->sum_ticket = 0u;
  }
}

__device__ __forceinline__ void mk_push(const MkParams& p, int nxt, int32_t j, bool up) {
  uint32_t* dn = p.pend[nxt] + (j >> 1);
  const uint32_t one = 1u << (16 * (j & 1));
  if (up) atomicAdd(dn, one);
  else atomicSub(dn, one);
}

__global__ void __launch_bounds__(256) k_mk_fire(const MkParams p) {
  __shared__ int cnt[FS_MAX_COMPARTMENTS];
  __shared__ bool last;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < FS_MAX_COMPARTMENTS) cnt[threadIdx.x] = 0;
  __syncthreads();
  MkScalars* S = p.S;
  const int64_t step = S->step;
  const double tau = S->tau;
  const uint64_t key = splitmix_step_key(p.seed, (uint64_t)step);
  const int nxt = (int)((step & 1) ^ 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nround = (p.n + stride - 1) / stride * stride;  // whole warps stay converged
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nround; i += stride) {
    int push = 0;
    int64_t e0 = 0, e1 = 0;
    if (i < p.n) {
      const double r = p.rates[i];
      if (r > 0.0) {
        const double q = -expm1(__dmul_rn(-r, tau));  // -np.expm1(-rates * tau)
        const double u = splitmix_uniform(key, (uint64_t)i);
        if (u < q) {
          const int s = p.states[i];
          const int ns = p.succ[s];
          p.states[i] = ns;
          atomicAdd(&cnt[ns], 1);
          atomicAdd(&cnt[s], -1);
          if ((ns == p.infectious) != (s == p.infectious)) {
            push = ns == p.infectious ? 1 : -1;
            e0 = __ldg(p.out_ro + i);
            e1 = __ldg(p.out_ro + i + 1);
          }
        }
      }
    }
    const bool wide = push && (e1 - e0 > 32);
    if (push && !wide)
      for (int64_t e = e0; e < e1; ++e) mk_push(p, nxt, __ldg(p.out_col + e), push > 0);
    unsigned wides = __ballot_sync(0xffffffffu, wide);
    while (wides) {  // hubs: the warp pushes 32 edges per iteration
      const int src = __ffs(wides) - 1;
      wides &= wides - 1;
      const int64_t a0 = __shfl_sync(0xffffffffu, e0, src), a1 = __shfl_sync(0xffffffffu, e1, src);
      const bool up = __shfl_sync(0xffffffffu, push, src) > 0;
      for (int64_t e = a0 + lane; e < a1; e += 32) mk_push(p, nxt, __ldg(p.out_col + e), up);
    }
  }
  __syncthreads();
  if (threadIdx.x < p.M && cnt[threadIdx.x]) atomicAdd(&S->delta[threadIdx.x], (unsigned long long)(long long)cnt[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&S->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {  // last CTA: fold the step into the scalars and the log
    const int64_t slot = step % p.log_cap;
    for (int c = 0; c < p.M; ++c) {
      const unsigned long long d = atomicExch(&S->delta[c], 0ull);
      S->counts[c] += (int64_t)d;
      p.log_counts[slot * FS_MAX_COMPARTMENTS + c] = S->counts[c];
    }
    S->step = step + 1;
    S->ticket = 0u;
  }
}

// counts from scratch: infectious in-neighbours of every node
__global__ void k_mk_init_counts(const MkParams p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int64_t e = __ldg(p.ro + i), e1 = __ldg(p.ro + i + 1); e < e1; ++e)
      c += p.states[__ldg(p.col + e)] == p.infectious;
    p.cnt[i] = (uint16_t)c;
    if ((i & 1) == 0) {
      p.pend[0][i >> 1] = kMkBias | (kMkBias << 16);
      p.pend[1][i >> 1] = kMkBias | (kMkBias << 16);
    }
  }
}

// numpy pairwise-sum tree of n values (host): leaves left to right, internal
// nodes grouped by height so each level only reads finished values
struct PwTree {
  std::vector<int64_t> leaf_lo;
  std::vector<int32_t> leaf_len;
  std::vector<int32_t> l, r, out, level;
  int build(int64_t lo, int64_t n, int* height) {
    if (n <= 128) {
      leaf_lo.push_back(lo);
      leaf_len.push_back((int32_t)n);
      *height = 0;
      return -(int)leaf_lo.size();  // provisional: leaves get ids after counting
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    int hl = 0, hr = 0;
    const int a = build(lo, n2, &hl);
    const int b = build(lo + n2, n - n2, &hr);
    l.push_back(a);
    r.push_back(b);
    *height = std::max(hl, hr) + 1;
    level.push_back(*height);
    return (int)l.size() - 1;
  }
};

}  // namespace fs

using namespace fs;

struct fs_markov {
  int device = 0, sms = 0;
  MkParams p{};
  MkScalars* S = nullptr;
  double* vals = nullptr;
  int64_t* leaf_lo = nullptr;
  int32_t* leaf_len = nullptr;
  int32_t *tl = nullptr, *tr = nullptr, *tout = nullptr, *lend = nullptr;
  int32_t *loc_l = nullptr, *loc_r = nullptr, *loc_out = nullptr, *blk_lvl = nullptr;
  uint16_t* cnt = nullptr;
  uint32_t* pend[2] = {nullptr, nullptr};
  double* log_clock = nullptr;
  double* log_tau = nullptr;
  int64_t* log_counts = nullptr;
  int32_t steps_per_batch = 50;
  int grid = 1;
  cudaStream_t cap = nullptr;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};  // by step parity at batch start
  int64_t h_step = 0;
};

namespace {

#define MK_CUDA(call)                                                                                         \
  do {                                                                                                        \
    cudaError_t err__ = (call);                                                                               \
    if (err__ != cudaSuccess) return set_error(FS_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(err__), __FILE__, __LINE__); \
  } while (0)

// scratch from the device's stream-ordered pool, kept between engines (the
// renewal engine sets the pool's release threshold; fs_engine.cu)
template <typename T>
int mk_alloc(T** p, size_t n) {
  if (cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T), (cudaStream_t)0) != cudaSuccess)
    return set_error(FS_ENOMEM, "cudaMalloc(%zu)", n * sizeof(T));
  return 0;
}

int mk_launch(fs_markov* e, int nsteps, cudaStream_t st) {
  for (int k = 0; k < nsteps; ++k) {
    k_mk_sum<<<e->p.nblocks, 256, 0, st>>>(e->p);
    k_mk_fire<<<e->grid, 256, 0, st>>>(e->p);
    ++e->h_step;
  }
  MK_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace

extern "C" {

int fs_markov_create(const fs_graph* g, const fs_model* m, const fs_markov_config* c, int32_t* states, double* rates,
                     const fs_scalars* scal, int device, fs_markov** out) {
  if (!g || !m || !c || !states || !rates || !scal || !out) return set_error(FS_EINVAL, "null argument");
  *out = nullptr;
  {
    cudaMemPool_t pool;
    unsigned long long keep = ~0ull;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess)
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (g->num_nodes < 1) return set_error(FS_EINVAL, "empty graph");
  if (!g->out_row_offsets || !g->out_col_indices) return set_error(FS_EINVAL, "the Markov engine needs the outgoing CSR");
  if (g->d_max >= 32768) return set_error(FS_EINVAL, "in-degree %d beyond the count encoding", g->d_max);
  if (m->shedding != FS_SHED_CONSTANT) return set_error(FS_EINVAL, "the Markovian engine requires constant transmission");
  for (int i = 0; i < m->num_compartments; ++i)
    if (m->comp[i].hazard != FS_HZ_NONE && m->comp[i].hazard != FS_HZ_EXPONENTIAL)
      return set_error(FS_EINVAL, "the Markovian engine requires exponential holding times");
  if (!(c->p_max > 0.0 && c->p_max < 1.0) || !(c->theta > 0.0) || !(c->tau_max > 0.0) || c->steps_per_batch < 1)
    return set_error(FS_EINVAL, "bad Markov config");
  cudaSetDevice(device);
  fs_markov* e = new fs_markov();
  e->device = device;
  e->sms = fs_device_sm_count(device);
  e->steps_per_batch = c->steps_per_batch;
  const int64_t n = g->num_nodes;
  MkParams& p = e->p;
  p.n = n;
  p.ro = g->row_offsets;
  p.col = g->col_indices;
  p.out_ro = g->out_row_offsets;
  p.out_col = g->out_col_indices;
  p.states = states;
  p.rates = rates;
  p.M = m->num_compartments;
  p.edge_from = m->edge_from;
  p.infectious = m->infectious;
  for (int i = 0; i < FS_MAX_COMPARTMENTS; ++i) {
    p.succ[i] = i < m->num_compartments ? m->comp[i].succ : i;
    p.has_nodal[i] = i < m->num_compartments && m->comp[i].hazard == FS_HZ_EXPONENTIAL;
    p.nodal_rate[i] = p.has_nodal[i] ? m->comp[i].p0 : 0.0;
  }
  p.beta = m->beta;
  p.w = g->weights_uniform ? (double)g->uniform_weight : 1.0;
  p.theta = c->theta;
  p.p_max = c->p_max;
  p.tau_max = c->tau_max;
  p.seed = scal->seed;
  int rc = 0;
#define MK_TRY(x) do { rc = (x); if (rc) { fs_markov_destroy(e); return rc; } } while (0)
  // the pairwise tree of numpy's sum over n rates
  PwTree t;
  int h = 0;
  const int root0 = t.build(0, n, &h);
  const int nleaf = (int)t.leaf_lo.size(), nint = (int)t.l.size();
  auto vid = [&](int id) { return id < 0 ? (-id - 1) : nleaf + id; };  // leaves first, then internal
  // leaf span of every internal node (children precede parents in t.l / t.r)
  std::vector<int> first(nint), last(nint);
  auto span_lo = [&](int id) { return id < 0 ? (-id - 1) : first[id]; };
  auto span_hi = [&](int id) { return id < 0 ? (-id - 1) : last[id]; };
  for (int i = 0; i < nint; ++i) {
    first[i] = span_lo(t.l[i]);
    last[i] = span_hi(t.r[i]);
  }
  const int nblocks = (nleaf + kMkLeafBlock - 1) / kMkLeafBlock;
  std::vector<std::vector<int>> loc(nblocks * kMkLvl);
  std::vector<int> top;
  for (int i = 0; i < nint; ++i) {
    const int b0 = first[i] / kMkLeafBlock, b1 = last[i] / kMkLeafBlock;
    if (b0 == b1 && t.level[i] <= kMkLvl) loc[(size_t)b0 * kMkLvl + (t.level[i] - 1)].push_back(i);
    else top.push_back(i);
  }
  std::vector<int32_t> ll, lr, lo_, blv((size_t)nblocks * (kMkLvl + 1));
  for (int b = 0; b < nblocks; ++b) {
    blv[(size_t)b * (kMkLvl + 1)] = (int32_t)ll.size();
    for (int h = 0; h < kMkLvl; ++h) {
      for (int i : loc[(size_t)b * kMkLvl + h]) {
        ll.push_back(vid(t.l[i]));
        lr.push_back(vid(t.r[i]));
        lo_.push_back(nleaf + i);
      }
      blv[(size_t)b * (kMkLvl + 1) + h + 1] = (int32_t)ll.size();
    }
  }
  std::stable_sort(top.begin(), top.end(), [&](int a, int b) { return t.level[a] < t.level[b]; });
  const int ntop = (int)top.size();
  std::vector<int32_t> hl(ntop), hr(ntop), ho(ntop), lend;
  for (int k = 0; k < ntop; ++k) {
    const int i = top[k];
    hl[k] = vid(t.l[i]);
    hr[k] = vid(t.r[i]);
    ho[k] = nleaf + i;
    if (k + 1 == ntop || t.level[top[k + 1]] != t.level[i]) lend.push_back(k + 1);
  }
  p.nleaf = nleaf;
  p.nlevels = (int)lend.size();
  p.root = vid(root0);
  p.nblocks = nblocks;
  const int nloc = (int)ll.size();
  MK_TRY(mk_alloc(&e->loc_l, nloc));
  MK_TRY(mk_alloc(&e->loc_r, nloc));
  MK_TRY(mk_alloc(&e->loc_out, nloc));
  MK_TRY(mk_alloc(&e->blk_lvl, blv.size()));
  if (nloc) {
    MK_CUDA(cudaMemcpy(e->loc_l, ll.data(), nloc * sizeof(int32_t), cudaMemcpyHostToDevice));
    MK_CUDA(cudaMemcpy(e->loc_r, lr.data(), nloc * sizeof(int32_t), cudaMemcpyHostToDevice));
    MK_CUDA(cudaMemcpy(e->loc_out, lo_.data(), nloc * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  MK_CUDA(cudaMemcpy(e->blk_lvl, blv.data(), blv.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  p.loc_l = e->loc_l;
  p.loc_r = e->loc_r;
  p.loc_out = e->loc_out;
  p.blk_lvl = e->blk_lvl;
  MK_TRY(mk_alloc(&e->vals, (size_t)nleaf + nint));
  MK_TRY(mk_alloc(&e->leaf_lo, nleaf));
  MK_TRY(mk_alloc(&e->leaf_len, nleaf));
  MK_TRY(mk_alloc(&e->tl, ntop));
  MK_TRY(mk_alloc(&e->tr, ntop));
  MK_TRY(mk_alloc(&e->tout, ntop));
  MK_TRY(mk_alloc(&e->lend, lend.size()));
  MK_CUDA(cudaMemcpy(e->leaf_lo, t.leaf_lo.data(), nleaf * sizeof(int64_t), cudaMemcpyHostToDevice));
  MK_CUDA(cudaMemcpy(e->leaf_len, t.leaf_len.data(), nleaf * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (ntop) {
    MK_CUDA(cudaMemcpy(e->tl, hl.data(), ntop * sizeof(int32_t), cudaMemcpyHostToDevice));
    MK_CUDA(cudaMemcpy(e->tr, hr.data(), ntop * sizeof(int32_t), cudaMemcpyHostToDevice));
    MK_CUDA(cudaMemcpy(e->tout, ho.data(), ntop * sizeof(int32_t), cudaMemcpyHostToDevice));
    MK_CUDA(cudaMemcpy(e->lend, lend.data(), lend.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  p.leaf_val = e->vals;
  p.leaf_lo = e->leaf_lo;
  p.leaf_len = e->leaf_len;
  p.tree_l = e->tl;
  p.tree_r = e->tr;
  p.tree_out = e->tout;
  p.level_end = e->lend;
  // counts, pending deltas, scalars, log
  const size_t cap = (size_t)((n + 127) / 128) * 128;
  MK_TRY(mk_alloc(&e->cnt, cap));
  MK_TRY(mk_alloc(&e->pend[0], cap / 2));
  MK_TRY(mk_alloc(&e->pend[1], cap / 2));
  p.cnt = e->cnt;
  p.pend[0] = e->pend[0];
  p.pend[1] = e->pend[1];
  MK_TRY(mk_alloc(&e->S, 1));
  MkScalars s0{};
  s0.clock = scal->clock;
  s0.step = scal->step;
  for (int i = 0; i < FS_MAX_COMPARTMENTS; ++i) s0.counts[i] = scal->counts[i];
  MK_CUDA(cudaMemcpy(e->S, &s0, sizeof s0, cudaMemcpyHostToDevice));
  p.S = e->S;
  p.log_cap = std::max<int64_t>(256, 4 * (int64_t)c->steps_per_batch);
  MK_TRY(mk_alloc(&e->log_clock, p.log_cap));
  MK_TRY(mk_alloc(&e->log_tau, p.log_cap));
  MK_TRY(mk_alloc(&e->log_counts, (size_t)p.log_cap * FS_MAX_COMPARTMENTS));
  p.log_clock = e->log_clock;
  p.log_tau = e->log_tau;
  p.log_counts = e->log_counts;
  e->grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8));
  e->h_step = scal->step;
  const int ib = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8));
  k_mk_init_counts<<<ib, 256>>>(p);
  MK_CUDA(cudaGetLastError());
  MK_CUDA(cudaStreamCreateWithFlags(&e->cap, cudaStreamNonBlocking));
  MK_CUDA(cudaDeviceSynchronize());
#undef MK_TRY
  *out = e;
  return 0;
}

void fs_markov_destroy(fs_markov* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  for (auto& x : e->exec) if (x) cudaGraphExecDestroy(x);
  if (e->cap) cudaStreamDestroy(e->cap);
  void* ptrs[] = {e->S, e->vals, e->leaf_lo, e->leaf_len, e->tl, e->tr, e->tout, e->lend, e->loc_l, e->loc_r,
                  e->loc_out, e->blk_lvl, e->cnt, e->pend[0],
                  e->pend[1], e->log_clock, e->log_tau, e->log_counts};
  cudaDeviceSynchronize();  // nothing of this engine still in flight on any stream
  for (void* q : ptrs) if (q) cudaFreeAsync(q, (cudaStream_t)0);
  cudaStreamSynchronize((cudaStream_t)0);
  delete e;
}

int fs_markov_step(fs_markov* e, int32_t nsteps, void* stream) {
  if (!e || nsteps < 0) return set_error(FS_EINVAL, "bad arguments");
  MK_CUDA(cudaSetDevice(e->device));
  return mk_launch(e, nsteps, (cudaStream_t)stream);
}

int fs_markov_run_batch(fs_markov* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  MK_CUDA(cudaSetDevice(e->device));
  cudaGraphExec_t& ex = e->exec[0];
  const int64_t h0 = e->h_step;
  if (!ex) {
    cudaGraph_t graph = nullptr;
    MK_CUDA(cudaStreamBeginCapture(e->cap, cudaStreamCaptureModeThreadLocal));
    int rc = mk_launch(e, e->steps_per_batch, e->cap);
    cudaError_t err = cudaStreamEndCapture(e->cap, &graph);
    e->h_step = h0;
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (err != cudaSuccess) return set_error(FS_ECUDA, "graph capture: %s", cudaGetErrorString(err));
    err = cudaGraphInstantiate(&ex, graph, 0);
    cudaGraphDestroy(graph);
    if (err != cudaSuccess) return set_error(FS_ECUDA, "graph instantiate: %s", cudaGetErrorString(err));
  }
  MK_CUDA(cudaGraphLaunch(ex, (cudaStream_t)stream));
  e->h_step = h0 + e->steps_per_batch;
  return 0;
}

int fs_markov_get_scalars(fs_markov* e, fs_scalars* out, void* stream) {
  if (!e || !out) return set_error(FS_EINVAL, "null argument");
  MK_CUDA(cudaSetDevice(e->device));
  MkScalars s;
  MK_CUDA(cudaMemcpyAsync(&s, e->S, sizeof s, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  MK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  std::memset(out, 0, sizeof *out);
  out->clock = s.clock;
  out->tau_next = s.tau;
  out->step = s.step;
  out->seed = e->p.seed;
  out->last_max_rate = 0.0f;
  out->started = s.step > 0;
  for (int i = 0; i < FS_MAX_COMPARTMENTS; ++i) out->counts[i] = s.counts[i];
  return 0;
}

int fs_markov_set_scalars(fs_markov* e, const fs_scalars* in, void* stream) {
  if (!e || !in) return set_error(FS_EINVAL, "null argument");
  MK_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  MkScalars s{};
  s.clock = in->clock;
  s.tau = in->tau_next;
  s.step = in->step;
  for (int i = 0; i < FS_MAX_COMPARTMENTS; ++i) s.counts[i] = in->counts[i];
  MK_CUDA(cudaMemcpyAsync(e->S, &s, sizeof s, cudaMemcpyHostToDevice, st));
  e->p.seed = in->seed;
  e->h_step = in->step;
  for (auto& x : e->exec) if (x) { cudaGraphExecDestroy(x); x = nullptr; }  // the seed is baked into the graph
  // states may have been edited: rebuild the counts
  const int ib = (int)std::max<int64_t>(1, std::min<int64_t>((e->p.n + 255) / 256, (int64_t)e->sms * 8));
  k_mk_init_counts<<<ib, 256, 0, st>>>(e->p);
  MK_CUDA(cudaGetLastError());
  MK_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int fs_markov_read_log(fs_markov* e, int64_t first_step, int32_t n, double* clocks, double* taus, int64_t* counts,
                       void* stream) {
  if (!e || n < 0 || n > e->p.log_cap) return set_error(FS_EINVAL, "bad log request");
  MK_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<double> lc(e->p.log_cap), lt(e->p.log_cap);
  std::vector<int64_t> lk((size_t)e->p.log_cap * FS_MAX_COMPARTMENTS);
  MK_CUDA(cudaMemcpyAsync(lc.data(), e->log_clock, lc.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  MK_CUDA(cudaMemcpyAsync(lt.data(), e->log_tau, lt.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  MK_CUDA(cudaMemcpyAsync(lk.data(), e->log_counts, lk.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  MK_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i) {
    const int64_t slot = (first_step + i) % e->p.log_cap;
    if (clocks) clocks[i] = lc[slot];
    if (taus) taus[i] = lt[slot];
    if (counts)
      for (int c = 0; c < e->p.M; ++c) counts[(size_t)i * e->p.M + c] = lk[slot * FS_MAX_COMPARTMENTS + c];
  }
  return 0;
}

int fs_markov_refresh_rates(fs_markov* e, void* stream) {
  // rates of the current states and influence (what R/markov.py:178 leaves in
  // state.rates after a step); the next step recomputes the same values
  if (!e) return set_error(FS_EINVAL, "null engine");
  MK_CUDA(cudaSetDevice(e->device));
  k_mk_rates<<<e->grid, 256, 0, (cudaStream_t)stream>>>(e->p);
  MK_CUDA(cudaGetLastError());
  return 0;
}

int fs_markov_influence(fs_markov* e, double* out, void* stream) {
  // influence = count * w (R/markov.py:68-81 for uniform weights), after the
  // pending pushes are folded: computed from the current states
  if (!e || !out) return set_error(FS_EINVAL, "null argument");
  MK_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int ib = (int)std::max<int64_t>(1, std::min<int64_t>((e->p.n + 255) / 256, (int64_t)e->sms * 8));
  k_mk_init_counts<<<ib, 256, 0, st>>>(e->p);  // counts from the states (pushes folded implicitly)
  MK_CUDA(cudaGetLastError());
  std::vector<uint16_t> c(e->p.n);
  MK_CUDA(cudaMemcpyAsync(c.data(), e->cnt, e->p.n * sizeof(uint16_t), cudaMemcpyDeviceToHost, st));
  MK_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < e->p.n; ++i) out[i] = (double)c[i] * e->p.w;
  return 0;
}

}  // extern "C"
