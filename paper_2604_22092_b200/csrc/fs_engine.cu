// fs_engine.cu — the fused renewal tau-leap for sm_100a and its C ABI.
//
// One launch = one `renewal_step` of the reference
// (/root/reference/pkg/src/spreadsim/renewal.py:483-580):
//   CSR pressure gather -> per-compartment rate (pressure / exponential /
//   log-normal, Weibull, Erlang hazard) -> Bernoulli on a counter-based
//   uniform -> successor state, age reset / advance / freeze -> next-step
//   infectivity -> block max-rate and count deltas -> the last CTA to finish
//   folds the per-CTA partials into the device scalars (clock, step, tau',
//   counts) and the per-step log.  Nothing round-trips to the host inside a
//   batch, so `run_batch` is one CUDA-graph replay.
//
// Gather encodings:
//   COUNT_SMEM / COUNT_GLOBAL — constant transmission and uniform weights:
//     every contribution is the same f32 value c or 0, so the CSR-order f32
//     fold equals ptab[k], the k-fold sequential f32 sum of c, where k is the
//     number of infectious in-neighbours.  Infectivity travels as a 1-bit
//     mask (N/8 bytes), staged whole into shared memory when it fits.
//   F32  — general weights / age-dependent shedding: per-node sequential
//     f32 fold of f32(inf[col]*w) in CSR order (no FMA), bit-exact.
//   PRE  — pressure gathered by the edge-chunked merge kernel beforehand.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <cstdlib>
#include <string>
#include <vector>
#include <algorithm>
#include "fs_device.cuh"
#include "fs_internal.h"

namespace fs {

thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCntStride = FS_MAX_COMPARTMENTS;
// shared-memory budget for the staged mask: leaves room for the static
// tables on a 227 KB CTA
constexpr size_t kMaxSmemMaskBytes = 188u * 1024u;  // + ~34 KB static (queues) <= 227 KB

enum Gather { G_COUNT_SMEM = 0, G_COUNT_GLOBAL = 1, G_F32 = 2, G_PRE = 3, G_INCR = 4 };
constexpr int32_t kEntryInvalid = INT32_MIN;  // age not known to follow its cohort (init, host edits)
constexpr int kMemoSlots = 2;                  // age-dependent compartments memoised per CTA
constexpr int kMemoW = 1 << 10;                // entry steps per compartment (direct-mapped ring)

constexpr uint32_t kDeltaBias = 0x8000u;  // pending delta d is stored as d + 0x8000 (|d| <= d_max < 2^15)
enum Strat { S_THREAD = 0, S_WARP = 1 };

// Device-side run scalars.  Two slots ping-pong (the host tracks which one
// is current): step k reads slot `in` and its CTA 0 writes slot `out`, so no
// CTA ever reads a slot being written.  `pending` = the count deltas and max
// rate of step s.step-1 still sit in an accumulator and are folded in by the
// next step (or by begin_batch / the host).
struct DevState {
  fs_scalars s;
  int pending;
  int pad_;
};
// per-step accumulator (ring of 3): every CTA adds its count deltas and maxes
// its max rate with non-returning atomics — no fence, no ticket, no tail CTA
struct StepAcc {
  unsigned max_bits;
  int pad_;
  unsigned long long d[FS_MAX_COMPARTMENTS];
};

struct StepParams {
  // graph (renewal.py:264-313 inputs)
  const int64_t* ro;
  const int32_t* ro32;     // int32 offsets when E < 2^31, else nullptr
  const int32_t* col;
  const void* w;          // f32 or bf16; unused when uniform
  int w_bf16;
  int w_uniform;
  float w_val;
  int64_t n;
  int64_t ntiles;         // ceil(N/32) of the local rows
  int64_t node_base;      // global id of local node 0 (partitioned runs; multiple of 32)
  int64_t tile_base;      // node_base / 32
  int64_t ntiles_mask;    // words of the (global) infectious mask
  // state
  void* states;
  void* ages;
  void* inf[2];
  uint32_t* mask[2];
  float* pressure;
  float* rates;
  const DevState* Sin;           // scalars as of this step's start
  DevState* Sout;                // written by CTA 0 for the next step
  StepAcc* acc;                  // ring of 3 accumulators
  // engine scratch
  double* log_clock;
  double* log_tau;
  int64_t* log_counts;
  int64_t log_cap;
  const float* ptab;
  int ptab_mul;                  // ptab[k] == f32(k * c) for every k <= d_max
  float ptab_c;
  const int32_t* active_tiles;   // compaction: tile ids, or nullptr
  const int64_t* num_active;
  const float* pre;              // G_PRE: gathered pressure
  int count_mode;
  // incremental count mode (G_INCR): per-node infectious in-neighbour count,
  // kept current by +-1 pushes along the outgoing edges of every node whose
  // infectious status changes
  uint16_t* cnt;                 // [N] counts as of the current step's start, minus pending deltas
  uint32_t* pend[2];             // [ceil(N/2)] words of biased u16 pending deltas, double-buffered by step parity
  const int64_t* out_ro;         // outgoing CSR of the local rows (the incoming one for symmetric graphs)
  const int32_t* out_col;        // global ids
  int world;                     // > 1: pushes go to the owner's pending deltas (peer_pend)
  int64_t part_chunk;            // nodes per rank
  uint32_t* peer_pend[2][FS_MAX_PARTITIONS];  // every rank's pending-delta arrays, by parity
  int stream_evict_first;        // CSR stream larger than L2: evict-first hint on column loads
  int host_parity;               // the host's mirror of (step & 1) for this launch (early loads), -1: none
  // age-cohort hazard memo: entry step of each node's
  // current compartment; the per-CTA memo itself lives in shared memory
  int32_t* entry;                // [N] or nullptr (memo off)
  unsigned long long* dbg;       // optional per-CTA %globaltimer stamps [grid][4]
  // model / config
  fs_model model;
  double eps, tau_max, delta;
  int rng;
  int hprec;
  float inf_val;                 // stored infectivity of an I node (count mode), promoted
};

// Per-CTA, per-step memo of nodal hazard rates by age cohort: every node
// that entered compartment c at step j carries the same age bits (the same
// f32 recurrence age += f32(tau) since), hence the same rate, so the f64
// hazard (R/hazards.py:122-132) runs once per (CTA, c, j) instead of once
// per node.  Entries are (step tag << 32 | rate bits); racing writers store
// identical values.  Results are bit-identical with or without it.
struct HazardMemo {
  unsigned long long e[kMemoSlots][kMemoW];
  int slot[FS_MAX_COMPARTMENTS];  // compartment -> memo slot, -1: not memoised
};

template <int BLOCK>
__device__ __forceinline__ void memo_init(HazardMemo& hm, const StepParams& p, int tid) {
  for (int i = tid; i < kMemoSlots * kMemoW; i += BLOCK) (&hm.e[0][0])[i] = ~0ull;  // tag 0xFFFFFFFF: stale
  if (tid == 0) {
    int next = 0;
    for (int c = 0; c < FS_MAX_COMPARTMENTS; ++c) {
      const bool costly = c < p.model.num_compartments && p.model.comp[c].hazard >= FS_HZ_LOGNORMAL;
      hm.slot[c] = (costly && next < kMemoSlots) ? next++ : -1;
    }
  }
}

struct MergeParams {
  const int64_t* ro;
  const int32_t* ro32;
  const int32_t* col;
  const void* w;
  int w_bf16;
  int w_uniform;
  float w_val;
  int64_t n;
  int64_t e;
  int64_t epb;
  int64_t nchunks;
  const int64_t* chunk_first;    // first node whose slice starts at/after chunk start
  const void* inf[2];            // general gather input (promoted on load)
  int inf_bf16;
  const uint32_t* mask[2];       // count gather input
  const float* ptab;
  const DevState* S;             // parity source; nullptr -> buffer 0
  float* out;
  int64_t nwords;
};

// ---------------------------------------------------------------------------
// L2 residency hints.  The infectious mask is read randomly ~d times per
// node per step and must stay in L2; the CSR column stream is read once per
// step and, when the working set exceeds L2, should not evict the mask.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_stream(int evict_first) {
  uint64_t a, b;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(a));
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(b));
  return evict_first ? a : b;
}
__device__ __forceinline__ uint32_t ldg_hint(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ldg_hint(const int32_t* p, uint64_t pol) {
  return (int32_t)ldg_hint(reinterpret_cast<const uint32_t*>(p), pol);
}

// ---------------------------------------------------------------------------
// gather primitives
// ---------------------------------------------------------------------------
template <bool SMEM>
__device__ __forceinline__ int mask_bit(const uint32_t* __restrict__ m, int32_t c) {
  uint32_t w = SMEM ? m[c >> 5] : ldg_hint(m + (c >> 5), l2_policy_last());
  return (int)((w >> (c & 31)) & 1u);
}

template <typename IT>
__device__ __forceinline__ float load_inf(const void* inf, int32_t c) {
  return to_f32<IT>(__ldg(reinterpret_cast<const IT*>(inf) + c));
}

__device__ __forceinline__ float load_w(const void* w, int w_bf16, int64_t e) {
  if (w_bf16) return __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(w) + e));
  return __ldg(reinterpret_cast<const float*>(w) + e);
}

// thread-per-node infectious-neighbour count (order-free integer sum)
template <bool SMEM>
__device__ __forceinline__ int count_thread(const int32_t* __restrict__ col, const uint32_t* m,
                                            int64_t lo, int64_t hi) {
  int cnt = 0;
  int64_t e = lo;
  for (; e + 4 <= hi; e += 4) {
    int32_t c0 = __ldg(col + e), c1 = __ldg(col + e + 1), c2 = __ldg(col + e + 2), c3 = __ldg(col + e + 3);
    cnt += mask_bit<SMEM>(m, c0) + mask_bit<SMEM>(m, c1) + mask_bit<SMEM>(m, c2) + mask_bit<SMEM>(m, c3);
  }
  for (; e < hi; ++e) cnt += mask_bit<SMEM>(m, __ldg(col + e));
  return cnt;
}

// warp-cooperative count of one slice; every lane returns the total
template <bool SMEM>
__device__ __forceinline__ int count_warp(const int32_t* __restrict__ col, const uint32_t* m,
                                          int64_t lo, int64_t hi, int lane) {
  int cnt = 0;
  for (int64_t e = lo + lane; e < hi; e += 32) cnt += mask_bit<SMEM>(m, __ldg(col + e));
  return __reduce_add_sync(kFull, cnt);
}

// ---------------------------------------------------------------------------
// TMA bulk staging of the infectious mask (cp.async.bulk + mbarrier)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// one elected thread launches the copy of `bytes` (16-byte multiple) in
// <= 64 KB pieces; every thread later waits on the barrier's phase 0
__device__ __forceinline__ void stage_mask_async(uint32_t* dst, const uint32_t* src, uint32_t bytes, uint64_t* bar) {
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 65536u) {
      const uint32_t len = min(65536u, bytes - off);
      tma_bulk_g2s(reinterpret_cast<char*>(dst) + off, reinterpret_cast<const char*>(src) + off, len, bar);
    }
  }
}

// Cluster variant: the CTA of rank r in a cluster of `csize` copies chunks
// r, r + csize, ... of the mask and multicasts each into every CTA of the
// cluster (same smem offset, same mbarrier offset), so the cluster reads the
// mask from L2 once instead of csize times.  Every CTA's barrier expects the
// full byte count.  Callers must cluster-sync between barrier init and this.
__device__ __forceinline__ void stage_mask_multicast(uint32_t* dst, const uint32_t* src, uint32_t bytes, uint64_t* bar,
                                                     uint32_t rank, uint32_t csize) {
  if (threadIdx.x == 0) {
    constexpr uint32_t kChunk = 16384u;
    const uint16_t cta_mask = (uint16_t)((1u << csize) - 1u);
    const uint32_t nchunks = (bytes + kChunk - 1) / kChunk;
    for (uint32_t c = rank; c < nchunks; c += csize) {
      const uint32_t off = c * kChunk, len = min(kChunk, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
              smem_u32(reinterpret_cast<char*>(dst) + off)),
          "l"(reinterpret_cast<const char*>(src) + off), "r"(len), "r"(smem_u32(bar)), "h"(cta_mask)
          : "memory");
    }
  }
}
// programmatic dependent launch: let the next step's CTAs launch now, and
// block until the previous grid's memory is visible
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// [lo, hi) of node n: int32 copy when present; neighbouring lanes share
// boundaries, so each lane loads one offset and takes hi from lane+1
__device__ __forceinline__ void load_slice(const int64_t* __restrict__ ro, const int32_t* __restrict__ ro32,
                                           int64_t n, bool valid, int lane, int64_t& lo, int64_t& hi) {
  int64_t v = 0;
  if (valid) v = ro32 ? (int64_t)__ldg(ro32 + n) : __ldg(ro + n);
  int64_t up = __shfl_down_sync(0xffffffffu, v, 1);
  const int next_valid = __shfl_down_sync(0xffffffffu, (int)valid, 1);
  if (valid && (lane == 31 || !next_valid)) up = ro32 ? (int64_t)__ldg(ro32 + n + 1) : __ldg(ro + n + 1);
  lo = v;
  hi = valid ? up : v;
}

// tile-cooperative count: the warp streams the contiguous edge range of its
// 32 nodes 32 edges per group, 8 groups per pass with every load of a pass
// in flight together (columns first, then the mask words they address),
// tests the source bits and ballots.  Lane g keeps group g's ballot word;
// afterwards every lane fetches only the words its own slice spans and
// popcounts them.  Integer counts are order-free: exact for any partition.
__device__ __forceinline__ uint32_t bmsk(int start, int width) {
  uint32_t r;
  asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(r) : "r"(start), "r"(width));
  return r;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

template <bool SMEM_MASK, bool COL_SMEM = false>
__device__ __forceinline__ int count_tile(const int32_t* __restrict__ col, const uint32_t* m, int64_t lo, int64_t hi,
                                          bool need, unsigned need_mask, int lane, uint64_t col_pol) {
  const int j0 = __ffs(need_mask) - 1, j1 = 31 - __clz(need_mask);
  const int64_t E0 = __shfl_sync(0xffffffffu, lo, j0), E1 = __shfl_sync(0xffffffffu, hi, j1);
  const int32_t* __restrict__ cp = col + E0;
  const uint32_t cp_s = COL_SMEM ? smem_u32(cp) : 0u;  // columns staged in shared memory
  const int L = (int)(E1 - E0);
  // my slice relative to E0 (empty for lanes that need no count)
  const int a = need ? (int)(lo - E0) : 0, b = need ? (int)(hi - E0) : 0;
  int cnt = 0;
  for (int w0 = 0; w0 < L; w0 += 1024) {  // windows of 32 groups
    const int wl = min(L - w0, 1024);
    unsigned mine = 0;
    for (int gb = 0; gb < wl; gb += 256) {
      uint32_t c[8], word[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = gb + 32 * u + lane;
        c[u] = e < wl ? (COL_SMEM ? lds_u32(cp_s + 4u * (uint32_t)(w0 + e)) : (uint32_t)ldg_hint(cp + w0 + e, col_pol))
                      : 0u;  // bits past the range are never counted
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) word[u] = SMEM_MASK ? m[c[u] >> 5] : ldg_hint(m + (c[u] >> 5), l2_policy_last());
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int g = gb + 32 * u;
        if (g >= wl) break;  // warp-uniform
        const unsigned W = __ballot_sync(0xffffffffu, __funnelshift_r(word[u], word[u], c[u]) & 1u);
        if (lane == (g >> 5)) mine = W;
      }
    }
    const int sa = max(a - w0, 0), sb = min(b - w0, wl);
    const int gf = sa >> 5;
    const int span = sa < sb ? ((sb - 1) >> 5) - gf + 1 : 0;
    const int most = __reduce_max_sync(0xffffffffu, span);
    for (int k = 0; k < most; ++k) {
      const int gq = gf + k;
      const unsigned W = __shfl_sync(0xffffffffu, mine, gq & 31);
      if (k < span) {
        const int lo_b = max(sa - 32 * gq, 0), hi_b = min(sb - 32 * gq, 32);
        cnt += __popc(W & bmsk(lo_b, hi_b - lo_b));
      }
    }
  }
  return cnt;
}

// thread-per-node sequential f32 fold in CSR order: acc = f32(acc + f32(inf*w))
// (renewal.py:289 + 60-68; T/test_renewal.py:27-37)
template <typename IT>
__device__ __forceinline__ float fold_thread(const int32_t* __restrict__ col, const void* inf,
                                             const void* w, int w_bf16, int w_uniform, float w_val,
                                             int64_t lo, int64_t hi) {
  float acc = 0.0f;
  for (int64_t e = lo; e < hi; ++e) {
    float wv = w_uniform ? w_val : load_w(w, w_bf16, e);
    acc = __fadd_rn(acc, __fmul_rn(load_inf<IT>(inf, __ldg(col + e)), wv));
  }
  return acc;
}

// warp-cooperative fold of one slice, still in CSR order: lanes load 32
// consecutive contributions, then every lane folds them in lane order
// (renewal.py:221-242 semantics; padding lanes contribute +0).
template <typename IT>
__device__ __forceinline__ float fold_warp(const int32_t* __restrict__ col, const void* inf,
                                           const void* w, int w_bf16, int w_uniform, float w_val,
                                           int64_t lo, int64_t hi, int lane) {
  float acc = 0.0f;
  for (int64_t base = lo; base < hi; base += 32) {
    int64_t e = base + lane;
    float v = 0.0f;
    if (e < hi) {
      float wv = w_uniform ? w_val : load_w(w, w_bf16, e);
      v = __fmul_rn(load_inf<IT>(inf, __ldg(col + e)), wv);
    }
    const int live = (hi - base) < 32 ? (int)(hi - base) : 32;
    for (int l = 0; l < live; ++l) acc = __fadd_rn(acc, __shfl_sync(kFull, v, l));
  }
  return acc;
}

// ---------------------------------------------------------------------------
// the fused step
// ---------------------------------------------------------------------------
template <typename ST, typename AT>
struct NodeIn {
  int s;
  float age;
  int64_t lo, hi;
};

constexpr int kQueue = 64;  // per-warp deferral queue capacity (entries)

// per-launch constants every phase needs
struct StepConst {
  double tau;
  float tau_f;
  uint64_t key, seed;
  int64_t step;
  int edge_from, infectious, shed;
  float beta_f;
  bool write_inf;
};

// shared-memory model tables + the per-warp deferral queues
template <int WARPS>
struct StepShared {
  int succ[FS_MAX_COMPARTMENTS], term[FS_MAX_COMPARTMENTS], kind[FS_MAX_COMPARTMENTS];
  double p0[FS_MAX_COMPARTMENTS], p1[FS_MAX_COMPARTMENTS];
  int cnt[FS_MAX_COMPARTMENTS];
  float wmax[WARPS];
  int q_node[WARPS][kQueue];
  int q_state[WARPS][kQueue];
  float q_age[WARPS][kQueue];
  float q_press[WARPS][kQueue];
};

template <int WARPS>
__device__ __forceinline__ void load_tables(const StepParams& p, StepShared<WARPS>& sh, int tid) {
  if (tid < FS_MAX_COMPARTMENTS) {
    const fs_compartment& c = p.model.comp[tid];
    sh.succ[tid] = c.succ;
    sh.term[tid] = c.terminal;
    sh.kind[tid] = c.hazard;
    sh.p0[tid] = c.p0;
    sh.p1[tid] = c.p1;
    sh.cnt[tid] = 0;
  }
}

__device__ __forceinline__ double next_tau(const StepParams& p, float max_rate) {
  // tau' = min(tau_max, eps / (max rate + delta)) in f64 (renewal.py:577-578)
  const double cand = __ddiv_rn(p.eps, __dadd_rn((double)max_rate, p.delta));
  return (p.tau_max <= cand) ? p.tau_max : cand;
}

__device__ __forceinline__ StepConst step_const(const StepParams& p, bool count_gather) {
  StepConst k;
  const DevState* I = p.Sin;  // final: the previous grid completed
  k.step = I->s.step;
  k.seed = I->s.seed;
  if (I->pending) {
    const StepAcc* A = p.acc + (k.step - 1) % 3;
    k.tau = next_tau(p, __uint_as_float(__ldcg(&A->max_bits)));
  } else {
    k.tau = I->s.tau_next;
  }
  k.tau_f = __double2float_rn(k.tau);  // np.float32(tau), renewal.py:541
  k.key = splitmix_step_key(k.seed, (uint64_t)k.step);
  k.edge_from = p.model.edge_from;
  k.infectious = p.model.infectious;
  k.shed = p.model.shedding;
  k.beta_f = __double2float_rn(p.model.beta);
  k.write_inf = !count_gather;
  return k;
}

// CTA 0 / thread 0, right after the dependency wait: publish the next
// step's scalars.  Folds the previous step's pending deltas into the counts
// (and the per-step log), advances the clock by this step's tau, and clears
// the accumulator the next step will use.
__device__ __forceinline__ void commit_step_start(const StepParams& p, const StepConst& k) {
  const DevState* I = p.Sin;
  DevState* O = p.Sout;
  O->s = I->s;
  const int M = p.model.num_compartments;
  if (I->pending) {
    const StepAcc* A = p.acc + (k.step - 1) % 3;
    const int64_t prev = (k.step - 1) % p.log_cap;
    for (int c = 0; c < M; ++c) {
      const int64_t v = I->s.counts[c] + (int64_t)__ldcg(&A->d[c]);
      O->s.counts[c] = v;
      p.log_counts[prev * kCntStride + c] = v;
    }
    O->s.last_max_rate = __uint_as_float(__ldcg(&A->max_bits));
  }
  const double clock1 = I->s.clock + k.tau;  // renewal.py:497-498
  O->s.clock = clock1;
  O->s.tau_next = k.tau;
  O->s.step = k.step + 1;
  O->s.started = 1;
  O->pending = 1;
  const int64_t slot = k.step % p.log_cap;
  p.log_clock[slot] = clock1;
  p.log_tau[slot] = k.tau;
  StepAcc* Z = p.acc + (k.step + 1) % 3;  // last read by the previous step
  Z->max_bits = 0u;
  for (int c = 0; c < FS_MAX_COMPARTMENTS; ++c) Z->d[c] = 0ull;
}

// next-step infectivity of a node in compartment ns at age nage (f32 gather;
// renewal.py:556-565, cast on store by the caller)
__device__ __forceinline__ float inf_value(const StepParams& p, const StepConst& k, int ns, float nage) {
  if (ns != k.infectious) return 0.0f;
  if (k.shed == FS_SHED_CONSTANT) return k.beta_f;
  return __double2float_rn(
      __dmul_rn(p.model.beta, shedding_f64(k.shed, p.model.shed_mu, p.model.shed_sigma, p.model.shed_peak, (double)nage)));
}

// phase B: settle `cnt` queued nodes of this warp, one per lane — rate
// (pressure or hazard), uniform, Bernoulli, successor / age / infectivity
// incremental counts: +-1 on node j's pending delta (buffer `nxt`), in this
// device's memory or, node-partitioned, the owner's — possibly a peer GPU's
// over NVLink.  Chunk boundaries are even, so the 16-bit lane
// of j is the same in global and owner-local numbering.
__device__ __forceinline__ void push_delta(const StepParams& p, int nxt, int32_t j, bool up) {
  const uint32_t one = 1u << (16 * (j & 1));
  uint32_t* dn;
  if (p.world > 1) {
    const int owner = (int)((int64_t)j / p.part_chunk);
    dn = p.peer_pend[nxt][owner] + (((int64_t)j - (int64_t)owner * p.part_chunk) >> 1);
  } else {
    dn = p.pend[nxt] + (j >> 1);
  }
  if (up) atomicAdd(dn, one);
  else atomicSub(dn, one);
}

template <typename ST, typename AT, typename IT, bool MAT, int WARPS>
__device__ __forceinline__ void drain_entries(const StepParams& p, const StepConst& k, StepShared<WARPS>& sh,
                                              const int* qn_node, const int* qn_state, const float* qn_age,
                                              const float* qn_press, int lane, int cnt, float& lmax,
                                              uint32_t* mask_nxt, IT* inf_nxt, HazardMemo* hm = nullptr) {
  __syncwarp();
  const bool ok = lane < cnt;
  int push = 0;  // +1 / -1: this node's infectious status changed
  const int n = ok ? qn_node[lane] : 0;
  const int s = ok ? qn_state[lane] : 0;
  const float age = ok ? qn_age[lane] : 0.0f;
  float rate = 0.0f;
  bool compute = false;
  unsigned long long* slot = nullptr;
  if (ok) {
    if (s == k.edge_from) {
      rate = qn_press[lane];
    } else if (hm && hm->slot[s] >= 0) {
      const int32_t j = p.entry[n];
      const int64_t since = k.step - (int64_t)j;
      compute = true;
      if (j != kEntryInvalid && since >= 0 && since < kMemoW) {
        slot = &hm->e[hm->slot[s]][(uint32_t)j & (kMemoW - 1)];
        const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(slot);
        if ((uint32_t)(v >> 32) == (uint32_t)k.step) {
          rate = __uint_as_float((uint32_t)v);
          compute = false;
        }
      }
    } else {
      rate = nodal_rate(sh.kind[s], sh.p0[s], sh.p1[s], age, p.hprec);
    }
  }
  if (compute) {
    rate = nodal_rate(sh.kind[s], sh.p0[s], sh.p1[s], age, p.hprec);
    // racing writers of one slot store identical bits
    if (slot) *reinterpret_cast<volatile unsigned long long*>(slot) = ((unsigned long long)(uint32_t)k.step << 32) | __float_as_uint(rate);
  }
  lmax = fmaxf(lmax, rate);
  bool fire = false;
  if (rate > 0.0f) {
    const uint64_t gid = (uint64_t)(n + p.node_base);  // RNG keyed by the global node id (rng.py:5-7)
    const double u = (p.rng == FS_RNG_SPLITMIX) ? splitmix_uniform(k.key, gid)
                                                : philox_uniform(k.seed, (uint64_t)k.step, gid);
    fire = bernoulli_fire(u, rate, k.tau);
  }
  if (ok) {
    int ns = s;
    float nage;
    if (fire) {
      ns = sh.succ[s];
      nage = 0.0f;
      reinterpret_cast<ST*>(p.states)[n] = (ST)ns;
      if (p.entry) p.entry[n] = (int32_t)k.step;  // age cohort of the new compartment
      atomicAdd(&sh.cnt[ns], 1);
      atomicAdd(&sh.cnt[s], -1);
      if (!k.write_inf && ((ns == k.infectious) != (s == k.infectious))) {
        atomicXor(mask_nxt + p.tile_base + (n >> 5), 1u << (n & 31));
        if (p.cnt) push = (ns == k.infectious) ? 1 : -1;  // incremental counts: pushes below
      }
    } else {
      nage = __fadd_rn(age, k.tau_f);  // queued nodes are never terminal
    }
    reinterpret_cast<AT*>(p.ages)[n] = from_f32<AT>(nage);
    if (k.write_inf) inf_nxt[n] = from_f32<IT>(inf_value(p, k, ns, nage));
    if (MAT) p.rates[n] = rate;
  }
  if (p.cnt) {
    // +-1 on every out-neighbour's pending delta.  Rows of <= 32 edges are
    // pushed by their own lane; longer rows (scale-free hubs) by the whole
    // warp, 32 edges per iteration, so one hub does not serialise the step.
    const int nxt = (int)((k.step & 1) ^ 1);
    int64_t e0 = 0, e1 = 0;
    if (push) {
      e0 = __ldg(p.out_ro + n);  // out-row of local node n
      e1 = __ldg(p.out_ro + n + 1);
    }
    const bool wide = push && (e1 - e0 > 32);
    if (push && !wide)
      for (int64_t e = e0; e < e1; ++e) push_delta(p, nxt, __ldg(p.out_col + e), push > 0);
    unsigned wides = __ballot_sync(kFull, wide);
    while (wides) {
      const int src = __ffs(wides) - 1;
      wides &= wides - 1;
      const int64_t a0 = __shfl_sync(kFull, e0, src), a1 = __shfl_sync(kFull, e1, src);
      const bool up = __shfl_sync(kFull, push, src) > 0;
      for (int64_t e = a0 + lane; e < a1; e += 32) push_delta(p, nxt, __ldg(p.out_col + e), up);
    }
  }
  __syncwarp();
}

// phase B on this warp's own queue
template <typename ST, typename AT, typename IT, bool MAT, int WARPS>
__device__ __forceinline__ void drain_queue(const StepParams& p, const StepConst& k, StepShared<WARPS>& sh, int warp,
                                            int lane, int cnt, float& lmax, uint32_t* mask_nxt, IT* inf_nxt,
                                            HazardMemo* hm = nullptr) {
  drain_entries<ST, AT, IT, MAT, WARPS>(p, k, sh, sh.q_node[warp], sh.q_state[warp], sh.q_age[warp], sh.q_press[warp],
                                        lane, cnt, lmax, mask_nxt, inf_nxt, hm);
}

// phase A outcome of one tile (pressure already gathered): cheap outcomes
// now, possible transitions appended to the warp queue (drained at 32)
template <typename ST, typename AT, typename IT, bool MAT, int WARPS>
__device__ __forceinline__ void tile_outcome(const StepParams& p, const StepConst& k, StepShared<WARPS>& sh, int warp,
                                             int lane, int64_t tile, int64_t n, bool valid, int s, float age,
                                             float pressure, int& qn, float& lmax, uint32_t* mask_nxt, IT* inf_nxt,
                                             HazardMemo* hm = nullptr) {
  const bool isS = s == k.edge_from;
  const bool term = valid && sh.term[s] != 0;
  const bool defer = valid && !term && (!isS || pressure > 0.0f);
  if (valid && !term && !defer) {  // S with zero pressure: rate 0, ages
    const float nage = __fadd_rn(age, k.tau_f);
    reinterpret_cast<AT*>(p.ages)[n] = from_f32<AT>(nage);
    if (k.write_inf) inf_nxt[n] = from_f32<IT>(inf_value(p, k, s, nage));
  } else if (term && k.write_inf) {
    inf_nxt[n] = from_f32<IT>(inf_value(p, k, s, age));
  }
  if (MAT && valid) {
    p.pressure[n] = pressure;
    if (!defer) p.rates[n] = 0.0f;
  }
  if (!k.write_inf) {
    // next-step mask word; deferred nodes are fixed up in phase B
    const unsigned word = __ballot_sync(0xffffffffu, valid && s == k.infectious);
    if (lane == 0) mask_nxt[p.tile_base + tile] = word;
  }
  const unsigned dm = __ballot_sync(0xffffffffu, defer);
  if (defer) {
    const int at = qn + __popc(dm & ((1u << lane) - 1u));
    sh.q_node[warp][at] = (int)n;
    sh.q_state[warp][at] = s;
    sh.q_age[warp][at] = age;
    sh.q_press[warp][at] = pressure;
  }
  qn += __popc(dm);
  if (qn >= 32) {
    drain_queue<ST, AT, IT, MAT, WARPS>(p, k, sh, warp, lane, 32, lmax, mask_nxt, inf_nxt, hm);
    if (lane < qn - 32) {
      sh.q_node[warp][lane] = sh.q_node[warp][32 + lane];
      sh.q_state[warp][lane] = sh.q_state[warp][32 + lane];
      sh.q_age[warp][lane] = sh.q_age[warp][32 + lane];
      sh.q_press[warp][lane] = sh.q_press[warp][32 + lane];
    }
    qn -= 32;
  }
}

// block max-rate / count deltas into this step's accumulator
template <int WARPS>
__device__ __forceinline__ void finish_step(const StepParams& p, const StepConst& k, StepShared<WARPS>& sh, int warp,
                                            int lane, float lmax) {
  constexpr unsigned FULL = 0xffffffffu;
#pragma unroll
  for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(FULL, lmax, o));
  if (lane == 0) sh.wmax[warp] = lmax;
  __syncthreads();
  if (warp != 0) return;
  float bmax = lane < WARPS ? sh.wmax[lane] : 0.0f;
#pragma unroll
  for (int o = 16; o; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(FULL, bmax, o));
  StepAcc* A = p.acc + k.step % 3;
  if (lane == 0 && bmax > 0.0f) atomicMax(&A->max_bits, __float_as_uint(bmax));  // rates >= 0: bit order == value order
  if (lane < p.model.num_compartments) {
    const int d = sh.cnt[lane];
    if (d) atomicAdd(&A->d[lane], (unsigned long long)(long long)d);
  }
}

// One launch = one reference renewal_step (renewal.py:483-580), two phases
// per warp:
//  A (per 32-node tile, dense): node loads (one tile ahead), pressure
//    gather, and the cheap outcomes: terminal nodes do nothing, S nodes with
//    zero pressure only age.  Every node that may fire (S with pressure > 0,
//    any nodal compartment) is appended to the warp's shared-memory queue;
//    the tile's next-step mask word assumes no deferred node changes
//    infectious status.
//  B (whenever >= 32 queued, and once at the end): 32 queued nodes at a time,
//    all lanes busy: rate (pressure or f64 hazard), counter-based uniform,
//    Bernoulli, successor / age writes, infectivity / mask fix-up.
// This general kernel serves every gather mode and strategy (and the
// compaction tile list); the streaming k_step_tma below is the fast path
// of the count gather.
template <typename ST, typename AT, typename IT, int GATHER, int STRAT, bool MAT, int BLOCK>
__global__ void __launch_bounds__(BLOCK, (BLOCK >= 1024 ? 1 : 2)) k_step(const StepParams p) {
  extern __shared__ __align__(16) uint32_t s_mask[];
  constexpr int WARPS = BLOCK / 32;
  __shared__ StepShared<WARPS> sh;
  __shared__ __align__(8) uint64_t s_bar;
  constexpr bool COUNT = (GATHER == G_COUNT_SMEM || GATHER == G_COUNT_GLOBAL);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  pdl_wait();
  if (GATHER == G_COUNT_SMEM && tid == 0) mbar_init(&s_bar, 1);
  load_tables<WARPS>(p, sh, tid);
  const StepConst k = step_const(p, COUNT || p.count_mode);
  if (blockIdx.x == 0 && tid == 0) commit_step_start(p, k);
  const int cur = (int)(k.step & 1);
  const uint32_t* mask_cur = p.mask[cur];
  uint32_t* mask_nxt = p.mask[cur ^ 1];
  const void* inf_cur = p.inf[cur];
  IT* inf_nxt = reinterpret_cast<IT*>(p.inf[cur ^ 1]);
  __syncthreads();
  // stage the whole infectious mask (N/8 bytes) in shared memory with TMA
  // bulk copies; the first tile's node loads below overlap the transfer
  if (GATHER == G_COUNT_SMEM) stage_mask_async(s_mask, mask_cur, (uint32_t)(((p.ntiles_mask + 3) & ~3LL) * 4), &s_bar);
  bool mask_ready = GATHER != G_COUNT_SMEM;
  const uint32_t* gmask = (GATHER == G_COUNT_SMEM) ? s_mask : mask_cur;
  float lmax = 0.0f;
  int qn = 0;  // queued entries of this warp (warp-uniform)

  const int64_t ntiles = p.active_tiles ? *p.num_active : p.ntiles;
  const int64_t stride = (int64_t)gridDim.x * WARPS;
  auto load_in = [&](int64_t tile, NodeIn<ST, AT>& in) {
    const int64_t n = tile * 32 + lane;
    const bool valid = n < p.n;
    in.s = valid ? (int)reinterpret_cast<const ST*>(p.states)[n] : -1;
    in.age = valid ? to_f32<AT>(reinterpret_cast<const AT*>(p.ages)[n]) : 0.0f;
    in.lo = in.hi = 0;
    if (GATHER == G_INCR) {  // lo <- count, hi <- pending delta (biased)
      if (valid) {
        in.lo = p.cnt[n];
        in.hi = reinterpret_cast<const uint16_t*>(p.pend[cur])[n];
      }
    } else if (GATHER != G_PRE) {
      load_slice(p.ro, p.ro32, n, valid, lane, in.lo, in.hi);
    }
  };
  auto tile_of = [&](int64_t t) -> int64_t { return p.active_tiles ? (int64_t)p.active_tiles[t] : t; };

  int64_t t = (int64_t)blockIdx.x * WARPS + warp;
  NodeIn<ST, AT> nxt{};
  int64_t tile_n = 0;
  if (t < ntiles) {
    tile_n = tile_of(t);
    load_in(tile_n, nxt);
  }
  for (; t < ntiles; t += stride) {
    const NodeIn<ST, AT> in = nxt;
    const int64_t tile = tile_n;
    if (t + stride < ntiles) {  // next tile's node loads overlap this tile
      tile_n = tile_of(t + stride);
      load_in(tile_n, nxt);
    }
    const int64_t n = tile * 32 + lane;
    const bool valid = n < p.n;
    const bool need = valid && (in.s == k.edge_from || MAT);

    float pressure = 0.0f;
    if (GATHER == G_INCR) {
      // fold the pushes of the previous step into the count (and clear them)
      uint32_t c = (uint32_t)in.lo;
      const uint32_t dl = (uint32_t)in.hi;
      if (valid && dl != kDeltaBias) {
        c = c + dl - kDeltaBias;
        p.cnt[n] = (uint16_t)c;
        reinterpret_cast<uint16_t*>(p.pend[cur])[n] = (uint16_t)kDeltaBias;
      }
      if (need) pressure = p.ptab_mul ? __fmul_rn((float)c, p.ptab_c) : __ldg(p.ptab + c);
    } else if (GATHER == G_PRE) {
      if (need) pressure = __ldg(p.pre + n);
    } else {
      if (GATHER == G_COUNT_SMEM && !mask_ready) {
        mbar_wait_parity(&s_bar, 0);
        mask_ready = true;
      }
      const unsigned todo = __ballot_sync(kFull, need);
      if (STRAT == S_THREAD) {
        if (GATHER == G_F32) {
          if (need) pressure = fold_thread<IT>(p.col, inf_cur, p.w, p.w_bf16, p.w_uniform, p.w_val, in.lo, in.hi);
        } else if (todo) {
          const int kk = count_tile<GATHER == G_COUNT_SMEM>(p.col, gmask, in.lo, in.hi, need, todo, lane,
                                                            l2_policy_stream(p.stream_evict_first));
          if (need) pressure = p.ptab_mul ? __fmul_rn((float)kk, p.ptab_c) : __ldg(p.ptab + kk);
        }
      } else {  // warp per node (LANE strategy)
        unsigned rest = todo;
        while (rest) {
          const int j = __ffs(rest) - 1;
          rest &= rest - 1;
          const int64_t lj = __shfl_sync(kFull, in.lo, j), hj = __shfl_sync(kFull, in.hi, j);
          float pj;
          if (GATHER == G_F32) {
            pj = fold_warp<IT>(p.col, inf_cur, p.w, p.w_bf16, p.w_uniform, p.w_val, lj, hj, lane);
          } else {
            const int kk = count_warp<GATHER == G_COUNT_SMEM>(p.col, gmask, lj, hj, lane);
            pj = p.ptab_mul ? __fmul_rn((float)kk, p.ptab_c) : __ldg(p.ptab + kk);
          }
          if (lane == j) pressure = pj;
        }
      }
    }
    tile_outcome<ST, AT, IT, MAT, WARPS>(p, k, sh, warp, lane, tile, n, valid, in.s, in.age, pressure, qn, lmax,
                                         mask_nxt, inf_nxt);
  }
  if (qn > 0) drain_queue<ST, AT, IT, MAT, WARPS>(p, k, sh, warp, lane, qn, lmax, mask_nxt, inf_nxt);
  // a warp without tiles still has to see the bulk copy land before exit
  if (GATHER == G_COUNT_SMEM && !mask_ready) mbar_wait_parity(&s_bar, 0);
  finish_step<WARPS>(p, k, sh, warp, lane, lmax);
}

// ---------------------------------------------------------------------------
// Step kernel of the incremental count mode (G_INCR, no compaction list).
// No gather: a node's infectious in-neighbour count is read like any other
// per-node field, so phase A is a coalesced stream over (state, age,
// count, pending delta) — 32-node tiles, lane per node, two tiles of loads
// in flight, 32-bit indexing, the step constants computed once per CTA.
// Phase B (the deferral queue: hazards, uniforms, Bernoulli, pushes) is the
// same as k_step's.
// ---------------------------------------------------------------------------
template <typename ST, typename AT, bool MAT, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 2) k_step_incr(const StepParams p) {
  constexpr int WARPS = BLOCK / 32;
  __shared__ StepShared<WARPS> sh;
  __shared__ StepConst s_k;
  __shared__ HazardMemo s_hm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_launch_dependents();
  load_tables<WARPS>(p, sh, tid);  // static model tables: before the dependency wait
  if (p.entry) memo_init<BLOCK>(s_hm, p, tid);
  HazardMemo* hmp = p.entry ? &s_hm : nullptr;
  pdl_wait();
  if (tid == 0) {
    s_k = step_const(p, true);
    if (blockIdx.x == 0) commit_step_start(p, s_k);
  }
  const ST* __restrict__ states = reinterpret_cast<const ST*>(p.states);
  const AT* __restrict__ ages = reinterpret_cast<const AT*>(p.ages);
  uint16_t* __restrict__ cnt = p.cnt;
  const uint32_t N = (uint32_t)p.n, ntiles = (uint32_t)p.ntiles;
  const uint32_t stride = gridDim.x * WARPS;
  struct In { int s; float age; uint32_t c, d; };
  // arrays are padded to whole 128-node units: every lane loads unconditionally
  auto load = [&](uint32_t t, const uint16_t* pend, In& in) {
    const uint32_t n = t * 32u + (uint32_t)lane;
    in.s = (int)states[n];
    in.age = to_f32<AT>(ages[n]);
    in.c = cnt[n];
    in.d = pend[n];
  };
  // the first two tiles' loads need only the buffer parity, which the host
  // knows: they overlap thread 0's scalar reads instead of waiting for them
  uint32_t t = blockIdx.x * WARPS + warp;
  In in0{}, in1{};
  if (p.host_parity >= 0) {
    const uint16_t* pend_h = reinterpret_cast<const uint16_t*>(p.pend[p.host_parity & 1]);
    if (t < ntiles) load(t, pend_h, in0);
    if (t + stride < ntiles) load(t + stride, pend_h, in1);
  }
  __syncthreads();
  const StepConst k = s_k;
  const int cur = (int)(k.step & 1);
  uint32_t* mask_nxt = p.mask[cur ^ 1];
  uint16_t* __restrict__ pend = reinterpret_cast<uint16_t*>(p.pend[cur]);
  if (cur != p.host_parity) {  // no host mirror, or out of step: load now
    if (t < ntiles) load(t, pend, in0);
    if (t + stride < ntiles) load(t + stride, pend, in1);
  }
  float lmax = 0.0f;
  int qn = 0;
  for (; t < ntiles; t += stride) {
    const In in = in0;
    in0 = in1;
    if (t + 2 * stride < ntiles) load(t + 2 * stride, pend, in1);
    const uint32_t n = t * 32u + (uint32_t)lane;
    const bool valid = n < N;
    uint32_t c = in.c;
    if (valid && in.d != kDeltaBias) {  // fold the previous step's pushes, clear them
      c = c + in.d - kDeltaBias;
      cnt[n] = (uint16_t)c;
      pend[n] = (uint16_t)kDeltaBias;
    }
    const int s = valid ? in.s : -1;
    const float pressure = (valid && (s == k.edge_from || MAT))
                               ? (p.ptab_mul ? __fmul_rn((float)c, p.ptab_c) : __ldg(p.ptab + c))
                               : 0.0f;
    tile_outcome<ST, AT, float, MAT, WARPS>(p, k, sh, warp, lane, (int64_t)t, (int64_t)n, valid, s, in.age, pressure,
                                            qn, lmax, mask_nxt, nullptr, hmp);
  }
  if (qn > 0) drain_queue<ST, AT, float, MAT, WARPS>(p, k, sh, warp, lane, qn, lmax, mask_nxt, nullptr, hmp);
  finish_step<WARPS>(p, k, sh, warp, lane, lmax);
}

// thread-per-node count over a slice staged in shared memory: lane-private
// loop, two edges per iteration; an odd tail reads the sentinel column
// `zero_col`, whose mask word is guaranteed zero
// U columns per round, all of a round's mask loads in flight together: the
// mask lookups (shared memory at N <~ 1.5e6, L2 beyond) are the dependent
// latency of the gather, so a degree-d slice costs ceil(d/U) round trips.
template <bool SMEM_MASK, int U>
__device__ __forceinline__ int count_slice_smem(uint32_t col_addr, int len, const uint32_t* m, uint32_t zero_col) {
  int cnt = 0;
  const uint64_t pol = SMEM_MASK ? 0ull : l2_policy_last();
  for (int i = 0; i < len; i += U) {
    uint32_t c[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (i + u < len) ? lds_u32(col_addr + 4u * (uint32_t)(i + u)) : zero_col;
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = SMEM_MASK ? m[c[u] >> 5] : ldg_hint(m + (c[u] >> 5), pol);
#pragma unroll
    for (int u = 0; u < U; ++u) cnt += (int)(__funnelshift_r(w[u], w[u], c[u]) & 1u);
  }
  return cnt;
}

// ---------------------------------------------------------------------------
// Streaming fast path of the count gather (PER_NODE strategy).
// Each warp owns a contiguous run of 32-node tiles and keeps TMA_SLOTS of
// them in flight: lane 0 issues cp.async.bulk copies of the tile's offsets,
// states, ages and contiguous column slice into a shared-memory slot whose
// mbarrier completes on the byte count, so ~TMA_SLOTS x 1.7 KB per warp
// stream from HBM with no registers held.  The gather then reads columns
// and the staged infectious mask from shared memory only.
// ---------------------------------------------------------------------------
#ifndef FS_GATHER_U_SMEM
#define FS_GATHER_U_SMEM 2
#endif
#ifndef FS_GATHER_U_GLOBAL
#define FS_GATHER_U_GLOBAL 2
#endif
constexpr int kGatherU_Smem = FS_GATHER_U_SMEM;
constexpr int kGatherU_Global = FS_GATHER_U_GLOBAL;

struct TmaLayout {
  int slots;        // buffers per warp
  int slot_bytes;   // bytes per buffer
  int ro_off, st_off, ag_off, col_off;  // byte offsets inside a buffer
  int col_cap;      // column entries a buffer holds
};

template <typename ST, typename AT, bool SMEM_MASK, bool MAT, bool PTAB_MUL, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1) k_step_tma(const StepParams p, const TmaLayout L) {
  extern __shared__ __align__(128) unsigned char dyn[];
  constexpr int WARPS = BLOCK / 32;
  __shared__ StepShared<WARPS> sh;
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ __align__(8) uint64_t t_bar[WARPS][4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 32-bit indices: N < 2^31 nodes (graph.py:51) and E < 2^31 on this path
  const int N = (int)p.n, ntiles = (int)p.ntiles;
  const int mask_words = ((int)p.ntiles_mask + 1 + 3) & ~3;  // >= one zero word past the last tile
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(dyn);
  unsigned char* wbuf = dyn + (SMEM_MASK ? mask_words * 4 : 0) + (size_t)warp * L.slots * L.slot_bytes;
  const uint32_t wbuf_s = smem_u32(wbuf);
  const uint32_t zero_col = (uint32_t)p.ntiles_mask * 32u;  // sentinel: its mask word is zero

  const uint32_t csize = SMEM_MASK ? cluster_size() : 1u;
  unsigned long long* dbg = nullptr;
  unsigned long long* const dbg_base = p.dbg;
  if (tid == 0 && SMEM_MASK) {
    mbar_init(&s_bar, 1);
    mbar_arrive_expect_tx(&s_bar, (uint32_t)mask_words * 4u);
  }
  if (lane == 0)
    for (int sl = 0; sl < L.slots; ++sl) mbar_init(&t_bar[warp][sl], 1);
  pdl_launch_dependents();
  load_tables<WARPS>(p, sh, tid);
  if (SMEM_MASK && csize > 1) cluster_sync_all();  // peers' barriers are armed before any multicast lands
  else __syncthreads();
  const ST* __restrict__ states = reinterpret_cast<const ST*>(p.states);
  const AT* __restrict__ ages = reinterpret_cast<const AT*>(p.ages);
  const int32_t* __restrict__ ro = p.ro32;

  // contiguous tile run of this warp; lane j holds the run's (j)th tile
  // boundary offset, so every tile's edge range is a shuffle away
  const int gw = blockIdx.x * WARPS + warp, nw = gridDim.x * WARPS;
  const int per = ntiles / nw, rem = ntiles % nw;  // balanced split
  const int t0 = gw * per + min(gw, rem), t1 = t0 + per + (gw < rem ? 1 : 0);
  const uint64_t col_pol = l2_policy_stream(p.stream_evict_first);
  int bnd_base = t0;
  int32_t bnd = (t0 + lane <= t1) ? __ldg(ro + min((t0 + lane) * 32, N)) : 0;  // first edge of tile t0+lane
  // lane 0 streams tile t's columns [ro[32t] & ~3, (ro[32t+32] + 3) & ~3)
  // into slot sl with one bulk copy completing on the slot's mbarrier
  auto issue_cols = [&](int t, int sl) {
    if (t - bnd_base >= 31) {  // refill the boundary window (warp-uniform)
      bnd_base = t;
      bnd = (t + lane <= t1) ? __ldg(ro + min((t + lane) * 32, N)) : 0;
    }
    const int j = t - bnd_base;
    const int32_t c0 = __shfl_sync(kFull, bnd, j) & ~3, c1 = (__shfl_sync(kFull, bnd, j + 1) + 3) & ~3;
    if (lane == 0) {
      const uint32_t bytes = 4u * (uint32_t)(c1 - c0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the slot
      mbar_arrive_expect_tx(&t_bar[warp][sl], bytes);
      if (bytes) tma_bulk_g2s_hint(wbuf + (size_t)sl * L.slot_bytes, p.col + c0, bytes, &t_bar[warp][sl], col_pol);
    }
  };
  // per-node inputs, coalesced loads two tiles ahead (arrays are padded to
  // whole tiles, so every lane loads unconditionally)
  struct In { int s; float age; int32_t lo, hi; };
  auto load_in = [&](int t, In& in) {
    const int n = t * 32 + lane;
    in.s = (int)states[n];
    in.age = to_f32<AT>(ages[n]);
    in.lo = __ldg(ro + min(n, N));
    in.hi = __ldg(ro + min(n + 1, N));
  };

  float lmax = 0.0f;
  int qn = 0;
  // the CSR is static: stream the first column slices before waiting on the
  // previous step (they overlap its tail under programmatic launch)
  for (int sl = 0; sl < L.slots; ++sl)
    if (t0 + sl < t1) issue_cols(t0 + sl, sl);
  pdl_wait();  // previous step complete: scalars, states, ages, mask are final
  const StepConst k = step_const(p, true);
  if (blockIdx.x == 0 && tid == 0) commit_step_start(p, k);
  if (dbg_base) {
    dbg = dbg_base + ((size_t)(k.step & 15) * gridDim.x + blockIdx.x) * 4;
    if (tid == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      dbg[0] = now;
    }
  }
  const int cur = (int)(k.step & 1);
  const uint32_t* mask_cur = p.mask[cur];
  uint32_t* mask_nxt = p.mask[cur ^ 1];
  if (SMEM_MASK) stage_mask_multicast(s_mask, mask_cur, (uint32_t)mask_words * 4u, &s_bar, cluster_rank(), csize);
  const uint32_t* gmask = SMEM_MASK ? s_mask : mask_cur;
  In in0{}, in1{};
  if (t0 < t1) load_in(t0, in0);
  if (t0 + 1 < t1) load_in(t0 + 1, in1);
  if (SMEM_MASK) mbar_wait_parity(&s_bar, 0);
  uint32_t phase_bits = 0;  // bit sl: parity of slot sl's next completion
  int sl = 0;
  for (int t = t0; t < t1; ++t) {
    const In in = in0;
    in0 = in1;
    if (t + 2 < t1) load_in(t + 2, in1);
    const int n = t * 32 + lane;
    const bool valid = n < N;
    const int s = valid ? in.s : -1;
    const bool need = valid && (s == k.edge_from || MAT);
    mbar_wait_parity(&t_bar[warp][sl], (phase_bits >> sl) & 1u);
    phase_bits ^= 1u << sl;
    float pressure = 0.0f;
    const int32_t cbase = __shfl_sync(kFull, in.lo, 0) & ~3;  // the slot holds columns from cbase
    if (need) {
      const int kk = count_slice_smem<SMEM_MASK, SMEM_MASK ? kGatherU_Smem : kGatherU_Global>(wbuf_s + (uint32_t)(sl * L.slot_bytes) + 4u * (uint32_t)(in.lo - cbase),
                                                 in.hi - in.lo, gmask, zero_col);
      pressure = PTAB_MUL ? __fmul_rn((float)kk, p.ptab_c) : __ldg(p.ptab + kk);
    }
    __syncwarp();
    // the slot is consumed: refill it with tile t + slots
    if (t + L.slots < t1) issue_cols(t + L.slots, sl);
    tile_outcome<ST, AT, float, MAT, WARPS>(p, k, sh, warp, lane, t, n, valid, s, in.age, pressure, qn, lmax,
                                            mask_nxt, nullptr);
    sl = (sl + 1 == L.slots) ? 0 : sl + 1;
  }
  if (qn > 0) drain_queue<ST, AT, float, MAT, WARPS>(p, k, sh, warp, lane, qn, lmax, mask_nxt, nullptr);
  if (dbg && lane == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicMax(dbg + 1, now);
    if (warp == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      dbg[2] = sm;
    }
  }
  if (SMEM_MASK && csize > 1) cluster_sync_all();  // no CTA exits while its multicasts may be in flight
  finish_step<WARPS>(p, k, sh, warp, lane, lmax);
  if (dbg && tid == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    dbg[3] = now;
  }
}

// ---------------------------------------------------------------------------
// edge-chunked merge gather (renewal.py:245-261, 291-302): warp per chunk of
// `epb` edges.  A node belongs to the chunk holding its first edge; slices
// of <= 32 edges are folded by one lane, longer or straddling slices by the
// whole warp, always in CSR order, so the result is bit-identical to the
// per-node fold.  Writes pressure for every node owning >= 1 edge.
// ---------------------------------------------------------------------------
template <typename IT, int MODE /*0 f32, 1 count-smem, 2 count-global*/, int BLOCK>
__global__ void __launch_bounds__(BLOCK, (BLOCK >= 1024 ? 1 : 2)) k_gather_merge(const MergeParams q) {
  extern __shared__ __align__(16) uint32_t s_mask[];
  constexpr int WARPS = BLOCK / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();
  const int cur = q.S ? (int)(q.S->s.step & 1) : 0;
  const uint32_t* mask_cur = q.mask[cur];
  const void* inf_cur = q.inf[cur];
  if (MODE == 1) {
    const int64_t nvec = q.nwords >> 2;
    const uint4* src4 = reinterpret_cast<const uint4*>(mask_cur);
    uint4* dst4 = reinterpret_cast<uint4*>(s_mask);
    for (int64_t i = tid; i < nvec; i += BLOCK) dst4[i] = __ldg(src4 + i);
    for (int64_t i = (nvec << 2) + tid; i < q.nwords; i += BLOCK) s_mask[i] = __ldg(mask_cur + i);
    __syncthreads();
  }
  const uint32_t* gmask = (MODE == 1) ? s_mask : mask_cur;
  for (int64_t c = (int64_t)blockIdx.x * WARPS + warp; c < q.nchunks; c += (int64_t)gridDim.x * WARPS) {
    const int64_t e1 = min(q.e, (c + 1) * q.epb);
    const int64_t n_lo = __ldg(q.chunk_first + c), n_hi = __ldg(q.chunk_first + c + 1);
    for (int64_t base = n_lo; base < n_hi; base += 32) {
      const int64_t n = base + lane;
      int64_t lo = 0, hi = 0;
      if (n < n_hi) { lo = __ldg(q.ro + n); hi = __ldg(q.ro + n + 1); }
      const bool small = (n < n_hi) && (hi - lo <= 32) && (hi <= e1);
      if (small) {
        float v;
        if (MODE == 0) v = fold_thread<IT>(q.col, inf_cur, q.w, q.w_bf16, q.w_uniform, q.w_val, lo, hi);
        else v = __ldg(q.ptab + count_thread<MODE == 1>(q.col, gmask, lo, hi));
        q.out[n] = v;
      }
      unsigned big = __ballot_sync(kFull, (n < n_hi) && !small);
      while (big) {
        const int j = __ffs(big) - 1;
        big &= big - 1;
        const int64_t lj = __shfl_sync(kFull, lo, j), hj = __shfl_sync(kFull, hi, j);
        float v;
        if (MODE == 0) v = fold_warp<IT>(q.col, inf_cur, q.w, q.w_bf16, q.w_uniform, q.w_val, lj, hj, lane);
        else v = __ldg(q.ptab + count_warp<MODE == 1>(q.col, gmask, lj, hj, lane));
        if (lane == j) q.out[n] = v;
      }
    }
  }
}

// incremental count mode: counts from scratch (engine start, host edits):
// cnt[n] = number of infectious in-neighbours in mask m; both pending-delta
// buffers cleared to the bias
__global__ void k_init_counts(const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                              const uint32_t* __restrict__ m, int64_t n, uint16_t* __restrict__ cnt,
                              uint32_t* __restrict__ d0, uint32_t* __restrict__ d1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int64_t e = __ldg(ro + i), e1 = __ldg(ro + i + 1); e < e1; ++e) {
      const int32_t j = __ldg(col + e);
      c += (int)((__ldg(m + (j >> 5)) >> (j & 31)) & 1u);
    }
    cnt[i] = (uint16_t)c;
    if ((i & 1) == 0) {
      d0[i >> 1] = kDeltaBias | (kDeltaBias << 16);
      d1[i >> 1] = kDeltaBias | (kDeltaBias << 16);
    }
  }
}

// first node n with row_offsets[n] >= chunk start, for every chunk boundary
__global__ void k_chunk_first(const int64_t* __restrict__ ro, int64_t n, int64_t e, int64_t epb,
                              int64_t nchunks, int64_t* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t target = (c == nchunks) ? e + 1 : c * epb;  // last boundary: past the end
    int64_t lo = 0, hi = n;  // search ro[0..n-1]
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (__ldg(ro + mid) < target) lo = mid + 1; else hi = mid;
    }
    out[c] = lo;
  }
}

// ptab[k] = k-fold sequential f32 sum of c (count-gather pressure table);
// *exact_mul = 1 when every entry equals the single product f32(k * c)
// (e.g. beta = 0.25 with unit weights), letting the kernels skip the lookup
__global__ void k_ptab(float* ptab, int64_t len, float c, int* exact_mul) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float acc = 0.0f;
    int ok = 1;
    ptab[0] = 0.0f;
    for (int64_t k = 1; k < len; ++k) {
      acc = __fadd_rn(acc, c);
      ptab[k] = acc;
      if (acc != __fmul_rn((float)k, c)) ok = 0;
    }
    *exact_mul = ok;
  }
}

// batch prologue (renewal.py:583-597): fold a pending step into the
// scalars, then reset tau unless carry_tau
__global__ void k_begin_batch(DevState* D, StepAcc* acc, int64_t* log_counts, int64_t log_cap,
                              int M, double eps, double tau_max, double delta, int carry_tau) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (D->pending) {
    const int64_t last = D->s.step - 1;
    const StepAcc* A = acc + last % 3;
    for (int c = 0; c < M; ++c) {
      D->s.counts[c] += (int64_t)A->d[c];
      log_counts[(last % log_cap) * kCntStride + c] = D->s.counts[c];
    }
    const float mx = __uint_as_float(A->max_bits);
    D->s.last_max_rate = mx;
    const double cand = __ddiv_rn(eps, __dadd_rn((double)mx, delta));
    D->s.tau_next = (tau_max <= cand) ? tau_max : cand;
    D->pending = 0;
  }
  if (!carry_tau) D->s.tau_next = tau_max;
  for (int j = 0; j < 3; ++j) {
    acc[j].max_bits = 0u;
    for (int c = 0; c < FS_MAX_COMPARTMENTS; ++c) acc[j].d[c] = 0ull;
  }
}

// compaction refresh at tile granularity: a 32-node tile is active if any of
// its nodes is non-terminal (renewal.py:426-432 at node granularity; results
// are identical because terminal nodes do rate-0 work either way)
template <typename ST>
__global__ void k_refresh_tiles(const ST* __restrict__ states, int64_t n, int64_t ntiles, uint32_t term_bits,
                                int32_t* __restrict__ tiles, int64_t* __restrict__ num_active) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t0 = warp_g * 32; t0 < ntiles; t0 += nwarps * 32) {
    // lane l inspects tile t0 + l
    const int64_t t = t0 + lane;
    bool act = false;
    if (t < ntiles) {
      for (int k = 0; k < 32; ++k) {
        const int64_t nd = t * 32 + k;
        if (nd >= n) break;
        if (!((term_bits >> (int)states[nd]) & 1u)) { act = true; break; }
      }
    }
    const unsigned b = __ballot_sync(kFull, act);
    int64_t base = 0;
    if (lane == 0 && b) base = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(num_active), (unsigned long long)__popc(b));
    base = __shfl_sync(kFull, base, 0);
    if (act) tiles[base + __popc(b & ((1u << lane) - 1u))] = (int32_t)t;
  }
}

__global__ void k_zero_i64(int64_t* p) { *p = 0; }

// copy the current double-buffer half (parity of S->step) onto the other
template <typename T>
__global__ void k_sync_buffers(const DevState* S, T* b0, T* b1, int64_t n) {
  const int cur = (int)(S->s.step & 1);
  const T* src = cur ? b1 : b0;
  T* dst = cur ? b0 : b1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

template <typename T>
__global__ void k_fill(T* p, int64_t n, T v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// count mode: mask <- (inf != 0); flags values that are neither 0 nor c
template <typename IT>
__global__ void k_load_mask(const IT* __restrict__ inf, int64_t n, float c, uint32_t* m0, uint32_t* m1,
                            int* bad) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ((n + 31) & ~31LL);
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = i < n ? to_f32<IT>(inf[i]) : 0.0f;
    const bool on = v != 0.0f;
    if (on && v != c) atomicExch(bad, 1);
    const unsigned w = __ballot_sync(kFull, on);
    if (lane == 0) { m0[i >> 5] = w; m1[i >> 5] = w; }
  }
}

template <typename IT>
__global__ void k_store_mask(const uint32_t* __restrict__ m, int64_t n, IT c, IT* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ((m[i >> 5] >> (i & 31)) & 1u) ? c : from_f32<IT>(0.0f);
}

// single-process exchange between the partition engines of one device (the
// virtual-rank emulation of fs_exchange_step used to test the partitioned
// kernels bit-exactly on one GPU): sum the count deltas and max the max-rate
// bits of slot `slot` over `count` accumulator rings, written back to all.
// The mask needs no exchange there: the engines share the mask buffers.
struct AccPtrs { StepAcc* a[FS_MAX_PARTITIONS]; };
__global__ void k_exchange_local(AccPtrs ptrs, int count, int slot) {
  const int t = threadIdx.x;
  if (t < FS_MAX_COMPARTMENTS) {
    unsigned long long sum = 0;
    for (int r = 0; r < count; ++r) sum += ptrs.a[r][slot].d[t];
    for (int r = 0; r < count; ++r) ptrs.a[r][slot].d[t] = sum;
  } else if (t == FS_MAX_COMPARTMENTS) {
    unsigned mx = 0;
    for (int r = 0; r < count; ++r) mx = max(mx, ptrs.a[r][slot].max_bits);
    for (int r = 0; r < count; ++r) ptrs.a[r][slot].max_bits = mx;
  }
}

// ---------------------------------------------------------------------------
// kernel selection
// ---------------------------------------------------------------------------
using StepFn = void (*)(const StepParams);
using MergeFn = void (*)(const MergeParams);

template <typename ST, typename AT, typename IT, bool MAT>
StepFn pick_step2(int gather, int strat, int& block) {
  switch (gather) {
    case G_COUNT_SMEM:
      block = 1024;
      return strat == S_WARP ? k_step<ST, AT, IT, G_COUNT_SMEM, S_WARP, MAT, 1024>
                             : k_step<ST, AT, IT, G_COUNT_SMEM, S_THREAD, MAT, 1024>;
    case G_COUNT_GLOBAL:
      block = 512;
      return strat == S_WARP ? k_step<ST, AT, IT, G_COUNT_GLOBAL, S_WARP, MAT, 512>
                             : k_step<ST, AT, IT, G_COUNT_GLOBAL, S_THREAD, MAT, 512>;
    case G_INCR:
      block = 512;
      return k_step<ST, AT, IT, G_INCR, S_THREAD, MAT, 512>;
    case G_F32:
      block = 512;
      return strat == S_WARP ? k_step<ST, AT, IT, G_F32, S_WARP, MAT, 512>
                             : k_step<ST, AT, IT, G_F32, S_THREAD, MAT, 512>;
    default:
      block = 512;
      return k_step<ST, AT, IT, G_PRE, S_THREAD, MAT, 512>;
  }
}

StepFn pick_step(bool mixed, int gather, int strat, bool mat, int& block) {
  if (mixed)
    return mat ? pick_step2<int8_t, __half, __nv_bfloat16, true>(gather, strat, block)
               : pick_step2<int8_t, __half, __nv_bfloat16, false>(gather, strat, block);
  return mat ? pick_step2<int32_t, float, float, true>(gather, strat, block)
             : pick_step2<int32_t, float, float, false>(gather, strat, block);
}

StepFn pick_stream(bool mixed, bool mat) {
  if (mixed) return mat ? k_step_incr<int8_t, __half, true, 512> : k_step_incr<int8_t, __half, false, 512>;
  return mat ? k_step_incr<int32_t, float, true, 512> : k_step_incr<int32_t, float, false, 512>;
}

using TmaFn = void (*)(const StepParams, const TmaLayout);

template <typename ST, typename AT, bool SM, bool MAT, int B>
TmaFn pick_tma3(bool ptab_mul) {
  return ptab_mul ? k_step_tma<ST, AT, SM, MAT, true, B> : k_step_tma<ST, AT, SM, MAT, false, B>;
}
template <typename ST, typename AT, int B>
TmaFn pick_tma2(bool smem_mask, bool mat, bool ptab_mul) {
  if (smem_mask) return mat ? pick_tma3<ST, AT, true, true, B>(ptab_mul) : pick_tma3<ST, AT, true, false, B>(ptab_mul);
  return mat ? pick_tma3<ST, AT, false, true, B>(ptab_mul) : pick_tma3<ST, AT, false, false, B>(ptab_mul);
}
TmaFn pick_tma(bool mixed, bool smem_mask, bool mat, bool ptab_mul, int block) {
  if (block == 768)
    return mixed ? pick_tma2<int8_t, __half, 768>(smem_mask, mat, ptab_mul) : pick_tma2<int32_t, float, 768>(smem_mask, mat, ptab_mul);
  return mixed ? pick_tma2<int8_t, __half, 512>(smem_mask, mat, ptab_mul) : pick_tma2<int32_t, float, 512>(smem_mask, mat, ptab_mul);
}

// widest 16-byte-aligned column span of any 32-node tile (TMA slot size)
__global__ void k_max_tile_span(const int32_t* __restrict__ ro32, int64_t n, int64_t ntiles, unsigned long long* out) {
  unsigned long long best = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = ro32[t * 32], e1 = ro32[min((t + 1) * 32, n)];
    const unsigned long long span = (unsigned long long)(((e1 + 3) & ~3LL) - (e0 & ~3LL));
    best = span > best ? span : best;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
    best = v > best ? v : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

MergeFn pick_merge(bool inf_bf16, int mode, int& block) {
  if (mode == 1) { block = 1024; return inf_bf16 ? k_gather_merge<__nv_bfloat16, 1, 1024> : k_gather_merge<float, 1, 1024>; }
  block = 512;
  if (mode == 2) return inf_bf16 ? k_gather_merge<__nv_bfloat16, 2, 512> : k_gather_merge<float, 2, 512>;
  return inf_bf16 ? k_gather_merge<__nv_bfloat16, 0, 512> : k_gather_merge<float, 0, 512>;
}

}  // namespace fs

// ===========================================================================
// engine object + C ABI
// ===========================================================================
using namespace fs;

struct fs_engine {
  int device = 0;
  int sms = 0;
  fs_graph g{};
  fs_model m{};
  fs_config c{};
  fs_state_buffers b{};
  bool count_mode = false;
  bool mask_smem = false;
  bool mixed = false;
  int gather = G_F32;
  int strat = S_THREAD;
  bool merge = false;
  int64_t ntiles = 0;
  // node partition (fs_engine_create_partitioned); defaults = whole graph
  int64_t node_base = 0;
  int64_t ntiles_mask = 0;   // words of the global infectious mask
  int rank = 0, world = 1;
  void* comm = nullptr;
  int64_t mask_seg_words = 0;  // words of mask each rank contributes to the all-gather      // ncclComm_t: per-step exchange after every step kernel
  int64_t h_step = 0;        // host mirror of the device step counter (exchange slot / mask parity)
  float inf_val = 0.0f;  // promoted stored value of an I node (count mode)
  // launch shapes
  StepFn step_fn[2] = {nullptr, nullptr};
  bool tma = false;       // streaming count-gather kernel (k_step_tma)
  TmaFn tma_fn[2] = {nullptr, nullptr};
  TmaLayout tl{};
  int tma_cluster = 1;    // CTAs sharing one multicast mask fetch
  bool pdl = true;        // programmatic dependent launch between steps
  int tma_block = 512;    // threads per CTA of the streaming kernel
  unsigned long long* dbg = nullptr;  // FS_DEBUG_TIMES: per-CTA timestamps
  int step_block = 512, step_grid = 0, step_grid_general = 0;
  size_t step_smem = 0, step_smem_general = 0;
  MergeFn merge_fn = nullptr;
  int merge_block = 512, merge_grid = 0;
  size_t merge_smem = 0;
  int64_t nchunks = 0;
  // engine-owned device scratch
  DevState* dstate = nullptr;  // [2] ping-pong run scalars
  int s_cur = 0;               // which slot is current (host-tracked parity)
  StepAcc* acc = nullptr;      // [3] per-step accumulators
  double* log_clock = nullptr;
  double* log_tau = nullptr;
  int64_t* log_counts = nullptr;
  int64_t log_cap = 0;
  float* ptab = nullptr;
  int64_t ptab_len = 0;
  int ptab_mul = 0;
  float ptab_c = 0.0f;
  int32_t* active_tiles = nullptr;
  int64_t* num_active = nullptr;
  int64_t* chunk_first = nullptr;
  float* pre = nullptr;
  int* bad_flag = nullptr;
  // CUDA graphs of one batch (index: materialise last step)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t batch_exec[2][2][6] = {};  // [materialise][scalar slot][step % 6]: parity and exchange slot are baked in
  bool compaction_ready = false;
  int stream_evict_first = 0;
  // incremental count mode
  int32_t* entry = nullptr;           // hazard memo: per-node entry step
  bool incr = false;
  uint32_t* peer_pend[2][FS_MAX_PARTITIONS] = {};  // partitioned incremental: every rank's delta arrays
  bool peers_linked = false;
  bool stream = false;         // k_step_stream fast path of the incremental mode
  StepFn stream_fn[2] = {nullptr, nullptr};
  int stream_grid = 0;
  uint16_t* cnt = nullptr;
  uint32_t* delta[2] = {nullptr, nullptr};
};

namespace {

#define FS_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t err__ = (call);                                                               \
    if (err__ != cudaSuccess)                                                                 \
      return set_error(FS_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(err__), \
                       __FILE__, __LINE__);                                                   \
  } while (0)

template <typename T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t err = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (err != cudaSuccess) return set_error(FS_ENOMEM, "cudaMalloc(%zu B): %s", count * sizeof(T), cudaGetErrorString(err));
  return 0;
}

StepParams make_step_params(const fs_engine* e, bool use_pre, bool use_active, int in_slot) {
  StepParams p{};
  p.ro = e->g.row_offsets;
  p.ro32 = e->g.row_offsets32;
  p.col = e->g.col_indices;
  p.w = e->g.weights;
  p.w_bf16 = e->g.weights_dtype == FS_BF16;
  p.w_uniform = e->g.weights_uniform;
  p.w_val = e->g.uniform_weight;
  p.n = e->g.num_nodes;
  p.ntiles = e->ntiles;
  p.node_base = e->node_base;
  p.tile_base = e->node_base / 32;
  p.ntiles_mask = e->ntiles_mask;
  p.states = e->b.states;
  p.ages = e->b.ages;
  p.inf[0] = e->b.infectivity[0];
  p.inf[1] = e->b.infectivity[1];
  p.mask[0] = e->b.imask[0];
  p.mask[1] = e->b.imask[1];
  p.pressure = e->b.pressure;
  p.rates = e->b.rates;
  p.Sin = e->dstate + in_slot;
  p.Sout = e->dstate + (in_slot ^ 1);
  p.acc = e->acc;
  p.log_clock = e->log_clock;
  p.log_tau = e->log_tau;
  p.log_counts = e->log_counts;
  p.log_cap = e->log_cap;
  p.ptab = e->ptab;
  p.ptab_mul = e->ptab_mul;
  p.ptab_c = e->ptab_c;
  p.active_tiles = (use_active && e->c.compaction) ? e->active_tiles : nullptr;
  p.num_active = e->num_active;
  p.pre = use_pre ? e->pre : nullptr;
  p.count_mode = e->count_mode;
  p.stream_evict_first = e->stream_evict_first;
  p.host_parity = (int)(e->h_step & 1);
  p.entry = e->entry;
  p.cnt = e->incr ? e->cnt : nullptr;
  p.pend[0] = e->delta[0];
  p.pend[1] = e->delta[1];
  p.out_ro = e->g.out_row_offsets;
  p.out_col = e->g.out_col_indices;
  p.world = e->incr ? e->world : 1;
  p.part_chunk = e->mask_seg_words * 32;
  for (int par = 0; par < 2; ++par)
    for (int r = 0; r < FS_MAX_PARTITIONS; ++r) p.peer_pend[par][r] = e->peer_pend[par][r];
  p.dbg = e->dbg;
  p.model = e->m;
  p.eps = e->c.epsilon;
  p.tau_max = e->c.tau_max;
  p.delta = e->c.delta;
  p.rng = e->c.rng;
  p.hprec = e->c.hazard_precision;
  p.inf_val = e->inf_val;
  return p;
}

MergeParams make_merge_params(const fs_engine* e) {
  MergeParams q{};
  q.ro = e->g.row_offsets;
  q.ro32 = e->g.row_offsets32;
  q.col = e->g.col_indices;
  q.w = e->g.weights;
  q.w_bf16 = e->g.weights_dtype == FS_BF16;
  q.w_uniform = e->g.weights_uniform;
  q.w_val = e->g.uniform_weight;
  q.n = e->g.num_nodes;
  q.e = e->g.num_edges;
  q.epb = e->c.edges_per_block;
  q.nchunks = e->nchunks;
  q.chunk_first = e->chunk_first;
  q.inf[0] = e->b.infectivity[0];
  q.inf[1] = e->b.infectivity[1];
  q.inf_bf16 = e->mixed;
  q.mask[0] = e->b.imask[0];
  q.mask[1] = e->b.imask[1];
  q.ptab = e->ptab;
  q.S = e->dstate + e->s_cur;
  q.out = e->pre;
  q.nwords = e->ntiles_mask;
  return q;
}

int launch_steps(fs_engine* e, int nsteps, bool materialize_last, bool use_active, cudaStream_t st) {
  if (e->incr && e->world > 1 && !e->peers_linked)
    return set_error(FS_ESTATE, "partitioned incremental engine: link the ranks' delta buffers first");
  for (int k = 0; k < nsteps; ++k) {
    const bool mat = materialize_last && (k == nsteps - 1);
    if (e->merge) {
      MergeParams q = make_merge_params(e);
      e->merge_fn<<<e->merge_grid, e->merge_block, e->merge_smem, st>>>(q);
    }
    StepParams p = make_step_params(e, e->merge, use_active, e->s_cur);
    if (e->stream && !p.active_tiles) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(e->stream_grid);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = 0;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = e->pdl ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      FS_CUDA(cudaLaunchKernelEx(&cfg, e->stream_fn[mat], p));
    } else if (e->tma && !p.active_tiles) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(e->step_grid);
      cfg.blockDim = dim3(e->tma_block);
      cfg.dynamicSmemBytes = e->step_smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = e->tma_cluster;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = e->pdl ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      FS_CUDA(cudaLaunchKernelEx(&cfg, e->tma_fn[mat], p, e->tl));
    }
    else
      e->step_fn[mat]<<<e->step_grid_general, e->step_block, e->step_smem_general, st>>>(p);
    e->s_cur ^= 1;
    if (e->comm) {
      // step h_step is complete on this rank: make its accumulator and the
      // next-step mask global
      const int slot = (int)(e->h_step % 3);
      uint32_t* mask_nxt = e->b.imask[(e->h_step & 1) ^ 1];
      // incremental counts travel as peer pushes during the step: only the
      // accumulator is reduced; otherwise the next-step mask is all-gathered
      const int rc = fs_exchange_step(e->comm, &e->acc[slot].d[0], &e->acc[slot].max_bits, e->incr ? nullptr : mask_nxt,
                                      e->mask_seg_words, e->rank, st);
      if (rc) return rc;
    }
    ++e->h_step;
  }
  FS_CUDA(cudaGetLastError());
  return 0;
}

int launch_begin_batch(fs_engine* e, cudaStream_t st) {
  k_begin_batch<<<1, 32, 0, st>>>(e->dstate + e->s_cur, e->acc, e->log_counts, e->log_cap, e->m.num_compartments,
                                  e->c.epsilon, e->c.tau_max, e->c.delta, e->c.carry_tau);
  if (e->c.compaction) {
    uint32_t term_bits = 0;
    for (int i = 0; i < e->m.num_compartments; ++i)
      if (e->m.comp[i].terminal) term_bits |= 1u << i;
    const int64_t n = e->g.num_nodes;
    // rates are zeroed once per batch under compaction (renewal.py:594)
    if (e->b.rates) k_fill<float><<<e->sms * 4, 256, 0, st>>>(e->b.rates, n, 0.0f);
    if (e->b.pressure) k_fill<float><<<e->sms * 4, 256, 0, st>>>(e->b.pressure, n, 0.0f);
    k_zero_i64<<<1, 1, 0, st>>>(e->num_active);
    const int blocks = (int)std::min<int64_t>((e->ntiles + 255) / 256 + 1, (int64_t)e->sms * 8);
    if (e->mixed)
      k_refresh_tiles<int8_t><<<blocks, 256, 0, st>>>((const int8_t*)e->b.states, n, e->ntiles, term_bits,
                                                      e->active_tiles, e->num_active);
    else
      k_refresh_tiles<int32_t><<<blocks, 256, 0, st>>>((const int32_t*)e->b.states, n, e->ntiles, term_bits,
                                                       e->active_tiles, e->num_active);
    // inactive tiles are never rewritten: make both buffers agree on them
    const int blocks2 = (int)std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8);
    if (e->count_mode)
      k_sync_buffers<uint32_t><<<blocks2, 256, 0, st>>>(e->dstate + e->s_cur, e->b.imask[0], e->b.imask[1], e->ntiles_mask);
    else if (e->mixed)
      k_sync_buffers<__nv_bfloat16><<<blocks2, 256, 0, st>>>(e->dstate + e->s_cur, (__nv_bfloat16*)e->b.infectivity[0],
                                                             (__nv_bfloat16*)e->b.infectivity[1], n);
    else
      k_sync_buffers<float><<<blocks2, 256, 0, st>>>(e->dstate + e->s_cur, (float*)e->b.infectivity[0], (float*)e->b.infectivity[1], n);
  }
  FS_CUDA(cudaGetLastError());
  return 0;
}

// hazard memo: every node's cohort unknown, every slot's tag stale
int reset_memo(fs_engine* e, cudaStream_t st) {
  if (!e->entry) return 0;
  const int64_t n = (e->g.num_nodes + 127) / 128 * 128;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8);
  k_fill<int32_t><<<std::max(1, blocks), 256, 0, st>>>(e->entry, n, kEntryInvalid);
  FS_CUDA(cudaGetLastError());
  return 0;
}

// incremental counts from the current mask (buffer of step parity `step`)
int recount(fs_engine* e, int64_t step, cudaStream_t st) {
  if (!e->incr) return 0;
  const int64_t n = e->g.num_nodes;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8);
  k_init_counts<<<std::max(1, blocks), 256, 0, st>>>(e->g.row_offsets, e->g.col_indices, e->b.imask[step & 1], n,
                                                     e->cnt, e->delta[0], e->delta[1]);
  FS_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace

extern "C" {

int fs_abi_version(void) { return FS_ABI_VERSION; }
const char* fs_last_error(void) { return g_last_error.c_str(); }

int fs_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

static int engine_create(const fs_graph* g, const fs_model* m, const fs_config* c, const fs_state_buffers* buf,
                         const fs_scalars* scal, int device, const fs_partition* part, fs_engine** out) {
  if (!g || !m || !c || !buf || !scal || !out) return set_error(FS_EINVAL, "null argument");
  *out = nullptr;
  if (g->num_nodes < 1 || g->num_nodes > 2147483647LL) return set_error(FS_EINVAL, "num_nodes %lld outside [1, 2^31-1]", (long long)g->num_nodes);
  if (m->num_compartments < 1 || m->num_compartments > FS_MAX_COMPARTMENTS)
    return set_error(FS_EINVAL, "num_compartments %d outside [1, %d]", m->num_compartments, FS_MAX_COMPARTMENTS);
  if (c->strategy < FS_PER_NODE || c->strategy > FS_MERGE) return set_error(FS_EINVAL, "strategy must be resolved (got %d)", c->strategy);
  if (c->steps_per_batch < 1) return set_error(FS_EINVAL, "steps_per_batch must be >= 1");
  if (c->edges_per_block < 1) return set_error(FS_EINVAL, "edges_per_block must be >= 1");
  if (!buf->states || !buf->ages) return set_error(FS_EINVAL, "state buffers missing");
  FS_CUDA(cudaSetDevice(device));
  fs_engine* e = new fs_engine();
  e->device = device;
  e->sms = fs_device_sm_count(device);
  e->g = *g;
  e->m = *m;
  e->c = *c;
  e->b = *buf;
  e->mixed = c->mixed_precision != 0;
  const int64_t n = g->num_nodes;
  e->ntiles = (n + 31) / 32;
  e->ntiles_mask = e->ntiles;
  e->h_step = scal->step;
  if (part) {
    if (part->node_base < 0 || part->node_base % 32 != 0 || part->num_nodes_global < part->node_base + n ||
        part->num_nodes_global > 2147483647LL || part->world < 1 || part->rank < 0 || part->rank >= part->world) {
      delete e;
      return set_error(FS_EINVAL, "bad partition (node_base %lld must be a multiple of 32, N_global %lld)",
                       (long long)part->node_base, (long long)part->num_nodes_global);
    }
    e->node_base = part->node_base;
    e->ntiles_mask = (part->num_nodes_global + 31) / 32;
    e->rank = part->rank;
    e->world = part->world;
    e->comm = part->comm;
    e->mask_seg_words = part->mask_segment_words;
    if ((e->comm || e->world > 1) && (e->mask_seg_words < 1 || e->mask_seg_words * e->world < e->ntiles_mask ||
                    e->node_base / 32 != (int64_t)e->rank * e->mask_seg_words)) {
      delete e;
      return set_error(FS_EINVAL, "partition: ranks must own equal mask segments of mask_segment_words words");
    }
  }
  const bool can_count = (m->shedding == FS_SHED_CONSTANT) && (g->weights_uniform || g->num_edges == 0);
  e->count_mode = can_count && c->count_gather != 0;
  if (part && !e->count_mode) { delete e; return set_error(FS_EINVAL, "partitioned runs need the count gather (constant transmission, uniform weights)"); }
  if (c->count_gather == 1 && !can_count) { delete e; return set_error(FS_EINVAL, "count gather requires constant transmission and uniform weights"); }
  if (e->count_mode && (!buf->imask[0] || !buf->imask[1])) { delete e; return set_error(FS_EINVAL, "count gather needs the two mask buffers"); }
  if (!e->count_mode && (!buf->infectivity[0] || !buf->infectivity[1])) { delete e; return set_error(FS_EINVAL, "f32 gather needs the two infectivity buffers"); }
  // stored value of an infectious node and the per-edge contribution
  {
    float bf = (float)m->beta;
    if (e->mixed) bf = __bfloat162float(__float2bfloat16_rn(bf));
    e->inf_val = bf;
  }
  e->mask_smem = e->count_mode && (size_t)e->ntiles_mask * 4 <= kMaxSmemMaskBytes;
  // incremental counts: count gather + an outgoing CSR to push along, single
  // partition, degrees below the 2^15 delta headroom
  const bool can_incr = e->count_mode && g->out_row_offsets && g->out_col_indices && g->d_max < 32768 &&
                        g->num_edges > 0 && (!part || part->mask_segment_words > 0);
  if (c->incremental == 1 && !can_incr) { delete e; return set_error(FS_EINVAL, "incremental counts need the count gather, an outgoing CSR, d_max < 32768 and one partition"); }
  e->incr = can_incr && c->incremental != 0;
  e->merge = c->strategy == FS_MERGE && g->num_edges > 0 && !e->incr;
  e->strat = c->strategy == FS_LANE ? S_WARP : S_THREAD;
  if (e->incr) e->gather = G_INCR;
  else if (e->merge) e->gather = G_PRE;
  else if (e->count_mode) e->gather = e->mask_smem ? G_COUNT_SMEM : G_COUNT_GLOBAL;
  else e->gather = G_F32;

  int rc = 0;
#define TRY(x) do { rc = (x); if (rc) { fs_engine_destroy(e); return rc; } } while (0)
  for (int mat = 0; mat < 2; ++mat) e->step_fn[mat] = pick_step(e->mixed, e->gather, e->strat, mat != 0, e->step_block);
  e->step_smem = (e->gather == G_COUNT_SMEM) ? (size_t)((e->ntiles_mask + 3) & ~3LL) * 4 : 0;
  int occ = 1;
  for (int mat = 0; mat < 2; ++mat) {
    if (e->step_smem > 0)
      TRY(cudaFuncSetAttribute((const void*)e->step_fn[mat], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->step_smem) == cudaSuccess ? 0 : set_error(FS_ECUDA, "smem attribute"));
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)e->step_fn[1], e->step_block, e->step_smem) != cudaSuccess || occ < 1) occ = 1;
  // the step loops over 32-node tiles; do not launch CTAs with no tile
  {
    const int64_t warps_needed = e->ntiles;
    const int64_t ctas_needed = (warps_needed + e->step_block / 32 - 1) / (e->step_block / 32);
    e->step_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)e->sms * occ, ctas_needed));
  }
  TRY(dalloc(&e->bad_flag, 1));
  if (e->count_mode) {
    e->ptab_len = (int64_t)g->d_max + 1;
    TRY(dalloc(&e->ptab, e->ptab_len));
    volatile float a_ = e->inf_val, w_ = g->uniform_weight;
    const float cval = a_ * w_;  // f32(inf * w): one IEEE single multiply
    FS_CUDA(cudaMemset(e->bad_flag, 0, sizeof(int)));
    k_ptab<<<1, 1>>>(e->ptab, e->ptab_len, cval, e->bad_flag);
    FS_CUDA(cudaMemcpy(&e->ptab_mul, e->bad_flag, sizeof(int), cudaMemcpyDeviceToHost));
    e->ptab_c = cval;
  }
  {
    // column stream + per-node arrays larger than half the L2: stream them
    // with evict-first so the randomly read mask keeps its lines
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    const double ws = 4.0 * (double)g->num_edges + 16.0 * (double)n;
    e->stream_evict_first = (l2 > 0 && ws > 0.5 * (double)l2) ? 1 : 0;
    if (getenv("FS_NO_EVICT_HINT")) e->stream_evict_first = 0;
  }
  e->step_grid_general = e->step_grid;
  e->step_smem_general = e->step_smem;
  // streaming fast path: count gather, PER_NODE, padded buffers, int32 offsets
  if (e->count_mode && !e->incr && c->strategy == FS_PER_NODE && !e->merge && g->row_offsets32 && g->padded && buf->padded &&
      g->num_edges > 0) {
    unsigned long long* d_span = nullptr;
    TRY(dalloc(&d_span, 1));
    FS_CUDA(cudaMemset(d_span, 0, sizeof(unsigned long long)));
    k_max_tile_span<<<(int)std::min<int64_t>((e->ntiles + 255) / 256, 4096), 256>>>(g->row_offsets32, n, e->ntiles, d_span);
    unsigned long long span = 0;
    FS_CUDA(cudaMemcpy(&span, d_span, sizeof(span), cudaMemcpyDeviceToHost));
    cudaFree(d_span);
    TmaLayout L{};
    L.ro_off = L.st_off = L.ag_off = L.col_off = 0;  // slots hold the column slice only
    L.col_cap = (int)std::min<unsigned long long>(span, 1ull << 20);
    L.slot_bytes = (int)((4 * (int64_t)L.col_cap + 127) & ~127LL);
    const size_t mask_bytes = (size_t)((e->ntiles_mask + 1 + 3) & ~3LL) * 4;  // + zero sentinel word
    cudaFuncAttributes fa{};
    if (getenv("FS_TMA_BLOCK")) e->tma_block = atoi(getenv("FS_TMA_BLOCK")) == 768 ? 768 : 512;
    const int warps = e->tma_block / 32;
    int dev_smem = 0;
    cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    for (int smem_mask = 1; smem_mask >= 0 && !e->tma; --smem_mask) {
      TmaFn f0 = pick_tma(e->mixed, smem_mask != 0, false, e->ptab_mul != 0, e->tma_block);
      if (cudaFuncGetAttributes(&fa, (const void*)f0) != cudaSuccess) break;
      const int max_slots = getenv("FS_TMA_SLOTS") ? atoi(getenv("FS_TMA_SLOTS")) : 4;
      for (int slots = std::min(4, std::max(2, max_slots)); slots >= 2; --slots) {
        const size_t dyn = (smem_mask ? mask_bytes : 0) + (size_t)warps * slots * L.slot_bytes;
        if (dyn + fa.sharedSizeBytes + 1024 > (size_t)dev_smem) continue;
        L.slots = slots;
        e->tl = L;
        e->tma = true;
        e->step_smem = dyn;
        for (int mat = 0; mat < 2; ++mat) {
          e->tma_fn[mat] = pick_tma(e->mixed, smem_mask != 0, mat != 0, e->ptab_mul != 0, e->tma_block);
          TRY(cudaFuncSetAttribute((const void*)e->tma_fn[mat], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) == cudaSuccess ? 0 : set_error(FS_ECUDA, "tma smem attribute"));
        }
        int tocc = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, (const void*)e->tma_fn[0], e->tma_block, dyn) != cudaSuccess || tocc < 1) tocc = 1;
        const int64_t ctas_needed = (e->ntiles + warps - 1) / warps;
        e->step_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)e->sms * tocc, ctas_needed));
        // pairs of CTAs share the mask fetch (cluster of 2 packs all 148 SMs)
        e->tma_cluster = (smem_mask && e->step_grid >= 2) ? 2 : 1;
        if (e->tma_cluster > 1) e->step_grid -= e->step_grid % e->tma_cluster;
        break;
      }
    }
  }
  if (e->merge) {
    const int mode = e->count_mode ? (e->mask_smem ? 1 : 2) : 0;
    e->merge_fn = pick_merge(e->mixed, mode, e->merge_block);
    e->merge_smem = mode == 1 ? (size_t)e->ntiles_mask * 4 : 0;
    if (e->merge_smem)
      TRY(cudaFuncSetAttribute((const void*)e->merge_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->merge_smem) == cudaSuccess ? 0 : set_error(FS_ECUDA, "smem attribute"));
    int mocc = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&mocc, (const void*)e->merge_fn, e->merge_block, e->merge_smem) != cudaSuccess || mocc < 1) mocc = 1;
    e->nchunks = (g->num_edges + c->edges_per_block - 1) / c->edges_per_block;
    const int64_t ctas_needed = (e->nchunks + e->merge_block / 32 - 1) / (e->merge_block / 32);
    e->merge_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)e->sms * mocc, ctas_needed));
  }

  TRY(dalloc(&e->dstate, 2));
  TRY(dalloc(&e->acc, 3));
  e->log_cap = std::max<int64_t>(256, 4 * (int64_t)c->steps_per_batch);
  TRY(dalloc(&e->log_clock, e->log_cap));
  TRY(dalloc(&e->log_tau, e->log_cap));
  TRY(dalloc(&e->log_counts, (size_t)e->log_cap * kCntStride));
  TRY(dalloc(&e->num_active, 1));
  if (c->compaction) TRY(dalloc(&e->active_tiles, e->ntiles));
  FS_CUDA(cudaMemset(e->acc, 0, 3 * sizeof(StepAcc)));
  FS_CUDA(cudaMemset(e->num_active, 0, sizeof(int64_t)));
  {
    DevState d0{};
    d0.s = *scal;
    d0.pending = 0;
    FS_CUDA(cudaMemcpy(e->dstate, &d0, sizeof(DevState), cudaMemcpyHostToDevice));
    e->s_cur = 0;
  }
  if (e->merge) {
    TRY(dalloc(&e->chunk_first, e->nchunks + 1));
    TRY(dalloc(&e->pre, n));
    FS_CUDA(cudaMemset(e->pre, 0, n * sizeof(float)));
    k_chunk_first<<<(int)std::min<int64_t>((e->nchunks + 256) / 256, 4096), 256>>>(g->row_offsets, n, g->num_edges,
                                                                                  c->edges_per_block, e->nchunks, e->chunk_first);
  }
  if (e->incr) {
    const size_t cap = (size_t)((n + 127) / 128) * 128;  // whole 128-node stream units
    TRY(dalloc(&e->cnt, cap));
    TRY(dalloc(&e->delta[0], cap / 2));
    TRY(dalloc(&e->delta[1], cap / 2));
    TRY(recount(e, scal->step, nullptr));
    // streaming kernel: per-node arrays readable to a multiple of 128 nodes
    if (buf->padded >= 2 && !getenv("FS_NO_STREAM")) {
      e->stream = true;
      for (int mat = 0; mat < 2; ++mat) e->stream_fn[mat] = pick_stream(e->mixed, mat != 0);
      int socc = 1;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&socc, (const void*)e->stream_fn[0], 512, 0) != cudaSuccess || socc < 1) socc = 1;
      if (getenv("FS_INCR_CTAS_PER_SM")) socc = std::max(1, std::min(socc, atoi(getenv("FS_INCR_CTAS_PER_SM"))));
      e->stream_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)e->sms * socc, (e->ntiles + 15) / 16));
    }
  }
  {
    // hazard memo for models with age-dependent holding times
    bool costly = false;
    for (int c2 = 0; c2 < m->num_compartments; ++c2) costly |= m->comp[c2].hazard >= FS_HZ_LOGNORMAL;
    // the memo pays off when a CTA holds many nodes of each age cohort
    // (large N); at N ~ 1e6 its setup costs more than it saves
    const char* mv = getenv("FS_MEMO");
    const bool want = mv ? atoi(mv) != 0 : (e->incr && n >= (int64_t)8 * 1024 * 1024);
    if (costly && want && !getenv("FS_NO_MEMO")) {
      TRY(dalloc(&e->entry, (size_t)((n + 127) / 128) * 128));
      TRY(reset_memo(e, nullptr));
    }
  }
  if (getenv("FS_NO_PDL")) e->pdl = false;
  if (getenv("FS_DEBUG_TIMES")) {
    TRY(dalloc(&e->dbg, (size_t)std::max(e->step_grid, e->step_grid_general) * 4 * 16));
    FS_CUDA(cudaMemset(e->dbg, 0, sizeof(unsigned long long) * std::max(e->step_grid, e->step_grid_general) * 4 * 16));
  }
  FS_CUDA(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
  FS_CUDA(cudaGetLastError());
  FS_CUDA(cudaDeviceSynchronize());
#undef TRY
  *out = e;
  return 0;
}

int fs_engine_create(const fs_graph* g, const fs_model* m, const fs_config* c, const fs_state_buffers* buf,
                     const fs_scalars* scal, int device, fs_engine** out) {
  return engine_create(g, m, c, buf, scal, device, nullptr, out);
}

int fs_engine_create_partitioned(const fs_graph* g, const fs_model* m, const fs_config* c,
                                 const fs_state_buffers* buf, const fs_scalars* scal, int device,
                                 const fs_partition* part, fs_engine** out) {
  if (!part) return set_error(FS_EINVAL, "null partition");
  return engine_create(g, m, c, buf, scal, device, part, out);
}

void fs_engine_destroy(fs_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  for (auto& a : e->batch_exec)
    for (auto& b : a)
      for (auto& x : b) if (x) cudaGraphExecDestroy(x);
  if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
  void* ptrs[] = {e->dstate, e->acc, e->log_clock, e->log_tau, e->log_counts, e->ptab,
                  e->active_tiles, e->num_active, e->chunk_first, e->pre, e->bad_flag,
                  e->cnt, e->delta[0], e->delta[1], e->entry};
  for (void* q : ptrs) if (q) cudaFree(q);
  delete e;
}

int fs_engine_uses_count_gather(const fs_engine* e) { return e && e->count_mode ? 1 : 0; }

int fs_engine_current_buffer(fs_engine* e, void* stream) {
  fs_scalars s;
  int rc = fs_engine_get_scalars(e, &s, stream);
  if (rc) return rc;
  return (int)(s.step & 1);
}

int fs_engine_begin_batch(fs_engine* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  FS_CUDA(cudaSetDevice(e->device));
  return launch_begin_batch(e, (cudaStream_t)stream);
}

int fs_engine_step(fs_engine* e, int32_t nsteps, int32_t materialize, int32_t use_active, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  if (nsteps < 0) return set_error(FS_EINVAL, "nsteps < 0");
  if (materialize && (!e->b.pressure || !e->b.rates)) return set_error(FS_EINVAL, "materialize needs pressure/rates buffers");
  FS_CUDA(cudaSetDevice(e->device));
  if (use_active && !e->c.compaction) return set_error(FS_EINVAL, "engine built without compaction");
  return launch_steps(e, nsteps, materialize != 0, use_active != 0, (cudaStream_t)stream);
}

int fs_engine_run_batch(fs_engine* e, int32_t materialize, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  if (materialize && (!e->b.pressure || !e->b.rates)) return set_error(FS_EINVAL, "materialize needs pressure/rates buffers");
  FS_CUDA(cudaSetDevice(e->device));
  // one graph per (materialise, starting scalar slot): the kernels' slot
  // pointers are baked in at capture
  const int s0 = e->s_cur;
  const int64_t h0 = e->h_step;
  // the exchange's accumulator slot and mask buffer are baked in at capture
  cudaGraphExec_t& exec = e->batch_exec[materialize ? 1 : 0][s0][(int)(h0 % 6)];
  if (!exec) {
    cudaGraph_t graph = nullptr;
    FS_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = launch_begin_batch(e, e->cap_stream);
    if (!rc) rc = launch_steps(e, e->c.steps_per_batch, materialize != 0, e->c.compaction != 0, e->cap_stream);
    cudaError_t err = cudaStreamEndCapture(e->cap_stream, &graph);
    e->s_cur = s0;  // capture does not execute
    e->h_step = h0;
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (err != cudaSuccess) return set_error(FS_ECUDA, "graph capture: %s", cudaGetErrorString(err));
    err = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (err != cudaSuccess) return set_error(FS_ECUDA, "graph instantiate: %s", cudaGetErrorString(err));
  }
  FS_CUDA(cudaGraphLaunch(exec, (cudaStream_t)stream));
  e->s_cur = s0 ^ (e->c.steps_per_batch & 1);
  e->h_step = h0 + e->c.steps_per_batch;
  return 0;
}

// current scalars with a pending step folded in (host side, no writes)
static int read_state(fs_engine* e, DevState* d, StepAcc* a, cudaStream_t st) {
  FS_CUDA(cudaMemcpyAsync(d, e->dstate + e->s_cur, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaMemcpyAsync(a, e->acc, 3 * sizeof(StepAcc), cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaStreamSynchronize(st));
  if (d->pending) {
    const StepAcc& A = a[(d->s.step - 1) % 3];
    for (int c = 0; c < e->m.num_compartments; ++c) d->s.counts[c] += (int64_t)A.d[c];
    float mx;
    std::memcpy(&mx, &A.max_bits, sizeof mx);
    d->s.last_max_rate = mx;
    const double cand = e->c.epsilon / ((double)mx + e->c.delta);  // same IEEE f64 ops as the device
    d->s.tau_next = (e->c.tau_max <= cand) ? e->c.tau_max : cand;
  }
  return 0;
}

int fs_engine_read_log(fs_engine* e, int64_t first_step, int32_t n, double* clocks, double* taus, int64_t* counts,
                       void* stream) {
  if (!e || n < 0) return set_error(FS_EINVAL, "bad log request");
  if (n > e->log_cap) return set_error(FS_EINVAL, "log request of %d steps exceeds capacity %lld", n, (long long)e->log_cap);
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  DevState d;
  StepAcc a[3];
  int rc0 = read_state(e, &d, a, st);
  if (rc0) return rc0;
  std::vector<double> lc(e->log_cap), lt(e->log_cap);
  std::vector<int64_t> lk((size_t)e->log_cap * kCntStride);
  FS_CUDA(cudaMemcpyAsync(lc.data(), e->log_clock, lc.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaMemcpyAsync(lt.data(), e->log_tau, lt.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaMemcpyAsync(lk.data(), e->log_counts, lk.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaStreamSynchronize(st));
  const int M = e->m.num_compartments;
  for (int i = 0; i < n; ++i) {
    const int64_t slot = (first_step + i) % e->log_cap;
    if (clocks) clocks[i] = lc[slot];
    if (taus) taus[i] = lt[slot];
    const bool last_pending = d.pending && first_step + i == d.s.step - 1;  // counts not yet folded on device
    if (counts)
      for (int c2 = 0; c2 < M; ++c2)
        counts[(size_t)i * M + c2] = last_pending ? d.s.counts[c2] : lk[slot * kCntStride + c2];
  }
  return 0;
}

int fs_engine_get_scalars(fs_engine* e, fs_scalars* out, void* stream) {
  if (!e || !out) return set_error(FS_EINVAL, "null argument");
  FS_CUDA(cudaSetDevice(e->device));
  DevState d;
  StepAcc a[3];
  int rc = read_state(e, &d, a, (cudaStream_t)stream);
  if (rc) return rc;
  *out = d.s;
  return 0;
}

int fs_engine_set_scalars(fs_engine* e, const fs_scalars* in, void* stream) {
  if (!e || !in) return set_error(FS_EINVAL, "null argument");
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  DevState d{};
  d.s = *in;
  d.pending = 0;
  // a pending step must be folded first so no count delta is lost
  DevState cur;
  StepAcc a[3];
  int rc = read_state(e, &cur, a, st);
  if (rc) return rc;
  if ((in->step ^ cur.s.step) & 1) {
    // the step parity selects the current infectivity / mask buffer: move it
    const int from = (int)(cur.s.step & 1), to = from ^ 1;
    if (e->count_mode) {
      const size_t bytes = (size_t)((e->ntiles_mask + 1 + 3) & ~3LL) * 4;
      FS_CUDA(cudaMemcpyAsync(e->b.imask[to], e->b.imask[from], bytes, cudaMemcpyDeviceToDevice, st));
    } else {
      const size_t bytes = (size_t)e->g.num_nodes * (e->mixed ? 2 : 4);
      FS_CUDA(cudaMemcpyAsync(e->b.infectivity[to], e->b.infectivity[from], bytes, cudaMemcpyDeviceToDevice, st));
    }
  }
  FS_CUDA(cudaMemcpyAsync(e->dstate + e->s_cur, &d, sizeof(DevState), cudaMemcpyHostToDevice, st));
  FS_CUDA(cudaMemsetAsync(e->acc, 0, 3 * sizeof(StepAcc), st));
  if ((in->step ^ cur.s.step) & 1) {  // pending deltas are indexed by step parity: rebuild
    rc = recount(e, in->step, st);
    if (rc) return rc;
  }
  if (in->step != cur.s.step) {  // memo tags and cohorts are relative to the step counter
    rc = reset_memo(e, st);
    if (rc) return rc;
  }
  FS_CUDA(cudaStreamSynchronize(st));
  e->h_step = in->step;
  return 0;
}

int fs_engine_load_infectivity(fs_engine* e, const void* inf, void* stream) {
  if (!e || !inf) return set_error(FS_EINVAL, "null argument");
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = e->g.num_nodes;
  if (e->count_mode) {
    FS_CUDA(cudaMemsetAsync(e->bad_flag, 0, sizeof(int), st));
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8);
    if (e->mixed)
      k_load_mask<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)inf, n, e->inf_val, e->b.imask[0] + e->node_base / 32,
                                                          e->b.imask[1] + e->node_base / 32, e->bad_flag);
    else
      k_load_mask<float><<<blocks, 256, 0, st>>>((const float*)inf, n, e->inf_val, e->b.imask[0] + e->node_base / 32,
                                                 e->b.imask[1] + e->node_base / 32, e->bad_flag);
    int bad = 0;
    FS_CUDA(cudaMemcpyAsync(&bad, e->bad_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    FS_CUDA(cudaStreamSynchronize(st));
    if (bad) return set_error(FS_EREPR, "infectivity values are not in {0, beta}: the count gather cannot represent them");
    {
      DevState d;
      StepAcc a[3];
      int rc = read_state(e, &d, a, st);
      if (!rc) rc = recount(e, d.s.step, st);
      if (rc) return rc;
    }
    return 0;
  }
  const size_t bytes = (size_t)n * (e->mixed ? 2 : 4);
  FS_CUDA(cudaMemcpyAsync(e->b.infectivity[0], inf, bytes, cudaMemcpyDeviceToDevice, st));
  FS_CUDA(cudaMemcpyAsync(e->b.infectivity[1], inf, bytes, cudaMemcpyDeviceToDevice, st));
  return 0;
}

int fs_engine_store_infectivity(fs_engine* e, void* out, void* stream) {
  if (!e || !out) return set_error(FS_EINVAL, "null argument");
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  fs_scalars s;
  int rc = fs_engine_get_scalars(e, &s, stream);
  if (rc) return rc;
  const int cur = (int)(s.step & 1);
  const int64_t n = e->g.num_nodes;
  if (e->count_mode) {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8);
    if (e->mixed)
      k_store_mask<__nv_bfloat16><<<blocks, 256, 0, st>>>(e->b.imask[cur] + e->node_base / 32, n, __float2bfloat16_rn(e->inf_val), (__nv_bfloat16*)out);
    else
      k_store_mask<float><<<blocks, 256, 0, st>>>(e->b.imask[cur] + e->node_base / 32, n, e->inf_val, (float*)out);
    FS_CUDA(cudaGetLastError());
    return 0;
  }
  FS_CUDA(cudaMemcpyAsync(out, e->b.infectivity[cur], (size_t)n * (e->mixed ? 2 : 4), cudaMemcpyDeviceToDevice, st));
  return 0;
}

int fs_engine_reset_age_memo(fs_engine* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  FS_CUDA(cudaSetDevice(e->device));
  return reset_memo(e, (cudaStream_t)stream);
}

int fs_engine_acc_get(fs_engine* e, uint64_t* out17, void* stream) {
  if (!e || !out17) return set_error(FS_EINVAL, "null argument");
  if (e->h_step < 1) return set_error(FS_ESTATE, "no step to exchange");
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  const StepAcc* A = e->acc + (e->h_step - 1) % 3;
  unsigned mb = 0;
  FS_CUDA(cudaMemcpyAsync(out17, &A->d[0], FS_MAX_COMPARTMENTS * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaMemcpyAsync(&mb, &A->max_bits, sizeof mb, cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaStreamSynchronize(st));
  out17[FS_MAX_COMPARTMENTS] = mb;
  return 0;
}

int fs_engine_acc_set(fs_engine* e, const uint64_t* in17, void* stream) {
  if (!e || !in17) return set_error(FS_EINVAL, "null argument");
  if (e->h_step < 1) return set_error(FS_ESTATE, "no step to exchange");
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  StepAcc* A = e->acc + (e->h_step - 1) % 3;
  const unsigned mb = (unsigned)in17[FS_MAX_COMPARTMENTS];
  FS_CUDA(cudaMemcpyAsync(&A->d[0], in17, FS_MAX_COMPARTMENTS * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  FS_CUDA(cudaMemcpyAsync(&A->max_bits, &mb, sizeof mb, cudaMemcpyHostToDevice, st));
  FS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int fs_engine_delta_buffers(fs_engine* e, void** out2) {
  if (!e || !out2) return set_error(FS_EINVAL, "null argument");
  if (!e->incr) return set_error(FS_ESTATE, "engine does not use incremental counts");
  out2[0] = e->delta[0];
  out2[1] = e->delta[1];
  return 0;
}

int fs_engine_set_peer_deltas(fs_engine* e, void* const* ptrs) {
  if (!e || !ptrs) return set_error(FS_EINVAL, "null argument");
  if (!e->incr || e->world < 2) return set_error(FS_ESTATE, "not a partitioned incremental engine");
  for (int par = 0; par < 2; ++par)
    for (int r = 0; r < e->world; ++r) {
      if (!ptrs[par * e->world + r]) return set_error(FS_EINVAL, "null delta buffer for rank %d", r);
      e->peer_pend[par][r] = static_cast<uint32_t*>(ptrs[par * e->world + r]);
    }
  if (e->peer_pend[0][e->rank] != e->delta[0] || e->peer_pend[1][e->rank] != e->delta[1])
    return set_error(FS_EINVAL, "rank %d's own entries must be its own delta buffers", e->rank);
  e->peers_linked = true;
  return 0;
}

int fs_ipc_get_handle(void* dptr, uint8_t* out, int32_t len) {
  if (!dptr || !out || len < (int32_t)sizeof(cudaIpcMemHandle_t)) return set_error(FS_EINVAL, "ipc handle buffer too small");
  cudaIpcMemHandle_t h;
  FS_CUDA(cudaIpcGetMemHandle(&h, dptr));
  memcpy(out, &h, sizeof h);
  return (int)sizeof h;
}

int fs_ipc_open_handle(const uint8_t* in, int32_t device, void** out) {
  if (!in || !out) return set_error(FS_EINVAL, "null argument");
  FS_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, in, sizeof h);
  FS_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int fs_ipc_close(void* dptr) {
  if (dptr) FS_CUDA(cudaIpcCloseMemHandle(dptr));
  return 0;
}

int fs_engines_exchange_local(fs_engine* const* engines, int32_t count, void* stream) {
  if (!engines || count < 1 || count > FS_MAX_PARTITIONS) return set_error(FS_EINVAL, "1..%d engines", FS_MAX_PARTITIONS);
  AccPtrs ptrs{};
  const int64_t h = engines[0]->h_step;
  for (int r = 0; r < count; ++r) {
    if (!engines[r] || engines[r]->h_step != h || engines[r]->device != engines[0]->device)
      return set_error(FS_EINVAL, "engines must be on one device and at the same step");
    ptrs.a[r] = engines[r]->acc;
  }
  if (h < 1) return set_error(FS_ESTATE, "no step to exchange");
  FS_CUDA(cudaSetDevice(engines[0]->device));
  k_exchange_local<<<1, 32, 0, (cudaStream_t)stream>>>(ptrs, count, (int)((h - 1) % 3));
  FS_CUDA(cudaGetLastError());
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// standalone pressure gather (renewal.py:264-313) on a caller buffer
// ---------------------------------------------------------------------------
namespace fs {
template <typename IT, int STRAT>
__global__ void __launch_bounds__(256) k_gather_nodes(const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                                                      const void* w, int w_bf16, int w_uniform, float w_val,
                                                      const void* inf, int64_t n, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp_g; t * 32 < n; t += nwarps) {
    const int64_t i = t * 32 + lane;
    int64_t lo = 0, hi = 0;
    if (i < n) { lo = __ldg(ro + i); hi = __ldg(ro + i + 1); }
    if (STRAT == S_THREAD) {
      if (i < n) out[i] = fold_thread<IT>(col, inf, w, w_bf16, w_uniform, w_val, lo, hi);
    } else {
      unsigned todo = __ballot_sync(kFull, i < n);
      float mine = 0.0f;
      while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t lj = __shfl_sync(kFull, lo, j), hj = __shfl_sync(kFull, hi, j);
        const float v = fold_warp<IT>(col, inf, w, w_bf16, w_uniform, w_val, lj, hj, lane);
        if (lane == j) mine = v;
      }
      if (i < n) out[i] = mine;
    }
  }
}
}  // namespace fs

extern "C" int fs_pressure_gather(const fs_graph* g, const void* inf, int32_t inf_dtype, float* out,
                                  int32_t strategy, int32_t lanes_per_node, int32_t edges_per_block,
                                  void* stream) {
  (void)lanes_per_node;  // lane width changes the partition only, never the bits
  if (!g || !out) return set_error(FS_EINVAL, "null argument");
  if (inf_dtype != FS_F32 && inf_dtype != FS_BF16) return set_error(FS_EINVAL, "infectivity dtype must be f32 or bf16");
  if (strategy < FS_PER_NODE || strategy > FS_MERGE) return set_error(FS_EINVAL, "strategy must be resolved");
  const int64_t n = g->num_nodes;
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return 0;
  if (g->num_edges == 0) { FS_CUDA(cudaMemsetAsync(out, 0, n * sizeof(float), st)); return 0; }
  if (!inf) return set_error(FS_EINVAL, "null infectivity");
  const bool bf = inf_dtype == FS_BF16;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    sms = std::max(1, fs_device_sm_count(dev));
  }
  if (strategy == FS_MERGE) {
    if (edges_per_block < 1) return set_error(FS_EINVAL, "edges_per_block must be >= 1");
    const int64_t nchunks = (g->num_edges + edges_per_block - 1) / edges_per_block;
    int64_t* cf = nullptr;
    FS_CUDA(cudaMallocAsync((void**)&cf, (nchunks + 1) * sizeof(int64_t), st));
    FS_CUDA(cudaMemsetAsync(out, 0, n * sizeof(float), st));
    k_chunk_first<<<(int)std::min<int64_t>((nchunks + 256) / 256, 4096), 256, 0, st>>>(g->row_offsets, n, g->num_edges,
                                                                                      edges_per_block, nchunks, cf);
    MergeParams q{};
    q.ro = g->row_offsets;
    q.col = g->col_indices;
    q.w = g->weights;
    q.w_bf16 = g->weights_dtype == FS_BF16;
    q.w_uniform = g->weights_uniform;
    q.w_val = g->uniform_weight;
    q.n = n;
    q.e = g->num_edges;
    q.epb = edges_per_block;
    q.nchunks = nchunks;
    q.chunk_first = cf;
    q.inf[0] = q.inf[1] = inf;
    q.inf_bf16 = bf;
    q.S = nullptr;
    q.out = out;
    int block = 512;
    MergeFn fn = pick_merge(bf, 0, block);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nchunks + block / 32 - 1) / (block / 32), (int64_t)sms * 2));
    fn<<<grid, block, 0, st>>>(q);
    FS_CUDA(cudaFreeAsync(cf, st));
  } else {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
    const int s = strategy == FS_LANE ? S_WARP : S_THREAD;
    if (bf) {
      if (s == S_WARP) k_gather_nodes<__nv_bfloat16, S_WARP><<<grid, 256, 0, st>>>(g->row_offsets, g->col_indices, g->weights, g->weights_dtype == FS_BF16, g->weights_uniform, g->uniform_weight, inf, n, out);
      else k_gather_nodes<__nv_bfloat16, S_THREAD><<<grid, 256, 0, st>>>(g->row_offsets, g->col_indices, g->weights, g->weights_dtype == FS_BF16, g->weights_uniform, g->uniform_weight, inf, n, out);
    } else {
      if (s == S_WARP) k_gather_nodes<float, S_WARP><<<grid, 256, 0, st>>>(g->row_offsets, g->col_indices, g->weights, g->weights_dtype == FS_BF16, g->weights_uniform, g->uniform_weight, inf, n, out);
      else k_gather_nodes<float, S_THREAD><<<grid, 256, 0, st>>>(g->row_offsets, g->col_indices, g->weights, g->weights_dtype == FS_BF16, g->weights_uniform, g->uniform_weight, inf, n, out);
    }
  }
  FS_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int fs_engine_debug_times(fs_engine* e, unsigned long long* out, int32_t max_ctas) {
  if (!e || !e->dbg) return set_error(FS_EINVAL, "engine built without FS_DEBUG_TIMES");
  const int n = std::min(max_ctas, e->step_grid);  // stamps of the streaming kernel, [16 steps][grid][4]
  FS_CUDA(cudaDeviceSynchronize());
  FS_CUDA(cudaMemcpy(out, e->dbg, sizeof(unsigned long long) * 4 * 16 * n, cudaMemcpyDeviceToHost));
  FS_CUDA(cudaMemset(e->dbg, 0, sizeof(unsigned long long) * 4 * 16 * n));
  return n;
}
