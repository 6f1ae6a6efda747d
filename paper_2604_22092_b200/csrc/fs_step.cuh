// fs_step.cuh — the step kernels of the renewal engine (templates), shared by
// the translation units that instantiate them (fs_step_*.cu) and the engine
// (fs_engine.cu), which launches them through the pick_* functions.
//
// One launch = one `renewal_step` of the reference
// (/root/reference/pkg/src/spreadsim/renewal.py:483-580); see fs_engine.cu
// and DESIGN.md §3 for the kernel families and gather encodings.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>
#include "fs_device.cuh"
#include "fs_internal.h"

namespace fs {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCntStride = FS_MAX_COMPARTMENTS;
// shared-memory budget for the staged mask: leaves room for the static
// tables on a 227 KB CTA
constexpr size_t kMaxSmemMaskBytes = 188u * 1024u;  // + ~34 KB static (queues) <= 227 KB

// G_F32M_*: the f32 fold with a nonzero-infectivity bitmap prefilter — the
// mask (staged in shared memory, or read from L2) says which in-neighbours
// carry infectivity; only those are gathered and folded
enum Gather { G_COUNT_SMEM = 0, G_COUNT_GLOBAL = 1, G_F32 = 2, G_PRE = 3, G_INCR = 4, G_F32M_SMEM = 5, G_F32M_GLOBAL = 6 };
constexpr int32_t kEntryInvalid = INT32_MIN;  // age not known to follow its cohort (init, host edits)
constexpr int kCohortSlots = 2;                // age-dependent compartments with a cohort table
constexpr int kCohortW = 1 << 10;              // cohorts (entry steps) per table: a ring

constexpr uint32_t kDeltaBias = 0x8000u;  // pending delta d is stored as d + 0x8000 (|d| <= d_max < 2^15)
// S_HYBRID: thread per node for slices of <= kWide edges, the whole warp for
// longer ones (scale-free hubs) — the edge-merge dispatch fused into the step
enum Strat { S_THREAD = 0, S_WARP = 1, S_HYBRID = 2 };
constexpr int kWide = 32;

// Device-side run scalars.  Two slots ping-pong (the host tracks which one
// is current): step k reads slot `in` and its CTA 0 writes slot `out`, so no
// CTA ever reads a slot being written.  `pending` = the count deltas and max
// rate of step s.step-1 still sit in an accumulator and are folded in by the
// next step (or by begin_batch / the host).
struct DevState {
  fs_scalars s;
  int pending;
  // uniform S age: the f32 bits of the storage-rounded age
  // every S node has, advanced by the step kernels that keep S ages as this
  // one scalar (k_step_incr<UNI>) instead of in the ages array
  uint32_t s_age_bits;
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
  int f32_mask;                  // f32 gather keeps the nonzero-infectivity mask (G_F32M_*)
  // fused edge-merge (S_HYBRID + G_F32M_*): the nodes with more than kWide
  // in-edges, heaviest first, are folded by the grid's warps round robin
  // before the tile sweep; a tile lane of such a node waits for its flag
  const int32_t* hub_list;
  int64_t nhubs;
  float* hub_pre;                // [N] pressure of the hubs (entries of hubs only)
  uint32_t* hub_flag;            // [N] step tag (step + 1) once hub_pre[n] holds this step's value
  // incremental count mode (G_INCR): per-node infectious in-neighbour count,
  // kept current by +-1 pushes along the outgoing edges of every node whose
  // infectious status changes
  uint16_t* cnt;                 // [N] counts as of the current step's start, minus pending deltas
  uint32_t* pend[2];             // [ceil(N/2)] words of biased u16 pending deltas, double-buffered by step parity
  const int64_t* out_ro;         // outgoing CSR of the local rows (the incoming one for symmetric graphs)
  const int32_t* out_col;        // global ids
  int world;                     // > 1: pushes go to the owner's pending deltas (peer_pend)
  int hubs;                      // some out-row exceeds 32 edges: warp-cooperative pushes
  int64_t part_bound[FS_MAX_PARTITIONS + 1];  // node range boundaries of the ranks
  uint32_t* remote_log;          // partitioned: per-step count of pushes sent to other ranks (log ring)
  uint32_t* peer_pend[2][FS_MAX_PARTITIONS];  // every rank's pending-delta arrays, by parity
  // bulk (mailbox) exchange of remote pushes: every rank's
  // mailbox, [parity][sender] regions of kMboxHdr + mbox_cap words; pushes to
  // other ranks are staged per warp in shared memory (stage_cap per owner)
  // and written to the owner's mailbox as coalesced peer stores
  uint32_t* peer_mbox[FS_MAX_PARTITIONS];
  int64_t mbox_cap;
  int bulk;
  int stage_cap;
  int rank;
  int stream_evict_first;        // CSR stream larger than L2: evict-first hint on column loads
  int host_parity;               // the host's mirror of (step & 1) for this launch (early loads), -1: none
  // age-cohort hazard memo: entry step of each node's
  // current compartment; the per-CTA memo itself lives in shared memory
  int32_t* entry;                // [N] or nullptr (cohort table off)
  unsigned long long* ctab;      // [2 parity][kCohortSlots][kCohortW] (step tag << 32 | rate bits)
  unsigned long long* cage;      // [2 parity][kCohortW] (step tag << 32 | f32 age bits)
  int ncslots;
  int cslot[FS_MAX_COMPARTMENTS];      // compartment -> table slot, -1: none
  int cslot_comp[kCohortSlots];        // table slot -> compartment
  unsigned long long* dbg;       // optional per-CTA %globaltimer stamps [grid][4]
  // model / config
  fs_model model;
  double eps, tau_max, delta;
  int rng;
  int hprec;
  float inf_val;                 // stored infectivity of an I node (count mode), promoted
  uint32_t term_bits;            // bit c: compartment c is terminal
};


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

// [lo, hi) of node n in two halves, so the loads of the next tile stay in
// flight while this one is processed: load_slice_raw issues them (lo <- the
// lane's own offset, hi <- offset n+1 where no neighbour lane holds it) and
// finish_slice, at the tile's turn, takes hi from lane+1
__device__ __forceinline__ void load_slice_raw(const int64_t* __restrict__ ro, const int32_t* __restrict__ ro32,
                                               int64_t n, int64_t N, bool valid, int lane, int64_t& lo, int64_t& hi) {
  lo = valid ? (ro32 ? (int64_t)__ldg(ro32 + n) : __ldg(ro + n)) : 0;
  hi = (valid && (lane == 31 || n + 1 >= N)) ? (ro32 ? (int64_t)__ldg(ro32 + n + 1) : __ldg(ro + n + 1)) : 0;
}
__device__ __forceinline__ void finish_slice(int64_t n, int64_t N, bool valid, int lane, int64_t lo, int64_t& hi) {
  const int64_t up = __shfl_down_sync(0xffffffffu, lo, 1);
  hi = !valid ? lo : ((lane == 31 || n + 1 >= N) ? hi : up);
}
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

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
// The loads of kFoldB edges are issued together (columns, then the gathered
// infectivities), so a slice costs ~2 memory round trips per kFoldB edges
// instead of 2 per edge; the adds stay one sequential chain in CSR order.
#ifndef FS_FOLD_B
#define FS_FOLD_B 8
#endif
constexpr int kFoldB = FS_FOLD_B;
template <typename IT>
__device__ __forceinline__ float fold_thread(const int32_t* __restrict__ col, const void* inf,
                                             const void* w, int w_bf16, int w_uniform, float w_val,
                                             int64_t lo, int64_t hi) {
  float acc = 0.0f;
  for (int64_t e = lo; e < hi; e += kFoldB) {
    int32_t c[kFoldB];
    float v[kFoldB];
#pragma unroll
    for (int u = 0; u < kFoldB; ++u) c[u] = (e + u < hi) ? __ldg(col + e + u) : 0;
#pragma unroll
    for (int u = 0; u < kFoldB; ++u) {
      if (e + u < hi) {
        const float wv = w_uniform ? w_val : load_w(w, w_bf16, e + u);
        v[u] = __fmul_rn(load_inf<IT>(inf, c[u]), wv);
      }
    }
#pragma unroll
    for (int u = 0; u < kFoldB; ++u)
      if (e + u < hi) acc = __fadd_rn(acc, v[u]);
  }
  return acc;
}

// the same fold with the nonzero-infectivity bitmap as a prefilter: a column
// whose mask bit is clear has infectivity exactly 0, so its contribution
// f32(0 * w) = +-0 leaves the accumulator unchanged (it is never -0: it starts
// at +0 and x + (-x) rounds to +0) — only the set bits are gathered and
// folded, still in CSR order.  Needs finite weights (0 * inf = NaN), which
// the engine checks before it selects this gather.
template <typename IT, bool SMEM>
__device__ __forceinline__ float fold_thread_masked(const int32_t* __restrict__ col, const uint32_t* m, const void* inf,
                                                    const void* w, int w_bf16, int w_uniform, float w_val,
                                                    int64_t lo, int64_t hi) {
  float acc = 0.0f;
  for (int64_t e = lo; e < hi; e += kFoldB) {
    int32_t c[kFoldB];
#pragma unroll
    for (int u = 0; u < kFoldB; ++u) c[u] = (e + u < hi) ? __ldg(col + e + u) : 0;
    uint32_t bits = 0;
#pragma unroll
    for (int u = 0; u < kFoldB; ++u)
      if (e + u < hi) bits |= (uint32_t)mask_bit<SMEM>(m, c[u]) << u;
    if (bits) {
      float v[kFoldB];
#pragma unroll
      for (int u = 0; u < kFoldB; ++u)
        if ((bits >> u) & 1u) v[u] = __fmul_rn(load_inf<IT>(inf, c[u]), w_uniform ? w_val : load_w(w, w_bf16, e + u));
#pragma unroll
      for (int u = 0; u < kFoldB; ++u)
        if ((bits >> u) & 1u) acc = __fadd_rn(acc, v[u]);
    }
  }
  return acc;
}

// One hub row [lo, hi) folded by the whole warp with the mask prefilter:
// passes of 8 x 32 coalesced column loads, mask tests and ballots; the lanes
// gather the infectivities of their set columns (in registers), stage them in
// shared memory in edge order, and lane 0 folds only the set positions, in
// CSR order, while the next pass's loads are in flight.  Every lane returns
// the sum.
constexpr int kHubPass = 256;
constexpr int kFoldStage = kHubPass;  // per-warp stage of the hub fold (floats)
template <typename IT, bool SMEM_MASK>
__device__ __forceinline__ float fold_hub_masked(const int32_t* __restrict__ col, const uint32_t* m, const void* inf,
                                                 const void* w, int w_bf16, int w_uniform, float w_val, int64_t lo,
                                                 int64_t hi, int lane, float* stage, uint64_t col_pol) {
  constexpr int U = kHubPass / 32;
  float acc = 0.0f;
  float v[U];
  unsigned bal[U];
  auto pass = [&](int64_t base) {
    uint32_t c[U], word[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + 32 * u + lane;
      c[u] = e < hi ? (uint32_t)ldg_hint(col + e, col_pol) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) word[u] = SMEM_MASK ? m[c[u] >> 5] : ldg_hint(m + (c[u] >> 5), l2_policy_last());
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + 32 * u + lane;
      const bool on = e < hi && ((word[u] >> (c[u] & 31)) & 1u);
      bal[u] = __ballot_sync(0xffffffffu, on);
      v[u] = on ? __fmul_rn(load_inf<IT>(inf, (int32_t)c[u]), w_uniform ? w_val : load_w(w, w_bf16, e)) : 0.0f;
    }
  };
  pass(lo);
  for (int64_t base = lo; base < hi; base += kHubPass) {
    unsigned sb[U];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      stage[32 * u + lane] = v[u];
      sb[u] = bal[u];
    }
    __syncwarp();
    if (base + kHubPass < hi) pass(base + kHubPass);  // in flight during the chain below
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        unsigned W = sb[u];
        while (W) {
          const int bit = __ffs(W) - 1;
          W &= W - 1;
          acc = __fadd_rn(acc, stage[32 * u + bit]);
        }
      }
    }
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu, acc, 0);
}

// infectious in-neighbours of one hub row, counted by the whole warp: passes
// of 8 x 32 coalesced column loads and mask tests (every lane returns the total)
template <bool SMEM_MASK>
__device__ __forceinline__ int count_hub(const int32_t* __restrict__ col, const uint32_t* m, int64_t lo, int64_t hi,
                                         int lane, uint64_t col_pol) {
  int cnt = 0;
  for (int64_t base = lo; base < hi; base += kHubPass) {
    uint32_t c[8], word[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = base + 32 * u + lane;
      c[u] = e < hi ? (uint32_t)ldg_hint(col + e, col_pol) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) word[u] = SMEM_MASK ? m[c[u] >> 5] : ldg_hint(m + (c[u] >> 5), l2_policy_last());
#pragma unroll
    for (int u = 0; u < 8; ++u) cnt += (base + 32 * u + lane < hi) ? (int)((word[u] >> (c[u] & 31)) & 1u) : 0;
  }
  return __reduce_add_sync(0xffffffffu, cnt);
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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
  bool write_mask;               // maintain the next-step mask words
};

// shared-memory model tables + the per-warp deferral queues
template <int WARPS>
struct StepShared {
  int succ[FS_MAX_COMPARTMENTS], term[FS_MAX_COMPARTMENTS], kind[FS_MAX_COMPARTMENTS];
  int cslot[FS_MAX_COMPARTMENTS];  // cohort-table slot per compartment (-1: none / table off)
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
    sh.cslot[tid] = p.ctab ? p.cslot[tid] : -1;
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
  k.write_mask = count_gather || p.f32_mask;
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
  if (p.remote_log) p.remote_log[(k.step + 1) % p.log_cap] = 0u;  // the next step's counter
  for (int c = 0; c < FS_MAX_COMPARTMENTS; ++c) Z->d[c] = 0ull;
}

// uniform S age (k_step_incr<UNI>): every S node that does not fire ages by
// f32(tau) and rounds to the storage type (renewal.py:540-542), so one scalar
// advances for all of them; CTA 0 publishes it with the step's other scalars
template <typename AT>
__device__ __forceinline__ void commit_s_age(const StepParams& p, const StepConst& k) {
  const float a = __uint_as_float(p.Sin->s_age_bits);
  p.Sout->s_age_bits = __float_as_uint(to_f32<AT>(from_f32<AT>(__fadd_rn(a, k.tau_f))));
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
// Cohort hazard table.  Every node that entered compartment c at step j
// carries, at step k, the same age bits a_j(k) — all non-terminal nodes add
// the same f32(tau) each step and round to the same storage type — hence the
// same rate.  While step k runs, its CTAs prepare the table of step k+1: for
// each live cohort j in (k+1-W, k], a_j(k+1) = round(a_j(k) + f32(tau_k))
// (0 for the cohort entering at k) and the f64 hazard of every age-dependent
// compartment at that age, tagged with k+1.  Step k+1 then looks rates up by
// the node's entry step instead of evaluating the hazard.  Tags make stale or
// never-prepared slots (engine start, host edits, other kernels) fall back to
// direct evaluation; a cohort's age chain restarts only from a fresh cohort.
// Results are bit-identical with or without the table.  The preparation runs
// in lane 31 of each warp's final drain (drain_entries, argument `prep`).

constexpr int kMboxHdr = 32;  // words before a sender's mailbox entries (word 0: the cursor)
// a warp's staging of remote pushes in shared memory: world counters, then
// world segments of `cap` entries ((owner-local id << 1) | up)
struct MboxStage {
  uint32_t* e;
  int* n;
  int cap;
};

// incremental counts: +-1 on node j's pending delta (buffer `nxt`), in this
// device's memory or, node-partitioned, the owner's — possibly a peer GPU's
// over NVLink.  Chunk boundaries are even, so the 16-bit lane
// of j is the same in global and owner-local numbering.
// Returns 1 when the push went to another rank.
__device__ __forceinline__ int push_delta(const StepParams& p, int nxt, int32_t j, bool up) {
  const uint32_t one = 1u << (16 * (j & 1));
  uint32_t* dn;
  int remote = 0;
  if (p.world > 1) {
    int owner = 0;  // ranges (equal or edge-balanced) by their boundaries
    for (int r = 1; r < p.world; ++r) owner += (int64_t)j >= p.part_bound[r];
    dn = p.peer_pend[nxt][owner] + (((int64_t)j - p.part_bound[owner]) >> 1);
    remote = (int64_t)j < p.node_base || (int64_t)j >= p.node_base + p.n;
  } else {
    dn = p.pend[nxt] + (j >> 1);
  }
  if (up) atomicAdd(dn, one);
  else atomicSub(dn, one);
  return remote;
}

// partitioned form with the bulk exchange: a push to another rank is staged
// in the warp's shared-memory segment of its owner (flushed by
// flush_stage); a full segment falls back to the direct peer atomic
__device__ __forceinline__ int push_delta_staged(const StepParams& p, int nxt, int32_t j, bool up, const MboxStage& sg) {
  int owner = 0;
  for (int r = 1; r < p.world; ++r) owner += (int64_t)j >= p.part_bound[r];
  const uint32_t jl = (uint32_t)((int64_t)j - p.part_bound[owner]);
  if (owner != p.rank) {
    const int at = atomicAdd(sg.n + owner, 1);
    if (at < sg.cap) {
      sg.e[owner * sg.cap + at] = (jl << 1) | (up ? 1u : 0u);
      return 1;
    }
  }
  uint32_t* dn = p.peer_pend[nxt][owner] + (jl >> 1);
  const uint32_t one = 1u << (16 * (jl & 1));
  if (up) atomicAdd(dn, one);
  else atomicSub(dn, one);
  return owner != p.rank;
}

// the warp's staged pushes to their owners' mailboxes (region [nxt][this
// rank]): one remote cursor atomic per owner, then coalesced peer stores;
// entries past the mailbox's capacity go as direct peer atomics.  The owner
// applies them after the step's exchange (k_apply_mailbox).  Warp-converged.
__device__ __forceinline__ void flush_stage(const StepParams& p, int nxt, const MboxStage& sg, int lane) {
  __syncwarp();
  for (int o = 0; o < p.world; ++o) {
    const int cnt = min(sg.n[o], sg.cap);
    if (cnt == 0) continue;
    uint32_t* hdr = p.peer_mbox[o] + ((size_t)nxt * p.world + p.rank) * (size_t)(kMboxHdr + p.mbox_cap);
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(hdr, (unsigned)cnt);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int i = lane; i < cnt; i += 32) {
      const uint32_t v = sg.e[o * sg.cap + i];
      const unsigned long long slot = base + (unsigned long long)i;
      if (slot < (unsigned long long)p.mbox_cap) {
        hdr[kMboxHdr + slot] = v;
      } else {
        const uint32_t jl = v >> 1;
        uint32_t* dn = p.peer_pend[nxt][o] + (jl >> 1);
        const uint32_t one = 1u << (16 * (jl & 1));
        if (v & 1u) atomicAdd(dn, one);
        else atomicSub(dn, one);
      }
    }
  }
  __syncwarp();
  if (lane < p.world) sg.n[lane] = 0;
  __syncwarp();
}

// PART: node-partitioned engine (pushes may go to other ranks; `sg.e` set:
// staged for the bulk exchange); false compiles the multi-rank code out
// CNT: a count-encoding kernel (no infectivity buffers): the f32 infectivity
// write-back is compiled out rather than skipped at run time
template <typename ST, typename AT, typename IT, bool MAT, int WARPS, bool HUBS = true, bool UNI = false, bool PART = true,
          bool CNT = false>
__device__ __forceinline__ void drain_entries(const StepParams& p, const StepConst& k, StepShared<WARPS>& sh,
                                              const int* qn_node, const int* qn_state, const float* qn_age,
                                              const float* qn_press, int lane, int cnt, float& lmax,
                                              uint32_t* mask_nxt, IT* inf_nxt, int prep = -1,
                                              MboxStage sg = MboxStage{nullptr, nullptr, 0}) {
  __syncwarp();
  const bool ok = lane < cnt;
  int push = 0;  // +1 / -1: this node's infectious status changed
  const int n = ok ? qn_node[lane] : 0;
  const int s = ok ? qn_state[lane] : 0;
  // UNI: phase A never loads ages; a queued nodal node loads its own here
  // (S ages are the uniform scalar and are not needed for S rates)
  const float age = !ok ? 0.0f
                        : UNI ? (s == k.edge_from ? 0.0f : to_f32<AT>(reinterpret_cast<const AT*>(p.ages)[n]))
                              : qn_age[lane];
  float rate = 0.0f;
  bool compute = false;
  if (ok) {
    if (s == k.edge_from) {
      rate = qn_press[lane];
    } else {
      compute = true;
      const int sl = sh.cslot[s];
      if (sl >= 0) {  // the cohort table prepared by the previous step
        const int32_t j = p.entry[n];
        const int64_t since = k.step - (int64_t)j;
        if (j != kEntryInvalid && since >= 1 && since < kCohortW) {
          const unsigned long long v =
              __ldg(p.ctab + ((size_t)(k.step & 1) * kCohortSlots + sl) * kCohortW + ((uint32_t)j & (kCohortW - 1)));
          if ((uint32_t)(v >> 32) == (uint32_t)k.step) {
            rate = __uint_as_float((uint32_t)v);
            compute = false;
          }
        }
      }
    }
  }
  // cohort-table preparation rides in lane 31 of a warp's final drain
  // (never a queued lane there: a final queue holds < 32 entries), through the
  // same hazard call, so it adds no latency.  Pair `prep` = (slot sl, cohort
  // idx) of step k+1's table (see the cohort-table comment above).
  const bool prep_lane = prep >= 0 && lane == 31;
  int hk = 0;
  double hp0 = 0.0, hp1 = 0.0;
  float ha = 0.0f;
  unsigned long long prep_age = ~0ull;
  if (compute) {
    hk = sh.kind[s];
    hp0 = sh.p0[s];
    hp1 = sh.p1[s];
    ha = age;
  }
  if (prep_lane) {
    const int idx = prep & (kCohortW - 1), sl = prep / kCohortW;
    const int par_c = (int)(k.step & 1);
    const int64_t j = (k.step + 1) - (((k.step + 1) - idx) & (kCohortW - 1));
    if (j == k.step) {
      prep_age = ((unsigned long long)(uint32_t)(k.step + 1) << 32) | __float_as_uint(0.0f);
    } else if (j < k.step) {
      const unsigned long long cur = p.cage[par_c * kCohortW + idx];
      if ((uint32_t)(cur >> 32) == (uint32_t)k.step)
        prep_age = ((unsigned long long)(uint32_t)(k.step + 1) << 32) |
                   __float_as_uint(to_f32<AT>(from_f32<AT>(__fadd_rn(__uint_as_float((uint32_t)cur), k.tau_f))));
    }
    if (prep_age != ~0ull) {
      const fs_compartment& cc = p.model.comp[p.cslot_comp[sl]];
      hk = cc.hazard;
      hp0 = cc.p0;
      hp1 = cc.p1;
      ha = __uint_as_float((uint32_t)prep_age);
    }
  }
  float hr = 0.0f;
  if (compute || prep_age != ~0ull) hr = nodal_rate(hk, hp0, hp1, ha, p.hprec);
  if (compute) rate = hr;
  if (prep_lane) {
    const int idx = prep & (kCohortW - 1), sl = prep / kCohortW;
    const int par_n = (int)(k.step & 1) ^ 1;
    p.ctab[((size_t)par_n * kCohortSlots + sl) * kCohortW + idx] =
        prep_age != ~0ull ? ((prep_age >> 32) << 32) | __float_as_uint(hr) : ~0ull;
    if (sl == 0) p.cage[par_n * kCohortW + idx] = prep_age;
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
      if ((CNT || !k.write_inf) && ((ns == k.infectious) != (s == k.infectious))) {
        atomicXor(mask_nxt + p.tile_base + (n >> 5), 1u << (n & 31));
        if (p.cnt) push = (ns == k.infectious) ? 1 : -1;  // incremental counts: pushes below
      }
    } else {
      nage = __fadd_rn(age, k.tau_f);  // queued nodes are never terminal
    }
    if (!UNI || fire || s != k.edge_from) reinterpret_cast<AT*>(p.ages)[n] = from_f32<AT>(nage);
    if (!CNT && k.write_inf) {
      const IT iv = from_f32<IT>(inf_value(p, k, ns, nage));
      inf_nxt[n] = iv;
      // f32 mask: phase A left this (deferred) node's bit clear
      if (k.write_mask && to_f32<IT>(iv) != 0.0f) atomicOr(mask_nxt + p.tile_base + (n >> 5), 1u << (n & 31));
    }
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
    const bool wide = HUBS && p.hubs && push && (e1 - e0 > 32);
    int remote = 0;  // pushes this lane sent to other ranks (partitioned runs)
    auto push1 = [&](int32_t j, bool up) -> int {
      if (!PART) {  // one partition: straight into the local pending delta
        const uint32_t one = 1u << (16 * (j & 1));
        if (up) atomicAdd(p.pend[nxt] + (j >> 1), one);
        else atomicSub(p.pend[nxt] + (j >> 1), one);
        return 0;
      }
      return sg.e ? push_delta_staged(p, nxt, j, up, sg) : push_delta(p, nxt, j, up);
    };
    // column loads are batched ahead of their atomics: a load-then-push loop
    // would wait one memory round trip per edge (each push needs its column)
    constexpr int kPB = 8;
    if (push && !wide) {
      for (int64_t b = e0; b < e1; b += kPB) {
        int32_t cj[kPB];
#pragma unroll
        for (int j = 0; j < kPB; ++j) cj[j] = (b + j < e1) ? __ldg(p.out_col + b + j) : -1;
#pragma unroll
        for (int j = 0; j < kPB; ++j)
          if (cj[j] >= 0) remote += push1(cj[j], push > 0);
      }
    }
    unsigned wides = HUBS ? __ballot_sync(kFull, wide) : 0u;
    while (HUBS && wides) {
      const int src = __ffs(wides) - 1;
      wides &= wides - 1;
      const int64_t a0 = __shfl_sync(kFull, e0, src), a1 = __shfl_sync(kFull, e1, src);
      const bool up = __shfl_sync(kFull, push, src) > 0;
      constexpr int kHB = 8;  // 8 x 32 edges of the hub row in flight per round
      for (int64_t b = a0 + lane; b < a1; b += 32 * kHB) {
        int32_t cj[kHB];
#pragma unroll
        for (int j = 0; j < kHB; ++j) cj[j] = (b + 32 * j < a1) ? __ldg(p.out_col + b + 32 * j) : -1;
#pragma unroll
        for (int j = 0; j < kHB; ++j)
          if (cj[j] >= 0) remote += push1(cj[j], up);
      }
    }
    if (PART && sg.e) flush_stage(p, nxt, sg, lane);
    if (PART && p.remote_log) {
      const int tot = __reduce_add_sync(kFull, remote);
      if (lane == 0 && tot) atomicAdd(p.remote_log + k.step % p.log_cap, (unsigned)tot);
    }
    // partitioned: the pushes into peer GPUs' memory are ordered before
    // anything this thread's rank does next — in particular before the NCCL
    // all-reduce the next step waits on — so they are visible to the owner
    if (PART && p.world > 1 && __any_sync(kFull, push != 0)) __threadfence_system();
  }
  __syncwarp();
}

// phase B on this warp's own queue
template <typename ST, typename AT, typename IT, bool MAT, int WARPS, bool HUBS = true, bool UNI = false, bool PART = true,
          bool CNT = false>
__device__ __forceinline__ void drain_queue(const StepParams& p, const StepConst& k, StepShared<WARPS>& sh, int warp,
                                            int lane, int cnt, float& lmax, uint32_t* mask_nxt, IT* inf_nxt,
                                            MboxStage sg = MboxStage{nullptr, nullptr, 0}) {
  drain_entries<ST, AT, IT, MAT, WARPS, HUBS, UNI, PART, CNT>(p, k, sh, sh.q_node[warp], sh.q_state[warp], sh.q_age[warp],
                                                         sh.q_press[warp], lane, cnt, lmax, mask_nxt, inf_nxt, -1, sg);
}

// phase A outcome of one tile (pressure already gathered): cheap outcomes
// now, possible transitions appended to the warp queue (drained at 32)
template <typename ST, typename AT, typename IT, bool MAT, int WARPS, bool HUBS = true, bool UNI = false, bool PART = true,
          bool CNT = false>
__device__ __forceinline__ void tile_outcome(const StepParams& p, const StepConst& k, StepShared<WARPS>& sh, int warp,
                                             int lane, uint32_t tile, uint32_t n, bool valid, int s, float age,
                                             float pressure, int& qn, float& lmax, uint32_t* mask_nxt, IT* inf_nxt,
                                             MboxStage sg = MboxStage{nullptr, nullptr, 0}) {
  const bool isS = s == k.edge_from;
  const bool term = valid && sh.term[s] != 0;
  const bool defer = valid && !term && (!isS || pressure > 0.0f);
  bool nz = false;  // f32 gather: this node's next-step infectivity is nonzero (deferred nodes: phase B)
  if (!UNI && valid && !term && !defer) {  // S with zero pressure: rate 0, ages (UNI: the uniform scalar)
    const float nage = __fadd_rn(age, k.tau_f);
    reinterpret_cast<AT*>(p.ages)[n] = from_f32<AT>(nage);
    if (!CNT && k.write_inf) {
      const IT iv = from_f32<IT>(inf_value(p, k, s, nage));
      inf_nxt[n] = iv;
      nz = to_f32<IT>(iv) != 0.0f;
    }
  } else if (!CNT && term && k.write_inf) {
    const IT iv = from_f32<IT>(inf_value(p, k, s, age));
    inf_nxt[n] = iv;
    nz = to_f32<IT>(iv) != 0.0f;
  }
  if (MAT && valid) {
    p.pressure[n] = pressure;
    if (!defer) p.rates[n] = 0.0f;
  }
  if (k.write_mask) {
    // next-step mask word; deferred nodes are fixed up in phase B
    const unsigned word = __ballot_sync(0xffffffffu, (!CNT && k.write_inf) ? nz : (valid && s == k.infectious));
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
    drain_queue<ST, AT, IT, MAT, WARPS, HUBS, UNI, PART, CNT>(p, k, sh, warp, lane, 32, lmax, mask_nxt, inf_nxt, sg);
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
  constexpr bool FMASK = (GATHER == G_F32M_SMEM || GATHER == G_F32M_GLOBAL);  // f32 fold, mask prefilter
  constexpr bool F32 = GATHER == G_F32 || FMASK;
  constexpr bool SMASK = (GATHER == G_COUNT_SMEM || GATHER == G_F32M_SMEM);   // mask staged in shared memory
  // hub fold stages: static, or behind the staged mask in dynamic shared
  // memory (a 1024-thread CTA's static tables would pass 48 KB)
  constexpr int kStage = kFoldStage;  // per-warp hub fold stage
  __shared__ __align__(16) float s_fold_static[(STRAT == S_HYBRID && FMASK && !SMASK) ? WARPS * kStage : 4];
  float* const s_fold = (STRAT == S_HYBRID && SMASK)
                            ? reinterpret_cast<float*>(s_mask + ((p.ntiles_mask + 3) & ~3LL))
                            : s_fold_static;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  pdl_wait();
  if (SMASK && tid == 0) mbar_init(&s_bar, 1);
  load_tables<WARPS>(p, sh, tid);
  const StepConst k = step_const(p, COUNT || (p.count_mode && !F32));
  if (blockIdx.x == 0 && tid == 0) commit_step_start(p, k);
  const int cur = (int)(k.step & 1);
  const uint32_t* mask_cur = p.mask[cur];
  uint32_t* mask_nxt = p.mask[cur ^ 1];
  const void* inf_cur = p.inf[cur];
  IT* inf_nxt = reinterpret_cast<IT*>(p.inf[cur ^ 1]);
  __syncthreads();
  // stage the whole infectious mask (N/8 bytes) in shared memory with TMA
  // bulk copies; the first tile's node loads below overlap the transfer
  if (SMASK) stage_mask_async(s_mask, mask_cur, (uint32_t)(((p.ntiles_mask + 3) & ~3LL) * 4), &s_bar);
  bool mask_ready = !SMASK;
  const uint32_t* gmask = SMASK ? s_mask : mask_cur;
  float lmax = 0.0f;
  int qn = 0;  // queued entries of this warp (warp-uniform)
  const uint32_t hub_tag = (uint32_t)k.step + 1u;
  if (STRAT == S_HYBRID) {
    // fused edge-merge: the hubs first, heaviest first, round robin over every
    // warp of the grid (all CTAs are resident: grid <= SMs x occupancy), so no
    // warp folds more than its share of hub edges; the tile sweep below reads
    // the results
    if (SMASK && !mask_ready) {
      mbar_wait_parity(&s_bar, 0);
      mask_ready = true;
    }
    const uint64_t pol = l2_policy_stream(p.stream_evict_first);
    for (int64_t h = (int64_t)blockIdx.x * WARPS + warp; h < p.nhubs; h += (int64_t)gridDim.x * WARPS) {
      const int32_t hn = __ldg(p.hub_list + h);
      const int hs = (int)reinterpret_cast<const ST*>(p.states)[hn];
      if (hs != k.edge_from && !MAT) continue;  // only S nodes' pressure is used (all of them materialised)
      const int64_t lo = p.ro32 ? (int64_t)__ldg(p.ro32 + hn) : __ldg(p.ro + hn);
      const int64_t hi = p.ro32 ? (int64_t)__ldg(p.ro32 + hn + 1) : __ldg(p.ro + hn + 1);
      float pr;
      if (COUNT) {
        const int kk = count_hub<SMASK>(p.col, gmask, lo, hi, lane, pol);
        pr = p.ptab_mul ? __fmul_rn((float)kk, p.ptab_c) : __ldg(p.ptab + kk);
      } else {
        pr = fold_hub_masked<IT, SMASK>(p.col, gmask, inf_cur, p.w, p.w_bf16, p.w_uniform, p.w_val, lo, hi, lane,
                                        s_fold + warp * kStage, pol);
      }
      if (lane == 0) {
        p.hub_pre[hn] = pr;
        st_release_u32(p.hub_flag + hn, hub_tag);
      }
    }
  }

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
      load_slice_raw(p.ro, p.ro32, n, p.n, valid, lane, in.lo, in.hi);  // finished at the tile's turn
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
    NodeIn<ST, AT> in = nxt;
    const int64_t tile = tile_n;
    const bool more = t + stride < ntiles;
    if (more) {  // next tile's node loads overlap this tile
      tile_n = tile_of(t + stride);
      load_in(tile_n, nxt);
    }
    const int64_t n = tile * 32 + lane;
    const bool valid = n < p.n;
    if (GATHER != G_INCR && GATHER != G_PRE) finish_slice(n, p.n, valid, lane, in.lo, in.hi);
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
      if (SMASK && !mask_ready) {
        mbar_wait_parity(&s_bar, 0);
        mask_ready = true;
      }
      const unsigned todo = __ballot_sync(kFull, need);
      if (STRAT == S_THREAD) {
        if (FMASK) {
          // (the tile-cooperative sweep, fold_tile_masked, measured slower
          // here: 40 vs 34 us at C2 with shedding — fewer sectors, more
          // instructions)
          if (need)
            pressure = fold_thread_masked<IT, SMASK>(p.col, gmask, inf_cur, p.w, p.w_bf16, p.w_uniform, p.w_val, in.lo,
                                                     in.hi);
        } else if (GATHER == G_F32) {
          if (need) pressure = fold_thread<IT>(p.col, inf_cur, p.w, p.w_bf16, p.w_uniform, p.w_val, in.lo, in.hi);
        } else if (todo) {
          const int kk = count_tile<GATHER == G_COUNT_SMEM>(p.col, gmask, in.lo, in.hi, need, todo, lane,
                                                            l2_policy_stream(p.stream_evict_first));
          if (need) pressure = p.ptab_mul ? __fmul_rn((float)kk, p.ptab_c) : __ldg(p.ptab + kk);
        }
      } else if (STRAT == S_HYBRID) {  // fused edge-merge: hubs from the pre-pass
        const bool wide = need && (in.hi - in.lo > kWide);
        if (need && !wide) {
          if (COUNT) {
            const int kk = count_thread<SMASK>(p.col, gmask, in.lo, in.hi);
            pressure = p.ptab_mul ? __fmul_rn((float)kk, p.ptab_c) : __ldg(p.ptab + kk);
          } else {
            pressure = fold_thread_masked<IT, SMASK>(p.col, gmask, inf_cur, p.w, p.w_bf16, p.w_uniform, p.w_val, in.lo,
                                                     in.hi);
          }
        }
        // hub lanes take the pre-pass's result.  The engine launches this
        // kernel cooperatively (every CTA resident), so each hub's warp runs
        // and the wait ends
        if (wide) {
          while (ld_acquire_u32(p.hub_flag + n) != hub_tag) {
          }
          pressure = __ldcg(p.hub_pre + n);
        }
      } else {  // warp per node (LANE strategy)
        unsigned rest = todo;
        while (rest) {
          const int j = __ffs(rest) - 1;
          rest &= rest - 1;
          const int64_t lj = __shfl_sync(kFull, in.lo, j), hj = __shfl_sync(kFull, in.hi, j);
          float pj;
          if (F32) {
            pj = fold_warp<IT>(p.col, inf_cur, p.w, p.w_bf16, p.w_uniform, p.w_val, lj, hj, lane);
          } else {
            const int kk = count_warp<GATHER == G_COUNT_SMEM>(p.col, gmask, lj, hj, lane);
            pj = p.ptab_mul ? __fmul_rn((float)kk, p.ptab_c) : __ldg(p.ptab + kk);
          }
          if (lane == j) pressure = pj;
        }
      }
    }
    // the next tile's first column line, while this tile's outcome and
    // drains run (its offsets were loaded at the top of this iteration)
    if (F32 && more && tile_n * 32 + lane < p.n) prefetch_l1(p.col + nxt.lo);
    tile_outcome<ST, AT, IT, MAT, WARPS>(p, k, sh, warp, lane, (uint32_t)tile, (uint32_t)n, valid, in.s, in.age, pressure, qn, lmax,
                                         mask_nxt, inf_nxt);
  }
  {
    // the final drain also prepares one (slot, cohort) pair of the next
    // step's cohort table in its idle lane 31 (as k_step_incr does)
    const int gw = (int)blockIdx.x * WARPS + warp;
    const int prep = (p.ctab && gw < kCohortW * p.ncslots) ? gw : -1;
    if (qn > 0 || prep >= 0)
      drain_entries<ST, AT, IT, MAT, WARPS>(p, k, sh, sh.q_node[warp], sh.q_state[warp], sh.q_age[warp],
                                            sh.q_press[warp], lane, qn, lmax, mask_nxt, inf_nxt, prep);
  }
  // a warp without tiles still has to see the bulk copy land before exit
  if (SMASK && !mask_ready) mbar_wait_parity(&s_bar, 0);
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
#ifndef FS_PF_DEPTH
#define FS_PF_DEPTH 2
#endif
// `cta` / `nctas`: this CTA and the CTAs sharing the engine `p` (the whole
// grid, or one member's CTAs of an ensemble launch)
// PERSIST: one CTA runs several steps in a row (k_step_incr_persist): the
// per-node arrays it rewrites are then read back inside the same kernel, so
// no load may take the non-coherent read-only path
template <typename ST, typename AT, bool MAT, bool MEMO, bool HUBS, bool UNI, int BLOCK, bool PART = false,
          bool PERSIST = false>
__device__ __forceinline__ void step_incr_body(const StepParams& p, const uint32_t cta, const uint32_t nctas) {
  constexpr int WARPS = BLOCK / 32;
  __shared__ StepShared<WARPS> sh;
  __shared__ StepConst s_k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // bulk exchange: this warp's staging of remote pushes (dynamic shared memory)
  MboxStage sg{nullptr, nullptr, 0};
  if (PART && p.bulk) {
    extern __shared__ __align__(16) uint32_t fs_dyn[];
    uint32_t* base = fs_dyn + (size_t)warp * p.world * (p.stage_cap + 1);
    sg.n = reinterpret_cast<int*>(base);
    sg.e = base + p.world;
    sg.cap = p.stage_cap;
    if (lane < p.world) sg.n[lane] = 0;
    __syncwarp();
  }
#if FS_STEP_PROBE  // build with -DFS_STEP_PROBE=1 and run with FS_DEBUG_TIMES=1 (scripts/cta_times_incr.py)
  __shared__ unsigned long long s_entry;
  if (p.dbg && tid == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    s_entry = now;
  }
#endif
  pdl_launch_dependents();
  load_tables<WARPS>(p, sh, tid);  // static model tables: before the dependency wait
  pdl_wait();
  if (tid == 0) {
    s_k = step_const(p, true);
    if (cta == 0) {
      commit_step_start(p, s_k);
      if (UNI) commit_s_age<AT>(p, s_k);
    }
  }
  using SP = std::conditional_t<PERSIST, const ST*, const ST* __restrict__>;
  using AP = std::conditional_t<PERSIST, const AT*, const AT* __restrict__>;
  SP states = reinterpret_cast<const ST*>(p.states);
  AP ages = reinterpret_cast<const AT*>(p.ages);
  uint16_t* __restrict__ cnt = p.cnt;
  const uint32_t N = (uint32_t)p.n, ntiles = (uint32_t)p.ntiles;
  const uint32_t stride = nctas * WARPS;
  struct In { int s; float age; uint32_t c, d; };
  // arrays are padded to whole 128-node units: every lane loads unconditionally
  auto load = [&](uint32_t t, const uint16_t* pend, In& in) {
    const uint32_t n = t * 32u + (uint32_t)lane;
    in.s = (int)states[n];
    if (!UNI) in.age = to_f32<AT>(ages[n]);  // UNI: queued nodal nodes load their age in phase B
    in.c = cnt[n];
    in.d = pend[n];
  };
  // the first two tiles' loads need only the buffer parity, which the host
  // knows: they overlap thread 0's scalar reads instead of waiting for them
  uint32_t t = cta * WARPS + warp;
  constexpr int PD = FS_PF_DEPTH;  // tiles in flight per warp (register ring, compile-time indices)
  In inq[PD];
#pragma unroll
  for (int i = 0; i < PD; ++i) inq[i] = In{};
  if (p.host_parity >= 0) {
    const uint16_t* pend_h = reinterpret_cast<const uint16_t*>(p.pend[p.host_parity & 1]);
#pragma unroll
    for (int i = 0; i < PD; ++i)
      if (t + i * stride < ntiles) load(t + i * stride, pend_h, inq[i]);
  }
  __syncthreads();
  const StepConst& k = s_k;  // read from shared memory where used: keeps the hot loop's registers free
#if FS_STEP_PROBE  // per-CTA stamps [smid | entry, work end, constants ready, finish]
  if (p.dbg && tid == 0) {
    unsigned long long now;
    unsigned sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    unsigned long long* dbg = p.dbg + ((size_t)(k.step & 15) * nctas + cta) * 4;
    dbg[0] = ((unsigned long long)sm << 48) | (s_entry & 0xFFFFFFFFFFFFull);
    dbg[2] = now;
  }
#endif
  const int cur = (int)(k.step & 1);
  uint32_t* mask_nxt = p.mask[cur ^ 1];
  uint16_t* __restrict__ pend = reinterpret_cast<uint16_t*>(p.pend[cur]);
  if (cur != p.host_parity) {  // no host mirror, or out of step: load now
#pragma unroll
    for (int i = 0; i < PD; ++i)
      if (t + i * stride < ntiles) load(t + i * stride, pend, inq[i]);
  }
  float lmax = 0.0f;
  int qn = 0;
#if FS_STEP_PROBE
  int pr_def = 0, pr_drains = 0;
#endif
  for (; t < ntiles; t += stride) {
    const In in = inq[0];
#pragma unroll
    for (int i = 0; i < PD - 1; ++i) inq[i] = inq[i + 1];
    if (t + PD * stride < ntiles) load(t + PD * stride, pend, inq[PD - 1]);
    const uint32_t n = t * 32u + (uint32_t)lane;
    const bool valid = n < N;
    uint32_t c = in.c;
    if (valid && in.d != kDeltaBias) {  // fold the previous step's pushes, clear them
      c = c + in.d - kDeltaBias;
      cnt[n] = (uint16_t)c;
      pend[n] = (uint16_t)kDeltaBias;
    }
    const int s = valid ? in.s : -1;
    if (UNI && !MAT) {
      // quiet tile: every lane absorbed, or S with no infectious in-neighbour
      // (rate 0, and its age is the uniform scalar) — nothing but the
      // next-step mask word to write
      const bool quiet = !valid || ((p.term_bits >> s) & 1u) || (s == k.edge_from && c == 0u);
      if (__all_sync(0xffffffffu, quiet)) {
        const unsigned word = __ballot_sync(0xffffffffu, valid && s == k.infectious);
        if (lane == 0) mask_nxt[p.tile_base + t] = word;
        continue;
      }
    }
    const float pressure = (valid && (s == k.edge_from || MAT))
                               ? (p.ptab_mul ? __fmul_rn((float)c, p.ptab_c) : __ldg(p.ptab + c))
                               : 0.0f;
#if FS_STEP_PROBE
    const int q0 = qn;
#endif
    tile_outcome<ST, AT, float, MAT, WARPS, HUBS, UNI, PART, true>(p, k, sh, warp, lane, t, n, valid, s, in.age,
                                                                   pressure, qn, lmax, mask_nxt, nullptr, sg);
#if FS_STEP_PROBE
    pr_def += qn - q0 + (qn < q0 ? 32 : 0);
    pr_drains += qn < q0;
#endif
  }
  {
    // the final drain also prepares one (slot, cohort) pair of step k+1's
    // cohort table in its idle lane 31 (qn < 32 here)
    const int gw = (int)cta * WARPS + warp;
    const int prep = (MEMO && gw < kCohortW * p.ncslots) ? gw : -1;
    if (qn > 0 || prep >= 0)
      drain_entries<ST, AT, float, MAT, WARPS, HUBS, UNI, PART, true>(p, k, sh, sh.q_node[warp], sh.q_state[warp],
                                                                 sh.q_age[warp], sh.q_press[warp], lane, qn, lmax,
                                                                 mask_nxt, nullptr, prep, sg);
  }
#if FS_STEP_PROBE  // per-warp [phase end, deferred << 20 | mid-loop drains] after the per-CTA block
  if (p.dbg && lane == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    unsigned long long* w = p.dbg + (size_t)16 * nctas * 4 +
                            (((size_t)(k.step & 15) * nctas + cta) * 32 + (size_t)warp * 2);
    w[0] = now;
    w[1] = ((unsigned long long)pr_def << 20) | (unsigned long long)(pr_drains + (qn > 0 ? 1 : 0));
  }
#endif
#if FS_STEP_PROBE
  if (p.dbg && lane == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicMax(p.dbg + ((size_t)(k.step & 15) * nctas + cta) * 4 + 1, now);
  }
#endif
  finish_step<WARPS>(p, k, sh, warp, lane, lmax);
#if FS_STEP_PROBE
  if (p.dbg && tid == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    p.dbg[((size_t)(k.step & 15) * nctas + cta) * 4 + 3] = now;
  }
#endif
}


template <typename ST, typename AT, bool MAT, bool MEMO, bool HUBS, bool UNI, int BLOCK, bool PART = false>
__global__ void __launch_bounds__(BLOCK, 2) k_step_incr(const StepParams p) {
  step_incr_body<ST, AT, MAT, MEMO, HUBS, UNI, BLOCK, PART>(p, blockIdx.x, gridDim.x);
}


// Ensemble launch (fs_ensemble, DESIGN.md §8 row 2): one step of every member
// engine in one grid.  Member m owns CTAs [m * ctas_per, (m + 1) * ctas_per)
// and runs exactly the single-engine step on its own parameters — its own
// buffers, scalars, accumulators, log and RNG seed — so every member is
// bit-identical to its engine stepped alone.
template <typename ST, typename AT, bool MAT, bool MEMO, bool HUBS, bool UNI, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 2) k_step_incr_multi(const StepParams* __restrict__ P, const uint32_t ctas_per) {
  const uint32_t m = blockIdx.x / ctas_per;
  step_incr_body<ST, AT, MAT, MEMO, HUBS, UNI, BLOCK>(P[m], blockIdx.x - m * ctas_per, ctas_per);
}

// Ensembles of small trials (every member fits one CTA): CTA m runs `nsteps`
// consecutive steps of member m — a block barrier between steps instead of
// a kernel boundary, since no other CTA touches the member's state.  P holds
// the members' parameters for the four (scalar slot, step parity) pairs,
// [pair][count]; step i of the batch uses pair (s0 ^ i&1, p0 ^ i&1) — the
// same parameters the per-step launches would pass, so the results are
// the same bits.  The cohort table is off (its slots are read through the
// non-coherent path); the engine only picks this form without it.
template <typename ST, typename AT, bool HUBS, bool UNI, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 2) k_step_incr_persist(const StepParams* __restrict__ P, const uint32_t count,
                                                                const int s0, const int p0, const int nsteps) {
  const uint32_t m = blockIdx.x;
  for (int i = 0; i < nsteps; ++i) {
    const int pair = ((s0 ^ (i & 1)) << 1) | (p0 ^ (i & 1));
    step_incr_body<ST, AT, false, false, HUBS, UNI, BLOCK, false, true>(P[(size_t)pair * count + m], 0u, 1u);
    __syncthreads();  // this step's writes (state, counts, pushes, accumulator, scalars) before the next step's reads
  }
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
    tile_outcome<ST, AT, float, MAT, WARPS, true, false, true, true>(p, k, sh, warp, lane, (uint32_t)t, (uint32_t)n, valid, s, in.age, pressure, qn, lmax,
                                            mask_nxt, nullptr);
    sl = (sl + 1 == L.slots) ? 0 : sl + 1;
  }
  if (qn > 0) drain_queue<ST, AT, float, MAT, WARPS, true, false, true, true>(p, k, sh, warp, lane, qn, lmax, mask_nxt, nullptr);
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


using StepFn = void (*)(const StepParams);
using MergeFn = void (*)(const MergeParams);
using TmaFn = void (*)(const StepParams, const TmaLayout);
using MultiFn = void (*)(const StepParams*, uint32_t);
using PersistFn = void (*)(const StepParams*, uint32_t, int, int, int);

// instantiation units
StepFn pick_step(bool mixed, int gather, int strat, bool mat, int& block);  // fs_step_general.cu
StepFn pick_stream(bool mixed, bool mat, bool memo, bool hubs, bool uni, bool part = false);  // fs_step_incr.cu
MultiFn pick_stream_multi(bool mixed, bool mat, bool memo, bool hubs, bool uni);    // fs_step_multi.cu
PersistFn pick_stream_persist(bool mixed, bool hubs, bool uni);                     // fs_step_multi.cu
MergeFn pick_merge(bool inf_bf16, int mode, int& block);                    // fs_step_incr.cu
TmaFn pick_tma(bool mixed, bool smem_mask, bool mat, bool ptab_mul, int block);  // fs_step_tma.cu

}  // namespace fs
