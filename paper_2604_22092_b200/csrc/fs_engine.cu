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
#include "fs_step.cuh"

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

// small host values (run scalars, the pressure table) written through a
// launch argument instead of a pageable cudaMemcpy, which waits for the
// device: creating an engine (e.g. the members of an ensemble) then queues
// its setup without ever blocking on the work queued before it
struct WordBlob { uint32_t w[512]; };
__global__ void k_put_words(uint32_t* __restrict__ dst, const WordBlob b, int nwords) {
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = b.w[i];
}

static int put_small(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes % 4 == 0 && bytes <= sizeof(WordBlob)) {
    WordBlob b;
    memcpy(b.w, src, bytes);
    k_put_words<<<1, 128, 0, st>>>(static_cast<uint32_t*>(dst), b, (int)(bytes / 4));
  }
  const cudaError_t err = (bytes % 4 == 0 && bytes <= sizeof(WordBlob))
                              ? cudaGetLastError()
                              : cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  return err == cudaSuccess ? 0 : set_error(FS_ECUDA, "put_small(%zu B): %s", bytes, cudaGetErrorString(err));
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

// host edited the states between steps: the next step writes the next mask
// from the edited states, so every node whose infectious status now differs
// from its bit in the current mask pushes +-1 into the pending deltas that
// step's successor folds — exactly the pushes a transition would have made
template <typename ST>
__global__ void k_edit_pushes(const ST* __restrict__ states, const uint32_t* __restrict__ mask_cur, int64_t n,
                              int infectious, const int64_t* __restrict__ out_ro, const int32_t* __restrict__ out_col,
                              uint32_t* __restrict__ pend_nxt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool now = (int)states[i] == infectious;
    const bool was = (mask_cur[i >> 5] >> (i & 31)) & 1u;
    if (now == was) continue;
    for (int64_t e = out_ro[i], e1 = out_ro[i + 1]; e < e1; ++e) {
      const int32_t j = out_col[e];
      const uint32_t one = 1u << (16 * (j & 1));
      if (now) atomicAdd(pend_nxt + (j >> 1), one);
      else atomicSub(pend_nxt + (j >> 1), one);
    }
  }
}

// min / max of the S nodes' age bits (f32 of the storage value; ages >= 0,
// so the bit order is the value order)
template <typename ST, typename AT>
__global__ void k_s_age_range(const ST* __restrict__ states, const AT* __restrict__ ages, int64_t n, int s_comp,
                              uint32_t* __restrict__ range) {
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if ((int)states[i] != s_comp) continue;
    const uint32_t b = __float_as_uint(to_f32<AT>(ages[i]));
    lo = min(lo, b);
    hi = max(hi, b);
  }
  if (lo != 0xFFFFFFFFu) {
    atomicMin(range, lo);
    atomicMax(range + 1, hi);
  }
}

// write the uniform S age into the ages array
template <typename ST, typename AT>
__global__ void k_fill_s_age(const ST* __restrict__ states, AT* __restrict__ ages, int64_t n, int s_comp,
                             const uint32_t* __restrict__ bits) {
  const AT a = from_f32<AT>(__uint_as_float(*bits));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if ((int)states[i] == s_comp) ages[i] = a;
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
// batch prologue (renewal.py:583-597): fold a pending step into the
// scalars, then reset tau unless carry_tau
__device__ __forceinline__ void begin_batch_one(DevState* D, StepAcc* acc, int64_t* log_counts, int64_t log_cap,
                                                int M, double eps, double tau_max, double delta, int carry_tau) {
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

__global__ void k_begin_batch(DevState* D, StepAcc* acc, int64_t* log_counts, int64_t log_cap,
                              int M, double eps, double tau_max, double delta, int carry_tau) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  begin_batch_one(D, acc, log_counts, log_cap, M, eps, tau_max, delta, carry_tau);
}

// the same for every member of an ensemble (thread m: member m)
struct MemberBatch {
  DevState* D[2];      // the member's two scalar slots
  StepAcc* acc;        // its accumulator ring
  int64_t* log_counts; // its row of the ensemble's count log
};
__global__ void k_begin_batch_multi(const MemberBatch* __restrict__ mb, int count, int slot, int64_t log_cap, int M,
                                    double eps, double tau_max, double delta, int carry_tau) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= count) return;
  begin_batch_one(mb[m].D[slot], mb[m].acc, mb[m].log_counts, log_cap, M, eps, tau_max, delta, carry_tau);
}

// cohort table reset (reset_memo): entry = step - 1 for nodes of age exactly 0
template <typename AT>
__global__ void k_memo_reset(const AT* __restrict__ ages, int64_t n, int64_t cap, int32_t j, int32_t* __restrict__ entry) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
    bool zero = false;  // +0 exactly (bit pattern)
    if (i < n) {
      if constexpr (sizeof(AT) == 4) zero = __float_as_uint(ages[i]) == 0u;
      else zero = __half_as_ushort(ages[i]) == 0;
    }
    entry[i] = zero ? j : kEntryInvalid;
  }
}
struct CohortSeed {
  int n;
  int kind[kCohortSlots];
  double p0[kCohortSlots], p1[kCohortSlots];
};
// the table of `step`: the slot of the cohort entered at step - 1 (age 0)
__global__ void k_memo_seed(unsigned long long* ctab, unsigned long long* cage, CohortSeed cs, int64_t step, int hprec) {
  const int t = threadIdx.x;
  const int par = (int)(step & 1);
  const uint32_t idx = (uint32_t)(step - 1) & (kCohortW - 1);
  const unsigned long long tag = (unsigned long long)(uint32_t)step << 32;
  if (t == 0) cage[par * kCohortW + idx] = tag | __float_as_uint(0.0f);
  if (t < cs.n)
    ctab[((size_t)par * kCohortSlots + t) * kCohortW + idx] = tag | __float_as_uint(nodal_rate(cs.kind[t], cs.p0[t], cs.p1[t], 0.0f, hprec));
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
    if (bad && on && v != c) atomicExch(bad, 1);  // bad == nullptr: any nonzero value (f32 mask)
    const unsigned w = __ballot_sync(kFull, on);
    if (lane == 0) { m0[i >> 5] = w; m1[i >> 5] = w; }
  }
}

// 1 in *bad when some weight is not finite (the f32 mask prefilter skips
// 0 * w, which is NaN for an infinite or NaN weight)
__global__ void k_any_nonfinite(const void* w, int bf16, int64_t e, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(w)[i]) : reinterpret_cast<const float*>(w)[i];
    if (!isfinite(v)) atomicExch(bad, 1);
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

// bulk exchange, owner side: after the step's exchange (every rank's step —
// hence every mailbox write — complete), fold the entries the senders left
// in this rank's mailbox [par][sender] into the pending deltas of that parity;
// the last CTA of each sender resets its cursor for the step after next
__global__ void k_apply_mailbox(uint32_t* __restrict__ mbox, int par, int world, int rank, int64_t cap,
                                uint32_t* __restrict__ pend, unsigned* __restrict__ ticket) {
  const int s = blockIdx.y;
  if (s == rank) return;  // the whole block: nothing is ever staged to oneself
  uint32_t* hdr = mbox + ((size_t)par * world + s) * (size_t)(kMboxHdr + cap);
  const int64_t n = min((int64_t)__ldcg(hdr), cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = __ldcg(hdr + kMboxHdr + i);
    const uint32_t jl = v >> 1;
    const uint32_t one = 1u << (16 * (jl & 1));
    if (v & 1u) atomicAdd(pend + (jl >> 1), one);
    else atomicSub(pend + (jl >> 1), one);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ticket + s, 1u) == gridDim.x - 1) {
      hdr[0] = 0u;
      ticket[s] = 0u;
      __threadfence();
    }
  }
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
  bool fmask = false;     // f32 gather with the nonzero-infectivity mask prefilter (G_F32M_*)
  bool fresh = false;     // built on a fresh state (FS_BUF_FRESH): its first infectivity load is trusted
  int32_t* hub_list = nullptr;  // fused edge-merge: nodes with in-degree > kWide, heaviest first
  int64_t nhubs = 0;
  float* hub_pre = nullptr;     // [N]
  uint32_t* hub_flag = nullptr; // [N]
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
  int64_t part_bound[FS_MAX_PARTITIONS + 1] = {};  // rank r owns [part_bound[r], part_bound[r+1])
  bool unequal_ranges = false;
  uint32_t* remote_log = nullptr;  // partitioned: per-step pushes sent to other ranks
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
  bool delta_ipc = false;             // delta buffers from cudaMalloc (exported over CUDA IPC)
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
  // pipelined batches: each replay records an event after its steps and the
  // final fold, so the host can read one batch's log while the next runs
  static constexpr int kBatchEv = 8;
  cudaEvent_t batch_ev[kBatchEv] = {};
  int64_t batch_ev_end[kBatchEv] = {};  // step count after the batch (-1: unused)
  int batch_ev_next = 0;
  cudaStream_t copy_stream = nullptr;
  cudaGraphExec_t batch_exec[2][2][6] = {};  // [materialise][scalar slot][step % 6]: parity and exchange slot are baked in
  bool compaction_ready = false;
  bool tiles_valid = false;  // active tile list matches the states (set by begin_batch / refresh_tiles)
  int stream_evict_first = 0;
  // incremental count mode
  int32_t* entry = nullptr;           // cohort table: per-node entry step
  unsigned long long* ctab = nullptr;  // [2][kCohortSlots][kCohortW]
  unsigned long long* cage = nullptr;  // [2][kCohortW]
  bool incr = false;
  uint32_t* peer_pend[2][FS_MAX_PARTITIONS] = {};  // partitioned incremental: every rank's delta arrays
  bool peers_linked = false;
  // bulk exchange: this rank's mailbox [2 parity][world sender]
  // x (kMboxHdr + mbox_cap) words, every rank's mailbox, the apply tickets
  uint32_t* mbox = nullptr;
  int64_t mbox_cap = 0;
  uint32_t* peer_mbox[FS_MAX_PARTITIONS] = {};
  unsigned* mbox_ticket = nullptr;
  bool bulk = false;
  int stage_cap = 0;
  size_t stream_smem = 0;
  bool stream = false;         // k_step_incr fast path of the incremental mode
  bool stream_part() const { return world > 1; }
  StepFn stream_fn[2] = {nullptr, nullptr};
  bool stream_memo = false, stream_hubs = false;  // k_step_incr variant flags
  // uniform S age: eligible when every step runs k_step_incr
  // and no transition re-enters S; on while every S node's age is equal
  bool uni_ok = false;
  bool s_uniform = false;
  uint32_t* uni_range = nullptr;  // [2] device scratch: min / max S-age bits
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

// Engine scratch comes from the device's stream-ordered pool, kept (not
// released to the driver) between engines: creating an engine per run
// (run_renewal, ensemble trials) then costs no cudaMalloc / cudaFree
// round trips.  Buffers exported over CUDA IPC use plain cudaMalloc.
static void keep_pool(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[device] = true;
}

template <typename T>
int dalloc(T** p, size_t count, bool ipc = false) {
  if (count == 0) count = 1;
  cudaError_t err = ipc ? cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T))
                        : cudaMallocAsync(reinterpret_cast<void**>(p), count * sizeof(T), (cudaStream_t)0);
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
  p.f32_mask = e->fmask;
  p.hub_list = e->hub_list;
  p.nhubs = e->nhubs;
  p.hub_pre = e->hub_pre;
  p.hub_flag = e->hub_flag;
  p.stream_evict_first = e->stream_evict_first;
  p.host_parity = (int)(e->h_step & 1);
  p.entry = e->entry;
  p.ctab = e->entry ? e->ctab : nullptr;
  p.cage = e->cage;
  p.ncslots = 0;
  for (int c = 0; c < FS_MAX_COMPARTMENTS; ++c) {
    p.cslot[c] = -1;
    if (c < e->m.num_compartments && e->m.comp[c].hazard >= FS_HZ_LOGNORMAL && p.ncslots < kCohortSlots) {
      p.cslot[c] = p.ncslots;
      p.cslot_comp[p.ncslots++] = c;
    }
  }
  p.cnt = e->incr ? e->cnt : nullptr;
  p.pend[0] = e->delta[0];
  p.pend[1] = e->delta[1];
  p.out_ro = e->g.out_row_offsets;
  p.out_col = e->g.out_col_indices;
  p.world = e->incr ? e->world : 1;
  p.hubs = e->g.d_max > 32 ? 1 : 0;  // local rows; partitioned rows of a symmetric graph mirror the degrees
  for (int r = 0; r <= FS_MAX_PARTITIONS; ++r) p.part_bound[r] = e->part_bound[r];
  p.remote_log = (e->incr && e->world > 1) ? e->remote_log : nullptr;
  for (int r = 0; r < FS_MAX_PARTITIONS; ++r) p.peer_mbox[r] = e->peer_mbox[r];
  p.mbox_cap = e->mbox_cap;
  p.bulk = e->bulk ? 1 : 0;
  p.stage_cap = e->stage_cap;
  p.rank = e->rank;
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
  p.term_bits = 0;
  for (int c = 0; c < e->m.num_compartments; ++c)
    if (e->m.comp[c].terminal) p.term_bits |= 1u << c;
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

// the mailbox entries of the step just run (h_step, before the host mirror
// advances) into this rank's pending deltas of the next parity
int apply_mailbox(fs_engine* e, cudaStream_t st) {
  const int par = (int)((e->h_step & 1) ^ 1);
  const int bx = std::max(1, std::min(64, 2 * e->sms / std::max(1, e->world)));
  k_apply_mailbox<<<dim3(bx, e->world), 256, 0, st>>>(e->mbox, par, e->world, e->rank, e->mbox_cap, e->delta[par],
                                                      e->mbox_ticket);
  FS_CUDA(cudaGetLastError());
  return 0;
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
      cfg.dynamicSmemBytes = e->bulk ? e->stream_smem : 0;  // the warps' push staging
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
    else if (e->strat == S_HYBRID) {
      // the one-launch edge-merge: tile lanes wait for hub results that other
      // CTAs of the grid produce, so the grid is launched cooperatively — all
      // CTAs resident together whatever else runs on the device
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(e->step_grid_general);
      cfg.blockDim = dim3(e->step_block);
      cfg.dynamicSmemBytes = e->step_smem_general;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      FS_CUDA(cudaLaunchKernelEx(&cfg, e->step_fn[mat], p));
    } else
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
      if (e->bulk) {
        const int rc2 = apply_mailbox(e, st);
        if (rc2) return rc2;
      }
    }
    ++e->h_step;
  }
  FS_CUDA(cudaGetLastError());
  return 0;
}

// compaction: rebuild the active tile list from the current states
// (refresh_active, renewal.py:426-432, at 32-node tile granularity)
int refresh_tiles(fs_engine* e, cudaStream_t st) {
  {
    uint32_t term_bits = 0;
    for (int i = 0; i < e->m.num_compartments; ++i)
      if (e->m.comp[i].terminal) term_bits |= 1u << i;
    const int64_t n = e->g.num_nodes;
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
    if (e->count_mode || e->fmask)
      k_sync_buffers<uint32_t><<<blocks2, 256, 0, st>>>(e->dstate + e->s_cur, e->b.imask[0], e->b.imask[1], e->ntiles_mask);
    if (e->count_mode)
      ;  // the mask is the whole infectivity
    else if (e->mixed)
      k_sync_buffers<__nv_bfloat16><<<blocks2, 256, 0, st>>>(e->dstate + e->s_cur, (__nv_bfloat16*)e->b.infectivity[0],
                                                             (__nv_bfloat16*)e->b.infectivity[1], n);
    else
      k_sync_buffers<float><<<blocks2, 256, 0, st>>>(e->dstate + e->s_cur, (float*)e->b.infectivity[0], (float*)e->b.infectivity[1], n);
  }
  FS_CUDA(cudaGetLastError());
  e->tiles_valid = true;
  return 0;
}

int launch_begin_batch(fs_engine* e, cudaStream_t st) {
  k_begin_batch<<<1, 32, 0, st>>>(e->dstate + e->s_cur, e->acc, e->log_counts, e->log_cap, e->m.num_compartments,
                                  e->c.epsilon, e->c.tau_max, e->c.delta, e->c.carry_tau);
  if (!e->c.compaction) {
    FS_CUDA(cudaGetLastError());
    return 0;
  }
  const int64_t n = e->g.num_nodes;
  // rates are zeroed once per batch under compaction (renewal.py:594)
  if (e->b.rates) k_fill<float><<<e->sms * 4, 256, 0, st>>>(e->b.rates, n, 0.0f);
  if (e->b.pressure) k_fill<float><<<e->sms * 4, 256, 0, st>>>(e->b.pressure, n, 0.0f);
  return refresh_tiles(e, st);
}

// hazard memo: every node's cohort unknown, every slot's tag stale
// `step` is the step the next launch runs.  A node whose age is exactly 0
// then is, for the table, a member of the cohort that "entered at step - 1"
// (its age chain from 0 is the one a fresh cohort follows), so it keeps
// table lookups instead of direct hazards — the seeds of a fresh state above
// all, every step until they transition; every other node's cohort is
// unknown.  The table of `step` is seeded with that cohort's slot (age 0,
// the hazards at age 0), everything else is stale.
int reset_memo(fs_engine* e, cudaStream_t st, int64_t step) {
  if (!e->entry) return 0;
  const int64_t n = e->g.num_nodes, cap = (n + 127) / 128 * 128;
  const int blocks = (int)std::min<int64_t>((cap + 255) / 256, (int64_t)e->sms * 8);
  FS_CUDA(cudaMemsetAsync(e->ctab, 0xFF, sizeof(unsigned long long) * 2 * kCohortSlots * kCohortW, st));
  FS_CUDA(cudaMemsetAsync(e->cage, 0xFF, sizeof(unsigned long long) * 2 * kCohortW, st));
  const int32_t j = (int32_t)(step - 1);
  if (e->mixed)
    k_memo_reset<__half><<<std::max(1, blocks), 256, 0, st>>>((const __half*)e->b.ages, n, cap, j, e->entry);
  else
    k_memo_reset<float><<<std::max(1, blocks), 256, 0, st>>>((const float*)e->b.ages, n, cap, j, e->entry);
  CohortSeed cs{};
  cs.n = 0;
  for (int c = 0; c < e->m.num_compartments && cs.n < kCohortSlots; ++c)
    if (e->m.comp[c].hazard >= FS_HZ_LOGNORMAL) {  // the table slots, as make_step_params numbers them
      cs.kind[cs.n] = e->m.comp[c].hazard;
      cs.p0[cs.n] = e->m.comp[c].p0;
      cs.p1[cs.n] = e->m.comp[c].p1;
      ++cs.n;
    }
  k_memo_seed<<<1, 32, 0, st>>>(e->ctab, e->cage, cs, step, e->c.hazard_precision);
  FS_CUDA(cudaGetLastError());
  return 0;
}

void drop_batch_graphs(fs_engine* e) {
  for (auto& a : e->batch_exec)
    for (auto& b : a)
      for (auto& x : b)
        if (x) { cudaGraphExecDestroy(x); x = nullptr; }
}

// S ages back into the ages array (the array is authoritative again for
// every node; the uniform scalar stays valid)
int sync_s_ages(fs_engine* e, cudaStream_t st) {
  if (!e->s_uniform) return 0;
  const int64_t n = e->g.num_nodes;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8));
  const uint32_t* bits = &e->dstate[e->s_cur].s_age_bits;
  if (e->mixed)
    k_fill_s_age<int8_t, __half><<<blocks, 256, 0, st>>>((const int8_t*)e->b.states, (__half*)e->b.ages, n,
                                                         e->m.edge_from, bits);
  else
    k_fill_s_age<int32_t, float><<<blocks, 256, 0, st>>>((const int32_t*)e->b.states, (float*)e->b.ages, n,
                                                         e->m.edge_from, bits);
  FS_CUDA(cudaGetLastError());
  return 0;
}

// the streaming step variants for the engine's current flags.  (A two-
// nodes-per-lane form — 64-node tiles, vector loads, SIMD halfword count
// folds — measured slower: C2 -3.5 %, C4 -10 %.)
void set_stream_fns(fs_engine* e, bool uni) {
  for (int mat = 0; mat < 2; ++mat) {
    e->stream_fn[mat] = pick_stream(e->mixed, mat != 0, e->stream_memo, e->stream_hubs, uni, e->world > 1);
    // the bulk exchange's per-warp push staging (dynamic shared memory on top
    // of the kernel's static tables: past the 48 KB default)
    if (e->stream_smem && e->stream_fn[mat])
      cudaFuncSetAttribute((const void*)e->stream_fn[mat], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->stream_smem);
  }
}

// (re)decide the uniform-S-age mode from the ages array (engine creation,
// host edits): on iff every S node holds the same age; the scalar is set to
// it.  Switching the mode switches the step kernel, so batch graphs go.
int recheck_uniform(fs_engine* e, cudaStream_t st) {
  if (!e->uni_ok) return 0;
  const int64_t n = e->g.num_nodes;
  const uint32_t init[2] = {0xFFFFFFFFu, 0u};
  FS_CUDA(cudaMemcpyAsync(e->uni_range, init, sizeof init, cudaMemcpyHostToDevice, st));
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8));
  if (e->mixed)
    k_s_age_range<int8_t, __half><<<blocks, 256, 0, st>>>((const int8_t*)e->b.states, (const __half*)e->b.ages, n,
                                                          e->m.edge_from, e->uni_range);
  else
    k_s_age_range<int32_t, float><<<blocks, 256, 0, st>>>((const int32_t*)e->b.states, (const float*)e->b.ages, n,
                                                          e->m.edge_from, e->uni_range);
  uint32_t r[2];
  FS_CUDA(cudaMemcpyAsync(r, e->uni_range, sizeof r, cudaMemcpyDeviceToHost, st));
  FS_CUDA(cudaStreamSynchronize(st));
  const bool none = r[0] == 0xFFFFFFFFu;  // no S node: any scalar will do
  const bool uni = none || r[0] == r[1];
  if (uni) {
    const uint32_t bits = none ? 0u : r[0];
    FS_CUDA(cudaMemcpyAsync(&e->dstate[e->s_cur].s_age_bits, &bits, sizeof bits, cudaMemcpyHostToDevice, st));
    FS_CUDA(cudaStreamSynchronize(st));
  }
  if (uni != e->s_uniform) {
    e->s_uniform = uni;
    drop_batch_graphs(e);
    set_stream_fns(e, uni);
  }
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

int fs_host_register(void* p, int64_t bytes) {
  if (!p || bytes <= 0) return set_error(FS_EINVAL, "fs_host_register: empty range");
  const cudaError_t e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(FS_ECUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
  }
  return 0;
}

int fs_host_unregister(void* p) {
  const cudaError_t e = cudaHostUnregister(p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(FS_ECUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
  }
  return 0;
}

// fused edge-merge: the nodes with more than kWide in-edges, heaviest first
// (fs_setup.cu: degree flags, compaction, descending sort by degree)
static int build_hub_list(fs_engine* e) {
  const int64_t n = e->g.num_nodes;
  int rc = dalloc(&e->hub_list, (size_t)n);
  if (!rc) rc = dalloc(&e->hub_pre, (size_t)n);
  if (!rc) rc = dalloc(&e->hub_flag, (size_t)n);
  if (rc) return rc;
  FS_CUDA(cudaMemset(e->hub_flag, 0, sizeof(uint32_t) * n));
  rc = fs_hub_list(e->g.row_offsets, n, kWide, e->hub_list, &e->nhubs, nullptr);
  if (rc) return rc;
  FS_CUDA(cudaDeviceSynchronize());
  return 0;
}

static int engine_create(const fs_graph* g, const fs_model* m, const fs_config* c, const fs_state_buffers* buf,
                         const fs_scalars* scal, int device, const fs_partition* part, fs_engine** out) {
  if (!g || !m || !c || !buf || !scal || !out) return set_error(FS_EINVAL, "null argument");
  *out = nullptr;
  keep_pool(device);
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
  e->fresh = (buf->padded & FS_BUF_FRESH) != 0;
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
    if (part->world > FS_MAX_PARTITIONS) { delete e; return set_error(FS_EINVAL, "at most %d partitions", FS_MAX_PARTITIONS); }
    if (part->range_bounds) {
      const int64_t* b = part->range_bounds;
      bool ok = b[0] == 0 && b[part->world] == part->num_nodes_global && b[part->rank] == part->node_base &&
                b[part->rank + 1] == part->node_base + n;
      for (int r = 0; r < part->world && ok; ++r) ok = b[r] < b[r + 1] && b[r] % 32 == 0;
      if (!ok) { delete e; return set_error(FS_EINVAL, "partition: bad range boundaries"); }
      for (int r = 0; r <= part->world; ++r) e->part_bound[r] = b[r];
      e->unequal_ranges = true;
    } else {
      if ((e->comm || e->world > 1) && (e->mask_seg_words < 1 || e->mask_seg_words * e->world < e->ntiles_mask ||
                      e->node_base / 32 != (int64_t)e->rank * e->mask_seg_words)) {
        delete e;
        return set_error(FS_EINVAL, "partition: ranks must own equal mask segments of mask_segment_words words");
      }
      for (int r = 0; r <= part->world; ++r)
        e->part_bound[r] = std::min<int64_t>((int64_t)r * e->mask_seg_words * 32, part->num_nodes_global);
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
  if (e->unequal_ranges && !e->incr) {
    delete e;
    return set_error(FS_EINVAL, "unequal partition ranges need incremental counts (the mask all-gather needs equal segments)");
  }
  // (The first fused MERGE form — hubs folded by the warp of their tile —
  // measured 2-3x slower than the 2-launch merge on BA graphs: the hubs are
  // the lowest node ids, so the first tiles' warps folded tens of thousands
  // of hub edges serially.  The hub pre-pass below spreads them over the grid.)
  int rc = 0;
#define TRY(x) do { rc = (x); if (rc) { fs_engine_destroy(e); return rc; } } while (0)
  TRY(dalloc(&e->bad_flag, 1));
  e->strat = c->strategy == FS_LANE ? S_WARP : S_THREAD;
  // f32 gather: keep a bitmap of the nodes with nonzero infectivity next to
  // the infectivity buffers and gather only those (fold_*_masked) — exact
  // for finite weights; one partition; not the warp-per-node LANE fold
  if (!e->count_mode && buf->imask[0] && buf->imask[1] && !part && e->strat != S_WARP && !getenv("FS_NO_F32_MASK")) {
    bool finite = true;
    if (g->num_edges > 0) {
      if (g->weights_uniform) {
        finite = std::isfinite(g->uniform_weight);
      } else {
        TRY(cudaMemset(e->bad_flag, 0, sizeof(int)) == cudaSuccess ? 0 : set_error(FS_ECUDA, "memset"));
        k_any_nonfinite<<<(int)std::min<int64_t>((g->num_edges + 255) / 256, (int64_t)e->sms * 8), 256>>>(
            g->weights, g->weights_dtype == FS_BF16, g->num_edges, e->bad_flag);
        int bad = 0;
        TRY(cudaMemcpy(&bad, e->bad_flag, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : set_error(FS_ECUDA, "nonfinite check"));
        finite = bad == 0;
      }
    }
    e->fmask = finite;
  }
  // EDGE_MERGE (scale-free graphs), the f32 gather with the mask or the count
  // gather: ONE launch — the grid's warps first fold / count the hub rows
  // (in-degree > kWide), heaviest first, round robin, then sweep the tiles,
  // reading the hubs' results (S_HYBRID).  f32 with
  // non-finite weights (or FS_MERGE_UNFUSED): the edge-chunked merge gather
  // kernel, then the step (2 launches).
  e->merge = c->strategy == FS_MERGE && g->num_edges > 0 && !e->incr && ((!e->fmask && !e->count_mode) || getenv("FS_MERGE_UNFUSED"));
  if (c->strategy == FS_MERGE && !e->merge && !e->incr && g->num_edges > 0) e->strat = S_HYBRID;
  if (e->merge) e->fmask = false;
  if (e->incr) e->gather = G_INCR;
  else if (e->merge) e->gather = G_PRE;
  else if (e->count_mode) e->gather = e->mask_smem ? G_COUNT_SMEM : G_COUNT_GLOBAL;
  else if (e->fmask)  // (+ the hub fold stages of 32 warps behind the mask)
    e->gather = (size_t)e->ntiles_mask * 4 + (e->strat == S_HYBRID ? 32u * kHubPass * 4u : 0u) <= kMaxSmemMaskBytes
                    ? G_F32M_SMEM : G_F32M_GLOBAL;
  else e->gather = G_F32;

  for (int mat = 0; mat < 2; ++mat) e->step_fn[mat] = pick_step(e->mixed, e->gather, e->strat, mat != 0, e->step_block);
  e->step_smem = (e->gather == G_COUNT_SMEM || e->gather == G_F32M_SMEM) ? (size_t)((e->ntiles_mask + 3) & ~3LL) * 4 : 0;
  if (e->gather == G_F32M_SMEM && e->strat == S_HYBRID)
    e->step_smem += (size_t)(e->step_block / 32) * kHubPass * sizeof(float);  // the hub fold stages behind the mask
  if (e->strat == S_HYBRID) TRY(build_hub_list(e));

  int occ = 1;
  for (int mat = 0; mat < 2; ++mat) {
    if (e->step_smem > 0)
      TRY(cudaFuncSetAttribute((const void*)e->step_fn[mat], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->step_smem) == cudaSuccess ? 0 : set_error(FS_ECUDA, "smem attribute"));
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)e->step_fn[1], e->step_block, e->step_smem) != cudaSuccess || occ < 1) occ = 1;
  {  // both variants must fit the grid (the cooperative launch of S_HYBRID checks it)
    int occ0 = occ;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, (const void*)e->step_fn[0], e->step_block, e->step_smem) == cudaSuccess && occ0 >= 1)
      occ = std::min(occ, occ0);
  }
  // the step loops over 32-node tiles; do not launch CTAs with no tile
  {
    const int64_t warps_needed = e->ntiles;
    const int64_t ctas_needed = (warps_needed + e->step_block / 32 - 1) / (e->step_block / 32);
    e->step_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)e->sms * occ, ctas_needed));
  }
  if (e->count_mode) {
    e->ptab_len = (int64_t)g->d_max + 1;
    TRY(dalloc(&e->ptab, e->ptab_len));
    volatile float a_ = e->inf_val, w_ = g->uniform_weight;
    const float cval = a_ * w_;  // f32(inf * w): one IEEE single multiply
    // the k-fold sequential f32 sums of c, on the host (IEEE single adds, no
    // contraction: volatile), and whether each equals f32(k * c)
    std::vector<float> tab((size_t)e->ptab_len);
    volatile float acc = 0.0f;
    int ok = 1;
    tab[0] = 0.0f;
    for (int64_t kk = 1; kk < e->ptab_len; ++kk) {
      acc = acc + cval;
      tab[(size_t)kk] = acc;
      volatile float prod = (float)kk * cval;
      if (acc != prod) ok = 0;
    }
    TRY(put_small(e->ptab, tab.data(), sizeof(float) * tab.size(), (cudaStream_t)0));
    e->ptab_mul = ok;
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
  if (e->count_mode && !e->incr && c->strategy == FS_PER_NODE && !e->merge && g->row_offsets32 && g->padded && (buf->padded & 3) &&
      g->num_edges > 0) {
    unsigned long long* d_span = nullptr;
    TRY(dalloc(&d_span, 1));
    FS_CUDA(cudaMemset(d_span, 0, sizeof(unsigned long long)));
    k_max_tile_span<<<(int)std::min<int64_t>((e->ntiles + 255) / 256, 4096), 256>>>(g->row_offsets32, n, e->ntiles, d_span);
    unsigned long long span = 0;
    FS_CUDA(cudaMemcpy(&span, d_span, sizeof(span), cudaMemcpyDeviceToHost));
    cudaFreeAsync(d_span, (cudaStream_t)0);
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
  if (e->world > 1) {
    TRY(dalloc(&e->remote_log, e->log_cap));
    FS_CUDA(cudaMemset(e->remote_log, 0, sizeof(uint32_t) * e->log_cap));
  }
  TRY(dalloc(&e->num_active, 1));
  if (c->compaction) TRY(dalloc(&e->active_tiles, e->ntiles));
  FS_CUDA(cudaMemset(e->acc, 0, 3 * sizeof(StepAcc)));
  FS_CUDA(cudaMemset(e->num_active, 0, sizeof(int64_t)));
  {
    DevState d0{};
    d0.s = *scal;
    d0.pending = 0;
    TRY(put_small(e->dstate, &d0, sizeof(DevState), (cudaStream_t)0));
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
    e->delta_ipc = e->world > 1 || part != nullptr;  // peers map these over CUDA IPC
    TRY(dalloc(&e->delta[0], cap / 2, e->delta_ipc));
    TRY(dalloc(&e->delta[1], cap / 2, e->delta_ipc));
    if (e->world > 1) {
      // bulk exchange: mailbox entries per sender and parity ~2 per local node
      // (clamped), exported over CUDA IPC like the delta buffers; used once
      // every rank's mailbox is linked (fs_engine_set_peer_mailboxes)
      // every rank must lay its mailbox out alike (senders index it with
      // their own copy of the capacity): sized from the largest range
      int64_t widest = 0;
      for (int r = 0; r < e->world; ++r) widest = std::max<int64_t>(widest, e->part_bound[r + 1] - e->part_bound[r]);
      const char* mc = getenv("FS_MBOX_CAP");
      e->mbox_cap = mc ? std::max<int64_t>(1, atoll(mc)) : std::max<int64_t>(65536, std::min<int64_t>(2 * widest, 1 << 24));
      const size_t words = (size_t)2 * e->world * (size_t)(kMboxHdr + e->mbox_cap);
      TRY(dalloc(&e->mbox, words, true));
      FS_CUDA(cudaMemset(e->mbox, 0, words * sizeof(uint32_t)));
      TRY(dalloc(&e->mbox_ticket, (size_t)e->world));
      FS_CUDA(cudaMemset(e->mbox_ticket, 0, sizeof(unsigned) * e->world));
      e->stage_cap = std::max(16, 512 / e->world - 1);  // 512 words of staging per warp
      e->stream_smem = (size_t)(512 / 32) * e->world * (e->stage_cap + 1) * sizeof(uint32_t);
    }
    TRY(recount(e, scal->step, nullptr));
    // streaming kernel: per-node arrays readable to a multiple of 128 nodes
    if ((buf->padded & 3) >= 2 && !getenv("FS_NO_STREAM")) {
      e->stream = true;
      e->stream_hubs = g->d_max > 32;
      set_stream_fns(e, false);
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
    // the cohort table is prepared inside the step kernel's final drains
    // (an idle lane, the same hazard call: DESIGN.md §3.3) — by the streaming
    // step and the general step, not the TMA count-gather kernel.  It
    // replaces the f64 hazard of every queued E / I node by a lookup: from
    // ~1.3e5 nodes on, where that outweighs the per-warp preparation (full
    // runs: 1e4 nodes 9.2 -> 8.2 us/step without it, 1e5 even, 3e5 11.6 ->
    // 9.8 and 1e6 24.8 -> 16.9 with it, scripts/diag_memo_size.py), for the
    // log-normal and the Weibull / Erlang hazards alike (C3 warm 81 -> 87,
    // e2e 38.9 -> 44.7 G-NUPS, flushed value -1 %)
    const char* mv = getenv("FS_MEMO");
    const bool preparer = e->stream || !e->tma;
    const bool want = mv ? atoi(mv) != 0 : (preparer && n >= (int64_t)1 << 17);
    if (costly && want && !getenv("FS_NO_MEMO")) {
      TRY(dalloc(&e->entry, (size_t)((n + 127) / 128) * 128));
      TRY(dalloc(&e->ctab, (size_t)2 * kCohortSlots * kCohortW));
      TRY(dalloc(&e->cage, (size_t)2 * kCohortW));
      TRY(reset_memo(e, nullptr, e->h_step));
      if (e->stream) {  // the memo's shared-memory table only in the variant that uses it
        e->stream_memo = true;
        set_stream_fns(e, false);
      }
    }
  }
  if (getenv("FS_NO_PDL")) e->pdl = false;
  {
    // uniform S age: only the streaming kernel keeps it, and only while no
    // transition leads back into S (SIS re-enters S with its own ages)
    bool reenter = m->comp[m->edge_from].terminal != 0;
    for (int c2 = 0; c2 < m->num_compartments; ++c2)
      if (c2 != m->edge_from && !m->comp[c2].terminal && m->comp[c2].succ == m->edge_from) reenter = true;
    e->uni_ok = e->stream && !c->compaction && !reenter && !getenv("FS_NO_UNI");
    if (e->uni_ok) {
      TRY(dalloc(&e->uni_range, 2));
      if (buf->padded & FS_BUF_FRESH) {  // every age is 0 (a fresh state): uniform, scalar 0
        e->s_uniform = true;
        set_stream_fns(e, true);
      } else {
        TRY(recheck_uniform(e, nullptr));
      }
    }
  }
  if (getenv("FS_DEBUG_TIMES")) {
    const size_t g = (size_t)std::max(std::max(e->step_grid, e->step_grid_general), e->stream_grid);
    TRY(dalloc(&e->dbg, g * (4 + 32) * 16));  // per-CTA block, then the per-warp block of the probe build
    FS_CUDA(cudaMemset(e->dbg, 0, sizeof(unsigned long long) * g * (4 + 32) * 16));
  }
  for (int i = 0; i < fs_engine::kBatchEv; ++i) e->batch_ev_end[i] = -1;
  // the capture / copy streams and batch events are made on first use
  // (ensemble members never need them).  The setup work above runs on the
  // legacy stream, which does not order against non-blocking streams (every
  // PyTorch pool stream is one): wait for it here — one host wait per
  // engine, the only one (small values go in by launch argument, put_small)
  FS_CUDA(cudaGetLastError());
  TRY(cudaStreamSynchronize((cudaStream_t)0) == cudaSuccess ? 0 : set_error(FS_ECUDA, "engine setup"));
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
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  for (auto& ev : e->batch_ev) if (ev) cudaEventDestroy(ev);
  cudaDeviceSynchronize();  // no kernel of this engine is still in flight on any stream
  void* ptrs[] = {e->dstate, e->acc, e->log_clock, e->log_tau, e->log_counts, e->ptab,
                  e->active_tiles, e->num_active, e->chunk_first, e->pre, e->bad_flag,
                  e->cnt, e->entry, e->ctab, e->cage, e->dbg, e->uni_range, e->remote_log,
                  e->hub_list, e->hub_pre, e->hub_flag, e->mbox_ticket};
  for (void* q : ptrs) if (q) cudaFreeAsync(q, (cudaStream_t)0);
  if (e->mbox) cudaFree(e->mbox);
  for (void* q : {(void*)e->delta[0], (void*)e->delta[1]})
    if (q) {
      if (e->delta_ipc) cudaFree(q);
      else cudaFreeAsync(q, (cudaStream_t)0);
    }
  cudaStreamSynchronize((cudaStream_t)0);
  delete e;
}

int fs_engine_uses_count_gather(const fs_engine* e) { return e && e->count_mode ? 1 : 0; }
int fs_engine_kernels_per_step(const fs_engine* e) { return e ? (e->merge ? 2 : 1) : 0; }

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
  if (use_active && !e->tiles_valid) {  // no batch boundary yet, or host-edited states
    const int rc = refresh_tiles(e, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return launch_steps(e, nsteps, materialize != 0, use_active != 0, (cudaStream_t)stream);
}

static int batch_resources(fs_engine* e) {
  if (e->cap_stream) return 0;
  FS_CUDA(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
  FS_CUDA(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < fs_engine::kBatchEv; ++i) FS_CUDA(cudaEventCreateWithFlags(&e->batch_ev[i], cudaEventDisableTiming));
  return 0;
}

int fs_engine_run_batch(fs_engine* e, int32_t materialize, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  if (materialize && (!e->b.pressure || !e->b.rates)) return set_error(FS_EINVAL, "materialize needs pressure/rates buffers");
  FS_CUDA(cudaSetDevice(e->device));
  {
    const int rc0 = batch_resources(e);
    if (rc0) return rc0;
  }
  // one graph per (materialise, starting scalar slot): the kernels' slot
  // pointers are baked in at capture
  const int s0 = e->s_cur;
  const int64_t h0 = e->h_step;
  // the exchange's accumulator slot and mask buffer are baked in at capture
  // baked in: the step parity (early loads) and, with a communicator, the
  // exchange slot step % 3 — so key by step % 6 only when exchanging
  cudaGraphExec_t& exec = e->batch_exec[materialize ? 1 : 0][s0][e->comm ? (int)(h0 % 6) : (int)(h0 & 1)];
  if (!exec) {
    cudaGraph_t graph = nullptr;
    FS_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = launch_begin_batch(e, e->cap_stream);
    if (!rc) rc = launch_steps(e, e->c.steps_per_batch, materialize != 0, e->c.compaction != 0, e->cap_stream);
    if (!rc) {
      // fold the last step's counts into the scalars and the log at the end
      // of the batch (what the next batch's prologue would do first), so the
      // batch's whole log is final when its graph completes
      k_begin_batch<<<1, 32, 0, e->cap_stream>>>(e->dstate + e->s_cur, e->acc, e->log_counts, e->log_cap,
                                                 e->m.num_compartments, e->c.epsilon, e->c.tau_max, e->c.delta, 1);
    }
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
  const int slot = e->batch_ev_next;
  e->batch_ev_next = (slot + 1) % fs_engine::kBatchEv;
  FS_CUDA(cudaEventRecord(e->batch_ev[slot], (cudaStream_t)stream));
  e->batch_ev_end[slot] = e->h_step;
  return 0;
}

int fs_engine_read_remote_pushes(fs_engine* e, int64_t first_step, int32_t n, uint32_t* out, void* stream) {
  if (!e || n < 0 || (n > 0 && !out)) return set_error(FS_EINVAL, "bad remote-push request");
  if (n > e->log_cap) return set_error(FS_EINVAL, "request of %d steps exceeds the log capacity", n);
  if (!e->remote_log) {
    for (int i = 0; i < n; ++i) out[i] = 0;
    return 0;
  }
  FS_CUDA(cudaSetDevice(e->device));
  std::vector<uint32_t> ring(e->log_cap);
  FS_CUDA(cudaMemcpyAsync(ring.data(), e->remote_log, ring.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                          (cudaStream_t)stream));
  FS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  for (int i = 0; i < n; ++i) out[i] = ring[(first_step + i) % e->log_cap];
  return 0;
}

int fs_engine_wait_log(fs_engine* e, int64_t first_step, int32_t n, double* clocks, double* taus, int64_t* counts) {
  if (!e || n < 0) return set_error(FS_EINVAL, "bad log request");
  if (n > e->log_cap) return set_error(FS_EINVAL, "log request of %d steps exceeds capacity %lld", n, (long long)e->log_cap);
  FS_CUDA(cudaSetDevice(e->device));
  const int64_t end = first_step + n;
  int slot = -1;
  for (int i = 0; i < fs_engine::kBatchEv; ++i)
    if (e->batch_ev_end[i] == end) slot = i;
  if (slot < 0) return set_error(FS_EINVAL, "no replayed batch ends at step %lld", (long long)end);
  if (e->h_step - first_step > e->log_cap)
    return set_error(FS_EINVAL, "steps %lld.. were overwritten in the log ring", (long long)first_step);
  FS_CUDA(cudaEventSynchronize(e->batch_ev[slot]));
  const int M = e->m.num_compartments;
  cudaStream_t cs = e->copy_stream;
  // the batch's slots of the ring, in at most two contiguous pieces
  std::vector<int64_t> lk((size_t)n * kCntStride);
  for (int64_t done = 0; done < n;) {
    const int64_t s0 = (first_step + done) % e->log_cap;
    const int64_t len = std::min<int64_t>(n - done, e->log_cap - s0);
    if (clocks) FS_CUDA(cudaMemcpyAsync(clocks + done, e->log_clock + s0, len * sizeof(double), cudaMemcpyDeviceToHost, cs));
    if (taus) FS_CUDA(cudaMemcpyAsync(taus + done, e->log_tau + s0, len * sizeof(double), cudaMemcpyDeviceToHost, cs));
    FS_CUDA(cudaMemcpyAsync(lk.data() + done * kCntStride, e->log_counts + s0 * kCntStride,
                            len * kCntStride * sizeof(int64_t), cudaMemcpyDeviceToHost, cs));
    done += len;
  }
  FS_CUDA(cudaStreamSynchronize(cs));
  if (counts)
    for (int i = 0; i < n; ++i)
      for (int c2 = 0; c2 < M; ++c2) counts[(size_t)i * M + c2] = lk[(size_t)i * kCntStride + c2];
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
    if (e->count_mode || e->fmask) {
      const size_t bytes = (size_t)((e->ntiles_mask + 1 + 3) & ~3LL) * 4;
      FS_CUDA(cudaMemcpyAsync(e->b.imask[to], e->b.imask[from], bytes, cudaMemcpyDeviceToDevice, st));
    }
    if (!e->count_mode) {
      const size_t bytes = (size_t)e->g.num_nodes * (e->mixed ? 2 : 4);
      FS_CUDA(cudaMemcpyAsync(e->b.infectivity[to], e->b.infectivity[from], bytes, cudaMemcpyDeviceToDevice, st));
    }
  }
  d.s_age_bits = cur.s_age_bits;  // the uniform S age is not part of fs_scalars
  FS_CUDA(cudaMemcpyAsync(e->dstate + e->s_cur, &d, sizeof(DevState), cudaMemcpyHostToDevice, st));
  FS_CUDA(cudaMemsetAsync(e->acc, 0, 3 * sizeof(StepAcc), st));
  if ((in->step ^ cur.s.step) & 1) {  // pending deltas are indexed by step parity: rebuild
    rc = recount(e, in->step, st);
    if (rc) return rc;
  }
  if (e->hub_flag && in->step != cur.s.step)  // hub tags are step numbers
    FS_CUDA(cudaMemsetAsync(e->hub_flag, 0, sizeof(uint32_t) * e->g.num_nodes, st));
  if (in->step != cur.s.step) {  // memo tags and cohorts are relative to the step counter
    rc = reset_memo(e, st, in->step);
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
  if (e->count_mode && e->fresh) {
    // a fresh state's infectivity is beta at the infectious seeds and 0
    // elsewhere by construction: no representability check, no host sync
    e->fresh = false;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8));
    if (e->mixed)
      k_load_mask<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)inf, n, e->inf_val, e->b.imask[0] + e->node_base / 32,
                                                          e->b.imask[1] + e->node_base / 32, nullptr);
    else
      k_load_mask<float><<<blocks, 256, 0, st>>>((const float*)inf, n, e->inf_val, e->b.imask[0] + e->node_base / 32,
                                                 e->b.imask[1] + e->node_base / 32, nullptr);
    FS_CUDA(cudaGetLastError());
    return recount(e, e->h_step, st);
  }
  e->fresh = false;
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
  if (e->fmask) {  // the nonzero bitmap of the loaded values, both parities
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8));
    if (e->mixed)
      k_load_mask<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)inf, n, 0.0f, e->b.imask[0], e->b.imask[1], nullptr);
    else
      k_load_mask<float><<<blocks, 256, 0, st>>>((const float*)inf, n, 0.0f, e->b.imask[0], e->b.imask[1], nullptr);
    FS_CUDA(cudaGetLastError());
  }
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

int fs_engine_states_edited(fs_engine* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reset_memo(e, st, e->h_step);  // edited nodes no longer follow their age cohorts
  if (!rc) rc = recheck_uniform(e, st);  // the caller synced S ages (fs_engine_sync_ages) before editing
  e->tiles_valid = false;       // an edit can revive nodes of an inactive tile
  if (rc || !e->incr) return rc;
  // under compaction, inactive tiles never fold their pending deltas: start
  // the edit from exact counts of the current mask (both delta buffers clean)
  if (e->c.compaction && (rc = recount(e, e->h_step, st))) return rc;
  if (e->world > 1) return set_error(FS_ESTATE, "host state edits are not supported on partitioned engines");
  const int cur = (int)(e->h_step & 1);
  const int64_t n = e->g.num_nodes;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)e->sms * 8));
  if (e->mixed)
    k_edit_pushes<int8_t><<<blocks, 256, 0, st>>>((const int8_t*)e->b.states, e->b.imask[cur], n, e->m.infectious,
                                                  e->g.out_row_offsets, e->g.out_col_indices, e->delta[cur ^ 1]);
  else
    k_edit_pushes<int32_t><<<blocks, 256, 0, st>>>((const int32_t*)e->b.states, e->b.imask[cur], n, e->m.infectious,
                                                   e->g.out_row_offsets, e->g.out_col_indices, e->delta[cur ^ 1]);
  FS_CUDA(cudaGetLastError());
  return 0;
}

int fs_engine_reset_age_memo(fs_engine* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  FS_CUDA(cudaSetDevice(e->device));
  const int rc = reset_memo(e, (cudaStream_t)stream, e->h_step);
  return rc ? rc : recheck_uniform(e, (cudaStream_t)stream);
}

int fs_engine_state_restored(fs_engine* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  FS_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  // every per-node array and the mask were overwritten: the incremental
  // counts and pending deltas are rebuilt from the current mask, the memo and
  // the active tiles are stale, and the S-age mode is re-decided
  int rc = reset_memo(e, st, e->h_step);
  if (!rc && e->incr) {
    if (e->world > 1) return set_error(FS_ESTATE, "restoring a partitioned engine is not supported");
    rc = recount(e, e->h_step, st);
  }
  if (!rc) rc = recheck_uniform(e, st);
  e->tiles_valid = false;
  return rc;
}

int fs_engine_sync_ages(fs_engine* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  FS_CUDA(cudaSetDevice(e->device));
  return sync_s_ages(e, (cudaStream_t)stream);
}

int fs_engine_uniform_s_age(const fs_engine* e) { return e && e->s_uniform ? 1 : 0; }

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
  for (int r = 0; r < count; ++r)  // the bulk exchange's mailboxes (h_step already advanced: step h-1 ran)
    if (engines[r]->bulk) {
      engines[r]->h_step -= 1;
      const int rc = apply_mailbox(engines[r], (cudaStream_t)stream);
      engines[r]->h_step += 1;
      if (rc) return rc;
    }
  return 0;
}

int fs_engine_mailbox(fs_engine* e, void** out, int64_t* words) {
  if (!e || !out) return set_error(FS_EINVAL, "null argument");
  if (!e->mbox) return set_error(FS_EINVAL, "engine has no mailbox (node-partitioned incremental engines only)");
  *out = e->mbox;
  if (words) *words = (int64_t)2 * e->world * (kMboxHdr + e->mbox_cap);
  return 0;
}

int fs_engine_set_peer_mailboxes(fs_engine* e, void* const* ptrs) {
  if (!e || !ptrs) return set_error(FS_EINVAL, "null argument");
  if (!e->mbox) return set_error(FS_EINVAL, "engine has no mailbox (node-partitioned incremental engines only)");
  if (ptrs[e->rank] != e->mbox) return set_error(FS_EINVAL, "ptrs[rank] must be this engine's own mailbox");
  for (int r = 0; r < e->world; ++r) {
    if (!ptrs[r]) return set_error(FS_EINVAL, "mailbox of rank %d missing", r);
    e->peer_mbox[r] = (uint32_t*)ptrs[r];
  }
  e->bulk = !getenv("FS_NO_BULK");
  drop_batch_graphs(e);  // captured launches bake the exchange in
  return 0;
}

int fs_engine_apply_mailbox(fs_engine* e, void* stream) {
  if (!e) return set_error(FS_EINVAL, "null engine");
  if (!e->bulk) return 0;
  if (e->h_step < 1) return set_error(FS_ESTATE, "no step to apply");
  FS_CUDA(cudaSetDevice(e->device));
  e->h_step -= 1;  // the step that ran
  const int rc = apply_mailbox(e, (cudaStream_t)stream);
  e->h_step += 1;
  return rc;
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
  const int n = e->stream ? e->stream_grid : e->step_grid;  // [16 steps][grid][4] of the kernel in use
  if (max_ctas < n) return set_error(FS_EINVAL, "fs_engine_debug_times: need room for %d CTAs", n);
  FS_CUDA(cudaDeviceSynchronize());
  FS_CUDA(cudaMemcpy(out, e->dbg, sizeof(unsigned long long) * (4 + 32) * 16 * n, cudaMemcpyDeviceToHost));
  FS_CUDA(cudaMemset(e->dbg, 0, sizeof(unsigned long long) * (4 + 32) * 16 * n));
  return n;
}

// ---------------------------------------------------------------------------
// Ensembles (R/analysis.py:97-130 `run_ensemble`): independent trials of one
// graph and model, stepped in lockstep by ONE grid per step.  Each member is
// an ordinary engine (its own states, ages, counts, scalars, seed); the
// ensemble launches k_step_incr_multi over a device array of the members'
// StepParams, so a step of R trials costs one launch instead of R, and a
// batch is one CUDA graph of steps_per_batch such launches between two
// batched count folds.  The members' per-step logs go to one [R][cap] ring
// owned by the ensemble, read back with three 2-D copies per batch.
// ---------------------------------------------------------------------------
struct fs_ensemble {
  int device = 0;
  int count = 0;
  std::vector<fs_engine*> members;
  MultiFn fn = nullptr;
  PersistFn persist = nullptr;    // small members: one CTA runs a whole batch of steps (k_step_incr_persist)
  StepFn member_fn = nullptr;     // the members' k_step_incr variant at creation
  uint32_t ctas_per = 1;
  int grid = 1;
  bool pdl = true;
  int M = 0, steps_per_batch = 0;
  double eps = 0, tau_max = 0, delta = 0;
  int carry_tau = 1;
  StepParams* dparams = nullptr;  // [2 scalar slot][2 step parity][count]
  MemberBatch* dbatch = nullptr;  // [count]
  double* log_clock = nullptr;    // [count][cap]
  double* log_tau = nullptr;      // [count][cap]
  int64_t* log_counts = nullptr;  // [count][cap][kCntStride]
  int64_t log_cap = 0;
  int s_cur = 0;
  int64_t h_step = 0;
  cudaStream_t cap_stream = nullptr, copy_stream = nullptr;
  cudaGraphExec_t exec[2][2] = {};  // [scalar slot][step parity] at the batch start
  static constexpr int kBatchEv = 8;
  cudaEvent_t ev[kBatchEv] = {};
  int64_t ev_end[kBatchEv] = {};
  int ev_next = 0;
};

extern "C" {

void fs_ensemble_destroy(fs_ensemble* x) {
  if (!x) return;
  cudaSetDevice(x->device);
  for (auto& a : x->exec)
    for (auto& g : a) if (g) cudaGraphExecDestroy(g);
  if (x->cap_stream) cudaStreamDestroy(x->cap_stream);
  if (x->copy_stream) cudaStreamDestroy(x->copy_stream);
  for (auto& ev : x->ev) if (ev) cudaEventDestroy(ev);
  cudaDeviceSynchronize();
  for (void* q : {(void*)x->dparams, (void*)x->dbatch, (void*)x->log_clock, (void*)x->log_tau, (void*)x->log_counts})
    if (q) cudaFreeAsync(q, (cudaStream_t)0);
  cudaStreamSynchronize((cudaStream_t)0);
  delete x;
}

int fs_ensemble_create(fs_engine* const* engines, int32_t count, fs_ensemble** out) {
  if (!out) return set_error(FS_EINVAL, "null output");
  *out = nullptr;
  if (!engines || count < 1) return set_error(FS_EINVAL, "an ensemble needs at least one engine");
  const fs_engine* e0 = engines[0];
  for (int i = 0; i < count; ++i) {
    const fs_engine* e = engines[i];
    if (!e) return set_error(FS_EINVAL, "null engine %d", i);
    if (!e->stream || e->c.compaction || e->world > 1 || e->comm || e->dbg)
      return set_error(FS_EINVAL, "ensemble member %d: needs the incremental streaming step (single partition, no compaction)", i);
    if (e->device != e0->device || e->g.num_nodes != e0->g.num_nodes || e->g.out_row_offsets != e0->g.out_row_offsets ||
        e->stream_fn[0] != e0->stream_fn[0] || e->c.steps_per_batch != e0->c.steps_per_batch ||
        e->m.num_compartments != e0->m.num_compartments || e->c.epsilon != e0->c.epsilon ||
        e->c.tau_max != e0->c.tau_max || e->c.delta != e0->c.delta || e->c.carry_tau != e0->c.carry_tau ||
        e->pdl != e0->pdl)
      return set_error(FS_EINVAL, "ensemble member %d: every member needs the same device, graph, model shape, config and step kernel", i);
    if (e->s_cur != e0->s_cur || e->h_step != e0->h_step)
      return set_error(FS_EINVAL, "ensemble member %d: members must be at the same step", i);
  }
  FS_CUDA(cudaSetDevice(e0->device));
  fs_ensemble* x = new fs_ensemble();
  int rc = 0;
#define TRY(v) do { rc = (v); if (rc) { fs_ensemble_destroy(x); return rc; } } while (0)
  x->device = e0->device;
  x->count = count;
  x->members.assign(engines, engines + count);
  x->member_fn = e0->stream_fn[0];
  x->fn = pick_stream_multi(e0->mixed, false, e0->stream_memo, e0->stream_hubs, e0->s_uniform);
  if (!x->fn) { delete x; return set_error(FS_EINVAL, "no ensemble step kernel for this engine variant"); }
  // members of at most 128 tiles (4096 nodes) without the cohort table: a
  // CTA per member steps the whole batch (no launch or grid boundary per
  // step); FS_ENSEMBLE_STEPWISE keeps one launch per step
  if (e0->ntiles <= 128 && !e0->stream_memo && !e0->stream_part() && !getenv("FS_ENSEMBLE_STEPWISE"))
    x->persist = pick_stream_persist(e0->mixed, e0->stream_hubs, e0->s_uniform);
  x->pdl = e0->pdl;
  x->M = e0->m.num_compartments;
  x->steps_per_batch = e0->c.steps_per_batch;
  x->eps = e0->c.epsilon;
  x->tau_max = e0->c.tau_max;
  x->delta = e0->c.delta;
  x->carry_tau = e0->c.carry_tau;
  x->s_cur = e0->s_cur;
  x->h_step = e0->h_step;
  // CTAs per member: enough warps for its tiles, the grid about one wave
  {
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)x->fn, 512, 0) != cudaSuccess || occ < 1) occ = 1;
    const int64_t need = (e0->ntiles + 15) / 16;
    const int64_t wave = ((int64_t)e0->sms * occ + count - 1) / count;
    x->ctas_per = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(need, wave));
    const int64_t grid = (int64_t)x->ctas_per * count;
    if (grid > INT32_MAX) { delete x; return set_error(FS_EINVAL, "ensemble grid too large"); }
    x->grid = (int)grid;
  }
  x->log_cap = e0->log_cap;
  TRY(dalloc(&x->log_clock, (size_t)count * x->log_cap));
  TRY(dalloc(&x->log_tau, (size_t)count * x->log_cap));
  TRY(dalloc(&x->log_counts, (size_t)count * x->log_cap * kCntStride));
  TRY(dalloc(&x->dparams, (size_t)4 * count));
  TRY(dalloc(&x->dbatch, (size_t)count));
  {
    std::vector<StepParams> hp((size_t)4 * count);
    std::vector<MemberBatch> hb((size_t)count);
    for (int i = 0; i < count; ++i) {
      fs_engine* e = engines[i];
      for (int s = 0; s < 2; ++s)
        for (int par = 0; par < 2; ++par) {
          StepParams p = make_step_params(e, false, false, s);
          p.host_parity = par;
          p.log_clock = x->log_clock + (size_t)i * x->log_cap;
          p.log_tau = x->log_tau + (size_t)i * x->log_cap;
          p.log_counts = x->log_counts + (size_t)i * x->log_cap * kCntStride;
          p.log_cap = x->log_cap;
          p.dbg = nullptr;
          hp[((size_t)s * 2 + par) * count + i] = p;
        }
      hb[i].D[0] = e->dstate;
      hb[i].D[1] = e->dstate + 1;
      hb[i].acc = e->acc;
      hb[i].log_counts = x->log_counts + (size_t)i * x->log_cap * kCntStride;
    }
    FS_CUDA(cudaMemcpy(x->dparams, hp.data(), hp.size() * sizeof(StepParams), cudaMemcpyHostToDevice));
    FS_CUDA(cudaMemcpy(x->dbatch, hb.data(), hb.size() * sizeof(MemberBatch), cudaMemcpyHostToDevice));
  }
  FS_CUDA(cudaStreamCreateWithFlags(&x->cap_stream, cudaStreamNonBlocking));
  FS_CUDA(cudaStreamCreateWithFlags(&x->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < fs_ensemble::kBatchEv; ++i) {
    FS_CUDA(cudaEventCreateWithFlags(&x->ev[i], cudaEventDisableTiming));
    x->ev_end[i] = -1;
  }
  FS_CUDA(cudaDeviceSynchronize());
#undef TRY
  *out = x;
  return 0;
}

int fs_ensemble_grid(const fs_ensemble* x, int32_t* ctas_per_member) {
  if (!x) return set_error(FS_EINVAL, "null ensemble");
  if (ctas_per_member) *ctas_per_member = (int32_t)x->ctas_per;
  return x->grid;
}

static int ensemble_launch_batch(fs_ensemble* x, cudaStream_t st) {
  const int tb = 128, mb = (x->count + tb - 1) / tb;
  k_begin_batch_multi<<<mb, tb, 0, st>>>(x->dbatch, x->count, x->s_cur, x->log_cap, x->M, x->eps, x->tau_max, x->delta,
                                         x->carry_tau);
  int s = x->s_cur;
  int64_t h = x->h_step;
  if (x->persist) {
    x->persist<<<x->count, 512, 0, st>>>(x->dparams, (uint32_t)x->count, s, (int)(h & 1), x->steps_per_batch);
    s ^= x->steps_per_batch & 1;
    h += x->steps_per_batch;
  }
  for (int k = 0; k < x->steps_per_batch && !x->persist; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(x->grid);
    cfg.blockDim = dim3(512);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = x->pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const StepParams* P = x->dparams + ((size_t)s * 2 + (size_t)(h & 1)) * x->count;
    FS_CUDA(cudaLaunchKernelEx(&cfg, x->fn, P, x->ctas_per));
    s ^= 1;
    ++h;
  }
  // the batch's last step folded into the scalars and the log (as the
  // single-engine batch graph ends)
  k_begin_batch_multi<<<mb, tb, 0, st>>>(x->dbatch, x->count, s, x->log_cap, x->M, x->eps, x->tau_max, x->delta, 1);
  FS_CUDA(cudaGetLastError());
  return 0;
}

int fs_ensemble_run_batch(fs_ensemble* x, void* stream) {
  if (!x) return set_error(FS_EINVAL, "null ensemble");
  for (fs_engine* e : x->members)
    if (e->s_cur != x->s_cur || e->h_step != x->h_step || e->stream_fn[0] != x->member_fn)
      return set_error(FS_ESTATE, "an ensemble member was stepped or edited outside the ensemble");
  FS_CUDA(cudaSetDevice(x->device));
  cudaGraphExec_t& exec = x->exec[x->s_cur][x->h_step & 1];
  if (!exec) {
    cudaGraph_t graph = nullptr;
    FS_CUDA(cudaStreamBeginCapture(x->cap_stream, cudaStreamCaptureModeThreadLocal));
    const int rc = ensemble_launch_batch(x, x->cap_stream);
    cudaError_t err = cudaStreamEndCapture(x->cap_stream, &graph);
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (err != cudaSuccess) return set_error(FS_ECUDA, "ensemble graph capture: %s", cudaGetErrorString(err));
    err = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (err != cudaSuccess) return set_error(FS_ECUDA, "ensemble graph instantiate: %s", cudaGetErrorString(err));
  }
  FS_CUDA(cudaGraphLaunch(exec, (cudaStream_t)stream));
  x->s_cur ^= (x->steps_per_batch & 1);
  x->h_step += x->steps_per_batch;
  for (fs_engine* e : x->members) {  // the members' host mirrors follow their device state
    e->s_cur = x->s_cur;
    e->h_step = x->h_step;
  }
  const int slot = x->ev_next;
  x->ev_next = (slot + 1) % fs_ensemble::kBatchEv;
  FS_CUDA(cudaEventRecord(x->ev[slot], (cudaStream_t)stream));
  x->ev_end[slot] = x->h_step;
  return 0;
}

int fs_ensemble_wait_log(fs_ensemble* x, int64_t first_step, int32_t n, double* clocks, double* taus, int64_t* counts) {
  if (!x || n < 0) return set_error(FS_EINVAL, "bad ensemble log request");
  if (n > x->log_cap) return set_error(FS_EINVAL, "log request of %d steps exceeds capacity %lld", n, (long long)x->log_cap);
  FS_CUDA(cudaSetDevice(x->device));
  const int64_t end = first_step + n;
  int slot = -1;
  for (int i = 0; i < fs_ensemble::kBatchEv; ++i)
    if (x->ev_end[i] == end) slot = i;
  if (slot < 0) return set_error(FS_EINVAL, "no ensemble batch ends at step %lld", (long long)end);
  if (x->h_step - first_step > x->log_cap)
    return set_error(FS_EINVAL, "steps %lld.. were overwritten in the log ring", (long long)first_step);
  FS_CUDA(cudaEventSynchronize(x->ev[slot]));
  const int R = x->count, M = x->M;
  cudaStream_t cs = x->copy_stream;
  // [R][n] clocks / taus and [R][n][kCntStride] counts, ring pieces as 2-D copies
  std::vector<int64_t> lk((size_t)R * n * kCntStride);
  for (int64_t done = 0; done < n;) {
    const int64_t s0 = (first_step + done) % x->log_cap;
    const int64_t len = std::min<int64_t>(n - done, x->log_cap - s0);
    if (clocks)
      FS_CUDA(cudaMemcpy2DAsync(clocks + done, (size_t)n * sizeof(double), x->log_clock + s0, (size_t)x->log_cap * sizeof(double),
                                (size_t)len * sizeof(double), (size_t)R, cudaMemcpyDeviceToHost, cs));
    if (taus)
      FS_CUDA(cudaMemcpy2DAsync(taus + done, (size_t)n * sizeof(double), x->log_tau + s0, (size_t)x->log_cap * sizeof(double),
                                (size_t)len * sizeof(double), (size_t)R, cudaMemcpyDeviceToHost, cs));
    FS_CUDA(cudaMemcpy2DAsync(lk.data() + done * kCntStride, (size_t)n * kCntStride * sizeof(int64_t),
                              x->log_counts + s0 * kCntStride, (size_t)x->log_cap * kCntStride * sizeof(int64_t),
                              (size_t)len * kCntStride * sizeof(int64_t), (size_t)R, cudaMemcpyDeviceToHost, cs));
    done += len;
  }
  FS_CUDA(cudaStreamSynchronize(cs));
  if (counts)
    for (size_t r = 0; r < (size_t)R; ++r)
      for (int i = 0; i < n; ++i)
        for (int c2 = 0; c2 < M; ++c2)
          counts[(r * n + i) * M + c2] = lk[(r * n + i) * kCntStride + c2];
  return 0;
}

}  // extern "C"
