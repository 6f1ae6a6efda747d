/*
 * flashspread.h — C ABI of libflashspread_b200.so, the sm_100a renewal
 * tau-leaping engine (FlashSpread, arxiv 2604.22092) behind the
 * `spreadsim.renewal` Python API.
 *
 * The reference package ships no native code: its hot path is the numpy
 * function `renewal_step` (/root/reference/pkg/src/spreadsim/renewal.py:483-580)
 * driven by `run_batch` / `run_renewal` (renewal.py:600-663).  Each entry
 * point below replaces one reference interface; the Python mirror in
 * paper_2604_22092_b200/renewal.py binds them with ctypes.
 *
 * Conventions
 *  - plain C types only; device pointers are raw addresses of CUDA memory
 *    owned by the caller (torch tensors) unless stated otherwise;
 *  - every function returns 0 on success and a negative FS_E* code on
 *    failure; fs_last_error() returns a thread-local message;
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *  - no C++ exception crosses the ABI.
 */
#ifndef FLASHSPREAD_H
#define FLASHSPREAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_ABI_VERSION 6
#define FS_MAX_COMPARTMENTS 16

/* error codes */
#define FS_OK 0
#define FS_EINVAL (-1)   /* bad argument (ValueError on the Python side) */
#define FS_ECUDA (-2)    /* CUDA runtime error */
#define FS_ENOMEM (-3)   /* device allocation failed */
#define FS_ESTATE (-4)   /* engine misuse (e.g. reconfigure after start) */
#define FS_ECONSERVE (-5)/* compartment counts no longer sum to N */
#define FS_EREPR (-6)    /* infectivity not representable by the count gather */

/* element types of the arrays that cross the boundary */
enum fs_dtype {
  FS_I8 = 1, FS_I32 = 2, FS_I64 = 3, FS_F16 = 4, FS_BF16 = 5,
  FS_F32 = 6, FS_F64 = 7, FS_U32 = 8, FS_U64 = 9
};

/* CSR traversal strategy — graph.py:61-67 `Strategy` */
enum fs_strategy { FS_PER_NODE = 0, FS_LANE = 1, FS_MERGE = 2, FS_AUTO = 3 };

/* holding-time hazard of a nodal compartment — models.py:35-51 `Holding`
 * (weibull / erlang are north_star extensions absent from the reference) */
enum fs_hazard {
  FS_HZ_NONE = 0,        /* absorbing, or the edge-driven S compartment */
  FS_HZ_EXPONENTIAL = 1, /* p0 = rate                                  */
  FS_HZ_LOGNORMAL = 2,   /* p0 = mu, p1 = sigma  (hazards.py:122-132)  */
  FS_HZ_WEIBULL = 3,     /* p0 = shape k, p1 = scale lambda            */
  FS_HZ_ERLANG = 4       /* p0 = shape k (integer), p1 = rate r        */
};

/* transmission profile s(tau) — hazards.py:161-218 `Shedding` */
enum fs_shedding { FS_SHED_CONSTANT = 0, FS_SHED_LN_HAZARD = 1, FS_SHED_DENSITY_PEAK = 2 };

/* counter-based uniform source */
enum fs_rng {
  FS_RNG_SPLITMIX = 0, /* reference mixer, rng.py:48-67 (bit-exact parity) */
  FS_RNG_PHILOX = 1    /* Philox4x32-10, key=seed, counter=(node, step)    */
};

/* precision of the hazard / shedding evaluation */
enum fs_hazard_precision { FS_HAZ_F64 = 0, FS_HAZ_F32 = 1 };

typedef struct fs_graph {
  int64_t num_nodes;
  int64_t num_edges;
  const int64_t* row_offsets;   /* device, int64[N+1] (graph.py:77-93)        */
  const int32_t* row_offsets32; /* optional int32 copy (E < 2^31) read by the
                                   hot kernels instead; NULL = use row_offsets */
  const int32_t* col_indices;   /* device, int32[E], slices sorted by source  */
  const void* weights;          /* device, f32[E] or bf16[E]; NULL if uniform */
  int32_t weights_dtype;        /* FS_F32 | FS_BF16                           */
  int32_t weights_uniform;      /* 1: every weight == uniform_weight          */
  float uniform_weight;         /* the common weight (already bf16-rounded in mixed mode) */
  int32_t d_max;                /* max in-degree                               */
  int32_t padded;               /* 1: row_offsets32 readable to N+9 entries and
                                   col_indices to E+4 (TMA bulk-copy slack)   */
  /* outgoing CSR (the transpose; the incoming arrays themselves for the
   * symmetric graphs of every reference generator), int64[N_global+1] /
   * int32[E]: the push targets of the incremental count mode; NULL = none */
  const int64_t* out_row_offsets;
  const int32_t* out_col_indices;
} fs_graph;

typedef struct fs_compartment {
  int32_t succ;      /* successor compartment when the transition fires */
  int32_t terminal;  /* absorbing: age frozen, rate 0                  */
  int32_t hazard;    /* enum fs_hazard                                  */
  int32_t pad_;
  double p0, p1;     /* hazard parameters, see enum fs_hazard           */
} fs_compartment;

typedef struct fs_model {   /* models.py:54-101 `ModelSpec` */
  int32_t num_compartments;
  int32_t edge_from;         /* S: rate = pressure  */
  int32_t edge_to;           /* first infected successor */
  int32_t infectious;        /* compartment exerting pressure */
  double beta;
  int32_t shedding;          /* enum fs_shedding */
  int32_t pad_;
  double shed_mu, shed_sigma;/* log-normal parameters of the profile */
  double shed_peak;          /* f(mode) for FS_SHED_DENSITY_PEAK     */
  fs_compartment comp[FS_MAX_COMPARTMENTS];
} fs_model;

typedef struct fs_config {  /* renewal.py:75-99 `RenewalConfig` (+ rng, hazard_precision) */
  double epsilon, tau_max, delta;
  int32_t steps_per_batch;
  int32_t strategy;          /* resolved enum fs_strategy (never FS_AUTO here) */
  int32_t compaction;
  int32_t mixed_precision;   /* states i8 / ages f16 / infectivity bf16        */
  int32_t lanes_per_node;
  int32_t edges_per_block;
  int32_t hazard_chunk;      /* accepted; results are chunk-independent        */
  int32_t chunk_skip;        /* accepted; results are skip-independent         */
  int32_t carry_tau;
  int32_t rng;               /* enum fs_rng                                    */
  int32_t hazard_precision;  /* enum fs_hazard_precision                       */
  int32_t count_gather;      /* -1 auto, 0 force general f32 gather, 1 require count gather */
  int32_t incremental;       /* count gather only: -1 auto, 0 off (gather the mask every step),
                                1 require — keep per-node infectious-neighbour counts current
                                by pushes along the outgoing CSR instead of re-gathering */
} fs_config;

/* device-resident engine scalars; mirrors the scalar fields of
 * `RenewalState` (renewal.py:114-126) */
typedef struct fs_scalars {
  double clock;         /* simulated time                         */
  double tau_next;      /* tau_prev of the reference: next step's tau */
  int64_t step;         /* step_counter                           */
  uint64_t seed;        /* RNG seed of the run                     */
  float last_max_rate;  /* max rate of the last step              */
  int32_t started;
  int64_t counts[FS_MAX_COMPARTMENTS];
} fs_scalars;

/* per-node state arrays (device, caller-owned) */
typedef struct fs_state_buffers {
  void* states;          /* int32[N] (int8[N] mixed)                         */
  void* ages;            /* f32[N]   (f16[N] mixed)                          */
  void* infectivity[2];  /* general gather: f32/bf16[N] double buffer         */
  uint32_t* imask[2];    /* count gather: infectious bit-mask double buffer,
                            uint32[ceil(N/32)] each, allocated to a 16-byte
                            multiple and 16-byte aligned (TMA bulk staging) */
  float* pressure;       /* f32[N], written on materialising steps            */
  float* rates;          /* f32[N], written on materialising steps            */
  int32_t padded;        /* 1: states/ages readable to a multiple of 32 nodes,
                            2: to a multiple of 128 nodes (streaming kernel);
                            | FS_BUF_FRESH: a fresh init_renewal_state —
                            every age 0, infectivity beta at the infectious
                            seeds — so the engine skips the checks that need
                            host round trips */
} fs_state_buffers;
#define FS_BUF_FRESH 4

/* node partition of a multi-GPU run: this
 * engine owns global nodes [node_base, node_base + g->num_nodes); its CSR
 * rows hold GLOBAL column ids; its mask buffers are global (every rank holds
 * the whole infectious mask, at least max(world * mask_segment_words,
 * ceil(N_global/32) + 1) words).  With `comm` (an ncclComm_t from
 * fs_comm_init) every step is followed by one NCCL group: all-reduce of the
 * count deltas and the max rate, in-place all-gather of the mask segments
 * (rank r owns words [r * mask_segment_words, (r+1) * mask_segment_words),
 * so node_base = r * 32 * mask_segment_words).  Without `comm` the engines of
 * one process share the mask buffers and call fs_engines_exchange_local.
 * Requires the count gather (constant transmission, uniform weights). */
#define FS_MAX_PARTITIONS 16
typedef struct fs_partition {
  int64_t node_base;
  int64_t num_nodes_global;
  int64_t mask_segment_words;
  int32_t rank, world;
  void* comm;
  /* world + 1 node boundaries (multiples of 32) of unequal, e.g. edge-
   * balanced, ranges; nullable: equal ranges of
   * mask_segment_words * 32 nodes.  Unequal ranges need incremental counts
   * (no mask all-gather). */
  const int64_t* range_bounds;
} fs_partition;

typedef struct fs_engine fs_engine;

int fs_abi_version(void);
const char* fs_last_error(void);
int fs_device_sm_count(int device);
/* page-lock / release a host range (cudaHostRegister), for callers that
 * upload the same host arrays repeatedly; the CSR upload itself goes through
 * fs_h2d_staged (registering fresh pages cost ~0.4 ms per MB on B200 hosts) */
int fs_host_register(void* p, int64_t bytes);
int fs_host_unregister(void* p);

/* Engine: renewal.py:321-355 `_build_plan` + the device side of
 * `init_renewal_state` (370-410).  Reads `*scal` (host) as the initial
 * scalars.  count_gather resolution: the bit-mask gather is used when the
 * transmission is constant and the weights uniform (exact). */
int fs_engine_create(const fs_graph* g, const fs_model* m, const fs_config* c,
                     const fs_state_buffers* buf, const fs_scalars* scal,
                     int device, fs_engine** out);
int fs_engine_create_partitioned(const fs_graph* g, const fs_model* m, const fs_config* c,
                                 const fs_state_buffers* buf, const fs_scalars* scal, int device,
                                 const fs_partition* part, fs_engine** out);
void fs_engine_destroy(fs_engine* e);
/* single-process partition exchange (the NCCL group's effect on engines that
 * share one device and their mask buffers): call after every engine ran the
 * same step */
int fs_engines_exchange_local(fs_engine* const* engines, int32_t count, void* stream);
/* Partitioned incremental counts: a rank whose node changes
 * infectious status pushes +-1 straight into the owner's pending-delta array —
 * in its own memory or a peer's over NVLink — during the step, so the only
 * per-step collective left is the tiny count / max-rate all-reduce.  Each
 * engine exposes its two delta buffers (by step parity); every engine must be
 * given all ranks' buffers, ptrs[parity * world + rank], before stepping:
 * the other engines' pointers directly (one device) or peer mappings from
 * fs_ipc_open_handle (one process per GPU). */
int fs_engine_delta_buffers(fs_engine* e, void** out2);
/* Bulk exchange of the pushes to other ranks: each warp
 * stages them in shared memory per owner and writes them, after each drain,
 * into the owner's mailbox with one remote cursor atomic per owner and
 * coalesced peer stores (instead of one NVLink atomic per push); after the
 * step's exchange every rank folds its mailbox into its pending deltas.
 * fs_engine_mailbox exposes this rank's mailbox (2 x world x (32 + cap)
 * words, for CUDA IPC export); fs_engine_set_peer_mailboxes(ptrs[world])
 * turns the mode on (ptrs[rank] = own mailbox; FS_NO_BULK keeps the direct
 * atomics).  Engines stepped with a communicator, or through
 * fs_engines_exchange_local, apply their mailbox automatically; with a
 * host-side exchange call fs_engine_apply_mailbox after it. */
int fs_engine_mailbox(fs_engine* e, void** out, int64_t* words);
int fs_engine_set_peer_mailboxes(fs_engine* e, void* const* ptrs);
int fs_engine_apply_mailbox(fs_engine* e, void* stream);
/* host-side step exchange (partitioned engines without a communicator): the
 * last step's accumulator — 16 count deltas and the max-rate bits, 17 u64 —
 * out to the host and, reduced over ranks, back before the next step */
int fs_engine_acc_get(fs_engine* e, uint64_t* out17, void* stream);
int fs_engine_acc_set(fs_engine* e, const uint64_t* in17, void* stream);
int fs_engine_set_peer_deltas(fs_engine* e, void* const* ptrs);
int fs_ipc_get_handle(void* dptr, uint8_t* out, int32_t len);
int fs_ipc_open_handle(const uint8_t* handle, int32_t device, void** out);
int fs_ipc_close(void* dptr);
/* NCCL communicator of a partitioned run: rank 0 makes the id (returns its
 * byte length, <= len), every rank calls fs_comm_init with it */
int fs_comm_unique_id(uint8_t* out, int32_t len);
int fs_comm_init(int32_t world, int32_t rank, const uint8_t* id, int32_t device, void** comm);
void fs_comm_destroy(void* comm);
/* 1 if the engine gathers from the infectious bit-mask, 0 for the f32 gather */
int fs_engine_uses_count_gather(const fs_engine* e);
/* Kernel launches one step issues (1: the fused step; 2: a separate
 * edge-chunked merge gather before it).  Diagnostic, for launch counting. */
int fs_engine_kernels_per_step(const fs_engine* e);
/* Uniform S age (SEIR / SIR: S is never re-entered, so every S node has the
 * same age, R/renewal.py:540-542).  While on, the step kernel keeps the S
 * age as one scalar and does not read or write it per node.
 * fs_engine_sync_ages writes it back into the ages array — call it before
 * reading or editing ages / states on the host; fs_engine_states_edited and
 * fs_engine_reset_age_memo re-decide the mode from the array afterwards.
 * Replaces nothing in the reference (an encoding of RenewalState.ages,
 * R/renewal.py:114-126). */
int fs_engine_sync_ages(fs_engine* e, void* stream);
/* The host overwrote the engine's state arrays and mask buffers wholesale
 * (a snapshot restore): rebuild the incremental counts from the current mask,
 * invalidate the hazard memo and the active tiles, re-decide the S-age mode.
 * Call after fs_engine_set_scalars.  No reference counterpart (the
 * reference's state is plain numpy arrays). */
int fs_engine_state_restored(fs_engine* e, void* stream);

/* Log of the replayed batch that ended at step first_step + n (a batch
 * launched by fs_engine_run_batch; the engine keeps the last 8): waits for
 * that batch only and copies its per-step clocks / taus / counts on a side
 * stream, so the next batch can already be running — the pipelined
 * run_renewal loop (R/renewal.py:632-663 reads the recorder after each
 * batch).  Every replayed batch ends by folding its last step's counts. */
int fs_engine_wait_log(fs_engine* e, int64_t first_step, int32_t n, double* clocks, double* taus, int64_t* counts);

/* ---- ensembles (R/analysis.py:97-130 run_ensemble, DESIGN.md §8 row 2) --- */
/* Independent trials of one graph and model stepped in lockstep by ONE grid
 * per step: every member is an ordinary engine (its own buffers, scalars and
 * seed) built with the incremental streaming step, all at the same step; a
 * member is bit-identical to its engine run alone.  Members must not be
 * stepped or edited while they belong to the ensemble (run_batch refuses);
 * destroy the ensemble before the engines. */
typedef struct fs_ensemble fs_ensemble;
int fs_ensemble_create(fs_engine* const* engines, int32_t count, fs_ensemble** out);
void fs_ensemble_destroy(fs_ensemble* x);
/* CTAs of one step launch (return value) and per member */
int fs_ensemble_grid(const fs_ensemble* x, int32_t* ctas_per_member);
/* one CUDA-graph batch of steps_per_batch lockstep steps of every member,
 * ending with every member's count fold (fs_engine_run_batch for R trials) */
int fs_ensemble_run_batch(fs_ensemble* x, void* stream);
/* per-member log of the batch ending at first_step + n: clocks[R][n],
 * taus[R][n], counts[R][n][M] (any may be NULL); waits for that batch only */
int fs_ensemble_wait_log(fs_ensemble* x, int64_t first_step, int32_t n, double* clocks, double* taus, int64_t* counts);
/* Partitioned runs: per-step count of the +-1 pushes this rank sent to other
 * ranks' pending deltas (over NVLink on a multi-GPU box), for steps
 * [first_step, first_step + n) still in the log ring. */
int fs_engine_read_remote_pushes(fs_engine* e, int64_t first_step, int32_t n, uint32_t* out, void* stream);
/* Mean device time of the per-step exchange (the NCCL group of the count /
 * max-rate all-reduces, plus the mask all-gather when seg_words > 0) over
 * `iters` back-to-back calls on `stream`, in microseconds. */
int fs_comm_time_exchange(void* comm, int32_t rank, int64_t seg_words, int32_t iters, void* stream, float* us);

/* ---- host side of the upload (fs_hostio.cpp) --------------------------- */
/* host -> device copy of a pageable array through the library's page-locked
 * staging slots, host threads filling one slot while the next is in flight */
int fs_h2d_staged(void* dst, const void* src, int64_t bytes, void* stream);
/* max in-degree of an int64 CSR (R/graph.py:194-201) and whether every f32
 * weight is equal (the uniform-weight scalar), with host threads */
int fs_host_csr_scan(const int64_t* row_offsets, int64_t n, const float* weights, int64_t num_edges, int64_t* d_max,
                     int32_t* uniform, float* w0);

/* ---- run setup on the device (fs_setup.cu) ------------------------------ */
/* Seed choice of init_renewal_state: the `count` nodes with the smallest
 * uniform_array(seed_key, 0, id) (R/renewal.py:162-169 _pick_seed_nodes,
 * seed_key = derive_seed(seed, 0x5EEDC0DE)), by a device radix select.  Each
 * chosen node gets states[i] = compartment (states may be null) and, when inf
 * is non-null, inf[i] = inf_value (cast on store); flags (nullable, u8[n])
 * receives 1 for chosen nodes.  Ties of the 53-bit uniform go to the smaller
 * id. */
int fs_seed_select(int64_t n, uint64_t seed_key, int64_t count, void* states, int32_t states_dtype,
                   int32_t compartment, void* inf, int32_t inf_dtype, float inf_value, uint8_t* flags,
                   void* stream);
/* the same selection for `trials` independent trials of one small graph
 * (N <= 4096) in one launch: trial t's states / infectivity at offset
 * t * stride, its pick key pick_keys[t] (host array) — the ensemble's
 * per-trial init_renewal_state (renewal.py:162-169) without host round trips */
int fs_seed_select_batch(int64_t n, int32_t trials, const uint64_t* pick_keys, int64_t count, void* states,
                         int64_t stride, int32_t states_dtype, int32_t compartment, void* inf, int32_t inf_dtype,
                         float inf_value, void* stream);
/* ids of the set flags in increasing order (sorted seed ids) */
int fs_flags_to_ids(const uint8_t* flags, int64_t n, int64_t* out_ids, int64_t* num_out, void* stream);
/* Is the incoming CSR its own transpose (an undirected graph, R/graph.py:
 * 221-231)?  Rows must be sorted by source (R/graph.py:141); *symmetric = 0
 * otherwise.  row_offsets32 (nullable) is preferred when given. */
int fs_check_symmetric(const int64_t* row_offsets, const int32_t* row_offsets32, const int32_t* col, int64_t n,
                       int64_t num_edges, int32_t* symmetric, void* stream);
/* int32 copy of int64 row offsets (E < 2^31) */
int fs_narrow_offsets(const int64_t* row_offsets, int64_t len, int32_t* out, void* stream);
/* fill n elements of elem_bytes (1, 2, 4, 8) with the low bytes of pattern */
int fs_fill(void* ptr, int64_t n, int32_t elem_bytes, uint64_t pattern, void* stream);
int fs_engine_uniform_s_age(const fs_engine* e);
/* which of the two infectivity / mask buffers holds the current step's input */
int fs_engine_current_buffer(fs_engine* e, void* stream);

/* renewal.py:583-597 `_begin_batch`: tau reset (carry_tau off) and, with
 * compaction, rates zeroing + active-tile refresh */
int fs_engine_begin_batch(fs_engine* e, void* stream);
/* renewal.py:483-580 `renewal_step` x nsteps, launched eagerly; the last
 * step materialises pressure/rates when `materialize` is nonzero; with
 * `use_active` only the tiles of the last begin_batch refresh are stepped
 * (the `active=` argument of renewal_step) */
int fs_engine_step(fs_engine* e, int32_t nsteps, int32_t materialize, int32_t use_active, void* stream);
/* renewal.py:600-629 `run_batch`: begin_batch + steps_per_batch steps,
 * replayed from a CUDA graph captured on first use */
int fs_engine_run_batch(fs_engine* e, int32_t materialize, void* stream);
/* Per-step log of steps [first_step, first_step+n): clock[n], tau[n] and
 * counts[n][M] (host arrays, any may be NULL) — the recorder of run_batch
 * (renewal.py:622-627).  The ring holds max(256, 4*steps_per_batch) steps. */
int fs_engine_read_log(fs_engine* e, int64_t first_step, int32_t n,
                       double* clocks, double* taus, int64_t* counts, void* stream);
int fs_engine_get_scalars(fs_engine* e, fs_scalars* out, void* stream);
int fs_engine_set_scalars(fs_engine* e, const fs_scalars* in, void* stream);
/* The engine memoises nodal hazards per age cohort (nodes that entered a
 * compartment at the same step share their age bit for bit): call this after
 * writing ages or states from outside the engine (host edits, snapshot
 * restores) so no node is assumed to follow its cohort. */
int fs_engine_reset_age_memo(fs_engine* e, void* stream);
/* the caller wrote `states` between steps: re-derive what the engine keeps
 * from them (age cohorts; with incremental counts, the pushes the edited
 * nodes' changes of infectious status imply for the step after next) */
int fs_engine_states_edited(fs_engine* e, void* stream);
/* re-derive the infectious mask / general buffer from a freshly uploaded
 * infectivity array (host edits between steps); `inf` has the storage dtype */
int fs_engine_load_infectivity(fs_engine* e, const void* inf, void* stream);
/* expand the current infectivity to the storage dtype (for reads) */
int fs_engine_store_infectivity(fs_engine* e, void* inf_out, void* stream);

/* renewal.py:264-313 `pressure_gather`: p_i = sum_e f32(inf[col[e]] * w[e])
 * folded in CSR order with an f32 accumulator, any strategy, bit-exact. */
int fs_pressure_gather(const fs_graph* g, const void* infectivity, int32_t inf_dtype,
                       float* out, int32_t strategy, int32_t lanes_per_node,
                       int32_t edges_per_block, void* stream);

/* rng.py:60-67 `uniform_array` (splitmix) or Philox4x32-10; streams==NULL
 * means streams = arange(n) */
int fs_uniform_fill(uint64_t seed, uint64_t step, const uint64_t* streams, int64_t n,
                    int32_t rng, double* out, void* stream);

/* hazards.py:122-132 `_hazard_f64` (and the weibull / erlang extensions):
 * out[i] = h(tau[i]) in f64 (precision FS_HAZ_F64) or fp32 math widened */
int fs_hazard_eval(const fs_compartment* c, const double* tau, int64_t n, double* out,
                   int32_t precision, void* stream);
/* hazards.py:108-119 `erfcx_stable` */
int fs_erfcx_eval(const double* z, int64_t n, double* out, void* stream);

/* renewal.py:426-432 `refresh_active`: sorted ids of non-terminal nodes.
 * `terminal` is a host array of num_compartments bytes. out_ids has N+pad
 * entries (zero-padded); *num_active is written (host). */
int fs_refresh_active(const void* states, int32_t states_dtype, int64_t n,
                      const uint8_t* terminal, int32_t num_compartments,
                      int32_t* out_ids, int64_t capacity, int64_t* num_active,
                      void* stream);


/* Random uniform-degree graph on the device (input construction for the
 * N = 1e8 / 1e9 configs; the reference's CPU generator gen_fixed_degree,
 * graph.py:289-328, does not scale there — DESIGN.md §8).  Union of d/2
 * keyed random Hamiltonian cycles (+ one perfect matching when d is odd);
 * shared edges dropped at both endpoints; slices sorted by source.  Writes
 * rows [row_lo, row_hi) of the incoming CSR with GLOBAL column ids:
 * row_offsets int64[rows+1] (local, from 0), col int32[col_capacity].  With
 * col == NULL only the offsets and *num_edges are produced (sizing call).
 * Every rank of a node-partitioned run generates its own rows, no exchange. */
int fs_gen_regular(int64_t n, int32_t k, uint64_t seed, int64_t row_lo, int64_t row_hi,
                   int64_t* row_offsets, int32_t* col, int64_t col_capacity, int64_t* num_edges,
                   void* stream);
/* Barabási–Albert preferential attachment (the model of the reference's
 * gen_barabasi_albert, R/graph.py:331-365: m-clique seed, each new node
 * attaches to m distinct nodes drawn from the endpoint list) and G(N, p)
 * with p = min(d_avg / (N-1), 1) (gen_erdos_renyi, R/graph.py:252-286), on
 * the device with counter-based draws (csrc/fs_gen_random.cu).  Same
 * output convention as fs_gen_regular: rows [row_lo, row_hi) of the
 * symmetric incoming CSR, global column ids, slices sorted; col == NULL is
 * the sizing call.  Deterministic for a seed; not the reference's numpy
 * stream, so parity is by the model's properties (tests/test_graphgen.py). */
int fs_gen_barabasi_albert(int64_t n, int32_t m, uint64_t seed, int64_t row_lo, int64_t row_hi,
                           int64_t* row_offsets, int32_t* col, int64_t col_capacity, int64_t* num_edges,
                           void* stream);
int fs_gen_erdos_renyi(int64_t n, double d_avg, uint64_t seed, int64_t row_lo, int64_t row_hi,
                       int64_t* row_offsets, int32_t* col, int64_t col_capacity, int64_t* num_edges,
                       void* stream);
/* host evaluation of one row of the same construction (tests); returns the
 * distinct degree and writes the sorted neighbours to out[k] */
int fs_gen_regular_row_host(int64_t n, int32_t k, uint64_t seed, int64_t node, int32_t* out);

/* ------------------------------------------------------------------------
 * Markovian tau-leaping engine (R/markov.py:34-228).
 * All-exponential models with constant transmission; influence = number of
 * infectious in-neighbours x the uniform weight, kept by pushes along the
 * outgoing CSR; tau = min(theta N / sum(rates), p_max / max(rates),
 * tau_max) with the sum in numpy's pairwise order (bit-identical to
 * R/markov.py:149-154).  `states` int32[N] and `rates` f64[N] are caller
 * owned; fs_scalars carries clock / step / seed / counts (tau_next = the tau
 * of the last step). */
typedef struct fs_markov_config {  /* R/markov.py:34-46 `MarkovConfig` */
  double theta, p_max, tau_max;
  int32_t steps_per_batch;
  int32_t pad_;
} fs_markov_config;
typedef struct fs_markov fs_markov;
int fs_markov_create(const fs_graph* g, const fs_model* m, const fs_markov_config* c, int32_t* states,
                     double* rates, const fs_scalars* scal, int device, fs_markov** out);
void fs_markov_destroy(fs_markov* e);
/* R/markov.py:143-181 `markov_step` x nsteps (eager) */
int fs_markov_step(fs_markov* e, int32_t nsteps, void* stream);
/* steps_per_batch steps as one CUDA-graph replay */
int fs_markov_run_batch(fs_markov* e, void* stream);
int fs_markov_get_scalars(fs_markov* e, fs_scalars* out, void* stream);
/* write scalars (and the seed); counts are rebuilt from the states */
int fs_markov_set_scalars(fs_markov* e, const fs_scalars* in, void* stream);
int fs_markov_read_log(fs_markov* e, int64_t first_step, int32_t n, double* clocks, double* taus,
                       int64_t* counts, void* stream);
/* recompute rates[] from the current states and influence (the state.rates
 * the reference holds after a step, R/markov.py:178) */
int fs_markov_refresh_rates(fs_markov* e, void* stream);
/* R/markov.py:68-81 `influence_gather` of the current states (host f64[N]) */
int fs_markov_influence(fs_markov* e, double* out, void* stream);

/* ------------------------------------------------------------------------
 * Device-side trajectory records and ensemble analysis (SURVEY.md §8f row
 * 4; the consumers of the per-step log).  Every pointer is device memory
 * unless noted; all arithmetic is f64. */

/* make_record (R/trajectory.py:31-61) for `trials` logs at once.  Trial t's
 * log is times[t*max_steps + s], counts[(t*max_steps + s)*ncomp + c] for
 * s < lens[t] (times non-decreasing, from 0).  grid f64[grid_points] is the
 * reference's np.linspace(0, t_final, grid_points).  Writes fractions
 * f64[trials][grid_points][ncomp] (grid-major, the memory order of the
 * reference's Fortran-order record; = f64(count) / f64(num_nodes) of the last
 * sample at or before each grid time, bit-identical to numpy) and, when
 * i_idx / r_idx >= 0, summary f64[trials][3] = peak_I, grid time of the first
 * peak, final_R (entries of an absent compartment are left untouched). */
int fs_traj_records(const double* times, const int64_t* counts, const int64_t* lens, int64_t trials,
                    int64_t max_steps, int32_t ncomp, const double* grid, int32_t grid_points,
                    int64_t num_nodes, int32_t i_idx, int32_t r_idx, double* fractions, double* summary,
                    void* stream);
/* x f64[runs][cols] -> out f64[cols] = x.mean(axis=0) (R/analysis.py:137-138;
 * sequential in run order, then / runs: bit-identical to numpy) */
int fs_ensemble_mean(const double* x, int64_t runs, int64_t cols, double* out, void* stream);
/* np.quantile(column, q, method="linear") of ncols columns of n values
 * (value i of column c at x[i*row_stride + c*col_stride]), 1 <= n <= 16384.
 * prev / next / gamma are HOST arrays of nq <= 8 entries: numpy's
 * _get_indexes (-1 = last) and _get_gamma for each quantile.  out
 * f64[nq][ncols]; numpy's _lerp, bit-identical (quantile_band
 * R/analysis.py:141-148, _percentile_ci :160-162). */
int fs_column_quantiles(const double* x, int64_t n, int64_t ncols, int64_t row_stride, int64_t col_stride,
                        int32_t nq, const int64_t* prev, const int64_t* next, const double* gamma,
                        double* out, void* stream);
/* The resampling loop of fidelity (R/analysis.py:226-240): ensembles a
 * f64[na][ncomp*grid_points], b f64[nb][...]; multinomial resample counts
 * int64[resamples][na] / [resamples][nb] (the reference's
 * _resample_weights draws, weights = count / n); per_run_peak / _final
 * f64[na] (fs_run_deviation; ignored when i_idx / r_idx < 0);
 * weights_scratch f64[resamples*(na+nb)].  samples f64[6][resamples]:
 * l_inf, l2, err_peak_i, err_final_r, w.per_run_peak, w.per_run_final. */
int fs_bootstrap_metrics(const double* a, int64_t na, const double* b, int64_t nb, int32_t ncomp,
                         int32_t grid_points, const int64_t* counts_a, const int64_t* counts_b,
                         int64_t resamples, int32_t i_idx, int32_t r_idx, const double* per_run_peak,
                         const double* per_run_final, double* weights_scratch, double* samples,
                         void* stream);
/* per run i: peak_dev[i] = |max_g a[i][i_idx][g] - ref_peak|, final_dev[i] =
 * |a[i][r_idx][G-1] - ref_final| (R/analysis.py:218-224; bit-identical) */
int fs_run_deviation(const double* a, int64_t runs, int32_t ncomp, int32_t grid_points, int32_t i_idx,
                     int32_t r_idx, double ref_peak, double ref_final, double* peak_dev, double* final_dev,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FLASHSPREAD_H */
