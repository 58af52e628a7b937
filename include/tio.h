/*
 * tio.h — C ABI of libtio, the B200 (sm_100a) lifetime / plan / migration
 * hot path.  Plain pointers and sizes only; no torch types.
 *
 * The reference (`offloader`, pure Python) has no FFI: its boundary is the
 * module API re-exported by pkg/src/offloader/__init__.py:4-65.  Each entry
 * point below names the reference function(s) it replaces; the Python shim
 * paper_2506_06472_b200/ (and INTEGRATION.md's ctypes stub) binds them with
 * the reference's names, argument meaning and exceptions.
 *
 * Conventions
 *   - return value: TIO_OK (0) or a negative TIO_ERR_* code; the message of
 *     the last failure on the calling thread is available via tio_last_error.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - memory kinds: TIO_MEM_HOST (pageable or pinned host pointers; copied to
 *     the device inside the call) or TIO_MEM_DEVICE (device pointers, used in
 *     place, must stay valid for the lifetime of the handle).
 *   - handles are opaque, owned by the library, freed with *_destroy.
 *   - integers are int64 (times in microseconds, sizes in bytes); the
 *     reference uses unbounded Python ints, callers must stay inside int64.
 */
#ifndef TIO_H_
#define TIO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TIO_ABI_VERSION 1

enum {
    TIO_OK = 0,
    TIO_ERR_INVALID = -1,        /* bad argument / handle (ValueError)                 */
    TIO_ERR_UNSATISFIABLE = -2,  /* planner.py:59-66 UnsatisfiableTraceError           */
    TIO_ERR_CHANNEL_CONFIG = -3, /* bandwidth.py:27-28 ChannelConfigError              */
    TIO_ERR_CUDA = -4,           /* CUDA runtime failure                               */
    TIO_ERR_NOMEM = -5,
    TIO_ERR_INTERNAL = -6,       /* planner.py:316-320 divergence assert / invariant   */
    TIO_ERR_OVERFLOW = -7,       /* value outside the int64 domain                     */
    TIO_ERR_SIMULATION = -8,     /* simulator.py:51-52 SimulationError                 */
    TIO_ERR_CONFIG = -9          /* simulator.py:55-56 ConfigurationError              */
};

enum { TIO_MEM_HOST = 0, TIO_MEM_DEVICE = 1 };
enum { TIO_KIND_INTERMEDIATE = 0, TIO_KIND_GLOBAL = 1 };
enum { TIO_DEST_NONE = 0, TIO_DEST_SSD = 1, TIO_DEST_CPU = 2 };

/* Column form of a trace (reference Trace, trace.py:87-110).  accesses of
 * tensor i are accesses[access_ptr[i] .. access_ptr[i+1]).  The trace must
 * satisfy validate_trace (trace.py:125-157); the library re-checks the
 * invariants its kernels depend on and fails with TIO_ERR_INVALID. */
typedef struct tio_trace_desc {
    int64_t num_kernels;
    const int64_t *duration_us;   /* [num_kernels]      */
    int64_t num_tensors;
    const int64_t *tensor_id;     /* [num_tensors]      */
    const int64_t *size_bytes;    /* [num_tensors]      */
    const int8_t *kind;           /* [num_tensors]      */
    const int64_t *access_ptr;    /* [num_tensors + 1]  */
    int64_t num_events;
    const int32_t *accesses;      /* [num_events] kernel indices */
} tio_trace_desc;

typedef struct tio_trace tio_trace;
typedef struct tio_plan tio_plan;

/* ChannelRates (bandwidth.py:178-214); rates in bytes/us, may be fractional
 * (durations use the exact binary value, like Fraction(float)). */
typedef struct tio_rates {
    double ssd_offload;
    double ssd_prefetch;
    int has_host;
    double host_offload;
    double host_prefetch;
} tio_rates;

/* Device views of the lifetime products (owned by the trace handle). */
typedef struct tio_lifetime_view {
    int64_t num_kernels, num_tensors, num_periods;
    int64_t iteration_us;          /* trace.py:106-107                         */
    const int64_t *starts;         /* [N+1] kernel start times, starts[N]=iter */
    const int64_t *timeline;       /* [N]   analysis.py:97-108                 */
    const int64_t *active;         /* [N]   analysis.py:111-117                */
    /* inactive periods in reference order (analysis.py:58-83) */
    const int64_t *period_tensor;  /* [P] tensor position in the trace         */
    const int32_t *period_start;   /* [P] start_kernel                         */
    const int32_t *period_end;     /* [P] end_kernel                           */
    const int8_t *period_wraps;    /* [P]                                      */
    const int64_t *tensor_period_ptr; /* [T+1] first period of each tensor     */
} tio_lifetime_view;

/* Summary of a finished plan. */
typedef struct tio_plan_info {
    int64_t num_commits;           /* rounds that committed (planner.py:336)  */
    int64_t num_entries;           /* 2 * num_commits                          */
    int64_t num_over;              /* over_capacity_kernels count              */
    int64_t capacity_bytes;
    int64_t residual_peak_bytes;   /* MemoryTimeline.peak()                    */
    int64_t planned_host_bytes;    /* planner.py:354-358                       */
    int64_t num_candidates;        /* inactive periods considered              */
    int64_t rounds;                /* evaluation rounds run on the device      */
    int64_t unsat_kernel;          /* set when TIO_ERR_UNSATISFIABLE           */
    int64_t unsat_bytes;
    int64_t loop_ns;               /* CUDA-event time of the round-loop kernel */
    /* round-loop phase profile (block 0, ns): prologue, evaluate, block
     * reduce, barrier 1, argmax, channel merge, residual, commit+barrier 2;
     * then dirty tiles, refits, sum of per-round max evaluate time,
     * per-thread-mode tiles, their refits, sum of per-round max dirty tiles
     * of one block */
    int64_t dbg[14];
} tio_plan_info;

/* One CommittedMigration (planner.py:97-111), commit order.  Relieved
 * kernels are up to two ranges [lo,hi] (tail, then head for wrap periods);
 * an empty range has lo > hi.  benefit = (benefit_hi << 64) | benefit_lo. */
typedef struct tio_commit {
    int64_t tensor_id;
    int64_t tensor_pos;
    int64_t start_kernel, end_kernel;
    int64_t wraps;
    int64_t destination;           /* TIO_DEST_SSD / TIO_DEST_CPU              */
    int64_t off_start, off_end, pre_start, pre_end;
    uint64_t benefit_lo, benefit_hi;
    int64_t cost;
    int64_t rel0_lo, rel0_hi, rel1_lo, rel1_hi;
} tio_commit;

/* One PlanEntry (planner.py:69-76), plan order (sorted, urgent marked). */
typedef struct tio_entry {
    int64_t tensor_id;
    int64_t tensor_pos;
    int64_t trigger_us;
    int64_t deadline_us;
    int32_t action;                /* 0 offload, 1 prefetch                    */
    int32_t target;                /* TIO_DEST_SSD / TIO_DEST_CPU; 0 = GPU     */
    int32_t urgent;
    int32_t pad;
} tio_entry;

int tio_abi_version(void);
/* Kernels libtio has launched in this process (the bench's gpu_launches). */
int tio_kernel_launches(int64_t *out);
/* Copies the last error message of this thread (NUL-terminated, truncated). */
int tio_last_error(char *buf, size_t len);
/* Loaded-code identification: device name, SM count, build arch. */
int tio_device_info(char *buf, size_t len);

/* ---- trace (replaces building a Trace + Trace.kernel_start_times) ------- */
int tio_trace_create(const tio_trace_desc *desc, int mem_kind, void *stream, tio_trace **out);
int tio_trace_destroy(tio_trace *t);

/* ---- lifetime stage --------------------------------------------------------
 * Replaces analysis.py:58-117 (compute_inactive_periods,
 * compute_memory_timeline, per_kernel_active_bytes) and trace.py:97-107.
 * Enqueues the lifetime kernels on `stream`; tio_lifetime_view synchronises
 * the stream and returns device pointers (valid until the next call or
 * destroy). */
int tio_lifetime(tio_trace *t, void *stream);
int tio_lifetime_view_get(tio_trace *t, void *stream, tio_lifetime_view *out);
/* period_interior_duration (analysis.py:86-94) of every period, in period
 * order, computed on the device from the start times: out = host [P]. */
int tio_period_interior(tio_trace *t, void *stream, int64_t *out);
/* Copy lifetime products to host buffers (any may be NULL). */
int tio_lifetime_copy_out(tio_trace *t, void *stream, int64_t *starts, int64_t *timeline,
                          int64_t *active, int64_t *period_tensor, int32_t *period_start,
                          int32_t *period_end, int8_t *period_wraps);

/* ---- planner -----------------------------------------------------------------
 * Replaces planner.py:267-370 plan_migrations (+ mark_urgent :373-397).
 * Runs the lifetime stage first if it has not run.  Returns
 * TIO_ERR_UNSATISFIABLE (info.unsat_kernel/unsat_bytes set, no plan handle)
 * when some kernel's active bytes exceed capacity, TIO_ERR_CHANNEL_CONFIG for
 * a non-positive rate. */
int tio_plan_create(tio_trace *t, int64_t capacity, const tio_rates *rates, int64_t host_cap,
                    void *stream, tio_plan **out, tio_plan_info *info);
/* Options of tio_plan_create2: max_rounds > 0 stops the greedy loop after
 * that many commits (the plan is then the reference's first max_rounds
 * commits; used to check a prefix of huge plans against the oracle);
 * warp_refit_max: reserved (ignored; the layout is kept for ABI stability). */
typedef struct tio_plan_opts {
    int64_t max_rounds;
    int32_t warp_refit_max;
    int32_t pad;
    /* Sharded planning: nranks > 1 makes this call rank `rank`
     * of nranks.  Every rank holds the whole replicated planner state (channels,
     * residual, critical prefix) but evaluates only the candidate tiles
     * t % nranks == rank; each round the ranks exchange their local best
     * (key + winner window) through the mailboxes and apply the same commit,
     * so every rank ends with the full plan.  mailbox: this rank's
     * tio_mailbox_bytes() of device memory (zeroed once); peer_mailboxes:
     * [nranks] device pointers of every rank's mailbox as mapped in this
     * process (CUDA IPC / peer access; [rank] = mailbox); epoch: 0 for the
     * first planning call over a mailbox, then previous epoch + previous
     * rounds + 2 (flags are compared against epoch + round + 1 and the message
     * slot is that tag's parity, so no reset is needed between calls).  A
     * peer that does not publish within 30 s ends the call with TIO_ERR_CUDA
     * ("rank exchange timed out").
     * blocks > 0 overrides the planner's grid (virtual ranks on one GPU). */
    int32_t nranks;
    int32_t rank;
    int32_t blocks;
    int32_t pad2;
    uint64_t epoch;
    void *mailbox;
    void *const *peer_mailboxes;
} tio_plan_opts;
/* device bytes of one rank's mailbox */
size_t tio_mailbox_bytes(void);
/* One rank's mailbox for sharded planning across processes (one process per
 * GPU: the per-round `allgather` of local bests): allocated and
 * zeroed on the current device; ipc_handle receives its CUDA IPC handle
 * (TIO_IPC_HANDLE_BYTES) for the other ranks, which map it with
 * tio_mailbox_open (peer access over NVLink enabled lazily).  Replaces no
 * reference function: the reference plans on one CPU thread
 * (planner.py:293-351). */
#define TIO_IPC_HANDLE_BYTES 64
int tio_mailbox_create(void **mailbox, unsigned char *ipc_handle);
int tio_mailbox_destroy(void *mailbox);
int tio_mailbox_open(const unsigned char *ipc_handle, void **mapped);
int tio_mailbox_close(void *mapped);
/* Sharded planning of one trace by `nranks` virtual ranks on THIS GPU (the
 * check of the multi-GPU protocol on one device): rank r runs as a separate
 * planner instance (own replicated state, own stream, its own cooperative
 * grid of SMs / nranks blocks), all concurrently, exchanging through
 * mailboxes in device memory.  out[r] / info[r]: each rank's plan. */
int tio_plan_create_virtual(tio_trace *t, int64_t capacity, const tio_rates *rates, int64_t host_cap,
                            const tio_plan_opts *opts, int32_t nranks, tio_plan **out, tio_plan_info *info);
int tio_plan_create2(tio_trace *t, int64_t capacity, const tio_rates *rates, int64_t host_cap,
                     const tio_plan_opts *opts, void *stream, tio_plan **out, tio_plan_info *info);
int tio_plan_info_get(tio_plan *p, tio_plan_info *out);
/* Host copies: commits[num_commits], entries[num_entries], residual[N],
 * over[num_over]; any may be NULL. */
int tio_plan_copy_out(tio_plan *p, void *stream, tio_commit *commits, tio_entry *entries,
                      int64_t *residual, int64_t *over);
/* write_plan (planner.py:402-420), byte-identical.  Call with buf=NULL to get
 * the size in *len; then with a buffer of that size. */
int tio_plan_write(tio_plan *p, void *stream, char *buf, size_t *len);
int tio_plan_destroy(tio_plan *p);

/* One-shot end-to-end call (the e2e bench leg): host trace in, host plan
 * entries out.  Equivalent to trace_create(HOST) + plan_create + copy_out. */
int tio_plan_host(const tio_trace_desc *desc, int64_t capacity, const tio_rates *rates,
                  int64_t host_cap, void *stream, tio_plan_info *info,
                  tio_entry *entries, int64_t entries_cap);

/* ---- migration engine scheduler -------------------------------------------
 * Replaces simulator.py:539-547 simulate / simulate_on_demand (an empty entry
 * list) and the `_Engine` semantics (simulator.py:178-528) that the runtime
 * engine executes: host C++ discrete-event model on host trace columns.
 * entries: plan entries (tensor_id, trigger_us, deadline_us, action, target
 * (1 SSD / 2 CPU for offloads), urgent); tensor_pos is ignored.
 * TIO_ERR_SIMULATION (SimulationError) when a kernel's active bytes exceed
 * capacity or the run gets stuck.  Per-kernel arrays may be NULL. */
typedef struct tio_sim_report {
    int64_t total_time, ideal_time, stall_time_total, peak_resident_bytes, emergency_offloads;
    int64_t channel_busy[4];   /* ssd.offload, ssd.prefetch, host.offload, host.prefetch: us booked in [0, total] */
    int64_t num_transfers;
} tio_sim_report;

int tio_simulate(const tio_trace_desc *trace, const tio_entry *entries, int64_t num_entries,
                 int64_t capacity, const tio_rates *rates, tio_sim_report *report,
                 int64_t *per_kernel_start, int64_t *stall_per_kernel, int64_t *per_kernel_resident);

/* Replaces simulator.py:549-560 simulate_layer_granularity (policy
 * simulator.py:95-177): no plan; when the memory-timeline peak exceeds
 * capacity, each layer block's still-needed tensors are offloaded to the SSD
 * tier as one batch when execution leaves the block, and prefetch batches run
 * one block ahead.  kernel_layer[N] / tensor_layer[T]: layer ids, INT64_MIN =
 * none (the caller applies any tensor layer map).  TIO_ERR_CONFIG
 * (ConfigurationError) for a missing layer id once the policy engages. */
int tio_simulate_layers(const tio_trace_desc *trace, const int64_t *kernel_layer, const int64_t *tensor_layer,
                        int64_t capacity, const tio_rates *rates, tio_sim_report *report,
                        int64_t *per_kernel_start, int64_t *stall_per_kernel, int64_t *per_kernel_resident);

/* ---- roofline sweep --------------------------------------------------------
 * Replaces roofline.py:39-125: total iteration time (us) under the roofline
 * policy at each bandwidth (bytes/us, both directions; exact ceil of bytes /
 * rate as transfer_duration), host trace columns in.  info: iteration length,
 * memory-timeline peak, pressured = peak > capacity (totals are then the
 * iteration length), period count and largest period size (for
 * saturation_bandwidth).  num_bandwidths = 0 fills info only. */
typedef struct tio_roofline_info {
    int64_t ideal_us, peak_bytes, pressured, num_periods, max_period_bytes;
} tio_roofline_info;

int tio_roofline(const tio_trace_desc *trace, int64_t capacity, const double *bandwidth, int64_t num_bandwidths,
                 int64_t *total_us, tio_roofline_info *info);

/* The engine program behind a run: every transfer the scheduler starts (in
 * start order) and every kernel's start time, model microseconds.
 * initial_loc[t]: 0 unallocated, 1 GPU, 2 SSD, 3 host at t = 0 (after plan
 * folding).  Call with transfers = NULL to get the count. */
typedef struct tio_transfer_rec {
    int64_t tensor_pos, tensor_id;
    int32_t action;             /* 0 offload, 1 prefetch */
    int32_t device;             /* TIO_DEST_SSD / TIO_DEST_CPU */
    int32_t urgent, emergency;
    int64_t start_us, end_us;
    int64_t after_kernel;       /* last kernel finished at start_us (-1: none) */
    int64_t tail;               /* 1: running at t = 0 (boundary-straddling, folded plan) */
    int64_t seq;                /* position in the engine's processing order (shared with kernel launches) */
} tio_transfer_rec;

int tio_schedule(const tio_trace_desc *trace, const tio_entry *entries, int64_t num_entries, int64_t capacity,
                 const tio_rates *rates, tio_transfer_rec *transfers, int64_t transfers_cap,
                 int64_t *num_transfers, int64_t *kernel_start, int64_t *kernel_seq, int8_t *initial_loc);

/* ---- migration engine executor ----------------------------------------------
 * tio_engine_replay runs one iteration of `trace` under the plan `entries` on
 * the device: the scheduler above decides every transfer (simulator.py
 * semantics); compute runs on its own stream as one placeholder kernel per
 * trace kernel that lasts its profiled duration x time_scale; every transfer
 * is a real copy between a device buffer (stream-ordered pool) and a 4 KB
 * aligned pinned host extent on the channel's side stream, gated by CUDA
 * events (no GDS on the target: both tiers land in pinned host memory).
 * With verify, every prefetched tensor is checked byte for byte against the
 * pattern it was written with.  Replaces the reference engine's execution
 * role (simulator.py:471-528 run); ideal = the same kernels, no transfers. */
typedef struct tio_engine_config {
    int64_t capacity;
    tio_rates rates;            /* rates the scheduler models (measured link) */
    double time_scale;          /* device us per trace us for the placeholder kernels */
    int verify;                 /* byte-check every prefetch */
    int measure_ideal;          /* also time the no-transfer run */
} tio_engine_config;

typedef struct tio_engine_stats {
    int64_t model_total_us, model_ideal_us, model_stall_us, model_peak_resident, emergency_offloads;
    double replay_ms, ideal_ms;                 /* CUDA-event device times */
    int64_t offload_bytes, prefetch_bytes, n_offloads, n_prefetches;
    double offload_busy_ms, prefetch_busy_ms;   /* sum of per-copy device times */
    int64_t peak_device_bytes;                  /* pool high-water during the replay */
    int64_t host_bytes;                         /* pinned host extents */
    int64_t verified_bytes, verify_mismatches;
} tio_engine_stats;

int tio_engine_replay(const tio_trace_desc *trace, const tio_entry *entries, int64_t num_entries,
                      const tio_engine_config *cfg, void *stream, tio_engine_stats *stats);

/* ---- online migration engine (a real training step) -------------------------
 * The engine program of tio_engine_replay, driven by the framework around
 * every operator of the real step instead of placeholder kernels
 * (simulator.py:178-528 `_Engine` semantics, PAPER.md:429-444 runtime):
 * create() schedules the plan once over the profiled durations; per step the
 * framework calls step_begin, then before_kernel(k) / after_kernel(k) around
 * kernel (operator) k of the profiled trace, then step_end.  Device memory
 * stays the framework's: the engine calls
 *   alloc_cb(user, tensor_pos, bytes, &dev_ptr)  when a prefetch starts (the
 *       framework allocates on the compute stream; the engine orders the copy
 *       after the compute stream's current position), and
 *   free_cb(user, tensor_pos, stream)            after an offload's D2H copy is
 *       enqueued on `stream` (the framework frees once that stream passes
 *       this point, e.g. record_stream + storage resize to 0).
 * Both return 0 on success.  bind() tells the engine the device address of
 * a tensor it may move (globals before the first step; tensors created by
 * kernel k via after_kernel).  Tiers: pinned host extents (4 KB aligned) on
 * one side stream per channel (ssd / host x offload / prefetch).
 * cfg.verify: checksum every tensor at offload and after prefetch, mismatches
 * counted on the device (tio_engine_stats_get). */
typedef int (*tio_alloc_cb)(void *user, int64_t tensor_pos, int64_t bytes, void **dev_ptr);
typedef int (*tio_free_cb)(void *user, int64_t tensor_pos, void *stream);
typedef struct tio_engine tio_engine;

typedef struct tio_engine_info_t {
    int64_t num_kernels, num_tensors, num_transfers, host_bytes;
    int64_t model_total_us, model_ideal_us, model_stall_us, model_peak_resident, emergency_offloads;
    int64_t model_offload_bytes, model_prefetch_bytes, model_offloads, model_prefetches;
} tio_engine_info_t;

typedef struct tio_engine_online_stats {
    int64_t steps, offload_bytes, prefetch_bytes, n_offloads, n_prefetches;   /* all steps */
    double last_offload_busy_ms, last_prefetch_busy_ms;                      /* last step, per-copy device time */
    int64_t last_offload_bytes, last_prefetch_bytes;
    int64_t verify, verify_mismatches;
    int64_t reconcile_transfers, reconcile_bytes;   /* step-boundary fix-ups (all steps) */
} tio_engine_online_stats;

int tio_engine_create(const tio_trace_desc *trace, const tio_entry *entries, int64_t num_entries,
                      const tio_engine_config *cfg, void *compute_stream, tio_alloc_cb alloc_cb, tio_free_cb free_cb,
                      void *user, tio_engine **out);
/* movable (optional, [num_tensors]): 1 for tensors the engine may move (bind these) */
int tio_engine_info(const tio_engine *eng, tio_engine_info_t *info, uint8_t *movable);
int tio_engine_bind(tio_engine *eng, int64_t n, const int64_t *tensor_pos, void *const *dev_ptr);
int tio_engine_step_begin(tio_engine *eng);
int tio_engine_before_kernel(tio_engine *eng, int64_t k);
int tio_engine_after_kernel(tio_engine *eng, int64_t k, int64_t n_new, const int64_t *new_pos, void *const *new_ptr);
/* done_stream (optional): made to wait for every transfer issued so far */
int tio_engine_step_end(tio_engine *eng, void *done_stream);
/* leave a step that failed (framework exception): waits for the engine's
 * streams; restore() then brings the globals back */
int tio_engine_step_abort(tio_engine *eng);
int tio_engine_stats_get(tio_engine *eng, tio_engine_online_stats *stats);
int tio_engine_destroy(tio_engine *eng);
/* Walk the engine program of `steps` consecutive steps without a device (no
 * CUDA calls; fake addresses): fails with the engine's own error when the
 * program would offload a tensor that is not resident, prefetch a resident
 * one or launch a kernel whose tensor is off the GPU.  Host-only. */
int tio_engine_check_program(const tio_trace_desc *trace, const tio_entry *entries, int64_t num_entries,
                             const tio_engine_config *cfg, int64_t steps, tio_engine_info_t *info);
/* between steps: bring every global whose latest copy is off the GPU back
 * (synchronous) and reset to the pre-steady-state (the next step sets it up) */
int tio_engine_restore(tio_engine *eng);
/* turn checksum verification on / off between steps */
int tio_engine_set_verify(tio_engine *eng, int verify);
/* the engine's verification checksum of a device buffer (order-independent
 * 64-bit sum of mixed words), written to *dev_out on `stream` */
int tio_checksum(const void *dev_ptr, int64_t bytes, unsigned long long *dev_out, void *stream);

/* K10: gather n device buffers into 4 KB-aligned extents of `staging`
 * (offsets[i] out) / scatter them back, with TMA bulk copies.  scratch: a
 * device buffer of >= 64 * n + 64 bytes for the segment tables. */
int tio_pack(const void *const *src, const int64_t *bytes, int64_t n, void *staging, int64_t *offsets,
             void *scratch, size_t scratch_bytes, void *stream);
int tio_unpack(const void *staging, const int64_t *offsets, void *const *dst, const int64_t *bytes, int64_t n,
               void *scratch, size_t scratch_bytes, void *stream);

/* ---- trace ingest (trace.py:160-275 parse_trace) ------------------------------
 * Multi-threaded host parse of a JSONL trace straight into columns.  Fast
 * format only: TIO_ERR_INVALID with *err_line for anything else (the caller
 * then uses the reference-exact parser for the error).  Model invariants are
 * checked by the caller.  threads <= 0: hardware concurrency. */
typedef struct tio_parsed_trace tio_parsed_trace;
int tio_trace_parse(const char *buf, size_t len, int threads, tio_parsed_trace **out, int64_t *err_line);
int tio_parsed_sizes(const tio_parsed_trace *p, int64_t *n_kernels, int64_t *n_tensors, int64_t *n_events,
                     int64_t *n_names, int64_t *names_bytes, int64_t *meta_bytes);
/* name table: names[name_off[i] .. name_off[i+1]) raw JSON string contents,
 * name_esc[i] = contains escapes; meta: raw JSON text of the header's meta. */
int tio_parsed_copy(const tio_parsed_trace *p, int64_t *k_index, int64_t *k_dur, int32_t *k_code,
                    int64_t *k_stage, int64_t *k_layer, int64_t *t_id, int64_t *t_size, int8_t *t_kind,
                    int64_t *t_layer, int64_t *ptr, int64_t *acc, char *names, int64_t *name_off,
                    uint8_t *name_esc, char *meta);
int tio_parsed_destroy(tio_parsed_trace *p);

/* ---- channel primitives (bandwidth.py:75-84) ------------------------------- */
/* ceil(nbytes / rate) exactly; TIO_ERR_CHANNEL_CONFIG for rate <= 0. */
int tio_transfer_duration(double rate, int64_t nbytes, int64_t *out);

/* ---- host channels and per-candidate helpers ---------------------------------
 * One serial migration channel with its bookings (BandwidthChannel,
 * bandwidth.py:47-164): bookings sorted by start (equal starts in insertion
 * order), periodic images at +-period (period <= 0: none) released with their
 * booking.  Host memory only; the planner's own channels live on the device.
 * Booking ids are > 0; images carry their booking's id as `owner`. */
typedef struct tio_channel tio_channel;
int tio_channel_create(double rate, int64_t period, tio_channel **out);          /* :47-73, ChannelConfigError */
int tio_channel_destroy(tio_channel *c);
int tio_channel_reserve_earliest(tio_channel *c, int64_t ready, int64_t nbytes, int64_t tensor_id,
                                 int64_t *id, int64_t *start, int64_t *end);    /* :88-100  */
int tio_channel_reserve_latest(tio_channel *c, int64_t deadline, int64_t not_before, int64_t nbytes,
                               int64_t tensor_id, int32_t *found, int64_t *id, int64_t *start,
                               int64_t *end);                                    /* :102-120 */
int tio_channel_record(tio_channel *c, int64_t start, int64_t end, int64_t tensor_id, int32_t shadow,
                       int64_t *id);                                             /* :129-137 */
int tio_channel_release(tio_channel *c, int64_t id);                             /* :122-127 */
int tio_channel_size(const tio_channel *c, int64_t *n);
int tio_channel_copy(const tio_channel *c, int64_t *start, int64_t *end, int64_t *tensor, int64_t *id,
                     int64_t *owner, int8_t *shadow);                            /* .reservations */
int tio_channel_busy(const tio_channel *c, int64_t w0, int64_t w1, int64_t *busy); /* :153-164 */
/* candidate_window (planner.py:147-176) on one channel pair; *ok = 0: None
 * (nothing stays booked), 1: both bookings live. */
int tio_candidate_window(tio_channel *off, tio_channel *pre, int64_t ready, int64_t deadline, int64_t nbytes,
                         int64_t iteration, int64_t tensor_id, int32_t *ok, int64_t *off_id, int64_t *off_end,
                         int64_t *pre_id, int64_t *pre_start);
/* _host_peak_occupancy (planner.py:179-186) */
int tio_host_peak_occupancy(const int64_t *s, const int64_t *e, const int64_t *sz, int64_t n, int64_t lo,
                            int64_t hi, int64_t *out);
/* candidate_benefit (planner.py:232-262): benefit = (hi << 64) | lo;
 * critical: optional [N] mask of the over-capacity covered kernels.
 * starts: [N+1] kernel start times (starts[N] = iteration). */
int tio_candidate_benefit(const int64_t *starts, const int64_t *dur, const int64_t *residual, int64_t N,
                          int64_t capacity, int32_t wraps, int64_t start_kernel, int64_t end_kernel, int64_t first,
                          int64_t last, int64_t lo, int64_t hi, int64_t size, uint64_t *benefit_lo,
                          uint64_t *benefit_hi, int8_t *critical);

#ifdef __cplusplus
}
#endif
#endif /* TIO_H_ */
