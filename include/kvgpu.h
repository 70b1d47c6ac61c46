/* kvgpu — B200 (sm_100a) engine for the Concur / kvadmit simulator hot path.
 *
 * This is the drop-in C boundary for the reference's hot path
 *   kvadmit::run_simulation(Population, Policy, CostParams, EngineParams)
 *   (/root/reference/proj/src/engine.hpp:75-78, engine.cpp:446-456)
 * and for the cache-policy seam it drives per event
 *   kvadmit::CacheTree (/root/reference/proj/src/cache_tree.hpp:94-198).
 *
 * Conventions follow the reference C ABI (/root/reference/proj/include/kvadmit/kvadmit.h):
 *   - every fallible call returns a status, 0 = success            (kvadmit.h:33-40)
 *   - kvg_last_error() is a thread-local message, never NULL        (kvadmit.h:44-45)
 *   - opaque handles are freed with their *_free function           (kvadmit.h:56-64)
 *   - exceptions never cross the ABI                                (capi.cpp:47-65)
 * Only plain C types cross this boundary (no torch / CUDA types). A handle is
 * bound to one CUDA device; separate handles may be driven from separate host
 * threads (one per GPU). Calls on one handle must be externally serialized.
 */
#ifndef KVGPU_KVGPU_H_
#define KVGPU_KVGPU_H_

#include <stddef.h>
#include <stdint.h>

#define KVG_API __attribute__((visibility("default")))

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors kva_status (kvadmit.h:33-40) plus KVG_ERR_CUDA. */
typedef enum kvg_status {
  KVG_OK = 0,
  KVG_ERR_CONFIG = 1,           /* bad configuration, argument, or request */
  KVG_ERR_IO = 2,               /* filesystem failure */
  KVG_ERR_HORIZON = 3,          /* a simulation exceeded its horizon guard */
  KVG_ERR_STATE = 4,            /* invariant violation or API misuse */
  KVG_ERR_MISSING_BASELINE = 5, /* kept for parity with kva_status */
  KVG_ERR_CUDA = 6              /* CUDA runtime failure or no device */
} kvg_status;

KVG_API const char* kvg_version(void);
/* Message for the most recent failure in this thread; never NULL. */
KVG_API const char* kvg_last_error(void);

/* ------------------------------------------------------------------ */
/* Inputs. Field meanings follow the reference structs cited per type. */
/* ------------------------------------------------------------------ */

/* workload.hpp:29-44 (Distribution). */
enum { KVG_DIST_CONSTANT = 0, KVG_DIST_UNIFORM = 1, KVG_DIST_LOGNORMAL = 2 };
typedef struct kvg_distribution {
  uint32_t kind; /* KVG_DIST_* */
  uint32_t _pad;
  double a; /* constant value | uniform min | lognormal mean */
  double b; /* uniform max | lognormal sigma */
} kvg_distribution;

/* workload.hpp:102-113 (WorkloadConfig). */
typedef struct kvg_workload_config {
  uint32_t agents;
  uint32_t shared_prompt; /* bool */
  uint64_t prompt_tokens;
  uint32_t steps;
  uint32_t _pad;
  kvg_distribution gen_tokens;
  kvg_distribution obs_tokens;
  kvg_distribution tool_latency;
  double tool_probability;
} kvg_workload_config;

/* workload.hpp:60-66 (StepPlan). */
typedef struct kvg_step_plan {
  uint64_t gen_tokens;
  uint64_t obs_tokens;
  double tool_latency;
  uint32_t has_tool; /* bool */
  uint32_t _pad;
} kvg_step_plan;

/* workload.hpp:115-128 (Population). Agent a's context is never materialised:
 * token p of agent a is p (p < prompt_tokens, shared prompt) or
 * ((a+1)<<32)|(p - shared_len) otherwise (workload.cpp:139-142, 167-171). */
typedef struct kvg_population {
  uint32_t agents;
  uint32_t steps; /* plans per agent (WorkloadConfig.steps) */
  uint64_t prompt_tokens;
  uint32_t shared_prompt; /* bool */
  uint32_t _pad;
  uint64_t shared_prompt_tokens; /* 0 when prompts are private */
  uint64_t stream_hash;          /* FNV-1a over sampled values */
  uint64_t peak_aggregate_tokens;
  kvg_step_plan* plans; /* agents*steps, row-major by agent */
} kvg_population;

/* controller.hpp:29-42 (ControllerConfig) and :49-62 (Policy). */
enum {
  KVG_POLICY_UNCONTROLLED = 0,
  KVG_POLICY_REQUEST_CAP = 1,
  KVG_POLICY_AGENT_CAP = 2,
  KVG_POLICY_AIMD = 3
};
typedef struct kvg_controller_config {
  double alpha, beta, u_low, u_high, h_thresh, w_min, w_max, initial_window,
      control_interval, signal_smoothing;
} kvg_controller_config;
typedef struct kvg_policy {
  uint32_t kind; /* KVG_POLICY_* */
  uint32_t cap;
  kvg_controller_config aimd;
} kvg_policy;

/* cost_model.hpp:26-36 (CostParams). */
typedef struct kvg_cost_params {
  double prefill_linear, prefill_quadratic, decode_base, decode_context,
      bytes_per_token, pcie_bandwidth, transfer_sync_overhead;
} kvg_cost_params;

/* metrics.hpp:57-63 (PhaseParams) and engine.hpp:29-41 (EngineParams). */
enum { KVG_EVICT_DISCARD = 0, KVG_EVICT_OFFLOAD = 1 };
typedef struct kvg_phase_params {
  double sat_threshold, hit_threshold;
  int32_t hysteresis;
  int32_t _pad;
} kvg_phase_params;
typedef struct kvg_engine_params {
  uint64_t capacity;  /* device pool, pages */
  uint64_t page_size; /* tokens per page */
  uint32_t eviction;  /* KVG_EVICT_* */
  uint32_t paranoid;  /* accepted for parity; device runs always self-check */
  double hit_window_decay;
  double horizon;
  kvg_phase_params phases;
} kvg_engine_params;

/* One simulation = one reference run_simulation() call. */
typedef struct kvg_sim_desc {
  const kvg_population* population;
  kvg_policy policy;
  kvg_cost_params cost;
  kvg_engine_params engine;
} kvg_sim_desc;

/* ------------------------------------------------------------------ */
/* Outputs (metrics.hpp:27-43, 77-83; engine.hpp:45-69).               */
/* ------------------------------------------------------------------ */

/* TraceRecord (metrics.hpp:27-39) with the TickHits pair (engine.hpp:45-48). */
typedef struct kvg_trace_row {
  double time, usage, hit_rate, window;
  uint64_t active, pending, decoded_cum, recompute_cum, transfers;
  double hit_matched, hit_requested;
} kvg_trace_row;

/* AgentStats (workload.hpp:75-82) plus the completion record the north star
 * asks for: simulated finish time and the event ordinal that finished it. */
typedef struct kvg_agent_stats {
  uint64_t generated_tokens, recompute_tokens, recompute_events, stall_events,
      pause_events;
  double wait_time;
  double finish_time;
  uint64_t finish_ordinal;
} kvg_agent_stats;

typedef struct kvg_ledger {
  double prefill_fresh, prefill_recompute, decode, transfer, tool_wait;
} kvg_ledger;

enum { KVG_PHASE_WARMUP = 0, KVG_PHASE_MIDDLE = 1, KVG_PHASE_COOLDOWN = 2 };
typedef struct kvg_phase_label {
  uint32_t phase;
  uint32_t _pad;
  double start, end;
} kvg_phase_label;

/* SimulationResult scalars (engine.hpp:50-69) plus hot-path counters. */
typedef struct kvg_sim_result {
  int32_t status; /* kvg_status of this simulation */
  uint32_t n_phases;
  kvg_ledger ledger;
  double makespan, device_busy, link_busy;
  uint64_t decoded_tokens, recompute_tokens, recompute_events, stall_events,
      offloaded_tokens, reloaded_tokens, discarded_tokens;
  double total_wait_time;
  uint64_t ticks;
  uint64_t workload_hash;
  /* hot-path counters (BASELINE.md §2 definitions) */
  uint64_t agent_steps;  /* successful dispatch_member calls */
  uint64_t lookups;      /* resolved prefix pages + terminating miss */
  uint64_t events;       /* processed (non-skipped) events */
  uint64_t evict_calls;  /* CacheTree::evict calls with needed > 0 */
  uint64_t evicted_pages;
  uint64_t cache_clock;  /* final CacheTree clock */
  uint64_t pool_used;    /* final resident pages */
  double hit_matched, hit_requested; /* final hit window */
  /* algorithmic-traffic counters (BASELINE.md §2 roofline definitions) */
  uint64_t hit_pages;       /* pages resolved by lookups (stamp refreshed)   */
  uint64_t created_pages;   /* pages inserted                                 */
  uint64_t refreshed_pages; /* resident pages refreshed by successful inserts */
  uint64_t evict_scanned;   /* resident pages scanned by eviction selects     */
  uint64_t agent_events;    /* agent state-machine advances                   */
  uint64_t device_cycles;   /* SM clock cycles this simulation ran (device)   */
  kvg_phase_label phases[3];
  /* status KVG_ERR_HORIZON: the event time that passed the horizon and the
   * agents still unfinished (HorizonError's message, engine.cpp:112-119) */
  double abort_time;
  uint64_t unfinished;
} kvg_sim_result;

/* Optional per-simulation event log (parity testing). */
enum {
  KVG_LOG_MATCH = 1,   /* agent, clock, a = matched tokens, b = host_matched */
  KVG_LOG_INSERT = 2,  /* agent, clock, a = ok,            b = stored     */
  KVG_LOG_EVICT = 3,   /* clock,        a = needed,        b = reclaimed  */
  KVG_LOG_VICTIM = 4,  /*               a = page key,      b = stamp      */
  KVG_LOG_FINISH = 5,  /* agent,        a = time bits,     b = ordinal    */
  KVG_LOG_DISCARD = 6, /* agent, clock, a = from page,     b = pages      */
  KVG_LOG_RELOAD = 7   /* agent, clock, a = promoted,      b = offloaded tokens of
                          the evictions the reload triggered                */
};
typedef struct kvg_log_record {
  uint32_t kind;
  uint32_t agent;
  uint64_t clock;
  uint64_t a, b;
} kvg_log_record;

/* ------------------------------------------------------------------ */
/* Host prologue: population build (workload.cpp:153-204).             */
/* ------------------------------------------------------------------ */

/* Fills *out; out->plans is allocated by the library and released with
 * kvg_population_free. Identical to the reference sampling stream bit for
 * bit (splitmix64 + libm Box-Muller, FNV-1a stream hash). */
KVG_API kvg_status kvg_build_population(const kvg_workload_config* cfg,
                                        uint64_t seed, kvg_population* out);
KVG_API void kvg_population_free(kvg_population* pop);

/* Reference calibration (cost_model.cpp:49-59) and defaults
 * (controller.hpp:29-42, metrics.hpp:57-63, engine.hpp:29-41). */
KVG_API void kvg_cost_params_init(kvg_cost_params* p);
KVG_API void kvg_controller_config_init(kvg_controller_config* c);
KVG_API void kvg_engine_params_init(kvg_engine_params* e);

/* ------------------------------------------------------------------ */
/* Batched simulation on one device.                                   */
/* ------------------------------------------------------------------ */

typedef struct kvg_batch kvg_batch;

enum { KVG_HOST_OUTPUTS_NONE = 0, KVG_HOST_OUTPUTS_STREAM = 1, KVG_HOST_OUTPUTS_COPY = 2 };
typedef struct kvg_batch_options {
  uint32_t warps_per_sim; /* 0 = automatic (1 for small sims, up to 32)   */
  uint32_t log_capacity;  /* per-sim event-log records; 0 disables logging */
  uint64_t trace_capacity;/* per-sim trace rows; 0 = automatic (grows)     */
  uint32_t host_outputs;  /* 1: kvg_batch_run also delivers results, agent
                             stats and trace rows into pinned host memory
                             before returning, the rows streamed by the
                             kernel while it runs (best for one blocking
                             call); 2 (KVG_HOST_OUTPUTS_COPY): the same, the
                             rows copied by one copy-engine DMA after the
                             kernel (no SM work: best when batches are
                             pipelined with kvg_batch_launch / _wait, the
                             DMA overlapping the next batch's kernel); 0:
                             outputs stay in HBM until first accessed */
  uint32_t verify;        /* 1: every prefix match is also re-derived by the
                             block-hash probe and checked (a mismatch fails
                             the simulation with KVG_ERR_STATE) */
} kvg_batch_options;

KVG_API void kvg_batch_options_init(kvg_batch_options* o);

/* Validates every descriptor (engine.cpp:446-452 semantics), copies the
 * populations to device memory and sizes the per-simulation workspaces. */
KVG_API kvg_status kvg_batch_create(int device, const kvg_sim_desc* sims,
                                    size_t n, const kvg_batch_options* opt,
                                    kvg_batch** out);
/* Runs every simulation to completion on the device (blocking). Re-runnable:
 * each call starts from the initial state. Returns KVG_ERR_HORIZON if any
 * simulation hit its horizon (per-sim status in kvg_batch_result), with the
 * partial results still readable, as run_simulation's partial_on_abort. */
KVG_API kvg_status kvg_batch_run(kvg_batch* b);
/* kvg_batch_run in two halves, so a caller can pipeline batches (create /
 * read back one batch while another runs; the reference's run_rows keeps its
 * thread pool busy the same way, experiment.cpp:75-108): kvg_batch_launch
 * enqueues the run on the batch's own stream and returns at once;
 * kvg_batch_wait blocks until it ends and then does everything kvg_batch_run
 * does after the kernels (trace regrow + re-run, host delivery, status). In
 * between, the batch's results / traces / stats are not readable
 * (KVG_ERR_CONFIG); kvg_batch_free waits for the launch. */
KVG_API kvg_status kvg_batch_launch(kvg_batch* b);
KVG_API kvg_status kvg_batch_wait(kvg_batch* b);
/* Device time of the last kvg_batch_run, milliseconds (CUDA events on the
 * launching stream): whole step (workspace init + kernels) and kernels only. */
KVG_API kvg_status kvg_batch_last_ms(const kvg_batch* b, double* ms);
/* Launch geometry of the one-warp (small-simulation) kernel: how many
 * simulations it runs, how many of its CTAs fit on one SM with this batch's
 * shared memory, and the SM count (one wave iff small_sims <= ctas * sms). */
KVG_API kvg_status kvg_batch_geometry(const kvg_batch* b, uint32_t* small_sims,
                                      uint32_t* small_ctas_per_sm, uint32_t* sms);
KVG_API kvg_status kvg_batch_timing(const kvg_batch* b, double* step_ms,
                                    double* kernel_ms);
/* Copies results device->host (done once per run, lazily). */
KVG_API kvg_status kvg_batch_result(kvg_batch* b, size_t i,
                                    kvg_sim_result* out);
KVG_API kvg_status kvg_batch_trace(kvg_batch* b, size_t i, kvg_trace_row* rows,
                                   size_t cap, size_t* n_rows);
KVG_API kvg_status kvg_batch_agent_stats(kvg_batch* b, size_t i,
                                         kvg_agent_stats* out, size_t cap,
                                         size_t* n_agents);
KVG_API kvg_status kvg_batch_log(kvg_batch* b, size_t i, kvg_log_record* out,
                                 size_t cap, size_t* n_records);
/* Every simulation's result of the last run, one call (cap >= n). */
KVG_API kvg_status kvg_batch_results(kvg_batch* b, kvg_sim_result* out, size_t cap);
/* Zero-copy view of simulation i's trace rows in the host block (valid until
 * the next run or free). */
KVG_API kvg_status kvg_batch_trace_view(kvg_batch* b, size_t i,
                                        const kvg_trace_row** rows, size_t* n_rows);
/* Host pointers to the run's output arrays (valid until the next run or
 * free). Zero-copy when the batch was created with host_outputs.
 *   results[i]  is simulation i's result (caller order, dense);
 *   stats_base / trace_base hold every simulation's agent stats / trace rows
 *   in padded per-simulation slices: simulation i's slice starts at the
 *   element index kvg_batch_offsets reports (not at a dense prefix sum). */
KVG_API kvg_status kvg_batch_outputs(kvg_batch* b, const kvg_sim_result** results,
                                     const kvg_trace_row** trace_base,
                                     const kvg_agent_stats** stats_base);
/* Element index of simulation i's first agent-stats record in stats_base and
 * of its first trace row in trace_base (see kvg_batch_outputs). */
KVG_API kvg_status kvg_batch_offsets(kvg_batch* b, size_t i, size_t* stats_index,
                                     size_t* trace_index);
KVG_API void kvg_batch_free(kvg_batch* b);

/* One-shot convenience: create, run, read scalar results, free. */
KVG_API kvg_status kvg_run_batch(int device, const kvg_sim_desc* sims,
                                 size_t n, kvg_sim_result* results);

/* Phase classification of a trace (metrics.cpp:41-81), host-side. */
KVG_API kvg_status kvg_classify_phases(const kvg_trace_row* rows, size_t n,
                                       double makespan,
                                       const kvg_phase_params* params,
                                       kvg_phase_label* out, size_t cap,
                                       size_t* n_out);

/* ------------------------------------------------------------------ */
/* Run artifacts (host-side), byte-identical to the reference's         */
/* execute_run output (experiment.cpp:161-170).                        */
/* ------------------------------------------------------------------ */

/* Summary (metrics.hpp:85-118), computed by kvg_summarize exactly as
 * summarize() does (engine.cpp:458-532). */
typedef struct kvg_summary {
  char name[128];
  char policy[64];
  uint64_t seed, agents;
  double makespan, throughput;
  uint64_t decoded_tokens, recompute_tokens, recompute_events, stall_events;
  double recompute_fraction, mean_hit_rate, mean_usage;
  kvg_ledger ledger;
  double device_busy, device_idle, link_busy, link_idle;
  uint64_t offloaded_tokens, reloaded_tokens, discarded_tokens;
  double total_wait_time;
  double warmup_duration, middle_duration, cooldown_duration, middle_fraction;
  double warmup_hit_rate, middle_hit_rate, cooldown_hit_rate, middle_usage_mean;
  uint64_t ticks, workload_hash;
} kvg_summary;

/* policy_name (controller.cpp:253-265). */
KVG_API kvg_status kvg_policy_name(const kvg_policy* p, char* out, size_t cap);
KVG_API kvg_status kvg_summarize(const kvg_sim_result* r, const kvg_trace_row* rows,
                                 size_t n, const char* name,
                                 const char* policy_label, uint64_t seed,
                                 uint32_t agents, kvg_summary* out);
/* export_trace (metrics.cpp:89-101), export_summary (:141-183),
 * export_phases (:266-276). */
KVG_API kvg_status kvg_write_trace_csv(const char* path, const kvg_trace_row* rows,
                                       size_t n);
KVG_API kvg_status kvg_write_summary(const char* path, const kvg_summary* s);
KVG_API kvg_status kvg_write_phases_csv(const char* path, const kvg_phase_label* p,
                                        size_t n);
/* trace.csv + summary.txt + phases.csv of one run into an existing `dir`. */
KVG_API kvg_status kvg_write_run_artifacts(const char* dir, const char* name,
                                           const char* policy_label, uint64_t seed,
                                           uint32_t agents, const kvg_sim_result* r,
                                           const kvg_trace_row* rows, size_t n,
                                           kvg_summary* out);

/* ------------------------------------------------------------------ */
/* Device-backed admission controllers: the reference's standalone     */
/* controller ABI (kvadmit.h:86-159) for N controllers at once, state   */
/* in HBM, each call one kernel over all of them.                       */
/* ------------------------------------------------------------------ */

enum { KVG_CMD_ADMIT = 0, KVG_CMD_PAUSE = 1, KVG_CMD_RESUME = 2 };
/* kva_command (kvadmit.h:123-126), same layout. */
typedef struct kvg_command {
  uint8_t kind; /* KVG_CMD_* */
  uint8_t _pad[3];
  uint32_t agent;
} kvg_command;

enum {
  KVG_CTL_ADD_PENDING = 0,      /* kva_controller_add_pending        */
  KVG_CTL_AGENT_FINISHED = 1,   /* kva_controller_on_agent_finished  */
  KVG_CTL_REQUEST_COMPLETE = 2, /* kva_controller_on_request_complete */
  KVG_CTL_TOOL_RETURN = 3       /* kva_controller_on_tool_return     */
};
typedef struct kvg_ctl_event {
  uint32_t controller, kind, agent, _pad;
} kvg_ctl_event;

typedef struct kvg_controllers kvg_controllers;
/* n controllers; controller i admits agents 0..total_agents[i]-1 under
 * policies[i] (validated like Policy::validate, controller.cpp:24-52). */
KVG_API kvg_status kvg_controllers_create(int device, size_t n, const kvg_policy* policies,
                                          const uint32_t* total_agents,
                                          kvg_controllers** out);
KVG_API void kvg_controllers_free(kvg_controllers* c);
/* update_window on every controller (usage[i], hit_rate[i]); window_out[i]
 * receives the post-update window as kva_controller_update_window reports
 * it (the display window). */
KVG_API kvg_status kvg_controllers_update_window(kvg_controllers* c, const double* usage,
                                                 const double* hit_rate, double* window_out);
/* One admission pass on every controller. at_boundary and commands are
 * concatenated per controller (controller i's slice starts at the sum of
 * total_agents[0..i) and is total_agents[i] long); n_out[i] = commands
 * controller i emitted. status[i] (optional) is KVG_ERR_STATE when the pass
 * emitted more commands than agents (possible only after API misuse put an
 * id on two lists; the reference fails that call, capi.cpp:228-236). */
KVG_API kvg_status kvg_controllers_admission_pass(kvg_controllers* c,
                                                  const uint8_t* at_boundary,
                                                  kvg_command* commands, size_t* n_out,
                                                  int32_t* status);
/* Applies events in submission order per controller; status[i] (optional)
 * is the kvg_status of event i (KVG_ERR_STATE for an unknown agent, like
 * UnknownAgent). */
KVG_API kvg_status kvg_controllers_apply(kvg_controllers* c, const kvg_ctl_event* events,
                                         size_t n_events, int32_t* status);
/* Per-controller state; any out-pointer may be NULL. */
KVG_API kvg_status kvg_controllers_state(const kvg_controllers* c, double* window,
                                         double* display_window, uint64_t* ticks,
                                         size_t* active, size_t* pending, size_t* paused);
KVG_API kvg_status kvg_controllers_active(const kvg_controllers* c, size_t i, uint32_t* out,
                                          size_t cap, size_t* n_out);

/* ------------------------------------------------------------------ */
/* Cache-policy seam: a device-resident paged prefix cache driven by a */
/* batch of CacheTree-style operations (cache_tree.hpp:96-167).        */
/* Sequences are owner-form: (agent, length) names the token sequence  */
/* agent `agent` would hold at that length under the population token */
/* scheme above, with the cache's shared prompt configuration.         */
/* ------------------------------------------------------------------ */

enum {
  KVG_OP_MATCH = 1,   /* match_prefix(seq)          -> r0 = matched, r1 = host_matched */
  KVG_OP_INSERT = 2,  /* insert(seq)                -> r0 = ok, r1 = inserted slots    */
  KVG_OP_EVICT = 3,   /* evict(arg)                 -> r0 = reclaimed                  */
  KVG_OP_PIN = 4,     /* pin(seq, arg tokens)                                          */
  KVG_OP_UNPIN = 5,   /* unpin(seq, arg tokens)     -> status on underflow             */
  KVG_OP_DISCARD = 6, /* discard_suffix(seq, arg)                                     */
  KVG_OP_RELOAD = 7   /* reload(seq, from=arg, max=arg2) -> r0 = promoted, r1 = offloaded
                         tokens of the evictions it triggered (offload mode)           */
};
typedef struct kvg_cache_op {
  uint32_t kind;
  uint32_t agent;
  uint64_t len; /* sequence length in tokens */
  uint64_t arg;
  uint64_t arg2;
} kvg_cache_op;
typedef struct kvg_cache_op_result {
  int32_t status;
  uint32_t _pad;
  uint64_t r0, r1;
  uint64_t clock, used;
  uint64_t victims_begin, victims_end; /* range into the victim list */
} kvg_cache_op_result;
typedef struct kvg_victim {
  uint64_t key;   /* (owner << 32) | page index; owner 0 = shared prompt */
  uint64_t stamp; /* last-access stamp at eviction */
} kvg_victim;

typedef struct kvg_cache kvg_cache;
KVG_API kvg_status kvg_cache_create(int device, uint64_t capacity,
                                    uint64_t page_size, uint32_t eviction,
                                    uint64_t prompt_tokens,
                                    uint32_t shared_prompt, uint32_t max_agents,
                                    kvg_cache** out);
/* Executes ops in order on the device. Victims of each op are appended to
 * the handle's victim list, ordered as the reference evicts them
 * (stamp ascending, deeper page first). */
KVG_API kvg_status kvg_cache_exec(kvg_cache* c, const kvg_cache_op* ops,
                                  size_t n, kvg_cache_op_result* results);
KVG_API kvg_status kvg_cache_victims(const kvg_cache* c, size_t begin,
                                     size_t end, kvg_victim* out);
KVG_API kvg_status kvg_cache_hit_window(const kvg_cache* c, double* matched,
                                        double* requested);
KVG_API void kvg_cache_free(kvg_cache* c);

/* Grid-wide page-table kernels (discard mode). kvg_cache_exec runs an EVICT
 * op as ONE cooperative launch over every SM (shared-memory radix-select
 * histograms merged once per digit pass) instead of on the one-CTA executor:
 *   KVG_GRID_AUTO   when the table has >= 4096 claimed buckets (default),
 *   KVG_GRID_NEVER  never, KVG_GRID_ALWAYS always.
 * record_victims = 0 stops appending victims to the handle's victim list
 * (bulk evictions of millions of pages; counts are still returned). */
enum { KVG_GRID_AUTO = 0, KVG_GRID_NEVER = 1, KVG_GRID_ALWAYS = 2 };
KVG_API kvg_status kvg_cache_configure(kvg_cache* c, uint32_t grid_mode,
                                       uint32_t record_victims);
/* n match_prefix calls (cache_tree.cpp:114-142) in one grid launch: agent
 * agents[i]'s owner-form sequence of lens[i] tokens. Leaves the cache (clock,
 * page stamps, summaries, hit window) and results[i] exactly as n successive
 * KVG_OP_MATCH ops through kvg_cache_exec would: query i runs at clock
 * clock0 + i + 1 and a page's final stamp is that of the last query covering
 * it. One warp per query over all SMs. Discard mode only. */
KVG_API kvg_status kvg_cache_match_batch(kvg_cache* c, const uint32_t* agents,
                                         const uint64_t* lens, size_t n,
                                         kvg_cache_op_result* results);
/* Device time (CUDA events on the launching stream) of the kernels of the
 * last kvg_cache_exec / kvg_cache_match_batch call, ms; grid_blocks = CTAs
 * of the last grid-wide eviction. */
KVG_API kvg_status kvg_cache_last_ms(const kvg_cache* c, double* ms, uint32_t* grid_blocks);

/* Test hook: the engine's ready-set walk (the smallest ready agent id >= from,
 * or 0xffffffff) in both device forms — the sweep kernel's and the
 * one-CTA-per-SM kernels' — over a caller's bitmap of n agents: rbits (one bit
 * per agent) and rl1 (one bit per non-empty rbits word). */
KVG_API kvg_status kvg_check_ready_next(int device, const uint32_t* rbits, const uint32_t* rl1,
                                        uint32_t n, const uint32_t* from, uint32_t nq,
                                        uint32_t* out_narrow, uint32_t* out_wide);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* KVGPU_KVGPU_H_ */
