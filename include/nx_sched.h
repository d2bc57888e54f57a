/* nx_sched.h — C-ABI of the B200 NexusSched hot path.
 *
 * Plain C: pointers, sizes, status codes; no torch / C++ types cross it.
 * Every entry point names the reference interface it replaces. Errors never
 * throw across the ABI; the status maps 1:1 onto the reference's exception
 * types (proj/src/*.cpp):
 *   NX_EINVAL   <- std::invalid_argument  (bad shapes / params / inputs)
 *   NX_ERUNTIME <- std::runtime_error     (config, I/O, prefill_priority cap)
 *   NX_ELOGIC   <- std::logic_error       (internal invariants)
 *   NX_ECUDA    no reference analogue: a CUDA call failed (no GPU, OOM, ...)
 * nx_last_error() returns the message of the calling thread's last failure.
 *
 * Threading: one stream per handle; handles are not shared between threads;
 * distinct handles are reentrant (proj/include/servesim/sim.h:78-100 —
 * run_simulation is reentrant).
 */
#ifndef NX_SCHED_H_
#define NX_SCHED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { NX_OK = 0, NX_EINVAL = 1, NX_ERUNTIME = 2, NX_ELOGIC = 3, NX_ECUDA = 4 };
enum { NX_DETERMINISTIC_FP64 = 0, NX_FAST_FP32 = 1 };

const char* nx_last_error(void);
/* sizeof of the ABI structs, in declaration order (nx_lens_problem,
 * nx_lens_plan, nx_route_group, nx_engine_report, nx_route_request,
 * nx_route_decision, nx_refit_problem, nx_refit_result, nx_replica_summary,
 * nx_request_record, nx_baseline_problem) — lets bindings verify their
 * layouts. */
int nx_abi_sizes(int64_t* out, int32_t n);
int nx_device_count(void);

/* ---- K1: batched perf-model evaluation ------------------------------------
 * Replaces servesim::throughput / predict_latency
 * (proj/include/servesim/perf_model.h:45-50, proj/src/perf_model.cpp:38-49).
 * params: n_params x 8 doubles in PerfParams order
 *         {tau0, w0, ws, tauB, tauS, p_max, kB, kS};
 * idx/b/s: n evaluation records (engine-params index, batch size, tokens).
 * out_T (and out_thr if non-NULL): n results.
 * mode NX_DETERMINISTIC_FP64: bit-identical expression order, no FMA;
 * NX_FAST_FP32: float math, <= 1e-4 relative.
 * Returns NX_EINVAL (like the reference's std::invalid_argument) if any
 * record has b < 1, s < b, idx out of range, or invalid params.
 * _dev variant: all pointers are device pointers, async on `stream`.
 * _host variant: host pointers; copies in/out are part of the call. */
int nx_perf_eval_dev(const double* params, int32_t n_params, const int32_t* idx,
                     const int32_t* b, const int32_t* s, double* out_T, double* out_thr,
                     int64_t n, int32_t mode, void* stream);
/* Stream-ordered variant: no host synchronisation; bit 0 of *dev_status (a
 * device word the caller zeroes) is set if any record or row is invalid. */
int nx_perf_eval_async(const double* params, int32_t n_params, const int32_t* idx,
                       const int32_t* b, const int32_t* s, double* out_T, double* out_thr,
                       int64_t n, int32_t mode, uint32_t* dev_status, void* stream);
int nx_perf_eval_host(const double* params, int32_t n_params, const int32_t* idx,
                      const int32_t* b, const int32_t* s, double* out_T, double* out_thr,
                      int64_t n, int32_t mode);

/* ---- K2: batched LENS scheduling decisions --------------------------------
 * Replaces servesim::schedule_step (proj/include/servesim/lens.h:114-124,
 * proj/src/lens.cpp:96-146): one independent decision per problem — the
 * candidate batch-size sweep, binary_search_budget per candidate
 * (lens.cpp:33-56), allocate_tokens/realize (:58-92) and the first-min /
 * early-exit selection. Run-queue requests need no per-request data (each
 * takes one decode token); waiters are given by their remaining prompt.
 * Status per problem mirrors the reference's exceptions: NX_EINVAL for an
 * invalid SchedulerConfig, SLOSpec, TradeoffModel or PerfParams, a
 * non-positive target, or (device limit) remaining < 1 / q_max, m_max >= 2^30. */
typedef struct nx_lens_problem {
  double params[8];                   /* PerfParams {tau0,w0,ws,tauB,tauS,p_max,kB,kS} */
  double ttft_slo_ms, tpot_slo_ms;    /* SLOSpec (lens.h:14-19) */
  double alpha_ms, beta, l_bar, td_min_ms; /* TradeoffModel (lens.h:22-38) */
  double eps_ratio, q_ref;            /* SchedulerConfig (lens.h:63-75) */
  int64_t m_max, q_max;
  int32_t n_search_iters;
  int32_t n_run;                      /* |run_q| */
  int32_t n_wait;                     /* |wait_q| (FCFS order) */
  int32_t pad_;
  int64_t wait_off;                   /* waiters at [wait_off, wait_off + n_wait) */
} nx_lens_problem;

typedef struct nx_lens_plan {         /* BatchPlan (lens.h:82-91) */
  int64_t b, s;
  double predicted_ms, target_ms;
  int32_t overload;                   /* run queue exceeded q_max: truncated decode plan */
  int32_t slo_risk;                   /* TargetLatency::slo_risk */
  int32_t n_decode;                   /* allocations [0, n_decode): run_q[i], 1 token */
  int32_t n_prefill;                  /* then wait_q[k], k < n_prefill, alloc_tokens[wait_off+k] tokens */
  int32_t status;                     /* NX_OK / NX_EINVAL */
  int32_t pad_;
} nx_lens_plan;

/* Device pointers, stream-ordered. wait_remaining: prompt_len - prefilled per
 * waiter (int32, >= 1). alloc_tokens: written for admitted waiters only. */
int nx_lens_schedule_dev(const nx_lens_problem* problems, int32_t n_problems,
                         const int32_t* wait_remaining, int64_t n_wait_total,
                         nx_lens_plan* plans, int32_t* alloc_tokens, void* stream);
/* Host pointers: copies in/out inside the call; returns the first failing
 * problem's status (all plans are still written). */
int nx_lens_schedule_host(const nx_lens_problem* problems, int32_t n_problems,
                          const int32_t* wait_remaining, int64_t n_wait_total,
                          nx_lens_plan* plans, int32_t* alloc_tokens);
/* The same with an evaluation mode: NX_DETERMINISTIC_FP64 (the two calls
 * above: bit-exact decisions) or NX_FAST_FP32 (every probe of the budget
 * search and the candidate errors in float; predicted_ms within 1e-4
 * relative of the fp64 model for the chosen plan; decisions can differ from
 * the deterministic mode where two candidates, or a probe and the target,
 * lie within float rounding of each other). Validation, the prefix and the
 * allocation lists are the deterministic mode's. Any other mode: NX_EINVAL. */
int nx_lens_schedule_mode_dev(const nx_lens_problem* problems, int32_t n_problems,
                              const int32_t* wait_remaining, int64_t n_wait_total,
                              nx_lens_plan* plans, int32_t* alloc_tokens, int32_t mode, void* stream);
int nx_lens_schedule_mode_host(const nx_lens_problem* problems, int32_t n_problems,
                               const int32_t* wait_remaining, int64_t n_wait_total,
                               nx_lens_plan* plans, int32_t* alloc_tokens, int32_t mode);

/* ---- K3: batched PRISM routing ---------------------------------------------
 * Replaces servesim::Router::route (proj/include/servesim/router.h:55-121,
 * proj/src/router.cpp:141-289). A group is one Router: its engines (in
 * registration order, <= 32), report table, session map, RNG and
 * round-robin cursor; its requests are routed in order, each decision
 * seeing the previous ones' dispatch echo (router.cpp:275-282) and session
 * memory (remember_session). Groups are independent (one warp each).
 * Policies: 0 prism, 1 round_robin, 2 session_affinity, 3 least_loaded,
 * 4 latency_based (the caller keeps the completion windows and passes each
 * engine's rolling mean; one request per group), 5 weighted.
 * Report rows and group state (l_bar_ema, rng, rr_next, session map) are
 * updated in place, as the Router's own state would be. */
typedef struct nx_route_group {
  double weights[4];                  /* RouterConfig (router.h:31-52) */
  double beta_aff, latency_knee, latency_scale_ms, load_half_ms, capacity_headroom,
      staleness_limit_ms;
  double ttft_slo_ms;                 /* SLOSpec::ttft_slo_ms */
  double l_bar_ema;                   /* router-side decode-length estimate (router.h:118) */
  uint64_t rng[4];                    /* weighted-policy xoshiro256++ state */
  uint64_t rr_next;                   /* round-robin cursor */
  int32_t policy, n_engines;
  int64_t engine_off;                 /* report rows [engine_off, +n_engines) */
  int64_t request_off;                /* requests [request_off, +n_requests) */
  int64_t session_off;                /* session map [session_off, +n_sessions) */
  int32_t n_requests, n_sessions;     /* n_sessions <= 100000 (router.h:107) */
} nx_route_group;

typedef struct nx_engine_report {     /* EngineReport (engine.h:50-67) + registration */
  double l_hat_ms, w_load_tokens, m_free_tokens, p_max, reported_at_ms;
  double static_weight;               /* RouterConfig::static_weights[engine_id] (1.0 if unset) */
  int64_t queue_len;
  int32_t engine_id;
  int32_t has_report;                 /* 0: no report received yet */
  double rolling_latency_ms;          /* latency_based only: the router's rolling e2e mean */
} nx_engine_report;

typedef struct nx_route_request {
  double now_ms;
  int64_t prompt_len;
  int32_t session;                    /* index into the group's session map */
  int32_t pad_;
} nx_route_request;

typedef struct nx_route_decision {    /* RouteDecision (router.h:67-72) */
  double score, factors[4];
  int32_t engine_id;
  int32_t degraded;
} nx_route_decision;

/* session_map: per group, engine index last routed for each session or -1. */
int nx_prism_route_dev(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                       const nx_route_request* requests, int32_t* session_map,
                       nx_route_decision* decisions, int32_t* group_status, void* stream);
int nx_prism_route_host(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                        int64_t n_reports, const nx_route_request* requests, int64_t n_requests,
                        int32_t* session_map, int64_t n_session_entries,
                        nx_route_decision* decisions, int32_t* group_status);
/* The same with an evaluation mode: NX_DETERMINISTIC_FP64 (the two calls
 * above: bit-exact choices) or NX_FAST_FP32 (the PRISM policy's scores,
 * factors and load ratios in float; choices can differ from the
 * deterministic mode where two engines' scores lie within float rounding;
 * the other policies are unchanged). Any other mode: NX_EINVAL. */
int nx_prism_route_mode_dev(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                            const nx_route_request* requests, int32_t* session_map,
                            nx_route_decision* decisions, int32_t* group_status, int32_t mode,
                            void* stream);
int nx_prism_route_mode_host(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                             int64_t n_reports, const nx_route_request* requests, int64_t n_requests,
                             int32_t* session_map, int64_t n_session_entries,
                             nx_route_decision* decisions, int32_t* group_status, int32_t mode);

/* ---- K4: batched learner refits ---------------------------------------------
 * Replaces OnlineLearner::update_linear / update_structural
 * (proj/include/servesim/learner.h:70-80, proj/src/learner.cpp:300-440) on
 * explicit windows: each problem is one learner whose ring holds
 * samples [sample_off, sample_off + n_samples) in chronological order (the
 * last long_window of them are the window). One warp per problem. */
typedef struct nx_refit_problem {
  double params[8];                   /* OnlineLearner::params() before the update */
  int64_t long_window, short_window, min_structural_samples;
  int64_t sample_off;
  int32_t n_samples;
  int32_t pad_;
} nx_refit_problem;

typedef struct nx_refit_result {
  double params[8];                   /* params() after the update */
  int64_t counters[7];                /* LearnerCounters increments (learner.h:26-34) */
  int32_t updated;                    /* the update's return value */
  int32_t status;                     /* NX_OK / NX_EINVAL (invalid sample / config) */
} nx_refit_result;

enum { NX_REFIT_LINEAR = 0, NX_REFIT_STRUCTURAL = 1 };

/* max_long_window: upper bound of problems[i].long_window (sizes the per-warp
 * scratch; a problem above it gets NX_EINVAL). */
int nx_refit_dev(int32_t kind, const nx_refit_problem* problems, int32_t n_problems,
                 const int32_t* sample_b, const int32_t* sample_s, const double* sample_y,
                 int64_t max_long_window, nx_refit_result* results, void* stream);
int nx_refit_host(int32_t kind, const nx_refit_problem* problems, int32_t n_problems,
                  const int32_t* sample_b, const int32_t* sample_s, const double* sample_y,
                  int64_t n_samples_total, nx_refit_result* results);

/* ---- scheduling building blocks (batched, host pointers) -------------------
 * The reference's free functions under schedule_step / Router::route /
 * TradeoffEstimator, evaluated on the device with the same core the
 * simulator uses; the C++ drop-in (include/nx_servesim.hpp) calls these.
 * Each returns the first failing record's status (all records written). */
typedef struct nx_target_query {      /* target_latency (lens.h:93-99) */
  double ttft_slo_ms, tpot_slo_ms, alpha_ms, beta, l_bar, td_min_ms, q_ref;
  int64_t wait_count;
  double target_ms;                   /* out */
  int32_t slo_risk, status;           /* out */
} nx_target_query;

typedef struct nx_budget_query {      /* binary_search_budget (lens.h:101-106) */
  double params[8];
  double target_ms;
  int64_t b, m_max, q_max, s_cap;     /* s_cap < 0: m_max */
  int32_t n_search_iters, status;     /* status out */
  int64_t budget;                     /* out */
} nx_budget_query;

typedef struct nx_allocate_problem {  /* allocate_tokens (lens.h:108-112) */
  int64_t b, s;
  int64_t wait_off;                   /* waiters' remaining prompts at [wait_off, +n_wait) */
  int32_t n_run, n_wait;
  int32_t n_prefill, status;          /* out: waiters admitted (tokens[wait_off + k]) */
} nx_allocate_problem;

typedef struct nx_score_query {       /* score_latency/load/capacity (router.h:57-66) */
  double l_hat_ms, w_load_tokens, m_free_tokens, p_max;
  double demand_tokens;
  double latency_knee, latency_scale_ms, ttft_slo_ms, load_half_ms, capacity_headroom;
  double latency, load, capacity;     /* out */
  int32_t status, pad_;
} nx_score_query;

#define NX_TRADEOFF_WINDOW 200        /* TradeoffEstimator::kWindow (lens.h:145) */
typedef struct nx_completion {        /* CompletionStats (lens.h:126-130) */
  double ttft_ms, tpot_ms;
  int64_t decode_len;
} nx_completion;

typedef struct nx_tradeoff_state {    /* TradeoffEstimator state (lens.h:132-151) */
  double alpha_ms, beta, l_bar, td_min_ms;
  int64_t degenerate_updates;
  double win_ttft[NX_TRADEOFF_WINDOW], win_tpot[NX_TRADEOFF_WINDOW];
  int32_t win_head, win_len;
  int64_t comp_off;                   /* this update's completions [comp_off, +n_new) */
  int32_t n_new, pad_;
} nx_tradeoff_state;

int nx_target_latency_host(nx_target_query* q, int32_t n);
int nx_budget_search_host(nx_budget_query* q, int32_t n);
int nx_allocate_tokens_host(nx_allocate_problem* p, int32_t n, const int32_t* wait_remaining,
                            int64_t n_wait_total, int32_t* tokens);
int nx_router_scores_host(nx_score_query* q, int32_t n);
int nx_tradeoff_update_host(nx_tradeoff_state* st, int32_t n, const nx_completion* completions,
                            int64_t n_completions);

/* schedule_baseline (proj/include/servesim/engine.h:68-79,
 * proj/src/engine.cpp:61-108): the prefill_priority and static_chunked engine
 * policies. Plan = the first n_decode runners (one decode token each), then
 * waiters k < n_prefill with tokens[wait_off + k]. Status: NX_ERUNTIME when
 * prefill_priority cannot fit the first prompt (the reference's
 * runtime_error), NX_ELOGIC for the lens policy, NX_EINVAL for an
 * allocate_tokens or predict_latency argument error. */
enum { NX_SCHED_LENS = 0, NX_SCHED_PREFILL_PRIORITY = 1, NX_SCHED_STATIC_CHUNKED = 2 };
typedef struct nx_baseline_problem {
  double params[8];                   /* learner's PerfParams */
  int64_t m_max, q_max, static_budget;
  int64_t wait_off;                   /* waiters' remaining prompts at [wait_off, +n_wait) */
  int32_t policy, engine_id;
  int32_t n_run, n_wait;
  int64_t b, s;                       /* out */
  double predicted_ms;                /* out */
  int32_t n_decode, n_prefill;        /* out */
  int32_t status, pad_;               /* out */
} nx_baseline_problem;

int nx_baseline_schedule_host(nx_baseline_problem* p, int32_t n, const int32_t* wait_remaining,
                              int64_t n_wait_total, int32_t* tokens);

/* ---- K5 (+K2/K3/K4 inside): batched replica simulation --------------------
 * Replaces servesim::run_simulation / sweep (proj/include/servesim/sim.h:
 * 78-100, proj/src/sim.cpp:245-347, 596-642): each config is a RunConfig JSON
 * document (RunConfig::from_json_text schema, proj/src/sim.cpp:454-582); one
 * replica per document. Workloads are synthesised on the host exactly like
 * the reference (arrival doubles come from host libm). */
typedef struct nx_sim* nx_sim_t;

typedef struct nx_replica_summary {
  int64_t arrived, completed, rejected, unfinished;
  int64_t events;        /* processed events (hashed) */
  int64_t decisions;     /* routes + executed batches = arrived + sum(samples) */
  uint64_t arrival_hash, event_hash;
  int32_t status;        /* NX_OK or the reference exception class */
  int32_t err_site;
} nx_replica_summary;

typedef struct nx_request_record { /* servesim::RequestRecord, metrics.h:12-20 */
  int64_t request_id;
  double arrival_ms, first_token_ms, completed_ms;
  int64_t prompt_tokens, output_tokens;
  int32_t engine_id, pad_;
} nx_request_record;

/* Parse + validate configs, synthesise workloads (host threads), pack the
 * SoA image into pinned host memory. No device work. */
int nx_sim_create_json(const char* const* configs, int32_t n_replicas, int32_t device,
                       int32_t host_threads, nx_sim_t* out);
/* A failed replica's status (NX_OK when it ran to completion) and the
 * reference's exception text for it (e.g. engine.cpp:75-78 "prefill_priority:
 * prompt exceeds m_max; raise m_max for engine 3") into buf[cap]. Valid after
 * the download. */
int nx_sim_error(nx_sim_t h, int32_t replica, char* buf, int64_t cap);
/* Workload generation again (build_workload, proj/src/sim.cpp:101-141) for
 * every replica on host threads, into the pinned input image; the parsed
 * configs are kept. Deterministic: the next run reproduces the same results.
 * May overlap a launch in flight: it rewrites the pinned image only after the
 * previous upload's copies have completed, so a caller can build the next
 * batch's inputs while the device runs this one. (bench.py times it inside
 * e2e, as the reference's run_simulation clock includes its workload build.) */
int nx_sim_rebuild_workloads(nx_sim_t h, int32_t host_threads);
/* Upload (H2D), launch, download (D2H) on the handle's stream; each is async.
 * nx_sim_last_kernel_ms covers the launch's state reset + the kernel. */
int nx_sim_upload(nx_sim_t h);
int nx_sim_launch(nx_sim_t h);
int nx_sim_download(nx_sim_t h);
int nx_sim_synchronize(nx_sim_t h);
/* upload + launch + download + synchronize */
int nx_sim_run(nx_sim_t h);
/* Device time of the last launch (CUDA events on the handle's stream). */
int nx_sim_last_kernel_ms(nx_sim_t h, float* ms);
/* Bytes moved per upload / download (e2e accounting). */
int nx_sim_io_bytes(nx_sim_t h, int64_t* h2d, int64_t* d2h);
int nx_sim_replica_count(nx_sim_t h);
int nx_sim_summaries(nx_sim_t h, nx_replica_summary* out);
/* Byte-identical to RunResult::summary_json (proj/src/sim.cpp:349-392). */
/* servesim::MetricsSummary of one replica (metrics.h / metrics.cpp:40-91),
 * computed on the device after the run (K7, device/summary.cu): nearest-rank
 * percentiles by radix selection, the means as the reference's left folds. */
typedef struct nx_replica_metrics {
  int64_t completed;
  double p50_e2e_ms, p90_e2e_ms, p50_ttft_ms, p50_tpot_ms;
  double mean_ttft_ms, mean_tpot_ms, slo_attainment_pct;
} nx_replica_metrics;
int nx_sim_metrics(nx_sim_t h, int32_t replica, nx_replica_metrics* out);
int nx_sim_summary_json(nx_sim_t h, int32_t replica, char* buf, int64_t cap, int64_t* len);
int nx_sim_records(nx_sim_t h, int32_t replica, nx_request_record* out, int64_t cap,
                   int64_t* n);
/* Work counters of a replica (roofline accounting): [0] executed steps,
 * [1] sum of batch sizes, [2] LENS candidate-window waiters scanned,
 * [3] linear-refit window samples, [4] structural-refit window samples,
 * [5] gauged (profiled) fits. */
int nx_sim_work(nx_sim_t h, int32_t replica, int64_t* out6);
/* SM cycles per phase of a replica (lane-0 clock64): [0] event selection +
 * hash, [1] routing + admission, [2] step planning, [3] step completion,
 * [4] state reports, [5] linear refits, [6] structural refits (on the refit
 * warp, overlapped with the event loop), [7] deliveries, [8] event loop
 * blocked on a pending refit, [9]-[15] refit internals (diagnostic) */
int nx_sim_phase_cycles(nx_sim_t h, int32_t replica, int64_t* out10);
/* %globaltimer (ns) at which the replica's CTA started and finished it
 * (diagnostic: per-replica latency under co-residency). */
int nx_sim_timeline(nx_sim_t h, int32_t replica, int64_t* begin_end_ns);
/* ---- observability (RunConfig.output / record_learner_history) ------------
 * Written by the device during the run when the config asks for them
 * (output.plans_jsonl, output.routing_jsonl, record_learner_history):
 * one plan row per started step (sim.cpp:149-158), one routing row per
 * arrival (sim.cpp:176-186), one learner snapshot per learner update event
 * (sim.cpp:322-327). */
typedef struct nx_plan_log_row {
  double sim_time_ms;
  int32_t engine_id, pad_;
  int64_t b, s;
  double predicted_ms, target_ms;
} nx_plan_log_row;
typedef struct nx_route_log_row {
  double sim_time_ms;
  int64_t request_id;
  int32_t chosen_engine, pad_;
  double s_latency, s_load, s_capacity, s_affinity, score;
} nx_route_log_row;
typedef struct nx_learner_snapshot {  /* LearnerSnapshot (sim.h:62-67) */
  int32_t engine_id, pad_;
  double sim_time_ms;
  int64_t samples_seen;
  double params[8];
} nx_learner_snapshot;
int nx_sim_plan_log(nx_sim_t h, int32_t replica, nx_plan_log_row* out, int64_t cap, int64_t* n);
int nx_sim_route_log(nx_sim_t h, int32_t replica, nx_route_log_row* out, int64_t cap, int64_t* n);
int nx_sim_learner_history(nx_sim_t h, int32_t replica, nx_learner_snapshot* out, int64_t cap,
                           int64_t* n);
/* Simulation::write_outputs (sim.cpp:393-413): summary.json, requests.csv and
 * the JSONL logs into the config's output.dir (no-op when it is empty). */
int nx_sim_write_outputs(nx_sim_t h, int32_t replica);
/* Learner state per engine: params[8] + samples + counters[7]. */
int nx_sim_learner(nx_sim_t h, int32_t replica, int32_t engine, double* params8,
                   int64_t* samples, int64_t* counters7);
void nx_sim_destroy(nx_sim_t h);

/* ---- K6: multi-GPU result gather ------------------------------------------
 * The per-replica nx_replica_summary array is the only data that crosses
 * GPUs (one collective per run; no per-step exchange). Device pointer to the
 * handle's summaries, filled by nx_sim_launch, for an NCCL all-gather. */
int nx_sim_summaries_dev(nx_sim_t h, void** dev_ptr, int64_t* bytes);
/* Device-to-device copy of those summaries into a caller buffer (e.g. the
 * send buffer of an ncclAllGather); ordered on the handle's stream. */
int nx_sim_copy_summaries(nx_sim_t h, void* dst_dev);
/* The gather itself over NCCL (libnccl.so.2 resolved at run time): rank 0
 * makes a unique id, the caller distributes it (any channel), every rank
 * joins, then one ncclAllGather of each rank's NxReplicaOut array (equal
 * replica counts per rank) into recv_dev (nranks x the _dev bytes), ordered
 * on the handle's stream. nx_gather_results of SURVEY §8(b). */
#define NX_NCCL_ID_BYTES 128
int nx_nccl_unique_id(char* id128);
int nx_nccl_comm_init(const char* id128, int32_t nranks, int32_t rank, int32_t device, void** comm);
int nx_nccl_comm_destroy(void* comm);
int nx_sim_gather_summaries(nx_sim_t h, void* comm, void* recv_dev);

/* ---- host utilities (reference workload generator semantics) -------------
 * synth_generate (proj/src/workload.cpp:137-166): prompts/outputs/session
 * ids for n requests. session_ids: n * 16-byte NUL-terminated strings. */
/* Parse a RunConfig JSON and synthesise its workload on the host only:
 * arrival fingerprint (sim.cpp:132-139), request and session counts. Raises
 * the reference's config errors (RunConfig::validate, sim.cpp:418-452). */
int nx_workload_info(const char* config_json, uint64_t* arrival_hash, int64_t* n_requests,
                     int64_t* n_sessions);
/* xoshiro256++ state of Rng(substream_seed(root_seed, tag, index))
 * (proj/include/servesim/rng.h): e.g. a Router's weighted-policy stream is
 * tag "router", index 0 (router.cpp:62-64). */
int nx_rng_state(uint64_t root_seed, const char* tag, uint64_t index, uint64_t* state4);
int nx_synth_generate(const char* scenario, int64_t n, uint64_t seed, int64_t* prompts,
                      int64_t* outputs, char* session_ids16);

#ifdef __cplusplus
}
#endif
#endif /* NX_SCHED_H_ */
