// Host/device shared layout of the replica batch in HBM.
//
// One replica = one independent servesim::Simulation (proj/src/sim.cpp:57-99).
// A batch of replicas is packed into structure-of-arrays pools; every per-engine
// and per-replica region is addressed by element offsets stored in the
// descriptors below. Plain C layout: compiled by both g++ and nvcc.
#pragma once
#include <stdint.h>

#define NX_MAX_ENGINES 32      /* one lane per engine in the warp-wide scans */
#define NX_TW_CAP 200          /* TradeoffEstimator::kWindow, proj/include/servesim/lens.h:145 */
#ifndef NX_EVLOG_CAP
#define NX_EVLOG_CAP (1 << 15) /* event-log ring entries per engine (power of two) */
#endif

/* Per-engine static description + pool offsets (one per engine, all replicas). */
typedef struct NxEngineDesc {
  double tp[8];            /* ground-truth PerfParams (engine.h:29) */
  double noise_sigma;
  double static_w;         /* router static weight for this engine (router.h:42) */
  int64_t period_us;       /* to_us(state_report_period_ms) */
  int64_t stale_us;        /* to_us(state_staleness_ms) */
  uint64_t rng[4];         /* xoshiro state for substream "engine-noise"/engine_id */
  int64_t wq_off;          /* wait-queue pool, capacity = replica n_req */
  int64_t rq_off;          /* run-queue pool, capacity = replica n_req */
  int64_t plan_off;        /* in-flight plan allocations, capacity = replica n_req */
  int64_t cache_off;       /* prefix-cache LRU arrays, capacity = replica n_sess */
  int64_t ring_off;        /* learner ring, capacity = long_window */
  int64_t tw_off;          /* tradeoff window, capacity = NX_TW_CAP */
  int64_t dq_off;          /* report deliveries FIFO, capacity = dq_cap */
  int64_t lat_off;         /* latency_based rolling window, capacity = lat_cap */
  int32_t engine_id, policy;
  int32_t kv_blocks, block_size, m_max, q_max, static_budget, wait_cap;
  int32_t dq_cap, lat_cap;
} NxEngineDesc;

typedef struct NxReplicaDesc {
  double ttft_slo, tpot_slo, eps_ratio, q_ref;
  double alpha, beta, l_bar, td_min;          /* TradeoffModel init */
  double weights[4], beta_aff, knee, scale_ms, load_half, headroom;
  double stale_limit, lat_window;
  uint64_t router_rng[4];
  int64_t duration_us;
  int64_t req_off;         /* request pools */
  int64_t sess_off;        /* router session map */
  int64_t scratch_off;     /* learner scratch, capacity = long_window doubles */
  int32_t n_eng, eng_base, n_req, n_sess;
  int32_t n_iters, route_policy;
  int32_t long_w, short_w, s_period, l_period, min_s;
  int32_t log_flags;       /* NX_LOG_* observability streams of this replica */
  int64_t plan_log_off, route_log_off, learn_log_off;  /* record offsets in the log pools */
  int64_t plan_log_cap, learn_log_cap;                 /* capacities (route log: n_req) */
} NxReplicaDesc;

/* Observability streams (proj/src/sim.cpp:149-158, 176-186, 322-327): written
   by the device as the events happen, formatted on the host. */
enum { NX_LOG_PLANS = 1, NX_LOG_ROUTES = 2, NX_LOG_LEARNER = 4 };
typedef struct NxPlanLog {   /* plans_jsonl row: the inflight plan of a started step */
  int64_t t_us;
  int32_t engine_id, b, s, pad_;
  double predicted_ms, target_ms;
} NxPlanLog;
typedef struct NxRouteLog {  /* routing_jsonl row: one RouteDecision */
  int64_t t_us;
  int32_t request, engine_id;
  double score, factors[4];
} NxRouteLog;
typedef struct NxLearnLog {  /* LearnerSnapshot after a learner update event */
  int64_t t_us, samples;
  int32_t engine_id, pad_;
  double params[8];
} NxLearnLog;

/* Per-replica result (device -> host). */
typedef struct NxReplicaOut {
  int64_t arrived, rejected, completed, pending, events;
  uint64_t event_hash;
  int32_t status;          /* 0 ok, 1 invalid_argument, 2 runtime_error, 3 logic_error */
  int32_t err_site;        /* NX_SITE_* where the error was raised */
  int64_t err_info;
  /* work counters for the roofline's algorithmic bytes:
     [0] executed steps, [1] sum of step batch sizes b, [2] sum of LENS
     candidate windows (waiters scanned), [3] linear-refit window samples,
     [4] structural-refit window samples (fits run), [5] gauged fits */
  int64_t work[6];
  /* SM cycles spent per phase (clock64, lane 0): [0] event selection + hash,
     [1] routing + admission, [2] step planning (LENS / baseline, KV trim,
     oracle), [3] step completion, [4] state reports, [5] linear refits,
     [6] structural refits (refit warp, overlapped), [7] report deliveries,
     [8] event-loop warp blocked on a pending refit, [9]-[15] refit internals */
  int64_t cycles[16];
  /* %globaltimer (ns) when the replica's CTA started and finished it */
  int64_t t_begin_ns, t_end_ns;
  int64_t n_plan_log, n_route_log, n_learn_log;  /* rows written to the logs */
} NxReplicaOut;

/* Per-replica metrics summary computed on the device (device/summary.cu):
   servesim::MetricsSummary (metrics.h) with engine counts by engine index. */
typedef struct NxReplicaMetrics {
  double p50_e2e, p90_e2e, p50_ttft, p50_tpot, mean_ttft, mean_tpot, slo_pct;
  int64_t completed;
  int32_t valid;           /* 0: a record's timestamps were out of order (metrics.cpp:13-16) */
  int32_t n_tpot;          /* multi-token requests */
  int32_t engine_count[NX_MAX_ENGINES];
} NxReplicaMetrics;

typedef struct NxEngineOut {
  double params[8];        /* learner's current PerfParams */
  int64_t samples;         /* OnlineLearner::samples_seen */
  int64_t counters[7];     /* LearnerCounters order (learner.h:26-34) */
  int64_t tradeoff_degenerate;
  double alpha, beta, l_bar;
} NxEngineOut;

/* The per-request fields every step touches, as one 16-byte record (one
   sector per request instead of one in each of four SoA arrays). */
typedef struct NxReqState {
  int32_t prefilled, decoded, prompt, target;
} NxReqState;

/* One logged event of an engine's stream (the engine-parallel event loop,
   device/sim_kernel.cu): its time, a reference to the event that pushed it
   (its parent: a log index in the same engine's stream, or a root event's
   sequence number) and its kind + flags. The reference's (time, sequence)
   order is recovered from these references (sim.cpp:50-55, 67-70). */
typedef struct NxEvLog {
  int64_t t;
  uint32_t par;
  uint32_t meta;
} NxEvLog;

/* Device pools (all pointers are device pointers). */
typedef struct NxPools {
  /* request inputs */
  const int64_t* arr_us; const double* arr_ms;
  const int32_t* session;
  NxReqState* req;             /* state (prefilled, decoded) + prompt, target */
  const NxReqState* req0;      /* launch image of req (prefilled = decoded = 0) */
  /* request state / outputs */
  int64_t* first_us; int64_t* done_us;
  int32_t* req_engine; uint8_t* kv_admitted;
  /* queues and plans */
  int32_t* wq; int32_t* rq; int32_t* plan_req; int32_t* plan_tok;
  int32_t* c_tokens; int32_t* c_prev; int32_t* c_next;
  int32_t* ring_b; int32_t* ring_s; double* ring_y;
  double* tw_ttft; double* tw_tpot;
  int64_t* dq_t; uint32_t* dq_seq; double* dq_sv; int64_t* dq_qlen;  /* dq_sv: 5 doubles per entry */
  double* lat_t; double* lat_e2e;
  int32_t* sess_engine;
  int32_t* records;
  double* scratch;               /* learner scratch: per CTA slot x engine warp */
  /* engine-parallel event loop, per CTA slot x engine (capacities below) */
  NxEvLog* evlog;                /* event-log ring per engine */
  int32_t* outbox;               /* completed requests per engine, 4 ints each */
  NxPlanLog* plan_stage;         /* per replica x engine plan rows (logging only) */
  NxLearnLog* learn_stage;       /* per replica x engine learner rows (logging only) */
  uint8_t* began;                /* per request: its arrival started a step (plan logging) */
  int64_t evlog_cap, outbox_cap, scratch_stride;
  int32_t slot_engines, slot_warps;  /* engines / engine warps per CTA slot */
  NxPlanLog* plan_log; NxRouteLog* route_log; NxLearnLog* learn_log;
  /* descriptors + outputs */
  const NxReplicaDesc* rep; const NxEngineDesc* eng;
  NxReplicaOut* rep_out; NxEngineOut* eng_out;
  NxReplicaMetrics* metrics;   /* device-side summaries (summary.cu) */
} NxPools;

enum {
  NX_SITE_NONE = 0,
  NX_SITE_BISECT = 1,        /* binary_search_budget invalid inputs (lens.cpp:36-38) */
  NX_SITE_ALLOCATE = 2,      /* allocate_tokens budget below queue needs (lens.cpp:61-63) */
  NX_SITE_PREFILL_CAP = 3,   /* prefill_priority prompt exceeds m_max (engine.cpp:74-79) */
  NX_SITE_SAMPLE = 4,        /* invalid LatencySample (learner.cpp:131-133) */
  NX_SITE_CAPACITY = 5,      /* score_capacity demand < 1 (router.cpp:54-56) */
  NX_SITE_OVERFLOW = 6,      /* device capacity exceeded (plan/delivery/latency ring) */
  NX_SITE_PARAMS = 7         /* predict_latency on invalid params (perf_model.cpp:26-28) */
};
