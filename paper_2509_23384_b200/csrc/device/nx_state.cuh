// Per-warp replica state staged in shared memory + the execution context.
//
// One warp simulates one replica. Lane 0 is the "sequential" owner of every
// shared scalar: all lanes run the same control flow and compute the same
// values from shared state, but only lane 0 stores (`put`), bracketed by
// __syncwarp so no lane reads a half-updated field. Lane-parallel sections
// (scans over engines, candidate batches, learner samples) write only
// lane-private slots and sync before anyone reads them.
#pragma once
#include "../nx_layout.h"
#include "nx_math.cuh"

// Optional out-of-line boundary for the large event handlers and refit
// stages (-DNX_OUTLINE: one copy each, ~2.5x smaller code). Measured slower
// per event on B200 than the fully inlined kernel (call overhead and a
// stack-resident Ctx outweigh the instruction-cache savings), so off by default.
#ifdef NX_OUTLINE
#define NX_COLD __noinline__
#else
#define NX_COLD
#endif

namespace nxd {

constexpr uint64_t kNoEvent = ~0ull;
constexpr int kFbTable = 1024;  // batch-factor table entries per learner fit
constexpr int kFitSmemS = 4096; // 1/f_S entries of the refit team's shared-memory fit tables
#ifndef NX_REFIT_WARPS
#define NX_REFIT_WARPS 3
#endif
constexpr int kRefitWarps = NX_REFIT_WARPS;  // structural-refit team per replica CTA (leader + helpers)
constexpr int kSimWarps = 1 + kRefitWarps;   // + the event-loop warp
constexpr int kMaxSmIds = 1024;              // %smid bound of the kernel's SM bookkeeping
constexpr int kSchedCtlInts = 3 + 2 * kMaxSmIds;

// One piece of fit work split across the refit team (nx_learner.cuh::team_work).
struct TeamTask {
  const double2* rec;
  const double* stab;
  const double* ifb;
  const int* pb;    // grouped sums: sample order by batch size / by distinct s
  const int* ps;
  const int* ob;
  const int* os;
  const int* us;
  double* ab;       // per-b / per-distinct-s aggregates
  double* as;
  double* part;     // rebuild partials of groups cut by chunk boundaries
  double kB;
  int n, tab, U;
  int op;           // 1 sample pass, 2 sum over b, 3 sum over s, 4 / 5 rebuild ab / as, -1 leave
};

// Scratch offsets (doubles) of the structural tier's grouped sums, after the
// s -> index table (nx_learner.cuh layout).
__host__ __device__ __forceinline__ int64_t group_base(int64_t W) { return 10 * W + kFbTable + 5120; }
__host__ __device__ __forceinline__ int64_t half_up(int64_t v) { return (v + 1) / 2; }
// Doubles of one warp's learner scratch for long_window W (nx_learner.cuh
// layout; host: capi.cpp fill_descriptors allocates two per replica).
__host__ __device__ __forceinline__ int64_t refit_scratch_stride(int64_t W) {
  const int64_t groups =
      2 * half_up(W) + half_up(kFbTable + 3) + half_up(W + 2) + 8 * kFbTable + 4 * W + 2 * 8 * 32 * kRefitWarps;
  return (group_base(W) + groups + 64 + 31) / 32 * 32;
}

// Engine scalars (EngineSim + OnlineLearner + TradeoffEstimator + router view)
struct EngSm {
  Params lp;                                   // learner current_ (learner.h:90)
  double alpha, beta, l_bar, td_min;           // TradeoffModel (lens.h:22-27)
  double plan_pred, plan_target, actual, learn_y;
  double lat_sum;
  double rep_lhat, rep_wload, rep_mfree, rep_pmax, rep_at;  // router's report copy
  uint64_t rng[4];
  double noise[32];                            // next oracle noise multipliers exp(sigma z)
  uint64_t step_t, learn_t, report_t;          // pending-event slots (kNoEvent = none)
  uint64_t dq_t0;                              // head of the delivery FIFO (cached)
  int64_t started_us, seen, rep_qlen, tw_degen;
  int32_t lin_left, str_left;                  // samples until the next linear / structural period
  int64_t cnt[7];                              // LearnerCounters
  // parent references of the pending events (sim_kernel.cu: log index of the
  // event that pushed them, kRootPar | seq of a root parent, kSelfRoot | seq
  // for the initial state reports)
  uint32_t step_seq, learn_seq, report_seq, dq_s0;
  uint32_t log_n;                              // events this engine has logged
  uint32_t last_fin_par;                       // key of the last step that completed requests
  uint64_t last_fin_t;                         // (kNoEvent: none)
  int64_t period_us;                           // state_report_period (shared-memory copy)
  int32_t eid1;                                // engine_id + 1 (event hash)
  int32_t wq_head, wq_len, rq_len;
  int32_t pinned, reserved, cache_blocks, lru_head, lru_tail;
  int32_t busy, plan_n, plan_b, plan_s, plan_wspan, plan_overload, plan_ndec;
  int32_t learn_b, learn_s;
  int32_t ring_size, ring_head, tw_head, tw_len, dq_head, dq_len, lat_head, lat_len;
  int32_t has_rep, noise_pos;
  int32_t refit_pending;                       // structural refit queued / running
  // decode-only step memo: T(R, R) under the learner params (valid while
  // lp_ver is unchanged) and under the ground truth
  int32_t lp_ver, memo_ver, memo_b, memo_tb;
  double memo_pred, memo_truth;
};

struct ErrSlot {                               // first error raised by one warp
  int32_t status, site;
  int64_t info;
  uint64_t t;                                  // key of the event that raised it
  uint32_t par;
  int32_t kind, eng;
};

constexpr int kPdMaxWarps = 9;                 // router + up to 8 engine warps per replica CTA

struct RepSm {
  uint64_t ev_hash, rr_next, rng[4];
  uint64_t next_arr;                           // arrival time at the cursor (cached)
  int64_t arrived, rejected, pending, n_rec, events, info;
  int64_t work[6];
  int64_t cycles[16];
  int64_t lcycles[16];                         // learner-internal timers (diagnostic build)
  int64_t t_begin_ns;
  int64_t n_plan_log, n_route_log, n_learn_log;
  double l_bar_ema;
  uint32_t next_seq;
  int32_t cursor, status, site;
  int32_t jq_head, jq_tail;                    // structural-refit job ring (warp 0 -> warp 1)
  int32_t jq_eng[64];
  TeamTask team;                               // refit leader -> helpers
  double team_part[kRefitWarps][11];           // per-warp fit-pass totals
  // engine-parallel event loop (sim_kernel.cu)
  ErrSlot err[kPdMaxWarps];
  uint64_t horizon;                            // engines process events with key < (horizon, arrival)
  uint64_t front[NX_MAX_ENGINES];              // next event time of each engine
  uint64_t kd_t;                               // drain key: last completion / last arrival
  uint32_t kd_par;
  int32_t kd_kind, kd_eng, kd_ready, kd_inf;
  int32_t final_mode, stop, parked, n_done, n_fin;
  int32_t all_arrived;
  uint32_t wpos[NX_MAX_ENGINES], mpos[NX_MAX_ENGINES];  // log entries written / merged
  int32_t ob_w[NX_MAX_ENGINES], ob_r[NX_MAX_ENGINES];   // outbox written / merged
  int32_t ps_w[NX_MAX_ENGINES], ps_r[NX_MAX_ENGINES];   // staged plan rows
  int32_t ls_w[NX_MAX_ENGINES], ls_r[NX_MAX_ENGINES];   // staged learner rows
  int32_t done[NX_MAX_ENGINES], fin[NX_MAX_ENGINES];
  int32_t am;                                  // arrivals merged
  uint64_t am_t;                               // time of the next routed, unmerged arrival
};

struct Ctx {
  const NxPools* P;
  const NxReplicaDesc* d;
  const NxEngineDesc* ed;  // this replica's engines
  RepSm* rs;
  EngSm* eng;
  int32_t* prefix;         // LENS prefix sums (union with chunk)
  double* chunk;           // 32 x 5 staging rows for exact-order folds
  double* scratch;         // learner scratch in HBM (fs cache, fb table, rows)
  double* lin_rows;        // this warp's linear-tier row buffer in the scratch
  int64_t roff, soff;
  int n_eng, n_req, n_sess, lane, prefix_cap;
  int worker;              // 0: event-loop warp, 1: structural-refit warp
  int log_flags;           // NX_LOG_* of this replica (register copy of the descriptor's)
  int team;                // warps in the refit team (1: the calling warp alone)
  double* fsm;             // shared-memory fit tables (1/f_B, then 1/f_S); nullptr: use scratch
  int fsm_cap;             // 1/f_S entries that fit in fsm
  ErrSlot* err;            // this warp's error slot
  uint32_t cur_ref;        // parent reference for events pushed by the current handler
  uint32_t cur_meta;       // log flags gathered while handling the current event
  int began;               // try_begin_step started a step and staged a plan row
  int inline_refit;        // structural refits run on the calling warp (no refit team)
  NxEvLog* elog;           // this CTA slot's event-log rings (engine e at e * evlog_cap)
  int32_t* obox;           // this CTA slot's outboxes
  int64_t ob_cap;          // outbox entries per engine
  NxEvLog* sring;          // shared-memory copies of the rings' most recent entries
  NxReqState* req;         // this replica's request state (shared memory or HBM)
  uint8_t* kva;            // this replica's KV-admitted flags (shared memory or HBM)
};

template <class T>
__device__ __forceinline__ void put(T& dst, T v) {
  __syncwarp();
  if (lane_id() == 0) dst = v;
  __syncwarp();
}

// Raise a reference exception: first error wins, replica stops.
__device__ __forceinline__ void fail(Ctx& c, int status, int site, int64_t info) {
  __syncwarp();
  if (c.lane == 0 && c.err->status == 0) {
    c.err->status = status;
    c.err->site = site;
    c.err->info = info;
  }
  __syncwarp();
}
__device__ __forceinline__ bool failed(const Ctx& c) {
  return *reinterpret_cast<const volatile int32_t*>(&c.err->status) != 0;
}

// Phase timers exist only in the diagnostic build (-DNX_TIMERS, made by
// tools/phase_report.py); the product kernel compiles every clock read and
// counter update away.
#ifdef NX_TIMERS
static __constant__ int nx_timers_on;
#else
constexpr int nx_timers_on = 0;
#endif

__device__ __forceinline__ long long nx_clock() {
#ifdef __CUDA_ARCH__
  return nx_timers_on ? clock64() : 0;
#else
  return 0;
#endif
}

__device__ __forceinline__ long long nx_globaltimer() {
  long long t = 0;
#ifdef __CUDA_ARCH__
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#endif
  return t;
}

// Phase timer: lane 0 charges the SM cycles of a scope to rs->cycles[k].
struct PhaseTimer {
  RepSm* rs;
  int k;
  long long t0;
  __device__ __forceinline__ PhaseTimer(RepSm* r, int kk) : rs(r), k(kk), t0(nx_clock()) {}
  __device__ __forceinline__ ~PhaseTimer() {
    if (nx_timers_on && lane_id() == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&rs->cycles[k]),
                static_cast<unsigned long long>(nx_clock() - t0));
  }
};

// counters shared by both warps of a replica CTA
__device__ __forceinline__ void count(int64_t& slot, int64_t v) {
  if (v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(&slot), static_cast<unsigned long long>(v));
}
__device__ __forceinline__ int32_t vload(const int32_t& x) {
  return *reinterpret_cast<const volatile int32_t*>(&x);
}
__device__ __forceinline__ void vstore(int32_t& x, int32_t v) {
  *reinterpret_cast<volatile int32_t*>(&x) = v;
}

}  // namespace nxd
