// K5 — batched discrete-event simulation: one CTA per replica, its engines
// simulated in parallel, one warp each.
//
// Each CTA runs one servesim::Simulation (proj/src/sim.cpp:245-347) to
// completion. The reference pops one std::priority_queue<SimEvent> in
// (time_us, sequence) order. Here the events are split by owner:
//
//  * engine events — step completion, learner update, state report, report
//    delivery (sim.cpp:196-243, 307-328) — touch only their engine's state
//    (queues, KV blocks, learner, noise stream, the router's copy of that
//    engine's report and latency window), so each engine warp runs its own
//    engines' events in their (time, sequence) order;
//  * arrivals (sim.cpp:168-194) read every engine's router-side state, so
//    the router warp handles them at a barrier: engines first process every
//    event ordered before the arrival (a time-window conservative parallel
//    discrete-event simulation whose windows end at arrival times).
//
// The reference's sequence numbers are never materialised. Every event keeps
// a reference to the event that pushed it (its parent), and sequence order
// between two events of equal time is the processing order of their parents
// (then push order), so the key comparison walks parent references (ev_less).
// Everything order-dependent across engines — the FNV event hash, the
// completion records, the router's l_bar EMA and session map, the
// observability logs — is produced by the router warp's merger, which
// consumes the engines' event logs in key order behind the engines' fronts.
//
// Inside an event an engine warp's lanes parallelise over candidate batch
// sizes (K2 LENS budget search), allocations (step completion) and learner
// samples (K4 refit, nx_learner.cuh, run by the engine's own warp); the
// router warp's lanes over engines (K3 PRISM scorer).
#ifndef NX_INLINE_EXPM1
#define NX_COMPACT_MATH 1  // one out-of-line expm1 (was ~180 KB of inlined copies)
#endif
#define NX_INLINE_REFIT 1  // structural refits run on the engine's own warp (record_sample)
#ifndef NX_SIM_LB_WARPS
#define NX_SIM_LB_WARPS 9  // warps per replica CTA the register budget is sized for (router + engine warps)
#endif
#include <stdlib.h>

#include "nx_learner.cuh"
#include "nx_lens.cuh"
#include "nx_router.cuh"

namespace nxd {

constexpr double kInf = __builtin_huge_val();

// Event references (see the file comment): a pending or logged event names
// its parent by the parent's index in the same engine's log, or by
// kRootPar | seq for a root parent (initial state report e: seq e; arrival i:
// seq E + i, sim.cpp:276-293). Initial state reports are roots themselves
// (kSelfRoot | seq).
constexpr uint32_t kRootPar = 0x80000000u, kSelfRoot = 0x40000000u, kSeqMask = 0x3fffffffu;
enum { kEvArrival = 0, kEvStep = 1, kEvReport = 2, kEvLearn = 3, kEvDeliver = 4 };  // sim.cpp:32-38
constexpr uint32_t kMetaPlan = 8u;   // log meta: the event started a step and staged a plan row
constexpr int kMetaFinShift = 8;     // log meta: requests a step completion finished
#ifndef NX_SRING
#define NX_SRING 256
#endif
constexpr int kRing = NX_SRING;      // shared-memory log entries per engine (merger's view)
// Phase timer slots of the diagnostic build (-DNX_TIMERS, tools/pdes_report.py)
enum {
  kTmMerge = 0, kTmRoute = 1, kTmPlan = 2, kTmComplete = 3, kTmReport = 4, kTmLinear = 5,
  kTmStructural = 6, kTmPark = 7, kTmRing = 8, kTmDrain = 9, kTmEvents = 10, kTmRouterIdle = 11,
  kTmFinal = 12, kTmWindows = 13, kTmNWindows = 14, kTmLearn = 15
};

// ---- small helpers ------------------------------------------------------------
// ceil(tokens / block) for tokens >= 0; block sizes are powers of two in
// practice (16), where a shift replaces the integer division sequence.
__device__ __forceinline__ int blocks_for(int tokens, int block) {
  const int t = tokens + block - 1;
  return (block & (block - 1)) == 0 ? t >> (__ffs(block) - 1) : t / block;
}
// (i + j) mod cap for 0 <= i, j <= cap (ring positions): a compare instead of
// a remainder by a runtime divisor.
__device__ __forceinline__ int ring_add(int i, int j, int cap) {
  const int t = i + j;
  return t >= cap ? t - cap : t;
}
// rr % n for the round-robin counter, 32-bit while it fits.
__device__ __forceinline__ int rr_mod(uint64_t rr, int n) {
  return rr < (1ull << 32) ? static_cast<int>(static_cast<uint32_t>(rr) % static_cast<uint32_t>(n))
                           : static_cast<int>(rr % static_cast<uint64_t>(n));
}
__device__ __forceinline__ int remaining(const Ctx& c, int r) {
  return c.req[r].prompt - c.req[r].prefilled;
}

// target_latency (lens.cpp:10-31) with the engine's tradeoff model
__device__ __forceinline__ double target_latency(const Ctx& c, const EngSm& g, int wait_count) {
  const NxReplicaDesc& d = *c.d;
  return lens_target(d.ttft_slo, d.tpot_slo, g.alpha, g.beta, g.l_bar, g.td_min, d.q_ref, wait_count);
}

// Prefix sums of the remaining prompts of the first `count` waiters of wq.
__device__ __forceinline__ void build_prefix(Ctx& c, const int32_t* wq, int count) {
  lens_prefix(c.lane, c.prefix, count, [&](int i) { return remaining(c, wq[i]); });
}
__device__ __forceinline__ int lower_bound_prefix(const int32_t* pre, int hi, int need) {
  return lens_lower_bound(pre, hi, need);
}

// Publishes a plan: n allocations whose first `ndec` are run-queue decodes.
__device__ __forceinline__ void set_plan(Ctx& c, EngSm& g, int n, int b, int s, double pred,
                                         double target, int wspan, int overload, int ndec) {
  __syncwarp();
  if (c.lane == 0) {
    g.plan_ndec = ndec;
    g.plan_n = n;
    g.plan_b = b;
    g.plan_s = s;
    g.plan_pred = pred;
    g.plan_target = target;
    g.plan_wspan = wspan;
    g.plan_overload = overload;
  }
  __syncwarp();
}

// Writes the run-queue decodes [0, R) of a plan.
__device__ __forceinline__ void write_decodes(Ctx& c, const int32_t* rq, int R, int32_t* preq,
                                              int32_t* ptok) {
  for (int i = c.lane; i < R; i += 32) {
    preq[i] = rq[i];
    ptok[i] = -1;
  }
}

// ---- K2: LENS schedule_step (lens.cpp:96-146) -----------------------------------
__device__ NX_COLD void plan_lens(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  const int R = g.rq_len, W = g.wq_len, qmax = ed.q_max, mmax = ed.m_max;
  const int32_t* wq = c.P->wq + ed.wq_off + g.wq_head;
  const int32_t* rq = c.P->rq + ed.rq_off;
  int32_t* preq = c.P->plan_req + ed.plan_off;
  int32_t* ptok = c.P->plan_tok + ed.plan_off;
  const Params P = g.lp;
  const double target = target_latency(c, g, W);
  if (R > qmax) {  // transient overload: truncated decode plan (lens.cpp:108-117)
    write_decodes(c, rq, qmax, preq, ptok);
    set_plan(c, g, qmax, qmax, qmax, predict(P, qmax, qmax), target, 0, 1, qmax);
    return;
  }
  if (!(target > 0.0)) {  // binary_search_budget precondition (lens.cpp:36-38)
    fail(c, 1, NX_SITE_BISECT, 0);
    return;
  }
  if (W == 0) {
    // Empty wait queue: the only candidate is B = R with S = R (avail = R),
    // so the sweep reduces to one prediction (lens.cpp:121-146).
    write_decodes(c, rq, R, preq, ptok);
    set_plan(c, g, R, R, R, predict(P, R, R), target, 0, 0, R);
    return;
  }
  const int span = ((R + W < qmax) ? R + W : qmax) - R;
  build_prefix(c, wq, span);
  if (c.lane == 0) count(c.rs->work[2], span);
  const int32_t* pre = c.prefix;
  const LensPick pick = lens_sweep(c.lane, P, R, span, mmax, c.d->n_iters, target, c.d->eps_ratio, pre);
  if (pick.budget < 0) {  // every candidate error was NaN: empty plan
    set_plan(c, g, 0, 0, 0, 0.0, target, 0, 0, 0);
    return;
  }
  const int best_budget = pick.budget;
  const double best_T = pick.T;
  const int need = best_budget - R;
  const int j = pick.j;
  write_decodes(c, rq, R, preq, ptok);
  for (int k = c.lane; k < j; k += 32) {  // allocate_tokens waiters (lens.cpp:71-77)
    const int rem = pre[k + 1] - pre[k];
    const int left = need - pre[k];
    preq[R + k] = wq[k];
    ptok[R + k] = rem < left ? rem : left;
  }
  set_plan(c, g, R + j, R + j, best_budget, best_T, target, j, 0, R);
}

// ---- baseline engine policies (engine.cpp:61-108) -------------------------------
__device__ NX_COLD void plan_baseline(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  const int R = g.rq_len, W = g.wq_len, qmax = ed.q_max, mmax = ed.m_max;
  const int32_t* wq = c.P->wq + ed.wq_off + g.wq_head;
  const int32_t* rq = c.P->rq + ed.rq_off;
  int32_t* preq = c.P->plan_req + ed.plan_off;
  int32_t* ptok = c.P->plan_tok + ed.plan_off;
  const Params P = g.lp;
  if (ed.policy == 1) {  // prefill_priority
    if (W > 0) {
      const int cnt = W < qmax ? W : qmax;
      build_prefix(c, wq, cnt);
      int j = 0;  // whole prompts while they fit under m_max
      for (int base = 0; base < cnt; base += 32) {
        const int k = base + c.lane;
        const unsigned ok = __ballot_sync(NX_FULL, k < cnt && c.prefix[k + 1] <= mmax);
        j += __popc(ok);
        if (ok != NX_FULL) break;
      }
      if (j == 0) {
        fail(c, 2, NX_SITE_PREFILL_CAP, ed.engine_id);
        return;
      }
      for (int k = c.lane; k < j; k += 32) {
        preq[k] = wq[k];
        ptok[k] = c.prefix[k + 1] - c.prefix[k];
      }
      const int s = c.prefix[j];
      set_plan(c, g, j, j, s, predict(P, j, s), 0.0, j, 0, 0);
    } else {
      write_decodes(c, rq, R, preq, ptok);
      set_plan(c, g, R, R, R, predict(P, R, R), 0.0, 0, 0, R);
    }
    return;
  }
  // static_chunked: allocate_tokens against a fixed budget
  const int b = (R + W < qmax) ? R + W : qmax;
  const int sb = (ed.static_budget < b) ? b : ed.static_budget;
  const int s = (mmax < sb) ? mmax : sb;
  if (b < R || s < b) {
    fail(c, 1, NX_SITE_ALLOCATE, b);
    return;
  }
  const int slots = b - R;
  const int budget = s - R;
  build_prefix(c, wq, slots);
  const int j = budget > 0 ? lower_bound_prefix(c.prefix, slots, budget) : 0;
  const int jj = j;  // waiters k < slots with prefix[k] < budget
  write_decodes(c, rq, R, preq, ptok);
  int part = 0;
  for (int k = c.lane; k < jj; k += 32) {
    const int rem = c.prefix[k + 1] - c.prefix[k];
    const int left = budget - c.prefix[k];
    const int take = rem < left ? rem : left;
    preq[R + k] = wq[k];
    ptok[R + k] = take;
    part += take;
  }
  const int stot = R + static_cast<int>(__reduce_add_sync(NX_FULL, static_cast<unsigned>(part)));
  const int n = R + jj;
  set_plan(c, g, n, n, stot, n > 0 ? predict(P, n, stot) : 0.0, 0.0, jj, 0, R);
}

// ---- trim_for_kv (engine.cpp:184-214) ----------------------------------------------
__device__ NX_COLD void trim_for_kv(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  int32_t* preq = c.P->plan_req + ed.plan_off;
  int32_t* ptok = c.P->plan_tok + ed.plan_off;
  const int n = g.plan_n, ndec = g.plan_ndec;
  __syncwarp();
  if (c.lane == 0) {
    int kept = ndec;  // decodes are always kept (growth already reserved)
    bool trimmed = false;
    for (int k = ndec; k < n; ++k) {
      const int r = preq[k];
      const int tok = ptok[k];
      bool keep;
      if (tok < 0 || c.kva[r]) {
        keep = true;
      } else if (trimmed) {
        keep = false;
      } else {
        const int foot = blocks_for(c.req[r].prompt + c.req[r].target, ed.block_size);
        const int fut = foot - blocks_for(c.req[r].prefilled + c.req[r].decoded,
                                          ed.block_size);
        if (static_cast<int64_t>(g.pinned) + g.reserved + fut <= ed.kv_blocks) {
          g.reserved += fut;
          c.kva[r] = 1;
          keep = true;
        } else {
          trimmed = true;
          keep = false;
        }
      }
      if (keep) {
        preq[kept] = r;
        ptok[kept] = tok;
        ++kept;
      }
    }
    if (kept != n) {
      int s = ndec;
      for (int k = ndec; k < kept; ++k) s += ptok[k];
      g.plan_n = kept;
      g.plan_b = kept;
      g.plan_s = s;
      g.plan_pred = kept > 0 ? predict(g.lp, kept, s) : 0.0;
    }
  }
  __syncwarp();
}

// Oracle noise (engine.cpp:128-132): the engine stream draws two uniforms per
// executed step; 32 steps' worth are drawn at once (lane 0, in stream order)
// and the Box-Muller + exp for each step runs on its own lane.
__device__ NX_COLD void refill_noise(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  __syncwarp();
  if (c.lane == 0) {
    Rng rng;
    for (int i = 0; i < 4; ++i) rng.s[i] = g.rng[i];
    for (int k = 0; k < 64; ++k) c.chunk[k] = rng.uniform();
    for (int i = 0; i < 4; ++i) g.rng[i] = rng.s[i];
  }
  __syncwarp();
  const double u1 = c.chunk[2 * c.lane], u2 = c.chunk[2 * c.lane + 1];
  const double z = sqrt(-2.0 * log(u1)) * cos((2.0 * 3.141592653589793) * u2);
  g.noise[c.lane] = exp(c.ed[e].noise_sigma * z);
  __syncwarp();
  if (c.lane == 0) g.noise_pos = 0;
  __syncwarp();
}

// ---- begin_step (engine.cpp:216-228) + step event (sim.cpp:143-166) ----------------
__device__ NX_COLD void try_begin_step(Ctx& c, int e, int64_t now_us) {
  EngSm& g = c.eng[e];
  __syncwarp();
  if (g.busy || (g.wq_len == 0 && g.rq_len == 0)) return;
  wait_refit(c, e);  // planning reads the learner's params
  PhaseTimer pt(c.rs, kTmPlan);
  const NxEngineDesc& ed = c.ed[e];
  const bool noisy = ed.noise_sigma != 0.0;
  const int R = g.rq_len;
  double truth;
  if (ed.policy == 0 && g.wq_len == 0 && R <= ed.q_max) {
    // Decode-only LENS step: with an empty wait queue the sweep has the single
    // candidate B = R, S = R (lens.cpp:121-146), and there is no prefill for
    // trim_for_kv to admit. The scheduler's and the oracle's predictions of
    // the same shape are independent chains, evaluated together.
    // Both values are memoised per engine: at low load R repeats for many
    // consecutive steps (same inputs, same value).
    const double bd = static_cast<double>(R);
    const bool hit_p = g.memo_b == R && g.memo_ver == g.lp_ver;
    const bool hit_t = g.memo_tb == R;
    const double pred = hit_p ? g.memo_pred : predict(g.lp, bd, bd);
    truth = hit_t ? g.memo_truth : predict(params_from(ed.tp), bd, bd);
    __syncwarp();
    if (c.lane == 0) {
      g.memo_b = R;
      g.memo_ver = g.lp_ver;
      g.memo_pred = pred;
      g.memo_tb = R;
      g.memo_truth = truth;
    }
    write_decodes(c, c.P->rq + ed.rq_off, R, c.P->plan_req + ed.plan_off, c.P->plan_tok + ed.plan_off);
    // BatchPlan::target_ms = target_latency(0 waiters) (lens.cpp:103-104);
    // validated configs make it positive (tpot, td_min > 0)
    set_plan(c, g, R, R, R, pred, target_latency(c, g, 0), 0, 0, R);
  } else {
    if (ed.policy == 0) plan_lens(c, e);
    else plan_baseline(c, e);
    if (failed(c) || g.plan_n == 0) return;
    if (g.plan_ndec < g.plan_n) trim_for_kv(c, e);
    if (g.plan_n == 0) return;
    truth = predict(params_from(ed.tp), g.plan_b, g.plan_s);  // oracle_latency (engine.cpp:128-132)
  }
  if (noisy && g.noise_pos >= 32) refill_noise(c, e);
  __syncwarp();
  if (c.lane == 0) {
    double actual = truth;
    if (noisy) actual = actual * g.noise[g.noise_pos++];
    const int64_t d = to_us(actual);
    g.busy = 1;
    g.started_us = now_us;
    g.actual = actual;
    g.step_t = static_cast<uint64_t>(now_us + (d > 1 ? d : 1));
    g.step_seq = c.cur_ref;  // pushed by the event being handled
    count(c.rs->work[0], 1);
    count(c.rs->work[1], g.plan_b);
  }
  if (c.log_flags & NX_LOG_PLANS) {  // plans_jsonl row (sim.cpp:149-158), staged per engine
    const int32_t k = c.rs->ps_w[e];
    if (k >= c.d->plan_log_cap) {
      fail(c, 1, NX_SITE_OVERFLOW, 1);
    } else {
      if (c.lane == 0) {
        NxPlanLog& L = c.P->plan_stage[c.d->plan_log_off * c.P->slot_engines + e * c.d->plan_log_cap + k];
        L.t_us = now_us;
        L.engine_id = ed.engine_id;
        L.b = g.plan_b;
        L.s = g.plan_s;
        L.pad_ = 0;
        L.predicted_ms = g.plan_pred;
        L.target_ms = g.plan_target;
        c.rs->ps_w[e] = k + 1;
      }
      c.began = 1;
      c.cur_meta |= kMetaPlan;
    }
  }
  __syncwarp();
}

// ---- prefix cache LRU (engine.cpp:284-305), lane 0 only ----------------------------
struct Lru {
  int32_t* tok;
  int32_t* prev;
  int32_t* next;
};
__device__ __forceinline__ Lru lru_of(const Ctx& c, int e) {
  const int64_t off = c.ed[e].cache_off;
  return {c.P->c_tokens + off, c.P->c_prev + off, c.P->c_next + off};
}
__device__ __forceinline__ void lru_unlink(EngSm& g, const Lru& L, int s) {
  const int p = L.prev[s], n = L.next[s];
  if (p >= 0) L.next[p] = n;
  else g.lru_head = n;
  if (n >= 0) L.prev[n] = p;
  else g.lru_tail = p;
  L.tok[s] = -1;
}
__device__ __forceinline__ void evict_to_fit(EngSm& g, const Lru& L, int kv_blocks, int pinned,
                                             int block) {
  while (g.cache_blocks > kv_blocks - pinned && g.lru_head >= 0) {
    const int v = g.lru_head;
    g.cache_blocks -= blocks_for(L.tok[v], block);
    lru_unlink(g, L, v);
  }
}
__device__ __forceinline__ void cache_insert(EngSm& g, const Lru& L, int s, int tokens,
                                             int kv_blocks, int pinned, int block) {
  if (L.tok[s] >= 0) {
    g.cache_blocks -= blocks_for(L.tok[s], block);
    lru_unlink(g, L, s);
  }
  L.tok[s] = tokens;
  L.prev[s] = g.lru_tail;
  L.next[s] = -1;
  if (g.lru_tail >= 0) L.next[g.lru_tail] = s;
  else g.lru_head = s;
  g.lru_tail = s;
  g.cache_blocks += blocks_for(tokens, block);
  evict_to_fit(g, L, kv_blocks, pinned, block);
}

// ---- admit (engine.cpp:139-169), lane 0 only ---------------------------------------
__device__ bool admit(Ctx& c, int e, int r) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  if (ed.wait_cap > 0 && g.wq_len >= ed.wait_cap) return false;
  const Lru L = lru_of(c, e);
  const int sess = c.P->session[c.roff + r];
  const int cached = L.tok[sess];
  if (cached >= 0) {
    const int prompt = c.req[r].prompt;
    const int credit = cached < prompt - 1 ? cached : prompt - 1;
    const int cb = blocks_for(credit, ed.block_size);
    if (credit > 0 && static_cast<int64_t>(g.pinned) + g.reserved + cb <= ed.kv_blocks) {
      g.cache_blocks -= blocks_for(cached, ed.block_size);
      lru_unlink(g, L, sess);
      c.req[r].prefilled = credit;
      g.pinned += cb;
    }
  }
  c.P->wq[ed.wq_off + g.wq_head + g.wq_len] = r;
  g.wq_len += 1;
  c.P->req_engine[c.roff + r] = e;
  return true;
}

// ---- TradeoffEstimator refit (lens.cpp:161-188), exact left folds --------------------
__device__ NX_COLD void tradeoff_refit(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  const int n = g.tw_len;
  if (n < 2) return;
  const double* tp = c.P->tw_ttft + ed.tw_off;
  const double* td = c.P->tw_tpot + ed.tw_off;
  const int head = g.tw_head;
  // lane 0 folds ttft, lane 1 folds tpot (window order: oldest first)
  double m = 0.0;
  if (c.lane < 2) {
    const double* src = c.lane == 0 ? tp : td;
    for (int i = 0; i < n; ++i) m += src[(head + i) % NX_TW_CAP];
  }
  const double dn = static_cast<double>(n);
  const double mtp = __shfl_sync(NX_FULL, m, 0) / dn;
  const double mtd = __shfl_sync(NX_FULL, m, 1) / dn;
  double acc = 0.0;  // lane 0: var, lane 1: cov
  if (c.lane < 2) {
    for (int i = 0; i < n; ++i) {
      const int k = (head + i) % NX_TW_CAP;
      const double dd = td[k] - mtd;
      acc += c.lane == 0 ? dd * dd : dd * (tp[k] - mtp);
    }
  }
  const double var = __shfl_sync(NX_FULL, acc, 0);
  const double cov = __shfl_sync(NX_FULL, acc, 1);
  const double sd = sqrt(var / dn);
  __syncwarp();
  if (c.lane == 0) {
    if (sd <= 0.15 * mtd) {
      g.tw_degen += 1;
    } else {
      const double slope = cov / var;
      const double nb = -slope;
      g.beta = (1e-3 < nb) ? nb : 1e-3;
      g.alpha = mtp + g.beta * mtd;
    }
  }
  __syncwarp();
}

// ---- complete_step (engine.cpp:230-282) + handle_step_complete (sim.cpp:196-224) ----
__device__ NX_COLD void step_complete(Ctx& c, int e, int64_t now_us) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  const NxPools& P = *c.P;
  const int64_t ro = c.roff;
  const int n = g.plan_n, block = ed.block_size;
  const int32_t* preq = P.plan_req + ed.plan_off;
  const int32_t* ptok = P.plan_tok + ed.plan_off;
  const double now = to_ms(now_us);
  const Lru L = lru_of(c, e);
  int* st_sess = reinterpret_cast<int*>(c.chunk);  // per-chunk staging for lane 0
  int* st_tok = st_sess + 32;
  int* st_pin = st_sess + 64;
  int* st_req = st_sess + 96;
  int pinned = g.pinned;
  int dsum = 0, n_fin = 0, n_first = 0;
  int g_ob_w = c.rs->ob_w[e];  // outbox cursor (lane 0's copy is the one written back)
  bool ovf = false;
  const long long t_cs = nx_clock();
  put(g.busy, 0);
  for (int base = 0; base < n; base += 32) {
    const int k = base + c.lane;
    int delta = 0, held = 0, r = -1, tokens = 0;
    bool first = false, fin = false;
    if (k < n) {
      r = preq[k];
      const int tok = ptok[k];
      const int4 q = *reinterpret_cast<const int4*>(&c.req[r]);  // one 16-B load
      int pre = q.x, dec = q.y;
      const int before = blocks_for(pre + dec, block);
      if (tok >= 0) pre += tok;
      else dec += 1;
      const int after = blocks_for(pre + dec, block);
      delta = after - before;
      *reinterpret_cast<int2*>(&c.req[r]) = make_int2(pre, dec);
      first = tok >= 0 && pre == q.z;
      fin = tok < 0 && dec == q.w;
      if (first) P.first_us[ro + r] = now_us;
      if (fin) {
        held = after;
        tokens = pre + dec;
      }
    }
    // pinned as seen by cache_insert of allocation k (after its own release)
    const int adj = delta - held;
    const int scan = warp_incl_scan(adj);
    const int pin_k = pinned + scan;
    pinned += __shfl_sync(NX_FULL, scan, 31);
    dsum += static_cast<int>(__reduce_add_sync(NX_FULL, static_cast<unsigned>(delta)));
    const unsigned finm = __ballot_sync(NX_FULL, fin);
    n_first += __popc(__ballot_sync(NX_FULL, first));
    if (finm) {
      __syncwarp();
      if (fin) {
        st_sess[c.lane] = P.session[ro + r];
        st_tok[c.lane] = tokens;
        st_pin[c.lane] = pin_k;
        st_req[c.lane] = r;
      }
      __syncwarp();
      if (c.lane == 0) {
        unsigned m = finm;
        while (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1;
          const int rr = st_req[l];
          cache_insert(g, L, st_sess[l], st_tok[l], ed.kv_blocks, st_pin[l], block);
          // CompletionStats + TradeoffEstimator EMA/window (lens.cpp:149-160)
          const int tgt = c.req[rr].target;
          const double first_ms = to_ms(P.first_us[ro + rr]);
          const double ttft = first_ms - P.arr_ms[ro + rr];
          const double tpot = tgt >= 2 ? (now - first_ms) / static_cast<double>(tgt - 1) : 0.0;
          const double lb = g.l_bar + 0.05 * (static_cast<double>(tgt) - g.l_bar);
          g.l_bar = (1.0 < lb) ? lb : 1.0;
          if (tgt >= 2) {
            int slot;
            if (g.tw_len < NX_TW_CAP) {
              slot = (g.tw_head + g.tw_len) % NX_TW_CAP;
              g.tw_len += 1;
            } else {
              slot = g.tw_head;
              g.tw_head = (g.tw_head + 1) % NX_TW_CAP;
            }
            P.tw_ttft[ed.tw_off + slot] = ttft;
            P.tw_tpot[ed.tw_off + slot] = tpot;
          }
          // RequestRecord + Router::on_completion (router.cpp:83-92): the
          // record, the router's l_bar EMA and session memory are applied by
          // the merger in global order (outbox); the latency window is this
          // engine's own
          P.done_us[ro + rr] = now_us;
          {
            int4* ob = reinterpret_cast<int4*>(c.obox) + static_cast<int64_t>(e) * c.ob_cap + g_ob_w;
            *ob = make_int4(rr, P.session[ro + rr], tgt, 0);
            ++g_ob_w;
          }
          if (c.d->route_policy == 4) {
            if (g.lat_len >= ed.lat_cap) {
              ovf = true;
            } else {
              const int slot = ring_add(g.lat_head, g.lat_len, ed.lat_cap);
              P.lat_t[ed.lat_off + slot] = now;
              P.lat_e2e[ed.lat_off + slot] = now - P.arr_ms[ro + rr];
              g.lat_len += 1;
              g.lat_sum += now - P.arr_ms[ro + rr];
            }
          }
        }
      }
      __syncwarp();
    }
    n_fin += __popc(finm);
  }
  __syncwarp();
  if (c.lane == 0) {
    g.pinned = pinned;
    g.reserved -= dsum;
    evict_to_fit(g, L, ed.kv_blocks, pinned, block);
    c.rs->ob_w[e] = g_ob_w;
  }
  __syncwarp();
  if (__any_sync(NX_FULL, ovf)) fail(c, 1, NX_SITE_OVERFLOW, 2);
  c.cur_meta |= static_cast<uint32_t>(n_fin) << kMetaFinShift;
  // run queue: drop finished (stable), then append new runners in plan order
  int32_t* rq = P.rq + ed.rq_off;
  int out = g.rq_len;
  if (n_fin) {
    out = 0;
    const int len = g.rq_len;
    for (int base = 0; base < len; base += 32) {
      const int i = base + c.lane;
      const int r = i < len ? rq[i] : 0;
      const bool keep = i < len && c.req[r].decoded != c.req[r].target;
      const unsigned m = __ballot_sync(NX_FULL, keep);
      __syncwarp();
      if (keep) rq[out + __popc(m & ((1u << c.lane) - 1))] = r;
      out += __popc(m);
      __syncwarp();
    }
  }
  if (n_first) {
    int32_t* wq = P.wq + ed.wq_off;
    for (int base = 0; base < n; base += 32) {
      const int k = base + c.lane;
      bool nr = false;
      int r = 0;
      if (k < n && ptok[k] >= 0) {
        r = preq[k];
        nr = c.req[r].prefilled == c.req[r].prompt;
      }
      const unsigned m = __ballot_sync(NX_FULL, nr);
      if (nr) rq[out + __popc(m & ((1u << c.lane) - 1))] = r;
      out += __popc(m);
    }
    __syncwarp();
    // wait queue: drop prefill-complete requests from the scheduled window,
    // keeping survivors in FCFS order at the window's tail
    if (c.lane == 0) {
      const int head = g.wq_head, span = g.plan_wspan;
      int wpos = head + span - 1;
      for (int i = span - 1; i >= 0; --i) {
        const int r = wq[head + i];
        if (c.req[r].prefilled != c.req[r].prompt) wq[wpos--] = r;
      }
      const int removed = wpos + 1 - head;
      g.wq_head = head + removed;
      g.wq_len -= removed;
    }
  }
  __syncwarp();
  if (c.lane == 0) {
    g.rq_len = out;
    // learner update event at the same timestamp (sim.cpp:216-221)
    g.learn_t = static_cast<uint64_t>(now_us);
    g.learn_seq = c.cur_ref;
    g.learn_b = g.plan_b;
    g.learn_s = g.plan_s;
    g.learn_y = g.actual;
  }
  __syncwarp();
  if (n_fin) tradeoff_refit(c, e);
  if (nx_timers_on && c.lane == 0) count(c.rs->cycles[kTmComplete], nx_clock() - t_cs);
  try_begin_step(c, e, now_us);
}

// ---- state report (sim.cpp:226-243, engine.cpp:307-332), lane 0 only -----------
__device__ NX_COLD void state_report(Ctx& c, int e, int64_t now_us) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  bool ovf = false;
  __syncwarp();
  if (c.lane == 0) {
    const double now = to_ms(now_us);
    double l_hat = 0.0;
    if (g.busy) {
      const double v = g.plan_pred - (now - to_ms(g.started_us));
      l_hat = (0.0 < v) ? v : 0.0;
    }
    double pending = 0.0, demand = 0.0;
    const int32_t* wq = c.P->wq + ed.wq_off + g.wq_head;
    for (int i = 0; i < g.wq_len; ++i) {
      const double rem = static_cast<double>(remaining(c, wq[i]));
      pending += rem;
      demand += rem + g.l_bar;
    }
    const int64_t q = static_cast<int64_t>(g.wq_len) + g.rq_len;
    const double w_load = pending + 32.0 * static_cast<double>(q);
    const double free_tok = static_cast<double>(static_cast<int64_t>(ed.kv_blocks - g.pinned) *
                                                static_cast<int64_t>(ed.block_size));
    const double mf = free_tok - demand;
    if (g.dq_len >= ed.dq_cap) {
      ovf = true;
    } else {
      const int slot = ring_add(g.dq_head, g.dq_len, ed.dq_cap);
      const int64_t o = ed.dq_off + slot;
      const int64_t dt = now_us + ed.stale_us;
      const uint32_t ds = c.cur_ref;  // delivery: first child of this report
      c.P->dq_t[o] = dt;
      c.P->dq_seq[o] = ds;
      double* sv = c.P->dq_sv + 5 * o;
      sv[0] = l_hat;
      sv[1] = w_load;
      sv[2] = (0.0 < mf) ? mf : 0.0;
      sv[3] = g.lp.p_max;
      sv[4] = now;
      c.P->dq_qlen[o] = q;
      if (g.dq_len == 0) {
        g.dq_t0 = static_cast<uint64_t>(dt);
        g.dq_s0 = ds;
      }
      g.dq_len += 1;
    }
    g.report_t = static_cast<uint64_t>(now_us + ed.period_us);
    g.report_seq = c.cur_ref;  // next report: second child
  }
  __syncwarp();
  if (__any_sync(NX_FULL, ovf)) fail(c, 1, NX_SITE_OVERFLOW, 3);
}

// ---- K3: Router::route (router.cpp:141-289) ------------------------------------

// lexicographic first minimum of (key, lane) over lanes with valid keys
__device__ __forceinline__ int warp_argmin_i64(int64_t key, bool valid) {
  int64_t v = valid ? key : INT64_MAX;
  int who = valid ? lane_id() : 64;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t ov = __shfl_xor_sync(NX_FULL, v, o);
    const int ow = __shfl_xor_sync(NX_FULL, who, o);
    if (ov < v || (ov == v && ow < who)) {
      v = ov;
      who = ow;
    }
  }
  return who;
}

__device__ int least_loaded(Ctx& c) {
  const int e = c.lane;
  const bool on = e < c.n_eng;
  int64_t len = 0;
  if (on && c.eng[e].has_rep) len = c.eng[e].rep_qlen;
  return warp_argmin_i64(len, on);
}

__device__ NX_COLD int route(Ctx& c, int rid, double now, double& score, double (&fac)[4]) {
  const NxReplicaDesc& d = *c.d;
  const int n = c.n_eng;
  const int sess = c.P->session[c.roff + rid];
  int32_t* sess_eng = c.P->sess_engine + c.soff;
  int chosen = 0;
  __syncwarp();
  switch (d.route_policy) {
    case 1: {  // round_robin
      chosen = rr_mod(c.rs->rr_next, n);
      put(c.rs->rr_next, c.rs->rr_next + 1);
      break;
    }
    case 2: {  // session_affinity
      const int se = sess_eng[sess];
      if (se >= 0) {
        chosen = se;
      } else {
        chosen = rr_mod(c.rs->rr_next, n);
        put(c.rs->rr_next, c.rs->rr_next + 1);
      }
      break;
    }
    case 3:
      chosen = least_loaded(c);
      break;
    case 4: {  // latency_based: rolling e2e window per engine (router.cpp:130-139)
      const int e = c.lane;
      double lat = kInf;
      if (e < n) {
        EngSm& g = c.eng[e];
        const NxEngineDesc& ed = c.ed[e];
        const double* lt = c.P->lat_t + ed.lat_off;
        const double* le = c.P->lat_e2e + ed.lat_off;
        const double horizon = now - d.lat_window;
        int head = g.lat_head, len = g.lat_len;
        double sum = g.lat_sum;
        while (len > 0 && lt[head] < horizon) {
          sum -= le[head];
          head = ring_add(head, 1, ed.lat_cap);
          --len;
        }
        g.lat_head = head;  // engine-owned fields: lane e is the only writer
        g.lat_len = len;
        g.lat_sum = sum;
        lat = len == 0 ? 0.0 : sum / static_cast<double>(len);
      }
      __syncwarp();
      // first strict minimum (NaN never wins)
      double v = (e < n && !isnan(lat)) ? lat : kInf;
      int who = e < n ? e : 64;
      if (e < n && isnan(lat)) who = 63;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(NX_FULL, v, o);
        const int ow = __shfl_xor_sync(NX_FULL, who, o);
        if (ov < v || (ov == v && ow < who)) {
          v = ov;
          who = ow;
        }
      }
      chosen = (v == kInf) ? 0 : who;
      break;
    }
    case 5: {  // weighted draw (router.cpp:186-203)
      if (c.lane == 0) {
        double total = 0.0;
        for (int e = 0; e < n; ++e) total += c.ed[e].static_w;
        Rng rng;
        for (int i = 0; i < 4; ++i) rng.s[i] = c.rs->rng[i];
        double draw = rng.uniform() * total;
        for (int i = 0; i < 4; ++i) c.rs->rng[i] = rng.s[i];
        chosen = n - 1;
        for (int e = 0; e < n; ++e) {
          draw -= c.ed[e].static_w;
          if (draw <= 0.0) {
            chosen = e;
            break;
          }
        }
      }
      chosen = __shfl_sync(NX_FULL, chosen, 0);
      __syncwarp();
      break;
    }
    default: {  // PRISM multiplicative score (router.cpp:205-284)
      const int prompt = c.req[rid].prompt;
      const double dem = static_cast<double>(prompt) + c.rs->l_bar_ema;
      const double demand = (1.0 < dem) ? dem : 1.0;
      const int e = c.lane;
      EngineView v;
      v.on = e < n;
      v.has_rep = false;
      v.lhat = v.wload = v.mfree = v.at = 0.0;
      v.pmax = 1.0;
      v.qlen = 0;
      v.id = 0x7fffffff;
      v.affine = false;
      if (v.on) {
        const EngSm& g = c.eng[e];
        v.has_rep = g.has_rep;
        v.lhat = g.rep_lhat;
        v.wload = g.rep_wload;
        v.mfree = g.rep_mfree;
        v.pmax = g.rep_pmax;
        v.at = g.rep_at;
        v.qlen = g.rep_qlen;
        v.id = c.ed[e].engine_id;
        v.affine = sess_eng[sess] == e;
      }
      RouterCfgD rc;
      for (int i = 0; i < 4; ++i) rc.w[i] = d.weights[i];
      rc.beta_aff = d.beta_aff;
      rc.knee = d.knee;
      rc.scale_ms = d.scale_ms;
      rc.load_half = d.load_half;
      rc.headroom = d.headroom;
      rc.stale_limit = d.stale_limit;
      rc.ttft_slo = d.ttft_slo;
      const PrismPick pk = prism_choose(rc, v, demand, now, n);
      chosen = pk.who;
      score = pk.score;
      for (int i = 0; i < 4; ++i) fac[i] = pk.f[i];
      __syncwarp();
      if (c.lane == 0) {  // dispatch echo (router.cpp:275-282)
        EngSm& g = c.eng[chosen];
        if (g.has_rep) {
          g.rep_qlen += 1;
          g.rep_wload += static_cast<double>(prompt) + 32.0;
        }
      }
      __syncwarp();
      break;
    }
  }
  __syncwarp();
  if (c.lane == 0) sess_eng[sess] = chosen;  // remember_session (router.cpp:107-122)
  __syncwarp();
  return chosen;
}


// LearnerSnapshot after a learner update event (sim.cpp:322-327), staged per
// engine; the merger emits the rows in event order.
__device__ void log_learner(Ctx& c, int e, int64_t now_us) {
  if (!(c.log_flags & NX_LOG_LEARNER) || failed(c)) return;
  const int32_t k = c.rs->ls_w[e];
  if (k >= c.d->learn_log_cap) {
    fail(c, 1, NX_SITE_OVERFLOW, 4);
    return;
  }
  __syncwarp();
  if (c.lane == 0) {
    const EngSm& g = c.eng[e];
    NxLearnLog& L = c.P->learn_stage[c.d->learn_log_off * c.P->slot_engines + e * c.d->learn_log_cap + k];
    L.t_us = now_us;
    L.samples = g.seen;
    L.engine_id = c.ed[e].engine_id;
    L.pad_ = 0;
    params_to(g.lp, L.params);
    c.rs->ls_w[e] = k + 1;
  }
  __syncwarp();
}

// ---- event keys ------------------------------------------------------------------
__device__ __forceinline__ uint64_t vload64(const uint64_t& x) {
  return *reinterpret_cast<const volatile uint64_t*>(&x);
}
__device__ __forceinline__ void vstore64(uint64_t& x, uint64_t v) {
  *reinterpret_cast<volatile uint64_t*>(&x) = v;
}
__device__ __forceinline__ uint32_t vloadu(const uint32_t& x) {
  return *reinterpret_cast<const volatile uint32_t*>(&x);
}

// CTA barrier reached from different code locations (the engine warps' park
// and the router's release): the non-.aligned form — __syncthreads() is
// barrier.sync.aligned, which requires every thread at the same instruction.
__device__ __forceinline__ void cta_barrier() { asm volatile("barrier.sync 0;" ::: "memory"); }

// Spin-wait watchdog: a warp that sees no progress from the others for
// 60 s is stuck on a protocol bug; trap (the launch fails with an error)
// instead of hanging the device.
__device__ unsigned long long* g_nx_dbg = nullptr;  // host-mapped dump (NX_DEBUG=1)
__device__ NX_COLD void dump_and_trap(const Ctx& c, int site) {
  unsigned long long* d = g_nx_dbg;
  if (d && atomicCAS(d, 0ull, 1ull) == 0ull) {
    const RepSm& R = *c.rs;
    d[1] = site; d[2] = threadIdx.x >> 5; d[3] = blockIdx.x;
    d[4] = R.horizon; d[5] = R.next_arr; d[6] = R.final_mode; d[7] = R.parked;
    d[8] = R.n_done; d[9] = R.n_fin; d[10] = R.kd_ready; d[11] = R.cursor; d[12] = R.am; d[13] = c.n_eng;
    d[14] = R.stop; d[15] = R.kd_inf;
    for (int e = 0; e < c.n_eng && e < 8; ++e) {
      const EngSm& g = c.eng[e];
      unsigned long long* q = d + 16 + 10 * e;
      q[0] = R.front[e]; q[1] = R.wpos[e]; q[2] = R.mpos[e]; q[3] = g.step_t; q[4] = g.report_t;
      q[5] = g.learn_t; q[6] = g.dq_t0; q[7] = R.done[e] | (R.fin[e] << 8) | (g.busy << 16);
      q[8] = g.log_n; q[9] = g.wq_len | (static_cast<unsigned long long>(g.rq_len) << 32);
    }
    __threadfence_system();
  }
  __trap();
}
__device__ __forceinline__ void spin_guard(const Ctx& c, long long t0, int site) {
  if (nx_globaltimer() - t0 > 20000000000ll) dump_and_trap(c, site);
}

struct EvKey {
  uint64_t t;
  uint32_t par;
  int kind, eng;
};

// Push order among one parent's children (sim.cpp:196-243): a step completion
// pushes its learner update, then the next step; a state report its delivery,
// then the next report; an arrival pushes one step.
__device__ __forceinline__ int child_of(int kind, uint32_t par) {
  return (kind == kEvReport || (kind == kEvStep && !(par & kRootPar))) ? 1 : 0;
}

// Ring-window error raised from single-lane code (no warp synchronisation).
__device__ __forceinline__ void raise_async(const Ctx& c, int site, int64_t info) {
  if (c.err->status == 0) {
    c.err->status = 3;
    c.err->site = site;
    c.err->info = 1000000 + info;
  }
}

__device__ EvKey parent_of(const Ctx& c, const EvKey& k) {
  EvKey p;
  p.eng = k.eng;
  if (k.par & kRootPar) {
    const uint32_t seq = k.par & kSeqMask;
    const bool rep = seq < static_cast<uint32_t>(c.n_eng);
    p.t = rep ? 0ull : static_cast<uint64_t>(c.P->arr_us[c.roff + (seq - c.n_eng)]);
    p.par = kSelfRoot | seq;
    p.kind = rep ? kEvReport : kEvArrival;
  } else {
    const uint32_t cap = static_cast<uint32_t>(NX_EVLOG_CAP);
    if (vloadu(c.rs->wpos[k.eng]) - k.par > cap - 2 * kRing) raise_async(c, NX_SITE_OVERFLOW, k.par);
    const NxEvLog L = c.elog[static_cast<int64_t>(k.eng) * cap + (k.par & (cap - 1))];
    p.t = static_cast<uint64_t>(L.t);
    p.par = L.par;
    p.kind = static_cast<int>(L.meta & 7u);
  }
  return p;
}

// Strict (time_us, sequence) order of two distinct events (sim.cpp:50-55):
// equal times are ordered like their parents were processed, then by push
// order — the sequence numbers' own definition (sim.cpp:67-70).
//
// State reports form one arithmetic chain per engine — report(e) at k·P_e,
// each pushed by the previous one, the first a root with seq e (sim.cpp:
// 236-242, 276-283) — and every engine's chain starts at 0, so equal-time
// reports of two engines are the common case; walking their parents would
// go all the way back to time 0. Closed form: with equal periods every
// ancestor pair ties and the roots decide (engine order); otherwise the
// parents' times k·P_e - P_e and k·P_f - P_f differ (larger period first).
__device__ bool ev_less(const Ctx& c, EvKey a, EvKey b) {
  if (a.t != b.t) return a.t < b.t;
  while (true) {
    if (a.kind == kEvReport && b.kind == kEvReport && a.eng != b.eng) {
      const int64_t pa = c.eng[a.eng].period_us, pb = c.eng[b.eng].period_us;
      if (a.t == 0 || pa == pb) return a.eng < b.eng;
      return pa > pb;
    }
    const bool ra = (a.par & kSelfRoot) != 0, rb = (b.par & kSelfRoot) != 0;
    if (ra || rb) return (ra && rb) ? (a.par & kSeqMask) < (b.par & kSeqMask) : ra;
    if (a.par == b.par && ((a.par & kRootPar) || a.eng == b.eng))
      return child_of(a.kind, a.par) < child_of(b.kind, b.par);
    a = parent_of(c, a);
    b = parent_of(c, b);
    if (a.t != b.t) return a.t < b.t;
  }
}

// The engine's next pending event (every lane computes the same).
__device__ EvKey next_event(const Ctx& c, int e) {
  const EngSm& g = c.eng[e];
  EvKey k;
  k.t = kNoEvent;
  k.par = 0;
  k.kind = -1;
  k.eng = e;
  auto take = [&](uint64_t t, uint32_t par, int kind) {
    if (t == kNoEvent) return;
    EvKey x;
    x.t = t;
    x.par = par;
    x.kind = kind;
    x.eng = e;
    if (t < k.t || (t == k.t && ev_less(c, x, k))) k = x;
  };
  take(g.step_t, g.step_seq, kEvStep);
  take(g.report_t, g.report_seq, kEvReport);
  take(g.learn_t, g.learn_seq, kEvLearn);
  take(g.dq_t0, g.dq_s0, kEvDeliver);
  return k;
}

__device__ __forceinline__ void note_error_key(Ctx& c, const EvKey& k) {
  __syncwarp();
  if (c.lane == 0 && c.err->status != 0 && c.err->kind < 0) {
    c.err->t = k.t;
    c.err->par = k.par;
    c.err->kind = k.kind;
    c.err->eng = k.eng;
  }
  __syncwarp();
}

// ---- engine warps ----------------------------------------------------------------
// One engine event: consume its slot, run the handler, log it for the merger.
__device__ NX_COLD void handle_engine_event(Ctx& c, int e, const EvKey& k) {
  EngSm& g = c.eng[e];
  const int64_t now = static_cast<int64_t>(k.t);
  int64_t dq_o = 0;  // the delivered report's slot
  if (k.kind == kEvDeliver) dq_o = c.ed[e].dq_off + g.dq_head;
  __syncwarp();
  if (c.lane == 0) {
    if (k.kind == kEvStep) g.step_t = kNoEvent;
    else if (k.kind == kEvReport) g.report_t = kNoEvent;
    else if (k.kind == kEvLearn) g.learn_t = kNoEvent;
    else {
      g.dq_head = ring_add(g.dq_head, 1, c.ed[e].dq_cap);
      g.dq_len -= 1;
      if (g.dq_len > 0) {
        const int64_t o = c.ed[e].dq_off + g.dq_head;
        g.dq_t0 = static_cast<uint64_t>(c.P->dq_t[o]);
        g.dq_s0 = c.P->dq_seq[o];
      } else {
        g.dq_t0 = kNoEvent;
      }
    }
  }
  __syncwarp();
  switch (k.kind) {
    case kEvStep:
      step_complete(c, e, now);
      break;
    case kEvReport: {
      PhaseTimer pt(c.rs, kTmReport);
      state_report(c, e, now);
      break;
    }
    case kEvLearn: {
      PhaseTimer pt(c.rs, kTmLearn);
      record_sample(c, e, g.learn_b, g.learn_s, g.learn_y);
      log_learner(c, e, now);
      break;
    }
    default: {  // report delivery -> Router::on_report (router.cpp:75-81)
      __syncwarp();
      if (c.lane == 0) {
        g.has_rep = 1;
        const double* dv = c.P->dq_sv + 5 * dq_o;
        g.rep_lhat = dv[0];
        g.rep_wload = dv[1];
        g.rep_mfree = dv[2];
        g.rep_pmax = dv[3];
        g.rep_at = dv[4];
        g.rep_qlen = c.P->dq_qlen[dq_o];
      }
      __syncwarp();
      break;
    }
  }
}

__device__ __forceinline__ bool engine_idle(const EngSm& g) {
  return g.wq_len == 0 && g.rq_len == 0 && !g.busy;
}

// No completion of engine e follows (final phase): inf = it stopped at the
// duration with requests still active.
__device__ void mark_done(Ctx& c, int e, bool inf) {
  __syncwarp();
  if (c.lane == 0 && !c.rs->done[e]) {
    c.rs->done[e] = inf ? 2 : 1;
    __threadfence_block();
    atomicAdd(&c.rs->n_done, 1);
  }
  __syncwarp();
}
__device__ void finish_engine(Ctx& c, int e) {
  mark_done(c, e, !engine_idle(c.eng[e]));
  __syncwarp();
  if (c.lane == 0 && !c.rs->fin[e]) {
    c.rs->fin[e] = 1;
    vstore64(c.rs->front[e], kNoEvent);
    __threadfence_block();
    atomicAdd(&c.rs->n_fin, 1);
  }
  __syncwarp();
}

enum { kParked = 0, kFinished = 1, kNeedDrain = 2, kBlocked = 3 };


// Final phase, engine e idle and its next event the state report k: the
// reference drops it iff no arrival is pending and no request is active
// anywhere at k (sim.cpp:295-300). Every arrival has been processed, so it
// is kept iff some engine still completes a request after k: one that
// stopped at the duration with requests active (done 2), one whose last
// completion follows k (done 1), or one still active whose front lies past
// k (its remaining completions come later). An active engine at or behind
// k leaves the decision open (-1): it is not blocked by this engine (its
// front is the lower one), so waiting cannot deadlock.
__device__ int drain_decide(const Ctx& c, const EvKey& k) {
  const RepSm& R = *c.rs;
  if (vload(R.kd_inf)) return 1;
  bool open = false;
  for (int f = 0; f < c.n_eng; ++f) {
    if (f == k.eng) continue;
    const uint64_t fr = vload64(R.front[f]);
    __threadfence_block();
    const int d = vload(R.done[f]);
    if (d == 2) return 1;
    if (d == 1) {
      const EngSm& g = c.eng[f];
      if (g.last_fin_t == kNoEvent) continue;
      EvKey kf;
      kf.t = g.last_fin_t;
      kf.par = g.last_fin_par;
      kf.kind = kEvStep;
      kf.eng = f;
      if (ev_less(c, k, kf)) return 1;
      continue;
    }
    if (fr > k.t) return 1;  // active with its front past k: it completes later
    open = true;
  }
  return open ? -1 : 0;
}

// Runs engine e's events in key order: before the arrival window's end
// (horizon) in the arrival phase; up to the duration in the final phase,
// where a state report is dropped once no request is pending or active
// (sim.cpp:295-300) — i.e. once its key passes the drain key.
__device__ __forceinline__ int advance(Ctx& c, int e, bool fm) {
  EngSm& g = c.eng[e];
  RepSm& R = *c.rs;
  const uint64_t H = R.horizon;
  const uint64_t duration = static_cast<uint64_t>(c.d->duration_us);
  const uint32_t cap = static_cast<uint32_t>(NX_EVLOG_CAP);
  while (true) {
    if (failed(c)) {
      if (fm) finish_engine(c, e);
      return fm ? kFinished : kParked;
    }
    if (fm && !vload(R.done[e]) && engine_idle(g)) mark_done(c, e, false);
    const EvKey k = next_event(c, e);
    if (c.lane == 0) vstore64(R.front[e], k.t);
    if (!fm) {
      if (k.t == kNoEvent || !(k.t < H || (k.t == H && (k.par & kSelfRoot)))) return kParked;
    } else {
      if (k.t == kNoEvent || k.t > duration) {
        finish_engine(c, e);
        return kFinished;
      }
      if (k.kind == kEvReport && vload(R.done[e]) == 1) {
        const int keep = drain_decide(c, k);
        if (keep < 0) return kNeedDrain;
        if (keep == 0) {  // dropped: nothing pending or active
          put(g.report_t, kNoEvent);
          continue;
        }
      }
    }
    const uint32_t idx = g.log_n;
    // the merger's shared-memory window of this engine's log must have room;
    // if not, yield to this warp's other engines (the merger may be waiting
    // on one of them)
    if (idx - vloadu(R.mpos[e]) >= static_cast<uint32_t>(kRing)) return kBlocked;
    c.cur_ref = idx;
    c.cur_meta = 0;
    c.began = 0;
    {
      PhaseTimer pt(c.rs, kTmEvents);
      handle_engine_event(c, e, k);
    }
    __syncwarp();
    if (c.lane == 0) {
      NxEvLog L;
      L.t = static_cast<int64_t>(k.t);
      L.par = k.par;
      L.meta = static_cast<uint32_t>(k.kind) | c.cur_meta;
      c.elog[static_cast<int64_t>(e) * cap + (idx & (cap - 1))] = L;
      c.sring[e * kRing + (idx & (kRing - 1))] = L;
      g.log_n = idx + 1;
      if (k.kind == kEvStep && (c.cur_meta >> kMetaFinShift) != 0) {
        g.last_fin_t = k.t;
        g.last_fin_par = k.par;
      }
      __threadfence_block();
      *reinterpret_cast<volatile uint32_t*>(&R.wpos[e]) = idx + 1;
    }
    __syncwarp();
    if (failed(c)) note_error_key(c, k);
  }
}

__device__ NX_COLD void engine_warp(Ctx& c, int w, int n_ew) {
  RepSm& R = *c.rs;
  long long t0 = nx_globaltimer();
  bool fm = vload(R.final_mode) != 0;
  while (true) {
    // One call site of advance (inlined). Passes over this warp's engines
    // until each has reached the window's horizon (arrival phase) or finished
    // (final phase); an engine that is blocked (log window full) or waiting
    // on a drain decision is retried after its warp-mates have run.
    bool done = true, progress = false;
    for (int e = w; e < c.n_eng; e += n_ew) {
      if (fm && vload(R.fin[e])) continue;
      const uint32_t before = c.eng[e].log_n;
      const int r = advance(c, e, fm);
      if (r == kBlocked || r == kNeedDrain) done = false;
      if (c.eng[e].log_n != before || r == kFinished) progress = true;
    }
    if (progress) t0 = nx_globaltimer();
    if (!done) {
      if (!progress) {
        PhaseTimer pt(c.rs, kTmRing);
        spin_guard(c, t0, __LINE__);
        __nanosleep(64);
      }
      continue;
    }
    if (fm) return;
    {
      PhaseTimer pt(c.rs, kTmPark);
      if (c.lane == 0) {
        __threadfence_block();
        atomicAdd(&R.parked, 1);
      }
      cta_barrier();  // released by the router once the window's arrivals are routed
    }
    if (vload(R.stop)) return;
    fm = vload(R.final_mode) != 0;
  }
}

// ---- router warp: merger, arrivals -----------------------------------------------
// Emits logged events in key order below the fronts: the FNV event hash
// (sim.cpp:302-305), records + Router::on_completion's l_bar EMA and session
// memory (router.cpp:83-92) in completion order, observability rows. Lane e
// holds the head of engine e's log, lane 31 the arrivals' (engines <= 31);
// the next event is a warp-wide time minimum (ties: ev_less), lane 0 folds it.
constexpr int kArrLane = 31;

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = __reduce_min_sync(NX_FULL, static_cast<uint32_t>(v >> 32));
  const uint32_t lo = __reduce_min_sync(NX_FULL, static_cast<uint32_t>(v >> 32) == hi ? static_cast<uint32_t>(v)
                                                                                      : 0xffffffffu);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ NX_COLD int merge_some(Ctx& c, int budget) {
  PhaseTimer pt(c.rs, kTmMerge);
  RepSm& R = *c.rs;
  const NxPools& P = *c.P;
  const int E = c.n_eng, lane = c.lane;
  const bool eng_lane = lane < E;
  uint64_t f = eng_lane ? vload64(R.front[lane]) : kNoEvent;
  if (lane == kArrLane) f = R.next_arr;
  const uint64_t F = warp_min_u64(f);
  __threadfence_block();
  const uint32_t lim = eng_lane ? vloadu(R.wpos[lane]) : 0u;
  __threadfence_block();
  uint32_t m = eng_lane ? R.mpos[lane] : 0u;
  int am = R.am;
  const int cursor = R.cursor;
  uint64_t ht = kNoEvent;  // this lane's head
  uint32_t hp = 0, hm = 0;
  auto load_head = [&]() {
    ht = kNoEvent;
    if (eng_lane) {
      if (m != lim) {
        const NxEvLog L = c.sring[lane * kRing + (m & (kRing - 1))];
        ht = static_cast<uint64_t>(L.t);
        hp = L.par;
        hm = L.meta;
      }
    } else if (lane == kArrLane && am < cursor) {
      ht = static_cast<uint64_t>(P.arr_us[c.roff + am]);
      hp = kSelfRoot | static_cast<uint32_t>(E + am);
      hm = kEvArrival;
    }
  };
  load_head();
  int n = 0;
  while (n < budget) {
    const bool valid = ht < F;
    const uint64_t tmin = warp_min_u64(valid ? ht : kNoEvent);
    if (tmin == kNoEvent) break;
    const unsigned cand = __ballot_sync(NX_FULL, valid && ht == tmin);
    int w = __ffs(cand) - 1;
    if (cand & (cand - 1)) {  // equal times: the (time, sequence) order decides
      EvKey best;
      best.t = tmin;
      best.par = __shfl_sync(NX_FULL, hp, w);
      best.kind = static_cast<int>(__shfl_sync(NX_FULL, hm, w) & 7u);
      best.eng = w == kArrLane ? 0 : w;
      unsigned rest = cand & (cand - 1);
      while (rest) {
        const int o = __ffs(rest) - 1;
        rest &= rest - 1;
        EvKey k;
        k.t = tmin;
        k.par = __shfl_sync(NX_FULL, hp, o);
        k.kind = static_cast<int>(__shfl_sync(NX_FULL, hm, o) & 7u);
        k.eng = o == kArrLane ? 0 : o;
        if (ev_less(c, k, best)) {
          best = k;
          w = o;
        }
      }
    }
    const uint32_t wm = __shfl_sync(NX_FULL, hm, w);
    ++n;
    if (lane == 0) {
      R.events += 1;
      const int kind = static_cast<int>(wm & 7u);
      if (w == kArrLane) {  // arrival
        const int rid = am;  // every lane tracks the arrivals cursor
        R.ev_hash = fnv_event(R.ev_hash, tmin, 0ull, 0ull, static_cast<uint64_t>(rid));
        if ((c.log_flags & NX_LOG_PLANS) && P.began[c.roff + rid]) {
          const int e = P.req_engine[c.roff + rid];
          const int64_t k = R.n_plan_log;
          if (k < c.d->plan_log_cap) {
            P.plan_log[c.d->plan_log_off + k] =
                P.plan_stage[c.d->plan_log_off * P.slot_engines + e * c.d->plan_log_cap + R.ps_r[e]];
            R.n_plan_log = k + 1;
          }
          R.ps_r[e] += 1;
        }
      } else {
        const int e = w;
        const EngSm& g = c.eng[e];
        R.ev_hash = fnv_event(R.ev_hash, tmin, static_cast<uint64_t>(kind), static_cast<uint64_t>(g.eid1), 0ull);
        if (kind == kEvStep) {
          const int nf = static_cast<int>(wm >> kMetaFinShift);
          if (nf) {
            const int4* ob = reinterpret_cast<const int4*>(c.obox) + static_cast<int64_t>(e) * c.ob_cap;
            const int r0 = R.ob_r[e];
            double lb = R.l_bar_ema;
            int64_t nr = R.n_rec;
            for (int j = 0; j < nf; ++j) {
              const int4 o = ob[r0 + j];
              P.records[c.roff + nr] = o.x;
              ++nr;
              const double le = lb + 0.05 * (static_cast<double>(o.z) - lb);
              lb = le < 1.0 ? 1.0 : le;
              P.sess_engine[c.soff + o.y] = e;
            }
            R.n_rec = nr;
            R.l_bar_ema = lb;
            R.ob_r[e] = r0 + nf;
          }
        }
        if (wm & kMetaPlan) {
          const int64_t k = R.n_plan_log;
          if (k < c.d->plan_log_cap) {
            P.plan_log[c.d->plan_log_off + k] =
                P.plan_stage[c.d->plan_log_off * P.slot_engines + e * c.d->plan_log_cap + R.ps_r[e]];
            R.n_plan_log = k + 1;
          }
          R.ps_r[e] += 1;
        }
        if (kind == kEvLearn && (c.log_flags & NX_LOG_LEARNER)) {
          const int64_t k = R.n_learn_log;
          if (k < c.d->learn_log_cap) {
            P.learn_log[c.d->learn_log_off + k] =
                P.learn_stage[c.d->learn_log_off * P.slot_engines + e * c.d->learn_log_cap + R.ls_r[e]];
            R.n_learn_log = k + 1;
          }
          R.ls_r[e] += 1;
        }
      }
    }
    if (w == kArrLane) {
      ++am;
    } else if (lane == w) {
      ++m;
      *reinterpret_cast<volatile uint32_t*>(&R.mpos[lane]) = m;  // frees the engine's ring slot
    }
    if (lane == w) load_head();
  }
  __syncwarp();
  if (lane == 0) {
    R.am = am;
    if (nx_timers_on) {
      R.lcycles[0] += 1;
      R.lcycles[1] += n;
      if (n == 0) R.lcycles[2] += 1;
    }
  }
  __syncwarp();
  return n;
}

// Every logged event and routed arrival merged (lane 0's view, broadcast).
__device__ bool merge_drained(Ctx& c) {
  bool all = true;
  if (c.lane == 0) {
    RepSm& R = *c.rs;
    for (int e = 0; e < c.n_eng; ++e) all &= R.mpos[e] == vloadu(R.wpos[e]);
    all &= R.am == R.cursor;
  }
  return __shfl_sync(NX_FULL, all ? 1 : 0, 0) != 0;
}

// The drain key (lane 0): state reports are dropped once no arrival is
// pending and no request is active — after the later of the last arrival and
// the last completion (sim.cpp:295-300).
__device__ void compute_drain(Ctx& c) {
  RepSm& R = *c.rs;
  if (c.lane == 0 && !R.kd_ready) {
    __threadfence_block();
    EvKey kd;
    kd.kind = -1;
    kd.t = 0;
    kd.par = 0;
    kd.eng = 0;
    if (c.n_req > 0) {
      kd.t = static_cast<uint64_t>(c.P->arr_us[c.roff + c.n_req - 1]);
      kd.par = kSelfRoot | static_cast<uint32_t>(c.n_eng + c.n_req - 1);
      kd.kind = kEvArrival;
    }
    bool inf = false;
    for (int e = 0; e < c.n_eng; ++e) {
      if (R.done[e] == 2) inf = true;
      const EngSm& g = c.eng[e];
      if (g.last_fin_t == kNoEvent) continue;
      EvKey k;
      k.t = g.last_fin_t;
      k.par = g.last_fin_par;
      k.kind = kEvStep;
      k.eng = e;
      if (kd.kind < 0 || ev_less(c, kd, k)) kd = k;
    }
    R.kd_t = kd.t;
    R.kd_par = kd.par;
    R.kd_kind = kd.kind;
    R.kd_eng = kd.eng;
    R.kd_inf = inf ? 1 : 0;
    __threadfence_block();
    vstore(R.kd_ready, 1);
  }
  __syncwarp();
}

// After the last arrival (or the first past the duration): no more windows.
__device__ void enter_final(Ctx& c) {
  RepSm& R = *c.rs;
  if (c.lane == 0) {
    R.final_mode = 1;
    R.next_arr = kNoEvent;
    R.all_arrived = R.pending == 0;
    if (R.pending > 0) {  // arrivals cut off by the duration stay pending: nothing is dropped
      R.kd_inf = 1;
      R.kd_ready = 1;
    }
  }
  __syncwarp();
}

// Arrivals at the window's end, in order (sim.cpp:168-194); engines are parked
// with every earlier event processed.
__device__ NX_COLD void route_arrivals(Ctx& c) {
  PhaseTimer pt(c.rs, kTmRoute);
  RepSm& R = *c.rs;
  const uint64_t t = R.horizon;
  const int64_t now = static_cast<int64_t>(t);
  while (R.cursor < c.n_req && static_cast<uint64_t>(c.P->arr_us[c.roff + R.cursor]) == t) {
    const int rid = R.cursor;
    __syncwarp();
    if (c.lane == 0) {
      R.cursor = rid + 1;
      R.arrived += 1;
      R.pending -= 1;
    }
    __syncwarp();
    c.cur_ref = kRootPar | static_cast<uint32_t>(c.n_eng + rid);
    c.cur_meta = 0;
    c.began = 0;
    EvKey ak;
    ak.t = t;
    ak.par = kSelfRoot | static_cast<uint32_t>(c.n_eng + rid);
    ak.kind = kEvArrival;
    ak.eng = 0;
    double score = 0.0, fac[4] = {1.0, 1.0, 1.0, 1.0};
    const int e = route(c, rid, to_ms(now), score, fac);
    if (c.lane == 0 && (c.log_flags & NX_LOG_ROUTES)) {  // routing_jsonl row (sim.cpp:176-186)
      NxRouteLog& L = c.P->route_log[c.d->route_log_off + R.n_route_log];
      L.t_us = now;
      L.request = rid;
      L.engine_id = c.ed[e].engine_id;
      L.score = score;
      for (int i = 0; i < 4; ++i) L.factors[i] = fac[i];
      R.n_route_log += 1;
    }
    if (failed(c)) {
      note_error_key(c, ak);
      return;
    }
    int ok = 0;
    if (c.lane == 0) {
      ok = admit(c, e, rid) ? 1 : 0;
      if (!ok) R.rejected += 1;
    }
    ok = __shfl_sync(NX_FULL, ok, 0);
    __syncwarp();
    if (ok) {
      try_begin_step(c, e, now);
      if (failed(c)) {
        note_error_key(c, ak);
        return;
      }
      __syncwarp();
      if (c.lane == 0) {
        if (c.began) c.P->began[c.roff + rid] = 1;
        const uint64_t st = c.eng[e].step_t;
        if (st < R.front[e]) vstore64(R.front[e], st);
      }
      __syncwarp();
    }
  }
  __syncwarp();
  const uint64_t nx = R.cursor < c.n_req ? static_cast<uint64_t>(c.P->arr_us[c.roff + R.cursor]) : kNoEvent;
  if (nx == kNoEvent || nx > static_cast<uint64_t>(c.d->duration_us)) {
    enter_final(c);
  } else if (c.lane == 0) {
    R.horizon = nx;
    R.next_arr = nx;
  }
  __syncwarp();
}

__device__ NX_COLD void router_warp(Ctx& c, int n_ew) {
  RepSm& R = *c.rs;
  const long long tw0 = nx_clock();
  while (!vload(R.final_mode)) {
    if (nx_timers_on && c.lane == 0) R.cycles[kTmNWindows] += 1;
    const long long twin = nx_clock();
    // merge behind the engines until every engine warp has parked
    long long t0 = nx_globaltimer();
    while (true) {
      const int n = merge_some(c, 32);
      if (vload(R.parked) == n_ew) break;
      if (n == 0) {
        PhaseTimer pt(c.rs, kTmRouterIdle);
        spin_guard(c, t0, __LINE__);
        __nanosleep(32);
      } else {
        t0 = nx_globaltimer();
      }
    }
    __threadfence_block();
    if (nx_timers_on && c.lane == 0) {  // window wall, and how much of it had a structural refit
      const long long dt = nx_clock() - twin;
      R.lcycles[6] += dt;
      if (R.lcycles[3]) {
        R.lcycles[4] += dt;
        R.lcycles[5] += 1;
        R.lcycles[3] = 0;
      }
    }
    {
      const long long tc = nx_clock();
      while (merge_some(c, 1 << 30) > 0) {
      }
      if (nx_timers_on && c.lane == 0) R.lcycles[7] += nx_clock() - tc;  // merge catch-up at the barrier
    }
    bool err = false;
    for (int w = 1; w <= n_ew; ++w) err |= R.err[w].status != 0;
    __syncwarp();
    if (c.lane == 0) R.parked = 0;
    if (err) {
      put(R.stop, 1);
    } else {
      route_arrivals(c);
      if (failed(c)) put(R.stop, 1);
    }
    __syncwarp();
    cta_barrier();  // release the engines into the next window
    if (vload(R.stop)) return;
  }
  const long long tf0 = nx_clock();
  if (nx_timers_on && c.lane == 0) R.cycles[kTmWindows] += tf0 - tw0;
  long long t0 = nx_globaltimer();
  while (true) {
    const int n = merge_some(c, 64);
    if (n > 0) t0 = nx_globaltimer();
    if (n == 0) {
      if (vload(R.n_fin) == c.n_eng) {
        __threadfence_block();
        if (merge_drained(c)) {
          if (nx_timers_on && c.lane == 0) R.cycles[kTmFinal] += nx_clock() - tf0;
          break;
        }
      } else {
        spin_guard(c, t0, __LINE__);
        __nanosleep(64);
      }
    }
  }
}

// ---- replica driver -------------------------------------------------------------
__device__ NX_COLD void init_replica(Ctx& c, int n_warps) {
  const NxReplicaDesc& d = *c.d;
  for (int e = c.lane; e < c.n_eng; e += 32) {
    EngSm& g = c.eng[e];
    const NxEngineDesc& ed = c.ed[e];
    // OnlineLearner::default_priors (learner.cpp:117-128)
    g.lp.p_max = 20.0; g.lp.kB = 0.1; g.lp.kS = 0.02; g.lp.tau0 = 5.0;
    g.lp.w0 = 0.0; g.lp.ws = 1.0; g.lp.tauB = 0.1; g.lp.tauS = 0.001;
    g.alpha = d.alpha; g.beta = d.beta; g.l_bar = d.l_bar; g.td_min = d.td_min;
    g.plan_pred = 0.0; g.plan_target = 0.0; g.actual = 0.0; g.learn_y = 0.0; g.lat_sum = 0.0;
    g.rep_lhat = 0.0; g.rep_wload = 0.0; g.rep_mfree = 0.0; g.rep_pmax = 1.0; g.rep_at = 0.0;
    for (int i = 0; i < 4; ++i) g.rng[i] = ed.rng[i];
    g.step_t = kNoEvent; g.learn_t = kNoEvent;
    g.report_t = 0; g.report_seq = kSelfRoot | static_cast<uint32_t>(e);  // initial reports: seq 0..E-1
    g.step_seq = 0; g.learn_seq = 0;
    g.started_us = 0; g.seen = 0; g.rep_qlen = 0; g.tw_degen = 0;
    g.lin_left = d.l_period; g.str_left = d.s_period;
    for (int i = 0; i < 7; ++i) g.cnt[i] = 0;
    g.wq_head = 0; g.wq_len = 0; g.rq_len = 0;
    g.pinned = 0; g.reserved = 0; g.cache_blocks = 0; g.lru_head = -1; g.lru_tail = -1;
    g.busy = 0; g.plan_n = 0; g.plan_b = 0; g.plan_s = 0; g.plan_wspan = 0; g.plan_overload = 0; g.plan_ndec = 0;
    g.learn_b = 0; g.learn_s = 0;
    g.ring_size = 0; g.ring_head = 0; g.tw_head = 0; g.tw_len = 0;
    g.dq_head = 0; g.dq_len = 0; g.lat_head = 0; g.lat_len = 0; g.has_rep = 0;
    g.dq_t0 = kNoEvent; g.dq_s0 = 0; g.noise_pos = 32; g.refit_pending = 0;
    g.lp_ver = 0; g.memo_ver = -1; g.memo_b = -1; g.memo_tb = -1; g.memo_pred = 0.0; g.memo_truth = 0.0;
    g.log_n = 0; g.last_fin_t = kNoEvent; g.last_fin_par = 0;
    g.period_us = ed.period_us; g.eid1 = ed.engine_id + 1;
    RepSm& R = *c.rs;
    R.front[e] = 0;  // the initial state report
    R.wpos[e] = 0; R.mpos[e] = 0;
    R.ob_w[e] = 0; R.ob_r[e] = 0; R.ps_w[e] = 0; R.ps_r[e] = 0; R.ls_w[e] = 0; R.ls_r[e] = 0;
    R.done[e] = 0; R.fin[e] = 0;
  }
  for (int w = c.lane; w < n_warps; w += 32) {
    ErrSlot& s = c.rs->err[w];
    s.status = 0; s.site = 0; s.info = 0; s.t = 0; s.par = 0; s.kind = -1; s.eng = 0;
  }
  if (c.lane == 0) {
    RepSm& R = *c.rs;
    R.ev_hash = 0xcbf29ce484222325ULL;
    R.rr_next = 0;
    for (int i = 0; i < 4; ++i) R.rng[i] = d.router_rng[i];
    R.arrived = 0; R.rejected = 0; R.pending = c.n_req; R.n_rec = 0; R.events = 0; R.info = 0;
    for (int i = 0; i < 6; ++i) R.work[i] = 0;
    for (int i = 0; i < 16; ++i) R.cycles[i] = 0;
    R.t_begin_ns = nx_globaltimer();
    R.n_plan_log = 0;
    R.n_route_log = 0;
    R.n_learn_log = 0;
    R.jq_head = 0;
    R.jq_tail = 0;
    R.l_bar_ema = 128.0;
    R.next_seq = 0;
    R.cursor = 0; R.status = 0; R.site = 0;
    R.final_mode = 0; R.stop = 0; R.parked = 0; R.n_done = 0; R.n_fin = 0; R.all_arrived = 0;
    R.kd_ready = 0; R.kd_inf = 0; R.kd_t = 0; R.kd_par = 0; R.kd_kind = -1; R.kd_eng = 0;
    R.am = 0; R.am_t = kNoEvent;
    const uint64_t a0 = c.n_req > 0 ? static_cast<uint64_t>(c.P->arr_us[c.roff]) : kNoEvent;
    R.next_arr = a0;
    R.horizon = a0;
  }
  __syncwarp();
  const uint64_t a0 = c.rs->next_arr;
  if (a0 == kNoEvent || a0 > static_cast<uint64_t>(c.d->duration_us)) enter_final(c);
  __syncwarp();
}

// The replica's first error in event order (every warp stops at its own first).
__device__ ErrSlot first_error(const Ctx& c, int n_warps) {
  ErrSlot best;
  best.status = 0;
  best.site = 0;
  best.info = 0;
  best.t = 0;
  best.par = 0;
  best.kind = -1;
  best.eng = 0;
  for (int w = 0; w < n_warps; ++w) {
    const ErrSlot& s = c.rs->err[w];
    if (s.status == 0) continue;
    bool take = best.status == 0;
    if (!take && s.kind >= 0 && best.kind >= 0) {
      EvKey a, b;
      a.t = s.t; a.par = s.par; a.kind = s.kind; a.eng = s.eng;
      b.t = best.t; b.par = best.par; b.kind = best.kind; b.eng = best.eng;
      take = ev_less(c, a, b);
    }
    if (take) best = s;
  }
  return best;
}

__device__ NX_COLD void write_outputs(Ctx& c, int r, int n_warps) {
  __syncwarp();
  NxReplicaOut& o = c.P->rep_out[r];
  if (c.lane == 0) {
    const RepSm& R = *c.rs;
    const ErrSlot err = first_error(c, n_warps);
    o.arrived = R.arrived;
    o.rejected = R.rejected;
    o.completed = R.n_rec;
    o.pending = R.pending;
    o.events = R.events;
    o.event_hash = R.ev_hash;
    o.status = err.status;
    o.err_site = err.site;
    o.err_info = err.info;
    for (int i = 0; i < 6; ++i) o.work[i] = R.work[i];
    for (int i = 0; i < 16; ++i) o.cycles[i] = R.cycles[i];
    if (nx_timers_on == 2)  // window counters instead of the phase-wall slots
      for (int i = 0; i < 4; ++i) o.cycles[12 + i] = R.lcycles[4 + i];
    if (nx_timers_on == 3)  // learner-internal timers in slots 8..15
      for (int i = 8; i < 16; ++i) o.cycles[i] = R.lcycles[i == 8 ? 7 : i];
    o.t_begin_ns = R.t_begin_ns;
    o.n_plan_log = R.n_plan_log;
    o.n_route_log = R.n_route_log;
    o.n_learn_log = R.n_learn_log;
    o.t_end_ns = nx_globaltimer();
  }
  for (int e = c.lane; e < c.n_eng; e += 32) {
    const EngSm& g = c.eng[e];
    NxEngineOut& eo = c.P->eng_out[c.d->eng_base + e];
    params_to(g.lp, eo.params);
    eo.samples = g.seen;
    for (int i = 0; i < 7; ++i) eo.counters[i] = g.cnt[i];
    eo.tradeoff_degenerate = g.tw_degen;
    eo.alpha = g.alpha;
    eo.beta = g.beta;
    eo.l_bar = g.l_bar;
  }
  __syncwarp();
}

__host__ __device__ __forceinline__ size_t align16(size_t v) { return (v + 15) & ~size_t(15); }
__host__ __device__ __forceinline__ size_t stage_bytes(int prefix_cap) {
  return align16(static_cast<size_t>(prefix_cap) * 4 > 32 * 5 * 8 ? static_cast<size_t>(prefix_cap) * 4
                                                                  : 32 * 5 * 8);
}
// Shared memory of a replica CTA without the engine warps' fit tables.
__host__ __device__ __forceinline__ size_t sim_smem_base(int max_eng, int prefix_cap) {
  return align16(sizeof(RepSm)) + kPdMaxWarps * stage_bytes(prefix_cap) +
         align16(sizeof(EngSm) * static_cast<size_t>(max_eng)) +
         sizeof(NxEvLog) * kRing * static_cast<size_t>(max_eng);
}

}  // namespace nxd

// One CTA per replica: warp 0 is the router (arrivals, merger), warps
// 1..n_ew each own the engines e with e % n_ew == warp - 1. CTAs pull replica
// indices (host order, longest expected first) from a global counter.
extern "C" __global__ void __launch_bounds__(32 * NX_SIM_LB_WARPS, 1)
nx_sim_kernel(const NxPools* __restrict__ pools, const int32_t* __restrict__ order, int n_rep,
              int* ctl, int prefix_cap, int max_eng, int n_ew, int fsm_cap, int req_cap) {
  using namespace nxd;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_slot;
  const int warp = threadIdx.x >> 5;
  const int n_warps = 1 + n_ew;
  Ctx c;
  c.P = pools;
  c.lane = lane_id();
  c.worker = warp;
  size_t off = 0;
  c.rs = reinterpret_cast<RepSm*>(smem);
  off += align16(sizeof(RepSm));
  c.chunk = reinterpret_cast<double*>(smem + off + warp * stage_bytes(prefix_cap));
  c.prefix = reinterpret_cast<int32_t*>(c.chunk);
  off += kPdMaxWarps * stage_bytes(prefix_cap);
  c.eng = reinterpret_cast<EngSm*>(smem + off);
  off += align16(sizeof(EngSm) * static_cast<size_t>(max_eng));
  c.sring = reinterpret_cast<NxEvLog*>(smem + off);
  off += sizeof(NxEvLog) * kRing * static_cast<size_t>(max_eng);
  // request state (prefilled, decoded, prompt, target) + KV-admitted flags of
  // the replica in shared memory when it fits (req_cap requests), else in HBM
  NxReqState* sreq = reinterpret_cast<NxReqState*>(smem + off);
  off += sizeof(NxReqState) * static_cast<size_t>(req_cap);
  uint8_t* skva = smem + off;
  off += align16(static_cast<size_t>(req_cap));

  c.fsm = (warp > 0 && fsm_cap >= 0)
              ? reinterpret_cast<double*>(smem + off) + static_cast<size_t>(warp - 1) * (kFbTable + fsm_cap)
              : nullptr;
  c.fsm_cap = fsm_cap < 0 ? 0 : fsm_cap;
  c.team = 1;
  c.inline_refit = 1;
  c.prefix_cap = prefix_cap;
  c.err = &c.rs->err[warp];
  const int64_t slot_e = static_cast<int64_t>(blockIdx.x) * pools->slot_engines;
  c.elog = pools->evlog + slot_e * NX_EVLOG_CAP;
  c.obox = pools->outbox + slot_e * pools->outbox_cap * 4;
  c.ob_cap = pools->outbox_cap;
  const int64_t ws = static_cast<int64_t>(blockIdx.x) * pools->slot_warps + (warp > 0 ? warp - 1 : 0);
  c.scratch = pools->scratch + ws * pools->scratch_stride;
  c.cur_ref = 0;
  c.cur_meta = 0;
  c.began = 0;
  while (true) {
    if (threadIdx.x == 0) s_slot = atomicAdd(&ctl[0], 1);
    __syncthreads();
    const int slot = s_slot;
    __syncthreads();
    if (slot >= n_rep) break;
    const int r = order[slot];
    c.d = pools->rep + r;
    c.ed = pools->eng + c.d->eng_base;
    c.n_eng = c.d->n_eng;
    c.n_req = c.d->n_req;
    c.n_sess = c.d->n_sess;
    c.log_flags = c.d->log_flags;
    c.roff = c.d->req_off;
    c.soff = c.d->sess_off;
    c.lin_rows = c.scratch + 6 * c.d->long_w + kFbTable;
    if (c.n_req <= req_cap) {
      c.req = sreq;
      c.kva = skva;
      for (int i = threadIdx.x; i < c.n_req; i += blockDim.x) {
        sreq[i] = pools->req0[c.roff + i];
        skva[i] = 0;
      }
    } else {
      c.req = pools->req + c.roff;
      c.kva = pools->kv_admitted + c.roff;
    }
    if (warp == 0) init_replica(c, n_warps);
    __syncthreads();
    if (warp == 0) router_warp(c, n_ew);
    else engine_warp(c, warp - 1, n_ew);
    __syncthreads();
    if (warp == 0) write_outputs(c, r, n_warps);
    __syncthreads();
  }
}

// Shared memory of one replica CTA without fit tables (host uses the same
// formula for its device-limit checks).
extern "C" size_t nx_sim_smem_per_warp(int max_engines, int prefix_cap) {
  return nxd::sim_smem_base(max_engines, prefix_cap);
}
// Doubles of one engine warp's shared-memory fit tables for fsm_cap 1/f_S entries.
extern "C" size_t nx_sim_req_smem_bytes(int req_cap) {
  return sizeof(NxReqState) * static_cast<size_t>(req_cap) + nxd::align16(static_cast<size_t>(req_cap));
}
extern "C" size_t nx_sim_fit_table_doubles(int fsm_cap) {
  return static_cast<size_t>(nxd::kFbTable + fsm_cap);
}

extern "C" cudaError_t nx_launch_sim(const NxPools* d_pools, const int32_t* d_order, int n_rep,
                                     int* d_next, int prefix_cap, int max_eng, int n_ew, int fsm_cap,
                                     int req_cap, size_t smem, int grid, cudaStream_t st) {
#ifdef NX_TIMERS
  const char* tm = getenv("NX_PHASE_TIMERS");
  const int timers = tm ? (tm[0] >= '1' && tm[0] <= '3' ? tm[0] - '0' : 0) : 0;
  cudaError_t terr = cudaMemcpyToSymbolAsync(nxd::nx_timers_on, &timers, sizeof timers, 0,
                                             cudaMemcpyHostToDevice, st);
  if (terr != cudaSuccess) return terr;
#endif
  cudaError_t err = cudaFuncSetAttribute(nx_sim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  if (const char* cv = getenv("NX_CARVEOUT")) {  // shared-memory share of L1 (percent; A/B knob)
    err = cudaFuncSetAttribute(nx_sim_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
    if (err != cudaSuccess) return err;
  }
  nx_sim_kernel<<<grid, 32 * (1 + n_ew), smem, st>>>(d_pools, d_order, n_rep, d_next, prefix_cap, max_eng, n_ew,
                                                      fsm_cap, req_cap);
  return cudaGetLastError();
}

extern "C" cudaError_t nx_sim_set_debug(unsigned long long* dev_ptr) {
  return cudaMemcpyToSymbol(nxd::g_nx_dbg, &dev_ptr, sizeof dev_ptr);
}

extern "C" cudaError_t nx_sim_occupancy(int warps_per_block, size_t smem, int* blocks_per_sm) {
  // dynamic shared memory above 48 KB must be opted into before the query
  cudaError_t err = cudaFuncSetAttribute(nx_sim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, nx_sim_kernel,
                                                       32 * warps_per_block, smem);
}
