// K5 — batched lockstep discrete-event simulation, one warp per replica.
//
// Each warp runs one servesim::Simulation (proj/src/sim.cpp:245-347) to
// completion. The reference's std::priority_queue<SimEvent> is replaced by
// per-engine event slots (step completion, learner update, state report,
// report-delivery FIFO head) plus an arrival cursor; the next event is a
// warp-wide (time_us, sequence) minimum, so the processing order — and hence
// the FNV event hash — equals the reference's. Inside an event the warp's
// lanes parallelise over engines (K3 PRISM scorer), candidate batch sizes
// (K2 LENS budget search), allocations (step completion) and learner samples
// (K4 refit, nx_learner.cuh).
#ifndef NX_INLINE_EXPM1
#define NX_COMPACT_MATH 1  // one out-of-line expm1 (was ~180 KB of inlined copies)
#endif
#include <stdlib.h>

#include "nx_learner.cuh"
#include "nx_lens.cuh"
#include "nx_router.cuh"

namespace nxd {

constexpr double kInf = __builtin_huge_val();

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
  return c.P->req[c.roff + r].prompt - c.P->req[c.roff + r].prefilled;
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
  if (c.lane == 0) c.rs->work[2] += span;
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
      if (tok < 0 || c.P->kv_admitted[c.roff + r]) {
        keep = true;
      } else if (trimmed) {
        keep = false;
      } else {
        const int foot = blocks_for(c.P->req[c.roff + r].prompt + c.P->req[c.roff + r].target, ed.block_size);
        const int fut = foot - blocks_for(c.P->req[c.roff + r].prefilled + c.P->req[c.roff + r].decoded,
                                          ed.block_size);
        if (static_cast<int64_t>(g.pinned) + g.reserved + fut <= ed.kv_blocks) {
          g.reserved += fut;
          c.P->kv_admitted[c.roff + r] = 1;
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
  PhaseTimer pt(c.rs, 2);
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
    g.step_seq = c.rs->next_seq++;
    c.rs->work[0] += 1;
    c.rs->work[1] += g.plan_b;
    if (c.log_flags & NX_LOG_PLANS) {  // plans_jsonl row (sim.cpp:149-158)
      const int64_t k = c.rs->n_plan_log;
      if (k >= c.d->plan_log_cap) {
        c.rs->status = 1;
        c.rs->site = NX_SITE_OVERFLOW;
      } else {
        NxPlanLog& L = c.P->plan_log[c.d->plan_log_off + k];
        L.t_us = now_us;
        L.engine_id = ed.engine_id;
        L.b = g.plan_b;
        L.s = g.plan_s;
        L.pad_ = 0;
        L.predicted_ms = g.plan_pred;
        L.target_ms = g.plan_target;
        c.rs->n_plan_log = k + 1;
      }
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
    const int prompt = c.P->req[c.roff + r].prompt;
    const int credit = cached < prompt - 1 ? cached : prompt - 1;
    const int cb = blocks_for(credit, ed.block_size);
    if (credit > 0 && static_cast<int64_t>(g.pinned) + g.reserved + cb <= ed.kv_blocks) {
      g.cache_blocks -= blocks_for(cached, ed.block_size);
      lru_unlink(g, L, sess);
      c.P->req[c.roff + r].prefilled = credit;
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
  const long long t_cs = nx_clock();
  put(g.busy, 0);
  for (int base = 0; base < n; base += 32) {
    const int k = base + c.lane;
    int delta = 0, held = 0, r = -1, tokens = 0;
    bool first = false, fin = false;
    if (k < n) {
      r = preq[k];
      const int tok = ptok[k];
      const int4 q = *reinterpret_cast<const int4*>(&P.req[ro + r]);  // one 16-B load
      int pre = q.x, dec = q.y;
      const int before = blocks_for(pre + dec, block);
      if (tok >= 0) pre += tok;
      else dec += 1;
      const int after = blocks_for(pre + dec, block);
      delta = after - before;
      *reinterpret_cast<int2*>(&P.req[ro + r]) = make_int2(pre, dec);
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
          const int tgt = P.req[ro + rr].target;
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
          // RequestRecord + Router::on_completion (router.cpp:83-92)
          P.done_us[ro + rr] = now_us;
          P.records[ro + c.rs->n_rec] = rr;
          c.rs->n_rec += 1;
          if (c.d->route_policy == 4) {
            if (g.lat_len >= ed.lat_cap) {
              c.rs->status = 1;
              c.rs->site = NX_SITE_OVERFLOW;
            } else {
              const int slot = ring_add(g.lat_head, g.lat_len, ed.lat_cap);
              P.lat_t[ed.lat_off + slot] = now;
              P.lat_e2e[ed.lat_off + slot] = now - P.arr_ms[ro + rr];
              g.lat_len += 1;
              g.lat_sum += now - P.arr_ms[ro + rr];
            }
          }
          const double le = c.rs->l_bar_ema + 0.05 * (static_cast<double>(tgt) - c.rs->l_bar_ema);
          c.rs->l_bar_ema = le < 1.0 ? 1.0 : le;
          P.sess_engine[c.soff + P.session[ro + rr]] = e;
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
  }
  __syncwarp();
  // run queue: drop finished (stable), then append new runners in plan order
  int32_t* rq = P.rq + ed.rq_off;
  int out = g.rq_len;
  if (n_fin) {
    out = 0;
    const int len = g.rq_len;
    for (int base = 0; base < len; base += 32) {
      const int i = base + c.lane;
      const int r = i < len ? rq[i] : 0;
      const bool keep = i < len && P.req[ro + r].decoded != P.req[ro + r].target;
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
        nr = P.req[ro + r].prefilled == P.req[ro + r].prompt;
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
        if (P.req[ro + r].prefilled != P.req[ro + r].prompt) wq[wpos--] = r;
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
    g.learn_seq = c.rs->next_seq++;
    g.learn_b = g.plan_b;
    g.learn_s = g.plan_s;
    g.learn_y = g.actual;
  }
  __syncwarp();
  if (n_fin) tradeoff_refit(c, e);
  if (nx_timers_on && c.lane == 0) c.rs->cycles[3] += nx_clock() - t_cs;
  try_begin_step(c, e, now_us);
}

// ---- state report (sim.cpp:226-243, engine.cpp:307-332), lane 0 only -----------
__device__ NX_COLD void state_report(Ctx& c, int e, int64_t now_us) {
  EngSm& g = c.eng[e];
  const NxEngineDesc& ed = c.ed[e];
  wait_refit(c, e);  // the report exports the learner's p_max
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
      c.rs->status = 1;
      c.rs->site = NX_SITE_OVERFLOW;
    } else {
      const int slot = ring_add(g.dq_head, g.dq_len, ed.dq_cap);
      const int64_t o = ed.dq_off + slot;
      const int64_t dt = now_us + ed.stale_us;
      const uint32_t ds = c.rs->next_seq++;
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
    g.report_seq = c.rs->next_seq++;
  }
  __syncwarp();
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
      const int prompt = c.P->req[c.roff + rid].prompt;
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

// LearnerSnapshot after a learner update event (sim.cpp:322-327): the
// structural refit record_sample may have queued is part of the update, so
// the snapshot waits for it (history recording trades overlap for order).
__device__ void log_learner(Ctx& c, int e, int64_t now_us) {
  if (!(c.log_flags & NX_LOG_LEARNER) || failed(c)) return;
  wait_refit(c, e);
  __syncwarp();
  if (c.lane == 0) {
    const int64_t k = c.rs->n_learn_log;
    if (k >= c.d->learn_log_cap) {
      c.rs->status = 1;
      c.rs->site = NX_SITE_OVERFLOW;
    } else {
      const EngSm& g = c.eng[e];
      NxLearnLog& L = c.P->learn_log[c.d->learn_log_off + k];
      L.t_us = now_us;
      L.samples = g.seen;
      L.engine_id = c.ed[e].engine_id;
      L.pad_ = 0;
      params_to(g.lp, L.params);
      c.rs->n_learn_log = k + 1;
    }
  }
  __syncwarp();
}

// ---- replica driver -------------------------------------------------------------
__device__ NX_COLD void init_replica(Ctx& c) {
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
    g.report_t = 0; g.report_seq = static_cast<uint32_t>(e);  // initial reports: seq 0..E-1
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
    R.next_seq = static_cast<uint32_t>(c.n_eng + c.n_req);  // arrival i carries seq E + i
    R.cursor = 0; R.status = 0; R.site = 0;
    R.next_arr = c.n_req > 0 ? static_cast<uint64_t>(c.P->arr_us[c.roff]) : kNoEvent;
  }
  __syncwarp();
}

__device__ void run_replica(Ctx& c) {
  const NxReplicaDesc& d = *c.d;
  const uint64_t duration = static_cast<uint64_t>(d.duration_us);
  while (!failed(c)) {
    long long t_sel = nx_clock();
    // ---- next event: warp-wide (time, seq) minimum over the slots ----
    uint64_t t = kNoEvent;
    uint32_t sq = 0xffffffffu;
    int kind = -1;
    if (c.lane < c.n_eng) {
      const EngSm& g = c.eng[c.lane];
      if (g.step_t != kNoEvent) { t = g.step_t; sq = g.step_seq; kind = 1; }
      if (g.report_t < t || (g.report_t == t && g.report_t != kNoEvent && g.report_seq < sq)) {
        t = g.report_t; sq = g.report_seq; kind = 2;
      }
      if (g.learn_t < t || (g.learn_t == t && g.learn_t != kNoEvent && g.learn_seq < sq)) {
        t = g.learn_t; sq = g.learn_seq; kind = 3;
      }
      if (g.dq_t0 < t || (g.dq_t0 == t && g.dq_t0 != kNoEvent && g.dq_s0 < sq)) {
        t = g.dq_t0; sq = g.dq_s0; kind = 4;
      }
    }
    if (c.lane == 0 && c.rs->next_arr != kNoEvent) {
      const uint64_t at = c.rs->next_arr;
      const uint32_t as = static_cast<uint32_t>(c.n_eng + c.rs->cursor);
      if (at < t || (at == t && as < sq)) { t = at; sq = as; kind = 0; }
    }
    const uint32_t hi = static_cast<uint32_t>(t >> 32), lo = static_cast<uint32_t>(t);
    const uint32_t mhi = __reduce_min_sync(NX_FULL, hi);
    const uint32_t mlo = __reduce_min_sync(NX_FULL, hi == mhi ? lo : 0xffffffffu);
    const bool tie = hi == mhi && lo == mlo;
    const uint32_t msq = __reduce_min_sync(NX_FULL, tie ? sq : 0xffffffffu);
    const uint64_t now_u = (static_cast<uint64_t>(mhi) << 32) | mlo;
    if (now_u == kNoEvent || now_u > duration) break;
    const unsigned win = __ballot_sync(NX_FULL, tie && sq == msq && kind >= 0);
    const int wl = __ffs(win) - 1;
    kind = __shfl_sync(NX_FULL, kind, wl);
    const int who = wl;  // engine index for engine events
    const int64_t now = static_cast<int64_t>(now_u);
    // ---- consume the slot ----
    int rid = 0;
    int64_t dq_o = 0;  // the delivered report's slot (read in case 4; no push in between)
    if (kind == 0) rid = c.rs->cursor;
    if (kind == 4) dq_o = c.ed[who].dq_off + c.eng[who].dq_head;
    __syncwarp();
    if (c.lane == 0) {
      EngSm& g = c.eng[kind == 0 ? 0 : who];
      if (kind == 0) {
        const int nc = c.rs->cursor + 1;
        c.rs->cursor = nc;
        c.rs->next_arr = nc < c.n_req ? static_cast<uint64_t>(c.P->arr_us[c.roff + nc]) : kNoEvent;
      }
      else if (kind == 1) g.step_t = kNoEvent;
      else if (kind == 2) g.report_t = kNoEvent;
      else if (kind == 3) g.learn_t = kNoEvent;
      else {
        g.dq_head = ring_add(g.dq_head, 1, c.ed[who].dq_cap);
        g.dq_len -= 1;
        if (g.dq_len > 0) {
          const int64_t o = c.ed[who].dq_off + g.dq_head;
          g.dq_t0 = static_cast<uint64_t>(c.P->dq_t[o]);
          g.dq_s0 = c.P->dq_seq[o];
        } else {
          g.dq_t0 = kNoEvent;
        }
      }
    }
    __syncwarp();
    // periodic reports keep no work alive (sim.cpp:295-300)
    if (kind == 2 && c.rs->pending == 0 && c.rs->arrived - c.rs->rejected - c.rs->n_rec == 0) continue;
    __syncwarp();
    if (c.lane == 0) {
      const uint64_t h = fnv_event(c.rs->ev_hash, now_u, static_cast<uint64_t>(kind),
                                   kind == 0 ? 0ull : static_cast<uint64_t>(c.ed[who].engine_id + 1),
                                   static_cast<uint64_t>(rid));
      c.rs->ev_hash = h;
      c.rs->events += 1;
      if (nx_timers_on) c.rs->cycles[0] += nx_clock() - t_sel;
    }
    __syncwarp();
    switch (kind) {
      case 0: {  // arrival (sim.cpp:168-194)
        __syncwarp();
        if (c.lane == 0) {
          c.rs->arrived += 1;
          c.rs->pending -= 1;
        }
        __syncwarp();
        int e, ok = 0;
        {
          PhaseTimer pt(c.rs, 1);
          double score = 0.0, fac[4] = {1.0, 1.0, 1.0, 1.0};
          e = route(c, rid, to_ms(now), score, fac);
          if (c.lane == 0 && (c.log_flags & NX_LOG_ROUTES)) {  // routing_jsonl row (sim.cpp:176-186)
            NxRouteLog& L = c.P->route_log[c.d->route_log_off + c.rs->n_route_log];
            L.t_us = now;
            L.request = rid;
            L.engine_id = c.ed[e].engine_id;
            L.score = score;
            for (int i = 0; i < 4; ++i) L.factors[i] = fac[i];
            c.rs->n_route_log += 1;
          }
          if (c.lane == 0 && !failed(c)) {
            ok = admit(c, e, rid) ? 1 : 0;
            if (!ok) c.rs->rejected += 1;
          }
        }
        if (failed(c)) break;
        ok = __shfl_sync(NX_FULL, ok, 0);
        __syncwarp();
        if (ok) try_begin_step(c, e, now);
        break;
      }
      case 1: {
        step_complete(c, who, now);
        // The learner update just queued at (now, seq) is the next event
        // unless another pending event shares this timestamp (all of those
        // carry smaller sequence numbers): then process it right here.
        if (failed(c)) break;
        bool other = false;
        if (c.lane < c.n_eng) {
          const EngSm& g = c.eng[c.lane];
          other = g.step_t == now_u || g.report_t == now_u || g.dq_t0 == now_u ||
                  (c.lane != who && g.learn_t == now_u);
        }
        if (c.lane == 0 && c.rs->next_arr == now_u) other = true;
        if (__any_sync(NX_FULL, other)) break;
        __syncwarp();
        if (c.lane == 0) {
          c.eng[who].learn_t = kNoEvent;
          c.rs->ev_hash = fnv_event(c.rs->ev_hash, now_u, 3ull,
                                    static_cast<uint64_t>(c.ed[who].engine_id + 1), 0ull);
          c.rs->events += 1;
        }
        __syncwarp();
        const EngSm& g = c.eng[who];
        record_sample(c, who, g.learn_b, g.learn_s, g.learn_y);
        log_learner(c, who, now);
        break;
      }
      case 2: {
        PhaseTimer pt(c.rs, 4);
        state_report(c, who, now);
        break;
      }
      case 3: {
        const EngSm& g = c.eng[who];
        record_sample(c, who, g.learn_b, g.learn_s, g.learn_y);
        log_learner(c, who, now);
        break;
      }
      case 4: {  // report delivery -> Router::on_report (router.cpp:75-81)
        PhaseTimer pt(c.rs, 7);
        __syncwarp();
        if (c.lane == 0) {
          EngSm& g = c.eng[who];
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
}

__device__ NX_COLD void write_outputs(Ctx& c, int r) {
  __syncwarp();
  NxReplicaOut& o = c.P->rep_out[r];
  if (c.lane == 0) {
    const RepSm& R = *c.rs;
    o.arrived = R.arrived;
    o.rejected = R.rejected;
    o.completed = R.n_rec;
    o.pending = R.pending;
    o.events = R.events;
    o.event_hash = R.ev_hash;
    o.status = R.status;
    o.err_site = R.site;
    o.err_info = R.info;
    for (int i = 0; i < 6; ++i) o.work[i] = R.work[i];
    for (int i = 0; i < 16; ++i) o.cycles[i] = R.cycles[i];
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

}  // namespace nxd

// One CTA per replica: warp 0 runs the event loop, warps 1..kRefitWarps run
// the queued structural refits. CTAs pull replica indices (host order, longest
// expected first) from a global counter so a long replica never idles others.
extern "C" __global__ void __launch_bounds__(32 * nxd::kSimWarps)
nx_sim_kernel(const NxPools* __restrict__ pools, const int32_t* __restrict__ order, int n_rep,
              int* ctl, int smem_per_cta, int prefix_cap, int max_eng, int n_excl) {
  using namespace nxd;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_slot;
  const int warp = threadIdx.x >> 5;
  Ctx c;
  c.P = pools;
  c.lane = lane_id();
  c.worker = warp;
  c.rs = reinterpret_cast<RepSm*>(smem);
  const size_t rep_bytes = (sizeof(RepSm) + 15) & ~size_t(15);
  const size_t stage = ((static_cast<size_t>(prefix_cap) * 4 > 32 * 5 * 8 ? static_cast<size_t>(prefix_cap) * 4
                                                                        : 32 * 5 * 8) + 15) & ~size_t(15);
  c.chunk = reinterpret_cast<double*>(smem + rep_bytes + warp * stage);
  c.prefix = reinterpret_cast<int32_t*>(c.chunk);
  c.eng = reinterpret_cast<EngSm*>(smem + rep_bytes + kSimWarps * stage);
  c.prefix_cap = prefix_cap;
  // the refit warps' fit tables follow the engine states (nx_sim_smem_per_warp)
  const size_t fit_off = (rep_bytes + kSimWarps * stage + sizeof(EngSm) * static_cast<size_t>(max_eng) + 15) &
                         ~size_t(15);
  c.fsm = warp == 1 ? reinterpret_cast<double*>(smem + fit_off) : nullptr;
  c.fsm_cap = kFitSmemS;
  c.team = kRefitWarps;
  (void)smem_per_cta;
  // Exclusive SMs for the longest replicas (order[0, n_excl)): under two
  // resident CTAs per SM an event loop runs ~1.3-1.8x slower than alone, and
  // the kernel ends with its longest replicas. The first CTA to arrive on
  // each of n_excl SMs takes one of them while its sibling on that SM waits;
  // then both join the shared queue order[n_excl, n). ctl: [0] shared
  // cursor, [1] exclusive cursor, [2] exclusive SMs claimed, then per-SM
  // arrival counts and states (0 unknown, 1 shared, 2 exclusive, 3 released).
  __shared__ int s_excl;
  int* sm_cnt = ctl + 3;
  int* sm_state = ctl + 3 + kMaxSmIds;
  unsigned smid = 0;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) {
    int excl = 0;
    if (n_excl > 0 && smid < static_cast<unsigned>(kMaxSmIds)) {
      const int k = atomicAdd(&sm_cnt[smid], 1);
      if (k == 0) {
        excl = atomicAdd(&ctl[2], 1) < n_excl;
        atomicExch(&sm_state[smid], excl ? 2 : 1);
      } else {
        int st;
        unsigned ns = 256;
        while ((st = atomicAdd(&sm_state[smid], 0)) == 0 || st == 2) {
          __nanosleep(ns);
          ns = ns < 8192 ? 2 * ns : 8192;
        }
      }
    }
    s_excl = excl;
  }
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) {
      int slot = n_rep;
      if (s_excl) {
        const int e = atomicAdd(&ctl[1], 1);
        if (e < n_excl) slot = e;
        // the exclusive replicas were already taken (a late-starting CTA:
        // others drained them): release the waiting sibling now, since the
        // release after a completed exclusive replica will not happen
        else atomicExch(&sm_state[smid], 3);
        s_excl = 0;  // one exclusive replica, then release the sibling
      }
      if (slot == n_rep) {
        const int k = n_excl + atomicAdd(&ctl[0], 1);
        if (k < n_rep) {
          slot = k;
        } else {  // shared queue drained: help with any exclusive ones left
          const int e = atomicAdd(&ctl[1], 1);
          if (e < n_excl) slot = e;
        }
      }
      s_slot = slot;
    }
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
    // learner scratch: the event loop (linear refits) and the refit leader;
    // helpers only read the leader's staged window
    c.scratch = pools->scratch + c.d->scratch_off + (warp == 0 ? 0 : 1) * refit_scratch_stride(c.d->long_w);
    c.lin_rows = c.scratch + 6 * c.d->long_w + kFbTable;
    if (warp == 0) init_replica(c);
    __syncthreads();
    if (warp == 0) {
      run_replica(c);
      for (int e = 0; e < c.n_eng; ++e) wait_refit(c, e);
      post_exit(c);
    } else if (warp == 1) {
      refit_worker(c);
    } else {
      team_helper(c);
    }
    __syncthreads();
    if (warp == 0) write_outputs(c, r);
    if (threadIdx.x == 0 && slot < n_excl && smid < static_cast<unsigned>(kMaxSmIds))
      atomicExch(&sm_state[smid], 3);  // exclusive replica done: wake the sibling
    __syncthreads();
  }
}

// Size of the per-CTA shared-memory slice (host uses the same formula).
extern "C" size_t nx_sim_smem_per_warp(int max_engines, int prefix_cap) {
  using namespace nxd;
  const size_t rep_bytes = (sizeof(RepSm) + 15) & ~size_t(15);
  const size_t stage = ((static_cast<size_t>(prefix_cap) * 4 > 32 * 5 * 8 ? static_cast<size_t>(prefix_cap) * 4
                                                                        : 32 * 5 * 8) + 15) & ~size_t(15);
  const size_t fit_off = (rep_bytes + kSimWarps * stage + sizeof(EngSm) * static_cast<size_t>(max_engines) + 15) &
                         ~size_t(15);
  return fit_off + sizeof(double) * (kFbTable + kFitSmemS);
}

extern "C" cudaError_t nx_launch_sim(const NxPools* d_pools, const int32_t* d_order, int n_rep,
                                     int* d_next, int smem_per_warp, int prefix_cap, int max_eng,
                                     int grid, int warps_per_block, int n_excl, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(smem_per_warp);  // one replica per CTA
#ifdef NX_TIMERS
  const char* tm = getenv("NX_PHASE_TIMERS");
  const int timers = tm && tm[0] == '1';
  cudaError_t terr = cudaMemcpyToSymbolAsync(nxd::nx_timers_on, &timers, sizeof timers, 0,
                                             cudaMemcpyHostToDevice, st);
  if (terr != cudaSuccess) return terr;
#endif
  cudaError_t err = cudaFuncSetAttribute(nx_sim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  nx_sim_kernel<<<grid, 32 * warps_per_block, smem, st>>>(d_pools, d_order, n_rep, d_next,
                                                          smem_per_warp, prefix_cap, max_eng, n_excl);
  return cudaGetLastError();
}

extern "C" cudaError_t nx_sim_occupancy(int warps_per_block, size_t smem, int* blocks_per_sm) {
  // dynamic shared memory above 48 KB must be opted into before the query
  cudaError_t err = cudaFuncSetAttribute(nx_sim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, nx_sim_kernel,
                                                       32 * warps_per_block, smem);
}
