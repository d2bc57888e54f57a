// TEST INFRASTRUCTURE — oracle/_ref driver.
//
// A C-ABI shim over the UNMODIFIED reference core (proj/src/*.cpp compiled in
// place by oracle/Makefile). It only calls the reference's public servesim::
// API (proj/include/servesim/*.h); it re-implements nothing. Used by tests/
// as the ground-truth checker and by bench.py's reference arm / cpu_baseline
// leg. Never linked into the product.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <stdexcept>
#include <algorithm>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "servesim/engine.h"
#include "servesim/learner.h"
#include "servesim/lens.h"
#include "servesim/metrics.h"
#include "servesim/perf_model.h"
#include "servesim/router.h"
#include "servesim/sim.h"

using namespace servesim;

namespace {
thread_local std::string g_err;

char* dup_string(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.data(), s.size() + 1);
  return out;
}

PerfParams params_from(const double* p) {
  PerfParams q;
  q.tau0 = p[0];
  q.w0 = p[1];
  q.ws = p[2];
  q.tauB = p[3];
  q.tauS = p[4];
  q.p_max = p[5];
  q.kB = p[6];
  q.kS = p[7];
  return q;
}

void params_to(const PerfParams& q, double* p) {
  p[0] = q.tau0;
  p[1] = q.w0;
  p[2] = q.ws;
  p[3] = q.tauB;
  p[4] = q.tauS;
  p[5] = q.p_max;
  p[6] = q.kB;
  p[7] = q.kS;
}

int64_t decisions_of(const RunResult& r) {
  const auto j = nlohmann::json::parse(r.summary_json);
  int64_t batches = 0;
  for (const auto& e : j["learners"]) batches += e["samples"].get<int64_t>();
  return r.arrived + batches;
}

// 0 ok, 1 invalid_argument, 2 runtime_error, 3 logic_error, 9 other
int classify(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::logic_error*>(&e)) return 3;
  if (dynamic_cast<const std::runtime_error*>(&e)) return 2;
  return 9;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// Runs servesim::run_simulation on a JSON RunConfig (RunConfig::from_json_text,
// src/sim.cpp:454). Returns a JSON document with counts, hashes, summary_json,
// decisions and (optionally) every RequestRecord.
int ref_run_json(const char* cfg_json, int with_records, char** out) {
  try {
    const RunConfig cfg = RunConfig::from_json_text(cfg_json);
    const RunResult r = run_simulation(cfg);
    nlohmann::ordered_json j;
    j["arrived"] = r.arrived;
    j["completed"] = r.completed;
    j["rejected"] = r.rejected;
    j["unfinished"] = r.unfinished;
    char hex[32];
    std::snprintf(hex, sizeof hex, "%016llx", (unsigned long long)r.arrival_hash);
    j["arrival_hash"] = hex;
    std::snprintf(hex, sizeof hex, "%016llx", (unsigned long long)r.event_hash);
    j["event_hash"] = hex;
    j["decisions"] = decisions_of(r);
    j["summary_json"] = r.summary_json;
    if (with_records) {
      std::vector<int64_t> id, eng, pt, ot;
      std::vector<double> arr, ft, done;
      for (const auto& rec : r.records) {
        id.push_back((int64_t)rec.request_id);
        eng.push_back(rec.engine_id);
        pt.push_back(rec.prompt_tokens);
        ot.push_back(rec.output_tokens);
        arr.push_back(rec.arrival_ms);
        ft.push_back(rec.first_token_ms);
        done.push_back(rec.completed_ms);
      }
      j["rec_id"] = id;
      j["rec_engine"] = eng;
      j["rec_prompt"] = pt;
      j["rec_output"] = ot;
      j["rec_arrival"] = arr;
      j["rec_first"] = ft;
      j["rec_done"] = done;
    }
    if (cfg.record_learner_history) {  // RunResult::learner_history (sim.cpp:322-327)
      nlohmann::ordered_json hist = nlohmann::ordered_json::array();
      for (const auto& h : r.learner_history) {
        double p8[8];
        params_to(h.params, p8);
        hist.push_back({h.engine_id, h.sim_time_ms, h.samples_seen, std::vector<double>(p8, p8 + 8)});
      }
      j["learner_history"] = hist;
    }
    *out = dup_string(j.dump());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Thread pool over independent run_simulation calls (run_simulation is
// reentrant: src/workload.cpp:17 is the only static, and it is const).
// Fills per-replica decisions and event hashes; returns wall seconds in *wall.
int ref_run_batch(const char* const* cfgs, int n, int threads,
                  int64_t* decisions, uint64_t* event_hash, double* wall) {
  std::vector<RunConfig> parsed;
  try {
    for (int i = 0; i < n; ++i) parsed.push_back(RunConfig::from_json_text(cfgs[i]));
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
  std::atomic<int> next{0};
  std::atomic<int> failed{0};
  const auto t0 = std::chrono::steady_clock::now();
  auto worker = [&]() {
    for (int i = next++; i < n; i = next++) {
      try {
        const RunResult r = run_simulation(parsed[i]);
        decisions[i] = decisions_of(r);
        event_hash[i] = r.event_hash;
      } catch (...) {
        decisions[i] = -1;
        failed++;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return failed ? 2 : 0;
}

// ---- unit-level entry points for golden-vector checks ----------------------

int ref_perf_eval(const double* params8, const int64_t* b, const int64_t* s,
                  int64_t n, double* out_T, double* out_thr) {
  try {
    const PerfParams p = params_from(params8);
    for (int64_t i = 0; i < n; ++i) {
      out_thr[i] = throughput(p, {b[i], s[i]});
      out_T[i] = predict_latency(p, {b[i], s[i]});
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

int ref_target_latency(int64_t wait_count, double ttft, double tpot,
                       const double* tm4, double q_ref, double* target,
                       int* risk) {
  try {
    TradeoffModel tm;
    tm.alpha_ms = tm4[0];
    tm.beta = tm4[1];
    tm.l_bar = tm4[2];
    tm.td_min_ms = tm4[3];
    const auto t = target_latency(wait_count, {ttft, tpot}, tm, q_ref);
    *target = t.target_ms;
    *risk = t.slo_risk;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

int ref_binary_search_budget(int64_t b, double target, const double* params8,
                             int64_t m_max, int64_t q_max, int n_iters,
                             int64_t s_cap, int64_t* out) {
  try {
    SchedulerConfig cfg;
    cfg.m_max = m_max;
    cfg.q_max = q_max;
    cfg.n_search_iters = n_iters;
    *out = binary_search_budget(b, target, params_from(params8), cfg, s_cap);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// schedule_step over explicit queues. wait_q/run_q given as (prompt, prefilled)
// pairs; ids are 1000+i for waiters and i for runners.
// Output: b, s, predicted, target, overload, and allocations (id, tokens, prefill).
int ref_schedule_step(const int64_t* w_prompt, const int64_t* w_prefilled,
                      int64_t n_wait, int64_t n_run, double ttft, double tpot,
                      const double* tm4, const double* params8, int64_t m_max,
                      int64_t q_max, int n_iters, double eps, double q_ref,
                      int64_t* out_bs, double* out_pt, int* out_overload,
                      int64_t* alloc_id, int64_t* alloc_tokens,
                      int* alloc_prefill) {
  try {
    std::vector<Request> store(static_cast<size_t>(n_wait + n_run));
    std::vector<const Request*> wait, run;
    for (int64_t i = 0; i < n_run; ++i) {
      Request& r = store[i];
      r.id = static_cast<uint64_t>(i);
      r.prompt_len = 64;
      r.prefilled = 64;
      r.state = RequestState::kRunning;
      run.push_back(&r);
    }
    for (int64_t i = 0; i < n_wait; ++i) {
      Request& r = store[n_run + i];
      r.id = static_cast<uint64_t>(1000 + i);
      r.prompt_len = w_prompt[i];
      r.prefilled = w_prefilled[i];
      wait.push_back(&r);
    }
    TradeoffModel tm;
    tm.alpha_ms = tm4[0];
    tm.beta = tm4[1];
    tm.l_bar = tm4[2];
    tm.td_min_ms = tm4[3];
    SchedulerConfig cfg;
    cfg.m_max = m_max;
    cfg.q_max = q_max;
    cfg.n_search_iters = n_iters;
    cfg.eps_ratio = eps;
    cfg.q_ref = q_ref;
    const BatchPlan plan = schedule_step(wait, run, {ttft, tpot}, tm,
                                         params_from(params8), cfg);
    out_bs[0] = plan.b;
    out_bs[1] = plan.s;
    out_pt[0] = plan.predicted_ms;
    out_pt[1] = plan.target_ms;
    *out_overload = plan.overload;
    for (size_t i = 0; i < plan.allocations.size(); ++i) {
      alloc_id[i] = static_cast<int64_t>(plan.allocations[i].request_id);
      alloc_tokens[i] = plan.allocations[i].tokens;
      alloc_prefill[i] = plan.allocations[i].is_prefill;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// schedule_baseline over explicit queues (ids as in ref_schedule_step).
// Output: b, s, predicted, and allocations (id, tokens, prefill).
int ref_schedule_baseline(int policy, const int64_t* w_prompt, const int64_t* w_prefilled,
                          int64_t n_wait, int64_t n_run, const double* params8, int64_t m_max,
                          int64_t q_max, int64_t static_budget, int engine_id, int64_t* out_bs,
                          double* out_pred, int64_t* alloc_id, int64_t* alloc_tokens,
                          int* alloc_prefill) {
  try {
    std::vector<Request> store(static_cast<size_t>(n_wait + n_run));
    std::vector<const Request*> wait, run;
    for (int64_t i = 0; i < n_run; ++i) {
      Request& r = store[i];
      r.id = static_cast<uint64_t>(i);
      r.prompt_len = 64;
      r.prefilled = 64;
      r.state = RequestState::kRunning;
      run.push_back(&r);
    }
    for (int64_t i = 0; i < n_wait; ++i) {
      Request& r = store[n_run + i];
      r.id = static_cast<uint64_t>(1000 + i);
      r.prompt_len = w_prompt[i];
      r.prefilled = w_prefilled[i];
      wait.push_back(&r);
    }
    EngineConfig cfg;
    cfg.engine_id = engine_id;
    cfg.m_max = m_max;
    cfg.q_max = q_max;
    cfg.static_budget = static_budget;
    const SchedulerPolicy pol = policy == 1   ? SchedulerPolicy::kPrefillPriority
                                : policy == 2 ? SchedulerPolicy::kStaticChunked
                                              : SchedulerPolicy::kLens;
    const BatchPlan plan = schedule_baseline(pol, wait, run, params_from(params8), cfg);
    out_bs[0] = plan.b;
    out_bs[1] = plan.s;
    *out_pred = plan.predicted_ms;
    for (size_t i = 0; i < plan.allocations.size(); ++i) {
      alloc_id[i] = static_cast<int64_t>(plan.allocations[i].request_id);
      alloc_tokens[i] = plan.allocations[i].tokens;
      alloc_prefill[i] = plan.allocations[i].is_prefill;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// PRISM route over a report table. state rows: l_hat, w_load, m_free, p_max,
// reported_at (5 doubles) + queue_len + has_report. Session affinity is given
// by `affine_engine` (engine id previously completing this session, or -1).
int ref_route(int policy, const double* router_cfg9, double ttft, double tpot,
              int n_engines, const int* engine_ids, const double* states5,
              const int64_t* queue_len, const int* has_report,
              int affine_engine, int64_t prompt_len, double now_ms,
              int* out_engine, double* out_score, double* out_factors,
              int* out_degraded) {
  try {
    RouterConfig cfg;
    cfg.policy = static_cast<RouterPolicy>(policy);
    for (int i = 0; i < 4; ++i) cfg.weights[i] = router_cfg9[i];
    cfg.beta_aff = router_cfg9[4];
    cfg.latency_knee = router_cfg9[5];
    cfg.latency_scale_ms = router_cfg9[6];
    cfg.load_half_ms = router_cfg9[7];
    cfg.capacity_headroom = router_cfg9[8];
    Router router(cfg, {ttft, tpot}, 1);
    for (int e = 0; e < n_engines; ++e) router.register_engine(engine_ids[e]);
    for (int e = 0; e < n_engines; ++e) {
      if (!has_report[e]) continue;
      EngineReport rep;
      rep.state.engine_id = engine_ids[e];
      rep.state.l_hat_ms = states5[5 * e + 0];
      rep.state.w_load_tokens = states5[5 * e + 1];
      rep.state.m_free_tokens = states5[5 * e + 2];
      rep.state.p_max = states5[5 * e + 3];
      rep.state.reported_at_ms = states5[5 * e + 4];
      rep.queue_len = queue_len[e];
      router.on_report(rep);
    }
    if (affine_engine >= 0) {
      router.on_completion(affine_engine, "sess", 1.0, 128, 0.0);
    }
    Request req;
    req.id = 1;
    req.session_id = "sess";
    req.prompt_len = prompt_len;
    const RouteDecision d = router.route(req, now_ms);
    *out_engine = d.engine_id;
    *out_score = d.score;
    for (int i = 0; i < 4; ++i) out_factors[i] = d.factors[i];
    *out_degraded = d.degraded;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Streams samples through an OnlineLearner (record_sample, src/learner.cpp:130)
// and returns the final params + counters.
int ref_learner_stream(const double* priors8, const int64_t* cfg5,
                       const int64_t* b, const int64_t* s, const double* y,
                       int64_t n, double* out_params8, int64_t* out_counters9) {
  try {
    LearnerConfig cfg;
    cfg.long_window = cfg5[0];
    cfg.short_window = cfg5[1];
    cfg.structural_period = cfg5[2];
    cfg.linear_period = cfg5[3];
    cfg.min_structural_samples = cfg5[4];
    OnlineLearner learner(params_from(priors8), cfg);
    for (int64_t i = 0; i < n; ++i) learner.record_sample({{b[i], s[i]}, y[i], 0.0});
    params_to(learner.params(), out_params8);
    const auto& c = learner.counters();
    out_counters9[0] = c.linear_updates;
    out_counters9[1] = c.structural_updates;
    out_counters9[2] = c.degenerate_updates;
    out_counters9[3] = c.rescale_updates;
    out_counters9[4] = c.clamp_events;
    out_counters9[5] = c.failed_fits;
    out_counters9[6] = c.low_identifiability;
    out_counters9[7] = learner.samples_seen();
    out_counters9[8] = learner.buffered();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Single structural update on a prepared window (fills the ring without
// triggering periodic updates, then calls update_structural()).
int ref_learner_structural(const double* priors8, int64_t window,
                           const int64_t* b, const int64_t* s, const double* y,
                           int64_t n, double* out_params8, int* accepted) {
  try {
    LearnerConfig cfg;
    cfg.long_window = window;
    cfg.short_window = std::min<int64_t>(64, window - 1);
    cfg.structural_period = 1 << 30;
    cfg.linear_period = (1 << 30) - 1;
    cfg.min_structural_samples = 1;
    OnlineLearner learner(params_from(priors8), cfg);
    for (int64_t i = 0; i < n; ++i) learner.record_sample({{b[i], s[i]}, y[i], 0.0});
    *accepted = learner.update_structural();
    params_to(learner.params(), out_params8);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Router over a sequence: registers engines (ids in order, static weights),
// replays completions (engine id, session "s<k>", decode length) through
// on_completion, installs reports, then routes the requests in order.
// Returns every RouteDecision and the final report view (dispatch echoes).
int ref_route_group(int policy, const double* router_cfg9, double ttft, double tpot,
                    uint64_t root_seed, int n_engines, const int* engine_ids,
                    const double* static_w, const double* states5, const int64_t* queue_len,
                    const int* has_report, int n_comp, const int* comp_engine,
                    const int* comp_session, const int64_t* comp_decode, int n_req,
                    const int64_t* req_prompt, const int* req_session, const double* req_now,
                    int* out_engine, double* out_score, double* out_factors, int* out_degraded,
                    double* out_states5, int64_t* out_qlen) {
  try {
    RouterConfig cfg;
    cfg.policy = static_cast<RouterPolicy>(policy);
    for (int i = 0; i < 4; ++i) cfg.weights[i] = router_cfg9[i];
    cfg.beta_aff = router_cfg9[4];
    cfg.latency_knee = router_cfg9[5];
    cfg.latency_scale_ms = router_cfg9[6];
    cfg.load_half_ms = router_cfg9[7];
    cfg.capacity_headroom = router_cfg9[8];
    for (int e = 0; e < n_engines; ++e)
      if (static_w[e] != 1.0) cfg.static_weights[engine_ids[e]] = static_w[e];
    Router router(cfg, {ttft, tpot}, root_seed);
    for (int e = 0; e < n_engines; ++e) router.register_engine(engine_ids[e]);
    for (int k = 0; k < n_comp; ++k)
      router.on_completion(comp_engine[k], "s" + std::to_string(comp_session[k]), 1.0,
                           comp_decode[k], 0.0);
    std::vector<EngineReport> view(n_engines);
    for (int e = 0; e < n_engines; ++e) {
      if (!has_report[e]) continue;
      EngineReport rep;
      rep.state.engine_id = engine_ids[e];
      rep.state.l_hat_ms = states5[5 * e + 0];
      rep.state.w_load_tokens = states5[5 * e + 1];
      rep.state.m_free_tokens = states5[5 * e + 2];
      rep.state.p_max = states5[5 * e + 3];
      rep.state.reported_at_ms = states5[5 * e + 4];
      rep.queue_len = queue_len[e];
      router.on_report(rep);
      view[e] = rep;
    }
    for (int k = 0; k < n_req; ++k) {
      Request req;
      req.id = static_cast<uint64_t>(k);
      req.session_id = "s" + std::to_string(req_session[k]);
      req.prompt_len = req_prompt[k];
      const RouteDecision d = router.route(req, req_now[k]);
      out_engine[k] = d.engine_id;
      out_score[k] = d.score;
      for (int i = 0; i < 4; ++i) out_factors[4 * k + i] = d.factors[i];
      out_degraded[k] = d.degraded;
      // mirror the dispatch echo into the returned view (router.cpp:275-282)
      if (cfg.policy == RouterPolicy::kPrism) {
        for (int e = 0; e < n_engines; ++e)
          if (engine_ids[e] == d.engine_id && has_report[e]) {
            view[e].queue_len += 1;
            view[e].state.w_load_tokens += static_cast<double>(req.prompt_len) + 32.0;
          }
      }
    }
    for (int e = 0; e < n_engines; ++e) {
      out_states5[5 * e + 0] = view[e].state.l_hat_ms;
      out_states5[5 * e + 1] = view[e].state.w_load_tokens;
      out_states5[5 * e + 2] = view[e].state.m_free_tokens;
      out_states5[5 * e + 3] = view[e].state.p_max;
      out_states5[5 * e + 4] = view[e].state.reported_at_ms;
      out_qlen[e] = view[e].queue_len;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Single linear update on a prepared window (same ring set-up as
// ref_learner_structural, then update_linear()).
int ref_learner_linear(const double* priors8, int64_t window, int64_t short_window,
                       const int64_t* b, const int64_t* s, const double* y, int64_t n,
                       double* out_params8, int* accepted, int64_t* out_counters7) {
  try {
    LearnerConfig cfg;
    cfg.long_window = window;
    cfg.short_window = short_window;
    cfg.structural_period = 1 << 30;
    cfg.linear_period = (1 << 30) - 1;
    cfg.min_structural_samples = 1;
    OnlineLearner learner(params_from(priors8), cfg);
    for (int64_t i = 0; i < n; ++i) learner.record_sample({{b[i], s[i]}, y[i], 0.0});
    *accepted = learner.update_linear();
    params_to(learner.params(), out_params8);
    const auto& c = learner.counters();
    const int64_t cv[7] = {c.linear_updates, c.structural_updates, c.degenerate_updates,
                           c.rescale_updates, c.clamp_events, c.failed_fits, c.low_identifiability};
    for (int i = 0; i < 7; ++i) out_counters7[i] = cv[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Structural update with explicit short window / min samples; counters out.
int ref_learner_structural2(const double* priors8, int64_t window, int64_t short_window,
                            int64_t min_samples, const int64_t* b, const int64_t* s,
                            const double* y, int64_t n, double* out_params8, int* accepted,
                            int64_t* out_counters7) {
  try {
    LearnerConfig cfg;
    cfg.long_window = window;
    cfg.short_window = short_window;
    cfg.structural_period = 1 << 30;
    cfg.linear_period = (1 << 30) - 1;
    cfg.min_structural_samples = min_samples;
    OnlineLearner learner(params_from(priors8), cfg);
    for (int64_t i = 0; i < n; ++i) learner.record_sample({{b[i], s[i]}, y[i], 0.0});
    *accepted = learner.update_structural();
    params_to(learner.params(), out_params8);
    const auto& c = learner.counters();
    const int64_t cv[7] = {c.linear_updates, c.structural_updates, c.degenerate_updates,
                           c.rescale_updates, c.clamp_events, c.failed_fits, c.low_identifiability};
    for (int i = 0; i < 7; ++i) out_counters7[i] = cv[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

}  // extern "C"
