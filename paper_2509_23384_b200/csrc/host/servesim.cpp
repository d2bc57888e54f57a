// C++ drop-in (include/nx_servesim.hpp) over the C-ABI: every model
// evaluation and scheduling decision is one batched device call
// (nx_perf_eval_host, nx_lens_schedule_host, nx_budget_search_host,
// nx_allocate_tokens_host, nx_target_latency_host, nx_prism_route_host,
// nx_router_scores_host, nx_tradeoff_update_host, nx_refit_host). The host
// keeps what the reference keeps in std containers: sample rings, report
// tables, session memory, completion windows — and JSON I/O.
#include "nx_servesim.hpp"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <list>
#include <stdexcept>

#include "frontend.hpp"
#include "json.hpp"
#include "nx_sched.h"

namespace servesim {
namespace {

// Re-raise a C-ABI status as the reference's exception class.
void raise(int rc) {
  if (rc == NX_OK) return;
  const std::string msg = nx_last_error();
  if (rc == NX_EINVAL) throw std::invalid_argument(msg);
  if (rc == NX_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

void pack(const PerfParams& p, double* out) {
  const double v[8] = {p.tau0, p.w0, p.ws, p.tauB, p.tauS, p.p_max, p.kB, p.kS};
  std::memcpy(out, v, sizeof v);
}
PerfParams unpack(const double* v) {
  PerfParams p;
  p.tau0 = v[0]; p.w0 = v[1]; p.ws = v[2]; p.tauB = v[3];
  p.tauS = v[4]; p.p_max = v[5]; p.kB = v[6]; p.kS = v[7];
  return p;
}

int32_t to_i32(int64_t v, const char* what) {
  if (v < INT32_MIN || v > INT32_MAX) throw std::invalid_argument(std::string(what) + ": device path needs 32-bit sizes");
  return static_cast<int32_t>(v);
}

// K1 over a span of shapes with one parameter row (perf_model.cpp:38-49).
void eval(const PerfParams& p, std::span<const BatchShape> shapes, double* T, double* thr) {
  const size_t n = shapes.size();
  std::vector<int32_t> idx(n, 0), b(n), s(n);
  for (size_t i = 0; i < n; ++i) {
    b[i] = to_i32(shapes[i].b, "BatchShape");
    s[i] = to_i32(shapes[i].s, "BatchShape");
  }
  double row[8];
  pack(p, row);
  raise(nx_perf_eval_host(row, 1, idx.data(), b.data(), s.data(), T, thr, static_cast<int64_t>(n),
                          NX_DETERMINISTIC_FP64));
}

}  // namespace

// ---- perf model -----------------------------------------------------------------
bool PerfParams::valid() const {
  return p_max > 0.0 && kB > 0.0 && kS > 0.0 && tau0 >= 0.0 && tauB >= 0.0 && tauS >= 0.0 &&
         ws > 0.0 && w0 >= 0.0;
}

std::string PerfParams::to_json() const {
  nlohmann::ordered_json j;
  j["tau0"] = tau0;
  j["w0"] = w0;
  j["ws"] = ws;
  j["tauB"] = tauB;
  j["tauS"] = tauS;
  j["p_max"] = p_max;
  j["kB"] = kB;
  j["kS"] = kS;
  return j.dump();
}

PerfParams PerfParams::from_json(const std::string& text) {
  const auto j = nlohmann::json::parse(text);
  PerfParams p;
  p.tau0 = j.at("tau0").get<double>();
  p.w0 = j.at("w0").get<double>();
  p.ws = j.at("ws").get<double>();
  p.tauB = j.at("tauB").get<double>();
  p.tauS = j.at("tauS").get<double>();
  p.p_max = j.at("p_max").get<double>();
  p.kB = j.at("kB").get<double>();
  p.kS = j.at("kS").get<double>();
  return p;
}

double throughput(const PerfParams& params, const BatchShape& shape) {
  double T = 0.0, thr = 0.0;
  eval(params, std::span<const BatchShape>(&shape, 1), &T, &thr);
  return thr;
}

double predict_latency(const PerfParams& params, const BatchShape& shape) {
  double T = 0.0;
  eval(params, std::span<const BatchShape>(&shape, 1), &T, nullptr);
  return T;
}

std::vector<double> predict_latency_batch(const PerfParams& params, std::span<const BatchShape> shapes) {
  std::vector<double> T(shapes.size());
  if (!shapes.empty()) eval(params, shapes, T.data(), nullptr);
  return T;
}

// goodness_of_fit (perf_model.cpp:51-70): predictions in one device launch,
// the sums folded in the reference's order.
double goodness_of_fit(const PerfParams& params, std::span<const LatencySample> samples) {
  if (samples.size() < 2) throw std::invalid_argument("goodness_of_fit needs at least 2 samples");
  std::vector<BatchShape> shapes(samples.size());
  for (size_t i = 0; i < samples.size(); ++i) shapes[i] = samples[i].shape;
  const std::vector<double> pred = predict_latency_batch(params, shapes);
  double mean = 0.0;
  for (const auto& s : samples) mean += s.observed_ms;
  mean /= static_cast<double>(samples.size());
  double ss_tot = 0.0, ss_res = 0.0;
  for (size_t i = 0; i < samples.size(); ++i) {
    const double r = samples[i].observed_ms - pred[i];
    ss_res += r * r;
    const double d = samples[i].observed_ms - mean;
    ss_tot += d * d;
  }
  if (ss_tot <= 0.0) throw std::invalid_argument("goodness_of_fit undefined: zero variance");
  return 1.0 - ss_res / ss_tot;
}

uint64_t substream_seed(uint64_t root, std::string_view tag, uint64_t index) {
  return nx::substream_seed(root, std::string(tag), index);
}

PerfParams perf_profile(const std::string& name) {
  const nx::Params p = nx::profile_params(name);
  PerfParams q;
  q.tau0 = p.tau0; q.w0 = p.w0; q.ws = p.ws; q.tauB = p.tauB;
  q.tauS = p.tauS; q.p_max = p.p_max; q.kB = p.kB; q.kS = p.kS;
  return q;
}

// ---- LENS ---------------------------------------------------------------------
TargetLatency target_latency(int64_t wait_count, const SLOSpec& slo, const TradeoffModel& tm,
                             double q_ref) {
  nx_target_query q{};
  q.ttft_slo_ms = slo.ttft_slo_ms;
  q.tpot_slo_ms = slo.tpot_slo_ms;
  q.alpha_ms = tm.alpha_ms;
  q.beta = tm.beta;
  q.l_bar = tm.l_bar;
  q.td_min_ms = tm.td_min_ms;
  q.q_ref = q_ref;
  q.wait_count = wait_count;
  raise(nx_target_latency_host(&q, 1));
  return {q.target_ms, q.slo_risk != 0};
}

int64_t binary_search_budget(int64_t b, double target_ms, const PerfParams& params,
                             const SchedulerConfig& cfg, int64_t s_cap) {
  nx_budget_query q{};
  pack(params, q.params);
  q.target_ms = target_ms;
  q.b = b;
  q.m_max = cfg.m_max;
  q.q_max = cfg.q_max;
  q.s_cap = s_cap;
  q.n_search_iters = cfg.n_search_iters;
  raise(nx_budget_search_host(&q, 1));
  return q.budget;
}

std::vector<Allocation> allocate_tokens(std::span<const Request* const> run_q,
                                        std::span<const Request* const> wait_q, int64_t b, int64_t s) {
  nx_allocate_problem p{};
  p.b = b;
  p.s = s;
  p.wait_off = 0;
  p.n_run = to_i32(static_cast<int64_t>(run_q.size()), "allocate_tokens");
  p.n_wait = to_i32(static_cast<int64_t>(wait_q.size()), "allocate_tokens");
  std::vector<int32_t> rem(wait_q.size()), tok(wait_q.size(), 0);
  for (size_t i = 0; i < wait_q.size(); ++i) rem[i] = to_i32(wait_q[i]->remaining_prompt(), "remaining prompt");
  raise(nx_allocate_tokens_host(&p, 1, rem.data(), static_cast<int64_t>(rem.size()), tok.data()));
  std::vector<Allocation> out;
  out.reserve(run_q.size() + static_cast<size_t>(p.n_prefill));
  for (const Request* r : run_q) out.push_back({r->id, 1, false});
  for (int32_t k = 0; k < p.n_prefill; ++k) out.push_back({wait_q[k]->id, tok[k], true});
  return out;
}

BatchPlan schedule_step(std::span<const Request* const> wait_q, std::span<const Request* const> run_q,
                        const SLOSpec& slo, const TradeoffModel& tm, const PerfParams& params,
                        const SchedulerConfig& cfg) {
  if (!cfg.valid()) throw std::invalid_argument("invalid SchedulerConfig");
  nx_lens_problem p{};
  pack(params, p.params);
  p.ttft_slo_ms = slo.ttft_slo_ms;
  p.tpot_slo_ms = slo.tpot_slo_ms;
  p.alpha_ms = tm.alpha_ms;
  p.beta = tm.beta;
  p.l_bar = tm.l_bar;
  p.td_min_ms = tm.td_min_ms;
  p.eps_ratio = cfg.eps_ratio;
  p.q_ref = cfg.q_ref;
  p.m_max = cfg.m_max;
  p.q_max = cfg.q_max;
  p.n_search_iters = cfg.n_search_iters;
  p.n_run = to_i32(static_cast<int64_t>(run_q.size()), "schedule_step");
  p.n_wait = to_i32(static_cast<int64_t>(wait_q.size()), "schedule_step");
  p.wait_off = 0;
  std::vector<int32_t> rem(wait_q.size()), tok(wait_q.size(), 0);
  for (size_t i = 0; i < wait_q.size(); ++i) rem[i] = to_i32(wait_q[i]->remaining_prompt(), "remaining prompt");
  nx_lens_plan plan{};
  raise(nx_lens_schedule_host(&p, 1, rem.data(), static_cast<int64_t>(rem.size()), &plan, tok.data()));
  BatchPlan out;
  out.b = plan.b;
  out.s = plan.s;
  out.predicted_ms = plan.predicted_ms;
  out.target_ms = plan.target_ms;
  out.overload = plan.overload != 0;
  out.allocations.reserve(static_cast<size_t>(plan.n_decode + plan.n_prefill));
  for (int32_t i = 0; i < plan.n_decode; ++i) out.allocations.push_back({run_q[i]->id, 1, false});
  for (int32_t k = 0; k < plan.n_prefill; ++k) out.allocations.push_back({wait_q[k]->id, tok[k], true});
  return out;
}

TradeoffEstimator::TradeoffEstimator(const TradeoffModel& initial)
    : model_(initial), win_ttft_(NX_TRADEOFF_WINDOW, 0.0), win_tpot_(NX_TRADEOFF_WINDOW, 0.0) {}

void TradeoffEstimator::update(std::span<const CompletionStats> completed) {
  nx_tradeoff_state st{};
  st.alpha_ms = model_.alpha_ms;
  st.beta = model_.beta;
  st.l_bar = model_.l_bar;
  st.td_min_ms = model_.td_min_ms;
  st.degenerate_updates = degenerate_updates_;
  std::copy(win_ttft_.begin(), win_ttft_.end(), st.win_ttft);
  std::copy(win_tpot_.begin(), win_tpot_.end(), st.win_tpot);
  st.win_head = win_head_;
  st.win_len = win_len_;
  st.comp_off = 0;
  st.n_new = to_i32(static_cast<int64_t>(completed.size()), "TradeoffEstimator::update");
  std::vector<nx_completion> comp(completed.size());
  for (size_t i = 0; i < completed.size(); ++i)
    comp[i] = {completed[i].ttft_ms, completed[i].tpot_ms, completed[i].decode_len};
  raise(nx_tradeoff_update_host(&st, 1, comp.data(), static_cast<int64_t>(comp.size())));
  model_.alpha_ms = st.alpha_ms;
  model_.beta = st.beta;
  model_.l_bar = st.l_bar;
  degenerate_updates_ = st.degenerate_updates;
  std::copy(st.win_ttft, st.win_ttft + NX_TRADEOFF_WINDOW, win_ttft_.begin());
  std::copy(st.win_tpot, st.win_tpot + NX_TRADEOFF_WINDOW, win_tpot_.begin());
  win_head_ = st.win_head;
  win_len_ = st.win_len;
}

// ---- router -----------------------------------------------------------------------
RouterPolicy router_policy_from_string(const std::string& name) {
  if (name == "prism") return RouterPolicy::kPrism;
  if (name == "round_robin") return RouterPolicy::kRoundRobin;
  if (name == "session_affinity") return RouterPolicy::kSessionAffinity;
  if (name == "least_loaded") return RouterPolicy::kLeastLoaded;
  if (name == "latency_based") return RouterPolicy::kLatencyBased;
  if (name == "weighted") return RouterPolicy::kWeighted;
  throw std::runtime_error("unknown router policy: " + name);
}

std::string to_string(RouterPolicy policy) {
  static const char* names[] = {"prism", "round_robin", "session_affinity", "least_loaded",
                                "latency_based", "weighted"};
  const int i = static_cast<int>(policy);
  return i >= 0 && i < 6 ? names[i] : "?";
}

namespace {
nx_score_query score_query(const StateVector& sv, const SLOSpec* slo, const RouterConfig& cfg,
                           double demand) {
  nx_score_query q{};
  q.l_hat_ms = sv.l_hat_ms;
  q.w_load_tokens = sv.w_load_tokens;
  q.m_free_tokens = sv.m_free_tokens;
  q.p_max = sv.p_max;
  q.demand_tokens = demand;
  q.latency_knee = cfg.latency_knee;
  q.latency_scale_ms = cfg.latency_scale_ms;
  q.ttft_slo_ms = slo ? slo->ttft_slo_ms : 1.0;
  q.load_half_ms = cfg.load_half_ms;
  q.capacity_headroom = cfg.capacity_headroom;
  return q;
}
}  // namespace

double score_latency(const StateVector& sv, const SLOSpec& slo, const RouterConfig& cfg) {
  nx_score_query q = score_query(sv, &slo, cfg, 1.0);
  raise(nx_router_scores_host(&q, 1));
  return q.latency;
}

double score_load(const StateVector& sv, const RouterConfig& cfg) {
  nx_score_query q = score_query(sv, nullptr, cfg, 1.0);
  raise(nx_router_scores_host(&q, 1));
  return q.load;
}

double score_capacity(const StateVector& sv, double req_demand_tokens, const RouterConfig& cfg) {
  nx_score_query q = score_query(sv, nullptr, cfg, req_demand_tokens);
  raise(nx_router_scores_host(&q, 1));
  return q.capacity;
}

Router::Router(const RouterConfig& cfg, const SLOSpec& slo, uint64_t root_seed) : cfg_(cfg), slo_(slo) {
  if (!cfg.valid()) throw std::invalid_argument("invalid RouterConfig");
  raise(nx_rng_state(root_seed, "router", 0, rng_.data()));
}

void Router::register_engine(int engine_id) {
  if (engines_.count(engine_id)) throw std::invalid_argument("engine registered twice");
  order_.push_back(engine_id);
  engines_[engine_id] = EngineInfo{};
}

void Router::on_report(const EngineReport& report) {
  auto it = engines_.find(report.state.engine_id);
  if (it == engines_.end()) throw std::invalid_argument("report from unregistered engine");
  it->second.report = report;
}

void Router::on_completion(int engine_id, const std::string& session_id, double e2e_ms,
                           int64_t decode_len, double now_ms) {
  auto it = engines_.find(engine_id);
  if (it == engines_.end()) return;
  it->second.latencies.emplace_back(now_ms, e2e_ms);
  it->second.latency_sum += e2e_ms;
  l_bar_ema_ += 0.05 * (static_cast<double>(decode_len) - l_bar_ema_);
  if (l_bar_ema_ < 1.0) l_bar_ema_ = 1.0;
  remember_session(session_id, engine_id);
}

// Session memory with the reference's LRU capacity (router.cpp:107-122).
void Router::remember_session(const std::string& session_id, int engine_id) {
  constexpr size_t kSessionCapacity = 100000;
  auto it = sessions_.find(session_id);
  if (it != sessions_.end()) {
    it->second = engine_id;
    session_lru_.erase(std::find(session_lru_.begin(), session_lru_.end(), session_id));
    session_lru_.push_back(session_id);
    return;
  }
  if (sessions_.size() >= kSessionCapacity) {
    sessions_.erase(session_lru_.front());
    session_lru_.pop_front();
  }
  session_lru_.push_back(session_id);
  sessions_[session_id] = engine_id;
}

double Router::score_affinity(int engine_id, const std::string& session_id) const {
  const auto it = sessions_.find(session_id);
  return it != sessions_.end() && it->second == engine_id ? cfg_.beta_aff : 1.0;
}

double Router::demand_estimate_tokens(int64_t prompt_len) const {
  return std::max(1.0, static_cast<double>(prompt_len) + l_bar_ema_);
}

// One Router::route (router.cpp:141-289) = one single-request group on K3.
RouteDecision Router::route(const Request& request, double now_ms) {
  if (order_.empty()) throw std::runtime_error("route: no engines registered");
  const int n = static_cast<int>(order_.size());
  nx_route_group g{};
  for (int i = 0; i < 4; ++i) g.weights[i] = cfg_.weights[i];
  g.beta_aff = cfg_.beta_aff;
  g.latency_knee = cfg_.latency_knee;
  g.latency_scale_ms = cfg_.latency_scale_ms;
  g.load_half_ms = cfg_.load_half_ms;
  g.capacity_headroom = cfg_.capacity_headroom;
  g.staleness_limit_ms = cfg_.staleness_limit_ms;
  g.ttft_slo_ms = slo_.ttft_slo_ms;
  g.l_bar_ema = l_bar_ema_;
  for (int i = 0; i < 4; ++i) g.rng[i] = rng_[i];
  g.rr_next = rr_next_;
  g.policy = static_cast<int32_t>(cfg_.policy);
  g.n_engines = n;
  g.n_requests = 1;
  g.n_sessions = 1;
  std::vector<nx_engine_report> rows(n);
  int32_t affine = -1;
  const auto sit = sessions_.find(request.session_id);
  for (int e = 0; e < n; ++e) {
    EngineInfo& info = engines_.at(order_[e]);
    nx_engine_report& r = rows[e];
    r.engine_id = order_[e];
    r.p_max = 1.0;
    const auto w = cfg_.static_weights.find(order_[e]);
    r.static_weight = w != cfg_.static_weights.end() ? w->second : 1.0;
    if (info.report) {
      const StateVector& sv = info.report->state;
      r.has_report = 1;
      r.l_hat_ms = sv.l_hat_ms;
      r.w_load_tokens = sv.w_load_tokens;
      r.m_free_tokens = sv.m_free_tokens;
      r.p_max = sv.p_max;
      r.reported_at_ms = sv.reported_at_ms;
      r.queue_len = info.report->queue_len;
    }
    if (cfg_.policy == RouterPolicy::kLatencyBased) {  // rolling window (router.cpp:130-139)
      auto& win = info.latencies;
      while (!win.empty() && win.front().first < now_ms - cfg_.latency_window_ms) {
        info.latency_sum -= win.front().second;
        win.pop_front();
      }
      r.rolling_latency_ms = win.empty() ? 0.0 : info.latency_sum / static_cast<double>(win.size());
    }
    if (sit != sessions_.end() && sit->second == order_[e]) affine = e;
  }
  nx_route_request q{};
  q.now_ms = now_ms;
  q.prompt_len = request.prompt_len;
  q.session = 0;
  nx_route_decision d{};
  int32_t status = 0;
  raise(nx_prism_route_host(&g, 1, rows.data(), n, &q, 1, &affine, 1, &d, &status));
  rr_next_ = g.rr_next;
  for (int i = 0; i < 4; ++i) rng_[i] = g.rng[i];
  for (int e = 0; e < n; ++e) {  // dispatch echo into the report view (router.cpp:275-282)
    EngineInfo& info = engines_.at(order_[e]);
    if (info.report) {
      info.report->queue_len = rows[e].queue_len;
      info.report->state.w_load_tokens = rows[e].w_load_tokens;
    }
  }
  RouteDecision out;
  out.engine_id = d.engine_id;
  out.score = d.score;
  for (int i = 0; i < 4; ++i) out.factors[i] = d.factors[i];
  out.degraded = d.degraded != 0;
  remember_session(request.session_id, out.engine_id);
  return out;
}

// ---- online learner ---------------------------------------------------------------
OnlineLearner::OnlineLearner(const PerfParams& priors, const LearnerConfig& cfg) : cfg_(cfg), current_(priors) {
  if (!cfg.valid()) throw std::invalid_argument("invalid LearnerConfig");
  if (!priors.valid()) throw std::invalid_argument("invalid learner priors");
  ring_.reserve(static_cast<size_t>(cfg.long_window));
}

PerfParams OnlineLearner::default_priors() {
  PerfParams p;
  p.p_max = 20.0;
  p.kB = 0.1;
  p.kS = 0.02;
  p.tau0 = 5.0;
  p.w0 = 0.0;
  p.ws = 1.0;
  p.tauB = 0.1;
  p.tauS = 0.001;
  return p;
}

void OnlineLearner::record_sample(const LatencySample& sample) {
  if (!(sample.observed_ms > 0.0) || !sample.shape.valid()) throw std::invalid_argument("invalid LatencySample");
  if (ring_.size() < static_cast<size_t>(cfg_.long_window)) {
    ring_.push_back(sample);
  } else {
    ring_[ring_head_] = sample;
    ring_head_ = (ring_head_ + 1) % ring_.size();
  }
  ++samples_seen_;
  if (samples_seen_ % cfg_.linear_period == 0) update_linear();
  if (samples_seen_ >= cfg_.min_structural_samples && samples_seen_ % cfg_.structural_period == 0)
    update_structural();
}

// One K4 refit on the ring's chronological window (learner.cpp:149-158).
bool OnlineLearner::refit(int kind) {
  const size_t n = ring_.size();
  std::vector<int32_t> b(n), s(n);
  std::vector<double> y(n);
  for (size_t i = 0; i < n; ++i) {
    const LatencySample& x = ring_[(ring_head_ + i) % n];
    b[i] = to_i32(x.shape.b, "LatencySample");
    s[i] = to_i32(x.shape.s, "LatencySample");
    y[i] = x.observed_ms;
  }
  nx_refit_problem p{};
  pack(current_, p.params);
  p.long_window = cfg_.long_window;
  p.short_window = cfg_.short_window;
  p.min_structural_samples = cfg_.min_structural_samples;
  p.sample_off = 0;
  p.n_samples = static_cast<int32_t>(n);
  nx_refit_result r{};
  raise(nx_refit_host(kind, &p, 1, b.data(), s.data(), y.data(), static_cast<int64_t>(n), &r));
  current_ = unpack(r.params);
  int64_t* c[7] = {&counters_.linear_updates, &counters_.structural_updates, &counters_.degenerate_updates,
                   &counters_.rescale_updates, &counters_.clamp_events, &counters_.failed_fits,
                   &counters_.low_identifiability};
  for (int i = 0; i < 7; ++i) *c[i] += r.counters[i];
  return r.updated != 0;
}

bool OnlineLearner::update_linear() { return refit(NX_REFIT_LINEAR); }
bool OnlineLearner::update_structural() { return refit(NX_REFIT_STRUCTURAL); }

double OnlineLearner::convergence_error(std::span<const LatencySample> probe) const {
  if (probe.empty()) throw std::invalid_argument("empty probe");
  std::vector<BatchShape> shapes(probe.size());
  for (size_t i = 0; i < probe.size(); ++i) shapes[i] = probe[i].shape;
  const std::vector<double> pred = predict_latency_batch(current_, shapes);
  double acc = 0.0;
  for (size_t i = 0; i < probe.size(); ++i)
    acc += std::fabs(pred[i] - probe[i].observed_ms) / probe[i].observed_ms;
  return acc / static_cast<double>(probe.size());
}

std::string OnlineLearner::to_json() const {
  nlohmann::ordered_json j;
  j["params"] = nlohmann::ordered_json::parse(current_.to_json());
  j["samples_seen"] = samples_seen_;
  j["buffered"] = buffered();
  j["linear_updates"] = counters_.linear_updates;
  j["structural_updates"] = counters_.structural_updates;
  j["degenerate_updates"] = counters_.degenerate_updates;
  j["rescale_updates"] = counters_.rescale_updates;
  j["clamp_events"] = counters_.clamp_events;
  j["failed_fits"] = counters_.failed_fits;
  j["low_identifiability"] = counters_.low_identifiability;
  return j.dump(2);
}

std::vector<LatencySample> load_samples_jsonl(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open samples file: " + path);
  std::vector<LatencySample> out;
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    try {
      const auto j = nlohmann::json::parse(line);
      LatencySample s;
      s.shape.b = j.at("b").get<int64_t>();
      s.shape.s = j.at("s").get<int64_t>();
      s.observed_ms = j.at("observed_ms").get<double>();
      s.sim_time_ms = j.value("sim_time_ms", 0.0);
      if (!s.shape.valid() || !(s.observed_ms > 0.0)) throw std::runtime_error("invariant violation");
      out.push_back(s);
    } catch (const std::exception& e) {
      throw std::runtime_error(path + ":" + std::to_string(lineno) + ": bad sample record: " + e.what());
    }
  }
  return out;
}

}  // namespace servesim

// =====================================================================================
// Engine policies, metrics, workload, simulation (engine.h, metrics.h, workload.h,
// sim.h). Metrics and workload synthesis are the host front-end's
// (csrc/host/report.cpp, frontend.cpp: reference semantics, host libm for the
// arrival doubles); run_simulation / sweep run on the lockstep kernel.
// =====================================================================================
#include "report.hpp"

#include <filesystem>
#include <sstream>

namespace servesim {

SchedulerPolicy scheduler_policy_from_string(const std::string& name) {
  if (name == "lens") return SchedulerPolicy::kLens;
  if (name == "prefill_priority") return SchedulerPolicy::kPrefillPriority;
  if (name == "static_chunked") return SchedulerPolicy::kStaticChunked;
  throw std::runtime_error("unknown scheduler policy: " + name);
}

std::string to_string(SchedulerPolicy policy) {
  switch (policy) {
    case SchedulerPolicy::kLens: return "lens";
    case SchedulerPolicy::kPrefillPriority: return "prefill_priority";
    case SchedulerPolicy::kStaticChunked: return "static_chunked";
  }
  return "?";
}

// ---- engine simulator (engine.cpp) ---------------------------------------------------
BatchPlan schedule_baseline(SchedulerPolicy policy, std::span<const Request* const> wait_q,
                            std::span<const Request* const> run_q, const PerfParams& params,
                            const EngineConfig& cfg) {
  nx_baseline_problem p{};
  pack(params, p.params);
  p.m_max = cfg.m_max;
  p.q_max = cfg.q_max;
  p.static_budget = cfg.static_budget;
  p.policy = policy == SchedulerPolicy::kPrefillPriority ? NX_SCHED_PREFILL_PRIORITY
             : policy == SchedulerPolicy::kStaticChunked ? NX_SCHED_STATIC_CHUNKED
                                                         : NX_SCHED_LENS;
  p.engine_id = cfg.engine_id;
  p.n_run = to_i32(static_cast<int64_t>(run_q.size()), "schedule_baseline");
  p.n_wait = to_i32(static_cast<int64_t>(wait_q.size()), "schedule_baseline");
  std::vector<int32_t> rem(wait_q.size()), tok(wait_q.size(), 0);
  for (size_t i = 0; i < wait_q.size(); ++i) rem[i] = to_i32(wait_q[i]->remaining_prompt(), "remaining prompt");
  const int rc = nx_baseline_schedule_host(&p, 1, rem.data(), static_cast<int64_t>(rem.size()), tok.data());
  if (rc == NX_ERUNTIME && p.status == NX_ERUNTIME)
    throw std::runtime_error("prefill_priority: prompt exceeds m_max; raise m_max for engine " +
                             std::to_string(cfg.engine_id));
  if (rc == NX_ELOGIC && p.status == NX_ELOGIC) throw std::logic_error("schedule_baseline called with lens policy");
  raise(rc);
  BatchPlan out;
  out.b = p.b;
  out.s = p.s;
  out.predicted_ms = p.predicted_ms;
  out.allocations.reserve(static_cast<size_t>(p.n_decode + p.n_prefill));
  for (int32_t i = 0; i < p.n_decode; ++i) out.allocations.push_back({run_q[i]->id, 1, false});
  for (int32_t k = 0; k < p.n_prefill; ++k) out.allocations.push_back({wait_q[k]->id, tok[k], true});
  return out;
}

EngineSim::EngineSim(const EngineConfig& cfg, const SLOSpec& slo, const SchedulerConfig& sched,
                     const TradeoffModel& tradeoff_init, const LearnerConfig& learner_cfg, uint64_t root_seed)
    : cfg_(cfg),
      slo_(slo),
      sched_(sched),
      learner_(OnlineLearner::default_priors(), learner_cfg),
      tradeoff_(tradeoff_init),
      noise_(substream_seed(root_seed, "engine-noise", static_cast<uint64_t>(cfg.engine_id))) {
  if (!cfg_.valid()) throw std::invalid_argument("invalid EngineConfig");
  sched_.m_max = cfg_.m_max;  // the engine's own batch caps win (engine.cpp:122-124)
  sched_.q_max = cfg_.q_max;
  if (!sched_.valid()) throw std::invalid_argument("invalid SchedulerConfig");
}

// Ground truth T_true(shape) * exp(sigma z) on the engine's noise stream
// (engine.cpp:128-132); T_true is a K1 launch.
double EngineSim::oracle_latency(const BatchShape& shape) {
  const double t = predict_latency(cfg_.true_params, shape);
  return cfg_.noise_sigma == 0.0 ? t : t * std::exp(cfg_.noise_sigma * noise_.normal());
}

int64_t EngineSim::cached_prefix_tokens(const std::string& session) const {
  const auto it = prefixes_.find(session);
  return it == prefixes_.end() ? 0 : it->second.tokens;
}

void EngineSim::drop_prefix(std::unordered_map<std::string, Prefix>::iterator it) {
  cached_ -= it->second.blocks;
  lru_.erase(it->second.stamp);
  prefixes_.erase(it);
}

// Reclaim least-recently-finished prefixes until the cache fits the free
// blocks (engine.cpp:285-292).
void EngineSim::shrink_cache() {
  while (cached_ > free_blocks() && !lru_.empty()) drop_prefix(prefixes_.find(lru_.begin()->second));
}

void EngineSim::keep_prefix(const std::string& session, int64_t tokens) {
  if (const auto it = prefixes_.find(session); it != prefixes_.end()) drop_prefix(it);
  const uint64_t stamp = next_stamp_++;
  prefixes_[session] = Prefix{tokens, blocks(tokens), stamp};
  lru_.emplace(stamp, session);
  cached_ += blocks(tokens);
  shrink_cache();
}

// admit (engine.cpp:139-169): a cached prefix of the session credits up to
// prompt - 1 tokens when its blocks fit beside the committed ones.
bool EngineSim::admit(Request* request, double now_ms) {
  (void)now_ms;
  if (request->state != RequestState::kWaiting) throw std::invalid_argument("admit: request not in waiting state");
  if (cfg_.wait_cap > 0 && static_cast<int64_t>(wait_q_.size()) >= cfg_.wait_cap) return false;
  if (const auto it = prefixes_.find(request->session_id); it != prefixes_.end()) {
    const int64_t credit = std::min(it->second.tokens, request->prompt_len - 1);
    const int64_t need = blocks(credit);
    if (credit > 0 && pinned_ + reserved_ + need <= cfg_.kv_blocks) {
      drop_prefix(it);
      request->prefilled = credit;
      request->precredited = credit;
      pinned_ += need;
    }
  }
  wait_q_.push_back(request);
  live_[request->id] = request;
  return true;
}

// trim_for_kv (engine.cpp:185-213): a waiter's first prefill reserves its
// whole footprint; the first one that does not fit ends the admissible FCFS
// prefix of new prefills (decodes and already-admitted prefills stay).
void EngineSim::admit_prefills(BatchPlan& plan) {
  std::vector<Allocation> keep;
  keep.reserve(plan.allocations.size());
  bool full = false;
  for (const Allocation& a : plan.allocations) {
    Request* r = live_.at(a.request_id);
    if (!a.is_prefill || r->kv_admitted) {
      keep.push_back(a);
      continue;
    }
    if (full) continue;
    const int64_t grow = blocks(r->prompt_len + r->target_decode) - blocks(r->prefilled + r->decoded);
    if (pinned_ + reserved_ + grow > cfg_.kv_blocks) {
      full = true;
      continue;
    }
    reserved_ += grow;
    r->kv_admitted = true;
    keep.push_back(a);
  }
  if (keep.size() == plan.allocations.size()) return;
  plan.allocations = std::move(keep);
  plan.b = static_cast<int64_t>(plan.allocations.size());
  plan.s = 0;
  for (const Allocation& a : plan.allocations) plan.s += a.tokens;
  plan.predicted_ms = plan.b > 0 ? predict_latency(learner_.params(), {plan.b, plan.s}) : 0.0;
}

std::optional<double> EngineSim::begin_step(double now_ms) {
  if (busy()) throw std::logic_error("begin_step on a busy engine");
  if (!has_work()) return std::nullopt;
  const std::vector<const Request*> run(run_q_.begin(), run_q_.end());
  const std::vector<const Request*> wait(wait_q_.begin(), wait_q_.end());
  BatchPlan plan = cfg_.scheduler_policy == SchedulerPolicy::kLens
                       ? schedule_step(wait, run, slo_, tradeoff_.model(), learner_.params(), sched_)
                       : schedule_baseline(cfg_.scheduler_policy, wait, run, learner_.params(), cfg_);
  if (plan.empty()) return std::nullopt;
  admit_prefills(plan);
  if (plan.empty()) return std::nullopt;
  const double actual = oracle_latency({plan.b, plan.s});
  step_ = Step{std::move(plan), now_ms, actual};
  return actual;
}

// complete_step (engine.cpp:226-283): token and block accounting per
// allocation, first-token / finish transitions, prefix caching of finished
// sessions, then one tradeoff refit over this step's completions.
StepOutcome EngineSim::complete_step(double now_ms) {
  if (!busy()) throw std::logic_error("complete_step on an idle engine");
  StepOutcome out;
  out.plan = std::move(step_->plan);
  out.actual_ms = step_->actual_ms;
  step_.reset();
  std::vector<CompletionStats> done;
  for (const Allocation& a : out.plan.allocations) {
    Request* r = live_.at(a.request_id);
    const int64_t before = blocks(r->prefilled + r->decoded);
    if (a.is_prefill) {
      r->prefilled += a.tokens;
      r->allocated_prefill += a.tokens;
    } else {
      r->decoded += 1;
      r->allocated_decode += 1;
    }
    const int64_t grew = blocks(r->prefilled + r->decoded) - before;
    pinned_ += grew;
    reserved_ -= grew;
    if (a.is_prefill) {
      if (r->prefilled != r->prompt_len) continue;
      r->state = RequestState::kRunning;
      r->first_token_ms = now_ms;
      out.first_tokens.push_back(r->id);
      wait_q_.erase(std::find(wait_q_.begin(), wait_q_.end(), r));
      run_q_.push_back(r);
    } else if (r->decoded == r->target_decode) {
      r->state = RequestState::kFinished;
      out.finished.push_back(r->id);
      CompletionStats c;
      c.ttft_ms = *r->first_token_ms - r->arrival_ms;
      c.decode_len = r->target_decode;
      c.tpot_ms = r->target_decode >= 2
                      ? (now_ms - *r->first_token_ms) / static_cast<double>(r->target_decode - 1)
                      : 0.0;
      done.push_back(c);
      pinned_ -= blocks(r->prefilled + r->decoded);
      keep_prefix(r->session_id, r->prefilled + r->decoded);
      run_q_.erase(std::find(run_q_.begin(), run_q_.end(), r));
      live_.erase(r->id);
    }
  }
  shrink_cache();
  if (!done.empty()) tradeoff_.update(done);
  return out;
}

// export_state (engine.cpp:307-332).
StateVector EngineSim::export_state(double now_ms) const {
  StateVector v;
  v.engine_id = cfg_.engine_id;
  v.reported_at_ms = now_ms;
  v.p_max = learner_.params().p_max;
  if (step_) v.l_hat_ms = std::max(0.0, step_->plan.predicted_ms - (now_ms - step_->started_ms));
  const double l_bar = tradeoff_.model().l_bar;
  double prefill = 0.0, demand = 0.0;
  for (const Request* r : wait_q_) {
    const double left = static_cast<double>(r->remaining_prompt());
    prefill += left;
    demand += left + l_bar;
  }
  v.w_load_tokens = prefill + 32.0 * static_cast<double>(wait_q_.size() + run_q_.size());
  v.m_free_tokens = std::max(0.0, static_cast<double>(free_blocks() * cfg_.block_size) - demand);
  return v;
}

// check_kv_consistency (engine.cpp:334-361).
void EngineSim::check_kv_consistency() const {
  int64_t held = 0;
  for (const auto& kv : live_) held += blocks(kv.second->prefilled + kv.second->decoded);
  if (held != pinned_) throw std::logic_error("kv accounting drift: pinned mismatch");
  if (pinned_ + free_blocks() != cfg_.kv_blocks) throw std::logic_error("kv conservation violated");
  if (pinned_ < 0 || reserved_ < 0 || cached_ < 0) throw std::logic_error("negative kv counter");
  if (pinned_ + reserved_ > cfg_.kv_blocks) throw std::logic_error("kv oversubscribed");
  if (cached_ > free_blocks()) throw std::logic_error("prefix cache exceeds free space");
  int64_t cache = 0;
  for (const auto& kv : prefixes_) cache += kv.second.blocks;
  if (cache != cached_) throw std::logic_error("kv accounting drift: cache mismatch");
}

// ---- metrics ------------------------------------------------------------------------
namespace {
nx::RecordRow row_of(const RequestRecord& r) {
  return {static_cast<int64_t>(r.request_id), r.arrival_ms, r.first_token_ms, r.completed_ms,
          r.prompt_tokens, r.output_tokens, r.engine_id};
}
std::vector<nx::RecordRow> rows_of(std::span<const RequestRecord> recs) {
  std::vector<nx::RecordRow> v;
  v.reserve(recs.size());
  for (const auto& r : recs) v.push_back(row_of(r));
  return v;
}
}  // namespace

RequestMetrics request_metrics(const RequestRecord& rec) {
  if (!(rec.arrival_ms <= rec.first_token_ms && rec.first_token_ms <= rec.completed_ms))
    throw std::invalid_argument("RequestRecord timestamps out of order");
  RequestMetrics m;
  m.ttft_ms = rec.first_token_ms - rec.arrival_ms;
  m.e2e_ms = rec.completed_ms - rec.arrival_ms;
  m.single_token = rec.output_tokens < 2;
  m.tpot_ms = m.single_token ? 0.0
                             : (rec.completed_ms - rec.first_token_ms) / static_cast<double>(rec.output_tokens - 1);
  return m;
}

double percentile(std::vector<double> values, double p) { return nx::percentile_nearest_rank(std::move(values), p); }

SloAttainment slo_attainment(std::span<const RequestRecord> records, const SLOSpec& slo) {
  if (records.empty()) return {100.0, true};
  return {nx::summarize_records(rows_of(records), slo.ttft_slo_ms, slo.tpot_slo_ms).slo_pct, false};
}

MetricsSummary summarize(std::span<const RequestRecord> records, const SLOSpec& slo) {
  const nx::Metrics m = nx::summarize_records(rows_of(records), slo.ttft_slo_ms, slo.tpot_slo_ms);
  MetricsSummary out;
  out.completed = m.completed;
  out.p50_e2e_ms = m.p50_e2e;
  out.p90_e2e_ms = m.p90_e2e;
  out.p50_ttft_ms = m.p50_ttft;
  out.p50_tpot_ms = m.p50_tpot;
  out.mean_ttft_ms = m.mean_ttft;
  out.mean_tpot_ms = m.mean_tpot;
  out.slo_attainment_pct = m.slo_pct;
  out.engine_share = m.engine_share;
  return out;
}

void write_requests_csv(const std::string& path, std::span<const RequestRecord> records) {
  nx::write_requests_csv(path, rows_of(records));
}

// ---- workload -----------------------------------------------------------------------
namespace {
ScenarioStats stats_of(const nx::Scenario& s) {
  ScenarioStats o;
  o.name = s.name;
  o.prompt = {s.prompt.mean, s.prompt.p99, s.prompt.std_dev};
  o.output = {s.output.mean, s.output.p99, s.output.std_dev};
  o.session_turn_prob = s.session_turn_prob;
  return o;
}
nx::Scenario scenario_of(const ScenarioStats& s) {
  nx::Scenario o;
  o.name = s.name;
  o.prompt = {s.prompt.mean, s.prompt.p99, s.prompt.std_dev};
  o.output = {s.output.mean, s.output.p99, s.output.std_dev};
  o.session_turn_prob = s.session_turn_prob;
  return o;
}
std::vector<TraceRecord> records_of(const std::vector<nx::TraceRow>& rows) {
  std::vector<TraceRecord> out;
  out.reserve(rows.size());
  for (const auto& r : rows) out.push_back({r.arrival_ms, r.session, r.prompt, r.output});
  return out;
}
std::vector<nx::TraceRow> trace_rows_of(const std::vector<TraceRecord>& recs) {
  std::vector<nx::TraceRow> out;
  out.reserve(recs.size());
  for (const auto& r : recs) out.push_back({r.arrival_ms, r.session_id, r.prompt_tokens, r.output_tokens});
  return out;
}
}  // namespace

std::vector<std::string> scenario_names() { return {"flowgpt", "coding", "sharegpt", "summarization"}; }

const ScenarioStats& scenario_by_name(const std::string& name) {
  static const std::map<std::string, ScenarioStats> table = [] {
    std::map<std::string, ScenarioStats> t;
    for (const auto& n : scenario_names()) t[n] = stats_of(nx::scenario_named(n));
    return t;
  }();
  const auto it = table.find(name);
  if (it == table.end()) throw std::runtime_error("unknown scenario: " + name);
  return it->second;
}

ScenarioStats load_scenario_json(const std::string& path) { return stats_of(nx::scenario_from_file(path)); }

std::vector<TraceRecord> load_trace(const std::string& path, bool* sorted_warning) {
  return records_of(nx::load_trace_rows(path, sorted_warning));
}

void write_trace(const std::string& path, const std::vector<TraceRecord>& records) {
  nx::write_trace_rows(path, trace_rows_of(records));
}

std::vector<TraceRecord> synth_generate(const ScenarioStats& stats, int64_t n, uint64_t seed) {
  if (!stats.valid()) throw std::invalid_argument("invalid ScenarioStats");
  return records_of(nx::synth_rows(scenario_of(stats), n, seed));
}

std::vector<TraceRecord> assign_arrivals(std::vector<TraceRecord> records, ArrivalMode mode, double rate_per_s,
                                         uint64_t seed, double time_scale, bool poisson) {
  std::vector<nx::TraceRow> rows = trace_rows_of(records);
  nx::assign_arrival_times(rows, mode == ArrivalMode::kTimestamp, rate_per_s, seed, time_scale, poisson);
  return records_of(rows);
}

// ---- simulation -----------------------------------------------------------------------
namespace {
nlohmann::ordered_json params_json(const PerfParams& p) { return nlohmann::ordered_json::parse(p.to_json()); }

PerfParams params_of(const nx::Params& p) {
  PerfParams q;
  q.tau0 = p.tau0; q.w0 = p.w0; q.ws = p.ws; q.tauB = p.tauB;
  q.tauS = p.tauS; q.p_max = p.p_max; q.kB = p.kB; q.kS = p.kS;
  return q;
}
}  // namespace

// RunConfig in the schema RunConfig::from_json_text reads (sim.cpp:454-582):
// every field explicit, so parsing it back yields this RunConfig exactly.
std::string RunConfig::to_json_text() const {
  nlohmann::ordered_json j;
  j["seed"] = seed;
  j["duration_ms"] = duration_ms;
  j["record_learner_history"] = record_learner_history;
  j["slo"] = {{"ttft_slo_ms", slo.ttft_slo_ms}, {"tpot_slo_ms", slo.tpot_slo_ms}};
  j["scheduler"] = {{"m_max", scheduler.m_max}, {"q_max", scheduler.q_max},
                    {"n_search_iters", scheduler.n_search_iters}, {"eps_ratio", scheduler.eps_ratio},
                    {"q_ref", scheduler.q_ref}};
  j["tradeoff"] = {{"alpha_ms", tradeoff.alpha_ms}, {"beta", tradeoff.beta}, {"l_bar", tradeoff.l_bar},
                   {"td_min_ms", tradeoff.td_min_ms}};
  j["learner"] = {{"long_window", learner.long_window}, {"short_window", learner.short_window},
                  {"structural_period", learner.structural_period}, {"linear_period", learner.linear_period},
                  {"min_structural_samples", learner.min_structural_samples}};
  nlohmann::ordered_json r;
  r["policy"] = to_string(router.policy);
  r["weights"] = std::vector<double>(router.weights.begin(), router.weights.end());
  r["beta_aff"] = router.beta_aff;
  r["latency_knee"] = router.latency_knee;
  r["latency_scale_ms"] = router.latency_scale_ms;
  r["load_half_ms"] = router.load_half_ms;
  r["capacity_headroom"] = router.capacity_headroom;
  r["staleness_limit_ms"] = router.staleness_limit_ms;
  r["latency_window_ms"] = router.latency_window_ms;
  nlohmann::ordered_json sw = nlohmann::ordered_json::object();
  for (const auto& [id, w] : router.static_weights) sw[std::to_string(id)] = w;
  r["static_weights"] = sw;
  j["router"] = r;
  nlohmann::ordered_json es = nlohmann::ordered_json::array();
  for (const auto& e : engines) {
    nlohmann::ordered_json x;
    x["engine_id"] = e.engine_id;
    x["true_params"] = params_json(e.true_params);
    x["noise_sigma"] = e.noise_sigma;
    x["kv_blocks"] = e.kv_blocks;
    x["block_size"] = e.block_size;
    x["m_max"] = e.m_max;
    x["q_max"] = e.q_max;
    x["scheduler_policy"] = to_string(e.scheduler_policy);
    x["static_budget"] = e.static_budget;
    x["state_report_period_ms"] = e.state_report_period_ms;
    x["state_staleness_ms"] = e.state_staleness_ms;
    x["wait_cap"] = e.wait_cap;
    es.push_back(x);
  }
  j["engines"] = es;
  j["workload"] = {{"scenario", workload.scenario}, {"scenario_file", workload.scenario_file},
                   {"trace", workload.trace_path},
                   {"mode", workload.mode == ArrivalMode::kQps ? "qps" : "timestamp"},
                   {"rate", workload.rate_per_s}, {"n", workload.n}, {"time_scale", workload.time_scale},
                   {"poisson", workload.poisson}};
  j["output"] = {{"dir", output.dir}, {"summary", output.summary}, {"requests_csv", output.requests_csv},
                 {"plans_jsonl", output.plans_jsonl}, {"routing_jsonl", output.routing_jsonl}};
  return j.dump();
}

RunConfig RunConfig::from_json_text(const std::string& text) {
  const nx::RunCfg c = nx::parse_run_config(text);  // reference defaults + validation
  RunConfig o;
  o.seed = c.seed;
  o.duration_ms = c.duration_ms;
  o.record_learner_history = c.record_learner_history;
  o.slo = {c.ttft_slo, c.tpot_slo};
  o.scheduler.m_max = c.m_max;
  o.scheduler.q_max = c.q_max;
  o.scheduler.n_search_iters = c.n_search_iters;
  o.scheduler.eps_ratio = c.eps_ratio;
  o.scheduler.q_ref = c.q_ref;
  o.tradeoff = {c.alpha, c.beta, c.l_bar, c.td_min};
  o.learner = {c.long_window, c.short_window, c.structural_period, c.linear_period, c.min_structural};
  o.router.policy = static_cast<RouterPolicy>(c.route_policy);
  for (int i = 0; i < 4; ++i) o.router.weights[i] = c.weights[i];
  o.router.beta_aff = c.beta_aff;
  o.router.latency_knee = c.knee;
  o.router.latency_scale_ms = c.scale_ms;
  o.router.load_half_ms = c.load_half;
  o.router.capacity_headroom = c.headroom;
  o.router.staleness_limit_ms = c.staleness_limit;
  o.router.latency_window_ms = c.latency_window;
  o.router.static_weights = c.static_weights;
  for (const auto& e : c.engines) {
    EngineConfig x;
    x.engine_id = e.engine_id;
    x.true_params = params_of(e.true_params);
    x.noise_sigma = e.noise_sigma;
    x.kv_blocks = e.kv_blocks;
    x.block_size = e.block_size;
    x.m_max = e.m_max;
    x.q_max = e.q_max;
    x.scheduler_policy = static_cast<SchedulerPolicy>(e.policy);
    x.static_budget = e.static_budget;
    x.state_report_period_ms = e.report_period_ms;
    x.state_staleness_ms = e.staleness_ms;
    x.wait_cap = e.wait_cap;
    o.engines.push_back(x);
  }
  o.workload.scenario = c.scenario;
  o.workload.scenario_file = c.scenario_file;
  o.workload.trace_path = c.trace_path;
  o.workload.mode = c.timestamp_mode ? ArrivalMode::kTimestamp : ArrivalMode::kQps;
  o.workload.rate_per_s = c.rate;
  o.workload.n = c.n;
  o.workload.time_scale = c.time_scale;
  o.workload.poisson = c.poisson;
  o.output = {c.out_dir, c.out_summary, c.out_requests_csv, c.out_plans_jsonl, c.out_routing_jsonl};
  return o;
}

RunConfig RunConfig::from_json_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open config: " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  try {
    return from_json_text(buf.str());
  } catch (const std::exception& e) {
    throw std::runtime_error(path + ": " + e.what());
  }
}

void RunConfig::validate() const {
  // the front-end's validator carries the reference's checks and messages
  // (RunConfig::validate, sim.cpp:418-452); reaching it through the JSON
  // form also exercises this config's round trip.
  if (engines.empty()) throw std::runtime_error("config: needs >= 1 engine");
  nx::validate_run_config(nx::parse_run_config(to_json_text()));
}

namespace {
void raise_replica(nx_sim_t h, int32_t r, const nx_replica_summary& s) {
  char buf[512];
  nx_sim_error(h, r, buf, sizeof buf);
  std::string msg = buf;
  if (msg.empty()) msg = "device replica failed";
  if (s.status == NX_EINVAL) throw std::invalid_argument(msg);
  if (s.status == NX_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

struct SimHandle {
  nx_sim_t h = nullptr;
  ~SimHandle() {
    if (h) nx_sim_destroy(h);
  }
};

RunResult result_of(nx_sim_t h, int32_t r, const nx_replica_summary& s) {
  RunResult out;
  out.arrived = s.arrived;
  out.completed = s.completed;
  out.rejected = s.rejected;
  out.unfinished = s.unfinished;
  out.arrival_hash = s.arrival_hash;
  out.event_hash = s.event_hash;
  std::vector<nx_request_record> recs(static_cast<size_t>(s.completed));
  int64_t n = 0;
  raise(nx_sim_records(h, r, recs.data(), s.completed, &n));
  for (const auto& x : recs)
    out.records.push_back({static_cast<uint64_t>(x.request_id), x.arrival_ms, x.first_token_ms, x.completed_ms,
                           x.prompt_tokens, x.output_tokens, x.engine_id});
  int64_t len = 0;
  raise(nx_sim_summary_json(h, r, nullptr, 0, &len));
  out.summary_json.assign(static_cast<size_t>(len) + 1, '\0');
  raise(nx_sim_summary_json(h, r, out.summary_json.data(), len + 1, &len));
  out.summary_json.resize(static_cast<size_t>(len));
  raise(nx_sim_learner_history(h, r, nullptr, 0, &n));
  std::vector<nx_learner_snapshot> hist(static_cast<size_t>(n));
  raise(nx_sim_learner_history(h, r, hist.data(), n, &n));
  for (const auto& x : hist) out.learner_history.push_back({x.engine_id, x.sim_time_ms, x.samples_seen, unpack(x.params)});
  return out;
}
}  // namespace

std::vector<RunResult> run_replicas(std::span<const RunConfig> cfgs, int device) {
  std::vector<std::string> texts;
  std::vector<const char*> ptrs;
  for (const auto& c : cfgs) {
    c.validate();
    texts.push_back(c.to_json_text());
  }
  for (const auto& t : texts) ptrs.push_back(t.c_str());
  SimHandle S;
  raise(nx_sim_create_json(ptrs.data(), static_cast<int32_t>(ptrs.size()), device, 1, &S.h));
  raise(nx_sim_run(S.h));
  std::vector<nx_replica_summary> sums(cfgs.size());
  raise(nx_sim_summaries(S.h, sums.data()));
  std::vector<RunResult> out;
  for (size_t r = 0; r < cfgs.size(); ++r) {
    if (sums[r].status != NX_OK) raise_replica(S.h, static_cast<int32_t>(r), sums[r]);
    const RunConfig& c = cfgs[r];
    RunResult res = result_of(S.h, static_cast<int32_t>(r), sums[r]);
    res.metrics = summarize(res.records, c.slo);
    if (!c.output.dir.empty()) raise(nx_sim_write_outputs(S.h, static_cast<int32_t>(r)));
    out.push_back(std::move(res));
  }
  return out;
}

RunResult run_simulation(const RunConfig& cfg) {
  return std::move(run_replicas(std::span<const RunConfig>(&cfg, 1))[0]);
}

SweepAxis sweep_axis_from_string(const std::string& name) {
  if (name == "rate") return SweepAxis::kRate;
  if (name == "policy") return SweepAxis::kPolicy;
  if (name == "budget") return SweepAxis::kBudget;
  throw std::runtime_error("unknown sweep axis: " + name);
}

// sweep (sim.cpp:608-642): every value that forms a valid config becomes one
// replica of a single device batch instead of one sequential run each;
// per-value failures are recorded in their rows.
SweepResult sweep(const RunConfig& base, SweepAxis axis, const std::vector<std::string>& values) {
  SweepResult out;
  out.axis = axis;
  std::vector<RunConfig> cfgs;
  std::vector<size_t> row_of_cfg;
  for (const std::string& value : values) {
    SweepRow row;
    row.value = value;
    try {
      RunConfig cfg = base;
      cfg.output.dir.clear();
      switch (axis) {
        case SweepAxis::kRate:
          cfg.workload.mode = ArrivalMode::kQps;
          cfg.workload.rate_per_s = std::stod(value);
          break;
        case SweepAxis::kPolicy: {
          const SchedulerPolicy policy = scheduler_policy_from_string(value);
          for (auto& e : cfg.engines) e.scheduler_policy = policy;
          break;
        }
        case SweepAxis::kBudget: {
          const int64_t budget = std::stoll(value);
          for (auto& e : cfg.engines) e.static_budget = budget;
          break;
        }
      }
      cfg.validate();
      cfgs.push_back(cfg);
      row_of_cfg.push_back(out.rows.size());
    } catch (const std::exception& e) {
      row.error = e.what();
    }
    out.rows.push_back(std::move(row));
  }
  // a workload that fails to build (e.g. an unreadable trace) fails only its
  // own row, like the reference's per-value try/catch (sim.cpp:608-642)
  {
    std::vector<RunConfig> keep;
    std::vector<size_t> keep_row;
    for (size_t k = 0; k < cfgs.size(); ++k) {
      const std::string t = cfgs[k].to_json_text();
      uint64_t ah = 0;
      int64_t nr = 0, ns = 0;
      if (nx_workload_info(t.c_str(), &ah, &nr, &ns) != NX_OK) {
        out.rows[row_of_cfg[k]].error = nx_last_error();
        continue;
      }
      keep.push_back(cfgs[k]);
      keep_row.push_back(row_of_cfg[k]);
    }
    cfgs = std::move(keep);
    row_of_cfg = std::move(keep_row);
  }
  if (cfgs.empty()) return out;
  std::vector<std::string> texts;
  std::vector<const char*> ptrs;
  for (const auto& c : cfgs) texts.push_back(c.to_json_text());
  for (const auto& t : texts) ptrs.push_back(t.c_str());
  SimHandle S;
  const int rc = nx_sim_create_json(ptrs.data(), static_cast<int32_t>(ptrs.size()), 0, 1, &S.h);
  if (rc != NX_OK) {  // a workload that fails to build fails its sweep rows
    const std::string msg = nx_last_error();
    for (size_t i : row_of_cfg) out.rows[i].error = msg;
    return out;
  }
  raise(nx_sim_run(S.h));
  std::vector<nx_replica_summary> sums(cfgs.size());
  raise(nx_sim_summaries(S.h, sums.data()));
  for (size_t k = 0; k < cfgs.size(); ++k) {
    SweepRow& row = out.rows[row_of_cfg[k]];
    try {
      if (sums[k].status != NX_OK) raise_replica(S.h, static_cast<int32_t>(k), sums[k]);
      row.result = result_of(S.h, static_cast<int32_t>(k), sums[k]);
      row.result.metrics = summarize(row.result.records, cfgs[k].slo);
      row.ok = true;
    } catch (const std::exception& e) {
      row.error = e.what();
    }
  }
  return out;
}

std::string sweep_csv(const SweepResult& result) {
  std::ostringstream out;
  out << "value,arrived,completed,rejected,unfinished,mean_ttft_ms,mean_tpot_ms,p50_e2e_ms,p90_e2e_ms,"
         "p50_ttft_ms,p50_tpot_ms,slo_attainment,arrival_hash,error\n";
  char buf[360];
  for (const auto& row : result.rows) {
    if (!row.ok) {
      out << row.value << ",,,,,,,,,,,,,\"" << row.error << "\"\n";
      continue;
    }
    const auto& r = row.result;
    const auto& m = r.metrics;
    std::snprintf(buf, sizeof buf, "%s,%lld,%lld,%lld,%lld,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f,%016llx,\n",
                  row.value.c_str(), static_cast<long long>(r.arrived), static_cast<long long>(r.completed),
                  static_cast<long long>(r.rejected), static_cast<long long>(r.unfinished), m.mean_ttft_ms,
                  m.mean_tpot_ms, m.p50_e2e_ms, m.p90_e2e_ms, m.p50_ttft_ms, m.p50_tpot_ms,
                  m.slo_attainment_pct, static_cast<unsigned long long>(r.arrival_hash));
    out << buf;
  }
  return out.str();
}

}  // namespace servesim
