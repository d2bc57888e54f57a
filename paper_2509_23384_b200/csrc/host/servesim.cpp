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
