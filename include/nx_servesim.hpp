// nx_servesim.hpp — C++ drop-in for the reference's perf-model, scheduler,
// router and learner interfaces (proj/include/servesim/{perf_model,lens,
// router,learner,rng,engine}.h), backed by the B200 path.
//
// Same namespace, type names, fields, defaults, signatures and exception
// classes as the reference, so its callers (and its own unit tests,
// tests/refsuite) compile unchanged against this header. Every model
// evaluation and scheduling decision runs on the device through the C-ABI
// (include/nx_sched.h); what stays on the host is object state the
// reference keeps in std containers (sample rings, completion windows,
// report tables, session maps) and JSON I/O.
//
// Link: paper_2509_23384_b200/_nxsched.so (which contains this API).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <deque>
#include <map>
#include <numbers>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <unordered_map>
#include <utility>
#include <vector>

namespace servesim {

// ---- perf model (perf_model.h:14-54) -----------------------------------------------
struct PerfParams {
  double tau0 = 0.0;
  double w0 = 0.0;
  double ws = 1.0;
  double tauB = 0.0;
  double tauS = 0.0;
  double p_max = 1.0;
  double kB = 1.0;
  double kS = 1.0;

  bool valid() const;
  std::string to_json() const;
  static PerfParams from_json(const std::string& text);
};

struct BatchShape {
  int64_t b = 1;
  int64_t s = 1;
  bool valid() const { return b >= 1 && s >= b; }
};

struct LatencySample {
  BatchShape shape;
  double observed_ms = 0.0;
  double sim_time_ms = 0.0;
};

double throughput(const PerfParams& params, const BatchShape& shape);
double predict_latency(const PerfParams& params, const BatchShape& shape);
double goodness_of_fit(const PerfParams& params, std::span<const LatencySample> samples);

// Batched forms (one device launch): out[i] for shapes[i].
std::vector<double> predict_latency_batch(const PerfParams& params, std::span<const BatchShape> shapes);

// ---- deterministic RNG (rng.h) -----------------------------------------------------
class Rng {
 public:
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s_) w = splitmix64(x);
  }
  uint64_t next_u64() {
    const uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
  }
  double uniform() { return (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return n ? next_u64() % n : 0; }
  double normal() {
    const double u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
  }
  static uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  const std::array<uint64_t, 4>& state() const { return s_; }

 private:
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  std::array<uint64_t, 4> s_{};
};

uint64_t substream_seed(uint64_t root, std::string_view tag, uint64_t index = 0);

// ---- engine-facing types (engine.h) -------------------------------------------------
enum class SchedulerPolicy { kLens, kPrefillPriority, kStaticChunked };
SchedulerPolicy scheduler_policy_from_string(const std::string& name);
std::string to_string(SchedulerPolicy policy);

PerfParams perf_profile(const std::string& name);

struct EngineConfig {
  int engine_id = 0;
  PerfParams true_params;
  double noise_sigma = 0.05;
  int64_t kv_blocks = 8192;
  int64_t block_size = 16;
  int64_t m_max = 8192;
  int64_t q_max = 256;
  SchedulerPolicy scheduler_policy = SchedulerPolicy::kLens;
  int64_t static_budget = 2048;
  double state_report_period_ms = 100.0;
  double state_staleness_ms = 0.0;
  int64_t wait_cap = 0;
  bool valid() const {
    return kv_blocks > 0 && block_size >= 1 && noise_sigma >= 0.0 && static_budget >= 1 &&
           static_budget <= m_max && m_max >= q_max && q_max >= 1 && state_report_period_ms > 0.0 &&
           state_staleness_ms >= 0.0 && wait_cap >= 0 && true_params.valid();
  }
};

struct StateVector {
  int engine_id = 0;
  double l_hat_ms = 0.0;
  double w_load_tokens = 0.0;
  double m_free_tokens = 0.0;
  double p_max = 1.0;
  double reported_at_ms = 0.0;
  bool valid() const {
    return l_hat_ms >= 0.0 && w_load_tokens >= 0.0 && m_free_tokens >= 0.0 && p_max > 0.0;
  }
};

struct EngineReport {
  StateVector state;
  int64_t queue_len = 0;
};

// ---- LENS (lens.h) -----------------------------------------------------------------
struct SLOSpec {
  double ttft_slo_ms = 2000.0;
  double tpot_slo_ms = 12.0;
  bool valid() const { return ttft_slo_ms > 0.0 && tpot_slo_ms > 0.0; }
};

struct TradeoffModel {
  double alpha_ms = 2000.0;
  double beta = 16.0;
  double l_bar = 128.0;
  double td_min_ms = 2.0;
  bool valid() const { return beta > 0.0 && l_bar >= 1.0 && td_min_ms > 0.0; }
  static TradeoffModel initial_for(const SLOSpec& slo) {
    TradeoffModel tm;
    tm.alpha_ms = 2.0 * slo.ttft_slo_ms;
    tm.beta = slo.ttft_slo_ms / slo.tpot_slo_ms;
    return tm;
  }
};

enum class RequestState { kWaiting, kRunning, kFinished };

struct Request {
  uint64_t id = 0;
  std::string session_id;
  int64_t prompt_len = 1;
  int64_t prefilled = 0;
  int64_t decoded = 0;
  int64_t target_decode = 1;
  int64_t precredited = 0;
  double arrival_ms = 0.0;
  std::optional<double> first_token_ms;
  RequestState state = RequestState::kWaiting;
  bool kv_admitted = false;
  int64_t allocated_prefill = 0;
  int64_t allocated_decode = 0;
  int64_t remaining_prompt() const { return prompt_len - prefilled; }
};

struct SchedulerConfig {
  int64_t m_max = 8192;
  int64_t q_max = 256;
  int n_search_iters = 10;
  double eps_ratio = 0.05;
  double q_ref = 16.0;
  bool valid() const {
    return m_max >= q_max && q_max >= 1 && n_search_iters >= 1 && eps_ratio > 0.0 &&
           eps_ratio < 1.0 && q_ref > 0.0;
  }
};

struct Allocation {
  uint64_t request_id = 0;
  int64_t tokens = 0;
  bool is_prefill = false;
};

struct BatchPlan {
  std::vector<Allocation> allocations;
  int64_t b = 0;
  int64_t s = 0;
  double predicted_ms = 0.0;
  double target_ms = 0.0;
  bool overload = false;
  bool empty() const { return allocations.empty(); }
};

struct TargetLatency {
  double target_ms = 0.0;
  bool slo_risk = false;
};

TargetLatency target_latency(int64_t wait_count, const SLOSpec& slo, const TradeoffModel& tm,
                             double q_ref);
int64_t binary_search_budget(int64_t b, double target_ms, const PerfParams& params,
                             const SchedulerConfig& cfg, int64_t s_cap = -1);
std::vector<Allocation> allocate_tokens(std::span<const Request* const> run_q,
                                        std::span<const Request* const> wait_q, int64_t b, int64_t s);
BatchPlan schedule_step(std::span<const Request* const> wait_q, std::span<const Request* const> run_q,
                        const SLOSpec& slo, const TradeoffModel& tm, const PerfParams& params,
                        const SchedulerConfig& cfg);

struct CompletionStats {
  double ttft_ms = 0.0;
  double tpot_ms = 0.0;
  int64_t decode_len = 0;
};

class TradeoffEstimator {
 public:
  explicit TradeoffEstimator(const TradeoffModel& initial);
  void update(std::span<const CompletionStats> completed);
  const TradeoffModel& model() const { return model_; }
  int64_t degenerate_updates() const { return degenerate_updates_; }

 private:
  TradeoffModel model_;
  std::vector<double> win_ttft_, win_tpot_;  // device-layout ring (NX_TRADEOFF_WINDOW)
  int32_t win_head_ = 0, win_len_ = 0;
  int64_t degenerate_updates_ = 0;
};

// ---- router (router.h) ----------------------------------------------------------
enum class RouterPolicy { kPrism, kRoundRobin, kSessionAffinity, kLeastLoaded, kLatencyBased, kWeighted };

RouterPolicy router_policy_from_string(const std::string& name);
std::string to_string(RouterPolicy policy);

struct RouterConfig {
  RouterPolicy policy = RouterPolicy::kPrism;
  std::array<double, 4> weights{1.0, 1.0, 1.0, 1.0};
  double beta_aff = 1.5;
  double latency_knee = 0.5;
  double latency_scale_ms = 0.0;
  double load_half_ms = 50.0;
  double capacity_headroom = 2.0;
  double staleness_limit_ms = 1000.0;
  double latency_window_ms = 2000.0;
  std::map<int, double> static_weights;
  bool valid() const {
    bool w_ok = true;
    for (double w : weights) w_ok = w_ok && w >= 0.0;
    return w_ok && beta_aff > 1.0 && latency_knee >= 0.0 && latency_scale_ms >= 0.0 &&
           load_half_ms > 0.0 && capacity_headroom >= 1.0 && staleness_limit_ms > 0.0 &&
           latency_window_ms > 0.0;
  }
};

double score_latency(const StateVector& sv, const SLOSpec& slo, const RouterConfig& cfg);
double score_load(const StateVector& sv, const RouterConfig& cfg);
double score_capacity(const StateVector& sv, double req_demand_tokens, const RouterConfig& cfg);

struct RouteDecision {
  int engine_id = -1;
  double score = 0.0;
  std::array<double, 4> factors{1.0, 1.0, 1.0, 1.0};
  bool degraded = false;
};

class Router {
 public:
  Router(const RouterConfig& cfg, const SLOSpec& slo, uint64_t root_seed);
  void register_engine(int engine_id);
  void on_report(const EngineReport& report);
  void on_completion(int engine_id, const std::string& session_id, double e2e_ms,
                     int64_t decode_len, double now_ms);
  RouteDecision route(const Request& request, double now_ms);
  double score_affinity(int engine_id, const std::string& session_id) const;
  double demand_estimate_tokens(int64_t prompt_len) const;
  size_t engine_count() const { return order_.size(); }

 private:
  struct EngineInfo {
    std::optional<EngineReport> report;
    std::deque<std::pair<double, double>> latencies;
    double latency_sum = 0.0;
  };
  void remember_session(const std::string& session_id, int engine_id);
  RouterConfig cfg_;
  SLOSpec slo_;
  std::array<uint64_t, 4> rng_{};
  uint64_t rr_next_ = 0;
  std::vector<int> order_;
  std::unordered_map<int, EngineInfo> engines_;
  std::unordered_map<std::string, int> sessions_;  // session -> engine id
  std::deque<std::string> session_lru_;
  double l_bar_ema_ = 128.0;
};

// ---- online learner (learner.h) ------------------------------------------------------
struct LearnerConfig {
  int64_t long_window = 4096;
  int64_t short_window = 64;
  int64_t structural_period = 1024;
  int64_t linear_period = 32;
  int64_t min_structural_samples = 256;
  bool valid() const {
    return long_window > 0 && short_window > 0 && structural_period > 0 && linear_period > 0 &&
           min_structural_samples > 0 && short_window < long_window &&
           linear_period < structural_period;
  }
};

struct LearnerCounters {
  int64_t linear_updates = 0;
  int64_t structural_updates = 0;
  int64_t degenerate_updates = 0;
  int64_t rescale_updates = 0;
  int64_t clamp_events = 0;
  int64_t failed_fits = 0;
  int64_t low_identifiability = 0;
};

class OnlineLearner {
 public:
  OnlineLearner(const PerfParams& priors, const LearnerConfig& cfg);
  static PerfParams default_priors();
  void record_sample(const LatencySample& sample);
  const PerfParams& params() const { return current_; }
  int64_t samples_seen() const { return samples_seen_; }
  int64_t buffered() const { return static_cast<int64_t>(ring_.size()); }
  const LearnerCounters& counters() const { return counters_; }
  const LearnerConfig& config() const { return cfg_; }
  bool update_linear();
  bool update_structural();
  double convergence_error(std::span<const LatencySample> probe) const;
  std::string to_json() const;

 private:
  bool refit(int kind);
  LearnerConfig cfg_;
  PerfParams current_;
  std::vector<LatencySample> ring_;
  size_t ring_head_ = 0;
  int64_t samples_seen_ = 0;
  LearnerCounters counters_;
};

std::vector<LatencySample> load_samples_jsonl(const std::string& path);

// ---- engine simulator (engine.h:68-180) ---------------------------------------------
// Host bookkeeping (queues, KV block counters, prefix cache) as in the
// reference; every scheduling decision, latency prediction, learner refit and
// tradeoff refit it makes is a device launch (schedule_step /
// nx_baseline_schedule_host / predict_latency / OnlineLearner /
// TradeoffEstimator). Inside simulations the same logic runs on the device
// (sim_kernel.cu); this class serves step-by-step callers.
struct StepOutcome {
  BatchPlan plan;
  double actual_ms = 0.0;
  std::vector<uint64_t> finished;
  std::vector<uint64_t> first_tokens;
};

BatchPlan schedule_baseline(SchedulerPolicy policy, std::span<const Request* const> wait_q,
                            std::span<const Request* const> run_q, const PerfParams& params,
                            const EngineConfig& cfg);

class EngineSim {
 public:
  EngineSim(const EngineConfig& cfg, const SLOSpec& slo, const SchedulerConfig& sched,
            const TradeoffModel& tradeoff_init, const LearnerConfig& learner_cfg, uint64_t root_seed);

  double oracle_latency(const BatchShape& shape);
  bool admit(Request* request, double now_ms);
  bool busy() const { return step_.has_value(); }
  bool has_work() const { return !wait_q_.empty() || !run_q_.empty(); }
  std::optional<double> begin_step(double now_ms);
  StepOutcome complete_step(double now_ms);
  StateVector export_state(double now_ms) const;
  int64_t queue_len() const { return static_cast<int64_t>(wait_q_.size() + run_q_.size()); }
  void record_learner_sample(const LatencySample& sample) { learner_.record_sample(sample); }

  const EngineConfig& config() const { return cfg_; }
  const SchedulerConfig& scheduler_config() const { return sched_; }
  OnlineLearner& learner() { return learner_; }
  const OnlineLearner& learner() const { return learner_; }
  TradeoffEstimator& tradeoff() { return tradeoff_; }
  const BatchPlan* inflight_plan() const { return step_ ? &step_->plan : nullptr; }

  int64_t used_blocks() const { return pinned_; }
  int64_t free_blocks() const { return cfg_.kv_blocks - pinned_; }
  int64_t reserved_blocks() const { return reserved_; }
  int64_t cache_blocks() const { return cached_; }
  int64_t cached_prefix_tokens(const std::string& session) const;
  void check_kv_consistency() const;

  const std::deque<Request*>& wait_queue() const { return wait_q_; }
  const std::vector<Request*>& run_queue() const { return run_q_; }

 private:
  struct Step {
    BatchPlan plan;
    double started_ms = 0.0, actual_ms = 0.0;
  };
  struct Prefix {  // a finished session's KV prefix, kept in free space
    int64_t tokens = 0, blocks = 0;
    uint64_t stamp = 0;  // insertion order; the smallest stamp is evicted first
  };
  int64_t blocks(int64_t tokens) const { return (tokens + cfg_.block_size - 1) / cfg_.block_size; }
  void drop_prefix(std::unordered_map<std::string, Prefix>::iterator it);
  void shrink_cache();
  void keep_prefix(const std::string& session, int64_t tokens);
  void admit_prefills(BatchPlan& plan);

  EngineConfig cfg_;
  SLOSpec slo_;
  SchedulerConfig sched_;
  OnlineLearner learner_;
  TradeoffEstimator tradeoff_;
  Rng noise_;
  std::deque<Request*> wait_q_;
  std::vector<Request*> run_q_;
  std::unordered_map<uint64_t, Request*> live_;
  std::optional<Step> step_;
  int64_t pinned_ = 0, reserved_ = 0, cached_ = 0;
  std::unordered_map<std::string, Prefix> prefixes_;
  std::map<uint64_t, std::string> lru_;  // stamp -> session
  uint64_t next_stamp_ = 0;
};

// ---- metrics (metrics.h) ---------------------------------------------------------------
struct RequestRecord {
  uint64_t request_id = 0;
  double arrival_ms = 0.0;
  double first_token_ms = 0.0;
  double completed_ms = 0.0;
  int64_t prompt_tokens = 0;
  int64_t output_tokens = 0;
  int engine_id = 0;
};

struct RequestMetrics {
  double ttft_ms = 0.0;
  double tpot_ms = 0.0;
  double e2e_ms = 0.0;
  bool single_token = false;
};

RequestMetrics request_metrics(const RequestRecord& rec);
double percentile(std::vector<double> values, double p);

struct SloAttainment {
  double percent = 100.0;
  bool empty = false;
};
SloAttainment slo_attainment(std::span<const RequestRecord> records, const SLOSpec& slo);

struct MetricsSummary {
  int64_t completed = 0;
  double p50_e2e_ms = 0.0;
  double p90_e2e_ms = 0.0;
  double p50_ttft_ms = 0.0;
  double p50_tpot_ms = 0.0;
  double mean_ttft_ms = 0.0;
  double mean_tpot_ms = 0.0;
  double slo_attainment_pct = 100.0;
  std::vector<std::pair<int, double>> engine_share;
};
MetricsSummary summarize(std::span<const RequestRecord> records, const SLOSpec& slo);
void write_requests_csv(const std::string& path, std::span<const RequestRecord> records);

// ---- workload (workload.h) -------------------------------------------------------------
struct TraceRecord {
  double arrival_ms = 0.0;
  std::string session_id;
  int64_t prompt_tokens = 1;
  int64_t output_tokens = 1;
};

struct LengthStats {
  double mean = 0.0;
  double p99 = 0.0;
  double std_dev = 0.0;
};

struct ScenarioStats {
  std::string name;
  LengthStats prompt;
  LengthStats output;
  double session_turn_prob = 0.0;
  bool valid() const {
    return prompt.mean > 0.0 && output.mean > 0.0 && prompt.p99 >= 0.0 && output.p99 >= 0.0 &&
           prompt.std_dev >= 0.0 && output.std_dev >= 0.0 && session_turn_prob >= 0.0 &&
           session_turn_prob <= 1.0;
  }
};

enum class ArrivalMode { kTimestamp, kQps };

const ScenarioStats& scenario_by_name(const std::string& name);
std::vector<std::string> scenario_names();
ScenarioStats load_scenario_json(const std::string& path);
std::vector<TraceRecord> load_trace(const std::string& path, bool* sorted_warning = nullptr);
void write_trace(const std::string& path, const std::vector<TraceRecord>& records);
std::vector<TraceRecord> synth_generate(const ScenarioStats& stats, int64_t n, uint64_t seed);
std::vector<TraceRecord> assign_arrivals(std::vector<TraceRecord> records, ArrivalMode mode,
                                         double rate_per_s, uint64_t seed, double time_scale = 1.0,
                                         bool poisson = false);

// ---- simulation (sim.h): runs on the lockstep kernel ---------------------------------
struct WorkloadConfig {
  std::string scenario;
  std::string scenario_file;
  std::string trace_path;
  ArrivalMode mode = ArrivalMode::kQps;
  double rate_per_s = 1.0;
  int64_t n = 100;
  double time_scale = 1.0;
  bool poisson = false;
};

struct OutputConfig {
  std::string dir;
  std::string summary = "summary.json";
  std::string requests_csv = "requests.csv";
  std::string plans_jsonl;
  std::string routing_jsonl;
};

struct RunConfig {
  uint64_t seed = 1;
  double duration_ms = 3.6e6;
  SLOSpec slo;
  SchedulerConfig scheduler;
  TradeoffModel tradeoff;
  LearnerConfig learner;
  RouterConfig router;
  std::vector<EngineConfig> engines;
  WorkloadConfig workload;
  OutputConfig output;
  bool record_learner_history = false;
  bool validate_invariants = false;

  void validate() const;
  static RunConfig from_json_text(const std::string& text);
  static RunConfig from_json_file(const std::string& path);
  // The RunConfig JSON document (RunConfig::from_json_text's schema) — what
  // the device batch entry point nx_sim_create_json consumes.
  std::string to_json_text() const;
};

struct LearnerSnapshot {
  int engine_id = 0;
  double sim_time_ms = 0.0;
  int64_t samples_seen = 0;
  PerfParams params;
};

struct RunResult {
  int64_t arrived = 0;
  int64_t completed = 0;
  int64_t rejected = 0;
  int64_t unfinished = 0;
  uint64_t arrival_hash = 0;
  uint64_t event_hash = 0;
  std::vector<RequestRecord> records;
  MetricsSummary metrics;
  std::vector<LearnerSnapshot> learner_history;
  std::string summary_json;
};

RunResult run_simulation(const RunConfig& cfg);
// Many configs as one device batch (one replica each); results in order.
std::vector<RunResult> run_replicas(std::span<const RunConfig> cfgs, int device = 0);

enum class SweepAxis { kRate, kPolicy, kBudget };
SweepAxis sweep_axis_from_string(const std::string& name);

struct SweepRow {
  std::string value;
  bool ok = false;
  std::string error;
  RunResult result;
};

struct SweepResult {
  SweepAxis axis;
  std::vector<SweepRow> rows;
};

SweepResult sweep(const RunConfig& base, SweepAxis axis, const std::vector<std::string>& values);
std::string sweep_csv(const SweepResult& result);

}  // namespace servesim
