// Host front-end implementation. See frontend.hpp for the reference map.
#include "frontend.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <fstream>
#include <numbers>
#include <sstream>
#include <stdexcept>

#include "json.hpp"

namespace nx {

double Xoshiro::normal() {
  // rng.h:41-45: sqrt(-2 log u1) * cos(2 pi u2); evaluation order preserved.
  const double u1 = uniform();
  const double u2 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}

uint64_t substream_seed(uint64_t root, const std::string& tag, uint64_t index) {
  uint64_t h = kFnvBasis;
  for (unsigned char c : tag) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  h ^= index + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  uint64_t x = root ^ h;
  return Xoshiro::mix(x);
}

Params profile_params(const std::string& name) {
  // Ground-truth tiers, proj/src/engine.cpp:34-59.
  Params p;
  p.w0 = 0.0;
  p.ws = 1.0;
  p.kB = 4.0;
  p.kS = 0.05;
  if (name == "fast") {
    p.p_max = 20.0; p.tau0 = 4.0; p.tauB = 0.08; p.tauS = 0.0004;
  } else if (name == "medium") {
    p.p_max = 10.0; p.tau0 = 5.0; p.tauB = 0.12; p.tauS = 0.0008;
  } else if (name == "slow") {
    p.p_max = 5.0; p.tau0 = 6.0; p.tauB = 0.18; p.tauS = 0.0016;
  } else {
    throw std::runtime_error("unknown perf profile: " + name);
  }
  return p;
}

Params learner_default_priors() {
  // OnlineLearner::default_priors, proj/src/learner.cpp:117-128.
  Params p;
  p.p_max = 20.0; p.kB = 0.1; p.kS = 0.02; p.tau0 = 5.0;
  p.w0 = 0.0; p.ws = 1.0; p.tauB = 0.1; p.tauS = 0.001;
  return p;
}

SchedPolicy sched_policy_from(const std::string& s) {
  if (s == "lens") return kLens;
  if (s == "prefill_priority") return kPrefillPriority;
  if (s == "static_chunked") return kStaticChunked;
  throw std::runtime_error("unknown scheduler policy: " + s);
}

RoutePolicy route_policy_from(const std::string& s) {
  static const char* names[] = {"prism", "round_robin", "session_affinity",
                                "least_loaded", "latency_based", "weighted"};
  for (int i = 0; i < 6; ++i)
    if (s == names[i]) return static_cast<RoutePolicy>(i);
  throw std::runtime_error("unknown router policy: " + s);
}

std::string route_policy_name(int32_t p) {
  static const char* names[] = {"prism", "round_robin", "session_affinity",
                                "least_loaded", "latency_based", "weighted"};
  return (p >= 0 && p < 6) ? names[p] : "?";
}

namespace {
using nlohmann::json;

template <class T>
T opt(const json& j, const char* key, T fallback) {
  return j.contains(key) ? j.at(key).get<T>() : fallback;
}

bool engine_valid(const EngineCfg& e) {
  // EngineConfig::valid, proj/include/servesim/engine.h:41-46
  return e.kv_blocks > 0 && e.block_size >= 1 && e.noise_sigma >= 0.0 &&
         e.static_budget >= 1 && e.static_budget <= e.m_max &&
         e.m_max >= e.q_max && e.q_max >= 1 && e.report_period_ms > 0.0 &&
         e.staleness_ms >= 0.0 && e.wait_cap >= 0 && e.true_params.valid();
}
}  // namespace

void validate_run_config(const RunCfg& c) {
  if (c.engines.empty()) throw std::runtime_error("config: needs >= 1 engine");
  if (!(c.duration_ms > 0)) throw std::runtime_error("config: duration_ms <= 0");
  if (!(c.ttft_slo > 0.0 && c.tpot_slo > 0.0))
    throw std::runtime_error("config: invalid slo");
  const bool sched_ok = c.m_max >= c.q_max && c.q_max >= 1 && c.n_search_iters >= 1 &&
                        c.eps_ratio > 0.0 && c.eps_ratio < 1.0 && c.q_ref > 0.0;
  if (!sched_ok) throw std::runtime_error("config: invalid scheduler");
  if (!(c.beta > 0.0 && c.l_bar >= 1.0 && c.td_min > 0.0))
    throw std::runtime_error("config: invalid tradeoff");
  const bool learner_ok = c.long_window > 0 && c.short_window > 0 &&
                          c.structural_period > 0 && c.linear_period > 0 &&
                          c.min_structural > 0 && c.short_window < c.long_window &&
                          c.linear_period < c.structural_period;
  if (!learner_ok) throw std::runtime_error("config: invalid learner");
  bool w_ok = true;
  for (double w : c.weights) w_ok = w_ok && w >= 0.0;
  const bool router_ok = w_ok && c.beta_aff > 1.0 && c.knee >= 0.0 &&
                         c.scale_ms >= 0.0 && c.load_half > 0.0 &&
                         c.headroom >= 1.0 && c.staleness_limit > 0.0 &&
                         c.latency_window > 0.0;
  if (!router_ok) throw std::runtime_error("config: invalid router");
  std::vector<int> ids;
  for (const auto& e : c.engines) {
    if (!engine_valid(e))
      throw std::runtime_error("config: invalid engine " + std::to_string(e.engine_id));
    ids.push_back(e.engine_id);
  }
  std::sort(ids.begin(), ids.end());
  if (std::adjacent_find(ids.begin(), ids.end()) != ids.end())
    throw std::runtime_error("config: duplicate engine_id");
  if (c.trace_path.empty() && c.scenario.empty() && c.scenario_file.empty())
    throw std::runtime_error("config: workload needs a scenario or trace");
  if (c.trace_path.empty() && c.n < 1)
    throw std::runtime_error("config: workload n must be >= 1");
  if (!c.timestamp_mode && !(c.rate > 0))
    throw std::runtime_error("config: qps mode needs rate > 0");
  if (c.timestamp_mode && c.trace_path.empty())
    throw std::runtime_error("config: timestamp mode needs a trace with recorded arrivals");
}

RunCfg parse_run_config(const std::string& text) {
  const json j = json::parse(text);
  RunCfg c;
  c.seed = opt<uint64_t>(j, "seed", c.seed);
  c.duration_ms = opt<double>(j, "duration_ms", c.duration_ms);
  if (j.contains("slo")) {
    const auto& s = j["slo"];
    c.ttft_slo = opt<double>(s, "ttft_slo_ms", c.ttft_slo);
    c.tpot_slo = opt<double>(s, "tpot_slo_ms", c.tpot_slo);
  }
  if (j.contains("scheduler")) {
    const auto& s = j["scheduler"];
    c.m_max = opt<int64_t>(s, "m_max", c.m_max);
    c.q_max = opt<int64_t>(s, "q_max", c.q_max);
    c.n_search_iters = opt<int32_t>(s, "n_search_iters", c.n_search_iters);
    c.eps_ratio = opt<double>(s, "eps_ratio", c.eps_ratio);
    c.q_ref = opt<double>(s, "q_ref", c.q_ref);
  }
  // TradeoffModel::initial_for(slo) precedes overrides (sim.cpp:475, lens.h:30-35)
  c.alpha = 2.0 * c.ttft_slo;
  c.beta = c.ttft_slo / c.tpot_slo;
  c.l_bar = 128.0;
  c.td_min = 2.0;
  if (j.contains("tradeoff")) {
    const auto& t = j["tradeoff"];
    c.alpha = opt<double>(t, "alpha_ms", c.alpha);
    c.beta = opt<double>(t, "beta", c.beta);
    c.l_bar = opt<double>(t, "l_bar", c.l_bar);
    c.td_min = opt<double>(t, "td_min_ms", c.td_min);
  }
  if (j.contains("learner")) {
    const auto& l = j["learner"];
    c.long_window = opt<int64_t>(l, "long_window", c.long_window);
    c.short_window = opt<int64_t>(l, "short_window", c.short_window);
    c.structural_period = opt<int64_t>(l, "structural_period", c.structural_period);
    c.linear_period = opt<int64_t>(l, "linear_period", c.linear_period);
    c.min_structural = opt<int64_t>(l, "min_structural_samples", c.min_structural);
  }
  if (j.contains("router")) {
    const auto& r = j["router"];
    c.route_policy = route_policy_from(opt<std::string>(r, "policy", "prism"));
    if (r.contains("weights")) {
      const auto& w = r["weights"];
      if (!w.is_array() || w.size() != 4)
        throw std::runtime_error("config: router.weights must have 4 entries");
      for (int i = 0; i < 4; ++i) c.weights[i] = w[i].get<double>();
    }
    c.beta_aff = opt<double>(r, "beta_aff", c.beta_aff);
    c.knee = opt<double>(r, "latency_knee", c.knee);
    c.scale_ms = opt<double>(r, "latency_scale_ms", c.scale_ms);
    c.load_half = opt<double>(r, "load_half_ms", c.load_half);
    c.headroom = opt<double>(r, "capacity_headroom", c.headroom);
    c.staleness_limit = opt<double>(r, "staleness_limit_ms", c.staleness_limit);
    c.latency_window = opt<double>(r, "latency_window_ms", c.latency_window);
    if (r.contains("static_weights")) {
      for (const auto& [key, value] : r["static_weights"].items())
        c.static_weights[std::stoi(key)] = value.get<double>();
    }
  }
  if (!j.contains("engines") || !j["engines"].is_array() || j["engines"].empty())
    throw std::runtime_error("config: engines array required");
  for (const auto& e : j["engines"]) {
    EngineCfg ec;
    ec.engine_id = opt<int32_t>(e, "engine_id", static_cast<int32_t>(c.engines.size()));
    if (e.contains("true_params")) {
      const auto& tp = e["true_params"];
      Params p;
      p.tau0 = tp.at("tau0").get<double>();
      p.w0 = tp.at("w0").get<double>();
      p.ws = tp.at("ws").get<double>();
      p.tauB = tp.at("tauB").get<double>();
      p.tauS = tp.at("tauS").get<double>();
      p.p_max = tp.at("p_max").get<double>();
      p.kB = tp.at("kB").get<double>();
      p.kS = tp.at("kS").get<double>();
      if (!p.valid()) throw std::invalid_argument("PerfParams JSON violates invariants");
      ec.true_params = p;
    } else {
      ec.true_params = profile_params(opt<std::string>(e, "profile", "medium"));
    }
    ec.noise_sigma = opt<double>(e, "noise_sigma", ec.noise_sigma);
    ec.kv_blocks = opt<int64_t>(e, "kv_blocks", ec.kv_blocks);
    ec.block_size = opt<int64_t>(e, "block_size", ec.block_size);
    ec.m_max = opt<int64_t>(e, "m_max", c.m_max);
    ec.q_max = opt<int64_t>(e, "q_max", c.q_max);
    ec.policy = sched_policy_from(opt<std::string>(e, "scheduler_policy", "lens"));
    ec.static_budget = opt<int64_t>(e, "static_budget", ec.static_budget);
    ec.report_period_ms = opt<double>(e, "state_report_period_ms", ec.report_period_ms);
    ec.staleness_ms = opt<double>(e, "state_staleness_ms", ec.staleness_ms);
    ec.wait_cap = opt<int64_t>(e, "wait_cap", ec.wait_cap);
    c.engines.push_back(ec);
  }
  if (j.contains("workload")) {
    const auto& w = j["workload"];
    c.scenario = opt<std::string>(w, "scenario", c.scenario);
    c.scenario_file = opt<std::string>(w, "scenario_file", c.scenario_file);
    c.trace_path = opt<std::string>(w, "trace", c.trace_path);
    const std::string mode = opt<std::string>(w, "mode", "qps");
    if (mode == "qps") c.timestamp_mode = false;
    else if (mode == "timestamp") c.timestamp_mode = true;
    else throw std::runtime_error("config: workload mode must be qps|timestamp");
    c.rate = opt<double>(w, "rate", c.rate);
    c.n = opt<int64_t>(w, "n", c.n);
    c.time_scale = opt<double>(w, "time_scale", c.time_scale);
    c.poisson = opt<bool>(w, "poisson", c.poisson);
  }
  c.record_learner_history = opt<bool>(j, "record_learner_history", c.record_learner_history);
  if (j.contains("output")) {  // OutputConfig (sim.cpp:570-579)
    const auto& o = j["output"];
    c.out_dir = opt<std::string>(o, "dir", c.out_dir);
    c.out_summary = opt<std::string>(o, "summary", c.out_summary);
    c.out_requests_csv = opt<std::string>(o, "requests_csv", c.out_requests_csv);
    c.out_plans_jsonl = opt<std::string>(o, "plans_jsonl", c.out_plans_jsonl);
    c.out_routing_jsonl = opt<std::string>(o, "routing_jsonl", c.out_routing_jsonl);
  }
  validate_run_config(c);
  return c;
}

// ---- workload ---------------------------------------------------------------

Scenario scenario_named(const std::string& name) {
  // Built-in statistics table (proj/src/workload.cpp:16-24): {mean, p99, std}.
  static const Scenario table[] = {
      {"flowgpt", {4089, 7014, 2061}, {177, 51, 200}, 0.7},
      {"coding", {440, 1131, 214}, {283, 1096, 233}, 0.2},
      {"sharegpt", {370, 1420, 351}, {249, 760, 170}, 0.5},
      {"summarization", {8936, 10171, 694}, {259, 587, 115}, 0.0},
  };
  for (const auto& s : table)
    if (s.name == name) return s;
  throw std::runtime_error("unknown scenario: " + name);
}

Scenario scenario_from_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open scenario file: " + path);
  json j;
  in >> j;
  Scenario s;
  s.name = j.at("name").get<std::string>();
  s.prompt = {j.at("prompt").at("mean").get<double>(), j.at("prompt").at("p99").get<double>(),
              j.at("prompt").at("std").get<double>()};
  s.output = {j.at("output").at("mean").get<double>(), j.at("output").at("p99").get<double>(),
              j.at("output").at("std").get<double>()};
  s.session_turn_prob = j.contains("session_turn_prob") ? j["session_turn_prob"].get<double>() : 0.0;
  const bool ok = s.prompt.mean > 0.0 && s.output.mean > 0.0 && s.prompt.p99 >= 0.0 &&
                  s.output.p99 >= 0.0 && s.prompt.std_dev >= 0.0 &&
                  s.output.std_dev >= 0.0 && s.session_turn_prob >= 0.0 &&
                  s.session_turn_prob <= 1.0;
  if (!ok) throw std::runtime_error("scenario stats invalid: " + path);
  return s;
}

namespace {
// Moment-matched truncated log-normal draw (proj/src/workload.cpp:26-48).
int64_t draw_tokens(const LengthStats& st, Xoshiro& rng) {
  if (st.std_dev <= 0.0) return std::max<int64_t>(1, llround(st.mean));
  const double ratio = st.std_dev / st.mean;
  const double sigma = std::sqrt(std::log1p(ratio * ratio));
  const double mu = std::log(st.mean) - 0.5 * sigma * sigma;
  const double x = std::exp(mu + sigma * rng.normal());
  const double cap = std::max(1.0, 4.0 * st.p99);
  return std::max<int64_t>(1, llround(std::min(x, cap)));
}
}  // namespace

std::vector<TraceRow> synth_rows(const Scenario& sc, int64_t n, uint64_t seed) {
  if (n < 1) throw std::invalid_argument("synth_generate: n must be >= 1");
  Xoshiro rng(substream_seed(seed, "workload"));
  std::deque<std::string> live;  // <= 64 recent sessions (workload.cpp:144)
  uint64_t next_session = 0;
  std::vector<TraceRow> rows;
  rows.reserve(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    TraceRow r;
    r.prompt = draw_tokens(sc.prompt, rng);
    r.output = draw_tokens(sc.output, rng);
    bool follow = false;
    if (!live.empty()) follow = rng.uniform() <= sc.session_turn_prob;
    if (follow) {
      r.session = live[rng.below(live.size())];
    } else {
      r.session = "s" + std::to_string(next_session++);
      live.push_back(r.session);
      if (live.size() > 64) live.pop_front();
    }
    rows.push_back(std::move(r));
  }
  return rows;
}

void assign_arrival_times(std::vector<TraceRow>& rows, bool timestamp_mode,
                          double rate, uint64_t seed, double time_scale,
                          bool poisson) {
  if (!timestamp_mode) {
    if (rate <= 0.0) throw std::runtime_error("qps mode requires rate > 0");
    const double gap = 1000.0 / rate;
    if (poisson) {
      Xoshiro rng(substream_seed(seed, "arrivals"));
      double t = 0.0;
      for (auto& r : rows) {
        r.arrival_ms = t;
        t += -gap * std::log(rng.uniform());
      }
    } else {
      for (size_t i = 0; i < rows.size(); ++i) rows[i].arrival_ms = static_cast<double>(i) * gap;
    }
    return;
  }
  if (time_scale <= 0.0) throw std::runtime_error("time_scale must be > 0");
  for (auto& r : rows) r.arrival_ms /= time_scale;
}

std::vector<TraceRow> load_trace_rows(const std::string& path, bool* sorted_warning) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open trace file: " + path);
  std::vector<TraceRow> rows;
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    try {
      const auto j = json::parse(line);
      TraceRow r;
      r.arrival_ms = j.at("arrival_ms").get<double>();
      r.session = j.at("session_id").get<std::string>();
      r.prompt = j.at("prompt_tokens").get<int64_t>();
      r.output = j.at("output_tokens").get<int64_t>();
      if (r.prompt < 1 || r.output < 1) throw std::runtime_error("token counts must be >= 1");
      rows.push_back(std::move(r));
    } catch (const std::exception& e) {
      throw std::runtime_error(path + ": line " + std::to_string(lineno) + ": " + e.what());
    }
  }
  auto earlier = [](const TraceRow& a, const TraceRow& b) { return a.arrival_ms < b.arrival_ms; };
  const bool sorted = std::is_sorted(rows.begin(), rows.end(), earlier);
  if (!sorted) std::stable_sort(rows.begin(), rows.end(), earlier);
  if (sorted_warning) *sorted_warning = !sorted;
  return rows;
}

void write_trace_rows(const std::string& path, const std::vector<TraceRow>& rows) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write trace file: " + path);
  for (const auto& r : rows) {
    nlohmann::ordered_json j;
    j["arrival_ms"] = r.arrival_ms;
    j["session_id"] = r.session;
    j["prompt_tokens"] = r.prompt;
    j["output_tokens"] = r.output;
    out << j.dump() << '\n';
  }
}

Workload build_workload(const RunCfg& c) {
  std::vector<TraceRow> rows;
  if (!c.trace_path.empty()) {
    rows = load_trace_rows(c.trace_path, nullptr);
    if (!c.timestamp_mode) assign_arrival_times(rows, false, c.rate, c.seed, 1.0, c.poisson);
    else assign_arrival_times(rows, true, 0.0, c.seed, c.time_scale, false);
  } else {
    const Scenario sc = !c.scenario_file.empty() ? scenario_from_file(c.scenario_file)
                                                 : scenario_named(c.scenario);
    rows = synth_rows(sc, c.n, c.seed);
    assign_arrival_times(rows, false, c.rate, c.seed, 1.0, c.poisson);
  }
  Workload w;
  const size_t n = rows.size();
  w.arrival_ms.resize(n);
  w.arrival_us.resize(n);
  w.prompt.resize(n);
  w.output.resize(n);
  w.session.resize(n);
  std::map<std::string, int32_t> intern;
  uint64_t h = kFnvBasis;
  for (size_t i = 0; i < n; ++i) {
    const TraceRow& r = rows[i];
    if (r.prompt > INT32_MAX / 2 || r.output > INT32_MAX / 2)
      throw std::invalid_argument("trace token counts exceed the device range");
    w.arrival_ms[i] = r.arrival_ms;
    w.arrival_us[i] = to_us(r.arrival_ms);
    w.prompt[i] = static_cast<int32_t>(r.prompt);
    w.output[i] = static_cast<int32_t>(r.output);
    auto [it, fresh] = intern.try_emplace(r.session, static_cast<int32_t>(w.session_names.size()));
    if (fresh) w.session_names.push_back(r.session);
    w.session[i] = it->second;
    // arrival fingerprint, proj/src/sim.cpp:132-139
    h = fnv1a_u64(h, static_cast<uint64_t>(w.arrival_us[i]));
    h = fnv1a_u64(h, static_cast<uint64_t>(r.prompt));
    h = fnv1a_u64(h, static_cast<uint64_t>(r.output));
    uint64_t sh = kFnvBasis;
    for (unsigned char ch : r.session) sh = fnv1a_u64(sh, ch);
    h = fnv1a_u64(h, sh);
  }
  w.arrival_hash = h;
  // prefill_priority must fit the longest prompt (proj/src/sim.cpp:248-262)
  int64_t max_prompt = 0;
  for (const auto& r : rows) max_prompt = std::max(max_prompt, r.prompt);
  for (const auto& e : c.engines) {
    if (e.policy == kPrefillPriority && max_prompt > e.m_max) {
      throw std::runtime_error("config: engine " + std::to_string(e.engine_id) +
                               " uses prefill_priority but m_max " + std::to_string(e.m_max) +
                               " < longest prompt " + std::to_string(max_prompt));
    }
  }
  return w;
}

}  // namespace nx
