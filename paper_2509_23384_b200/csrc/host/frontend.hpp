// Host front-end: RunConfig JSON -> flat replica description + host-generated
// workload. This is the part of the reference that stays on the host
// (config parsing, workload synthesis — arrival doubles must come
// from host libm so TTFT sums match exactly).
//
// Mirrors, by behaviour (not by code):
//   RunConfig::from_json_text / validate   proj/src/sim.cpp:418-582
//   build_workload + arrival hash          proj/src/sim.cpp:101-141
//   synth_generate / assign_arrivals       proj/src/workload.cpp:137-197
//   load_trace                             proj/src/workload.cpp:83-121
//   Rng / substream_seed                   proj/include/servesim/rng.h:12-72
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace nx {

// ---- xoshiro256++ stream (proj/include/servesim/rng.h:12-72) ---------------
struct Xoshiro {
  uint64_t s[4];
  static uint64_t mix(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  explicit Xoshiro(uint64_t seed) {
    for (int i = 0; i < 4; ++i) s[i] = mix(seed);
  }
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t out = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
  }
  double uniform() {  // (0, 1]
    return (static_cast<double>(next() >> 11) + 1.0) * 0x1.0p-53;
  }
  uint64_t below(uint64_t n) { return n ? next() % n : 0; }
  double normal();  // Box-Muller, two uniforms
};
uint64_t substream_seed(uint64_t root, const std::string& tag, uint64_t index = 0);

// ---- configuration (value types of proj/include/servesim/*.h) --------------
struct Params {  // PerfParams field order; 64 B, identical layout on device
  double tau0 = 0.0, w0 = 0.0, ws = 1.0, tauB = 0.0, tauS = 0.0;
  double p_max = 1.0, kB = 1.0, kS = 1.0;
  bool valid() const {
    return p_max > 0.0 && kB > 0.0 && kS > 0.0 && tau0 >= 0.0 && tauB >= 0.0 &&
           tauS >= 0.0 && ws > 0.0 && w0 >= 0.0;
  }
};
Params profile_params(const std::string& name);  // "fast" | "medium" | "slow"
Params learner_default_priors();

enum SchedPolicy : int32_t { kLens = 0, kPrefillPriority = 1, kStaticChunked = 2 };
enum RoutePolicy : int32_t {
  kPrism = 0, kRoundRobin = 1, kSessionAffinity = 2,
  kLeastLoaded = 3, kLatencyBased = 4, kWeighted = 5
};
SchedPolicy sched_policy_from(const std::string& s);
RoutePolicy route_policy_from(const std::string& s);
std::string route_policy_name(int32_t p);

struct EngineCfg {
  int32_t engine_id = 0;
  Params true_params;
  double noise_sigma = 0.05;
  int64_t kv_blocks = 8192, block_size = 16, m_max = 8192, q_max = 256;
  int32_t policy = kLens;
  int64_t static_budget = 2048;
  double report_period_ms = 100.0, staleness_ms = 0.0;
  int64_t wait_cap = 0;
};

struct RunCfg {
  uint64_t seed = 1;
  double duration_ms = 3.6e6;
  double ttft_slo = 2000.0, tpot_slo = 12.0;
  int64_t m_max = 8192, q_max = 256;
  int32_t n_search_iters = 10;
  double eps_ratio = 0.05, q_ref = 16.0;
  double alpha = 2000.0, beta = 16.0, l_bar = 128.0, td_min = 2.0;
  int64_t long_window = 4096, short_window = 64, structural_period = 1024,
          linear_period = 32, min_structural = 256;
  int32_t route_policy = kPrism;
  double weights[4] = {1.0, 1.0, 1.0, 1.0};
  double beta_aff = 1.5, knee = 0.5, scale_ms = 0.0, load_half = 50.0,
         headroom = 2.0, staleness_limit = 1000.0, latency_window = 2000.0;
  std::map<int, double> static_weights;
  std::vector<EngineCfg> engines;
  // workload
  std::string scenario, scenario_file, trace_path;
  bool timestamp_mode = false;
  double rate = 1.0;
  int64_t n = 100;
  double time_scale = 1.0;
  bool poisson = false;
  // observability (RunConfig::record_learner_history, OutputConfig; sim.h)
  bool record_learner_history = false;
  std::string out_dir, out_summary = "summary.json", out_requests_csv = "requests.csv";
  std::string out_plans_jsonl, out_routing_jsonl;
};

// Throws std::runtime_error / std::invalid_argument with the reference's
// messages for the cases the reference rejects.
RunCfg parse_run_config(const std::string& json_text);
void validate_run_config(const RunCfg& cfg);

// ---- workload ---------------------------------------------------------------
struct LengthStats { double mean, p99, std_dev; };
struct Scenario {
  std::string name;
  LengthStats prompt, output;
  double session_turn_prob;
};
Scenario scenario_named(const std::string& name);
Scenario scenario_from_file(const std::string& path);

struct Workload {
  std::vector<double> arrival_ms;
  std::vector<int64_t> arrival_us;     // llround(ms * 1000), proj/src/sim.cpp:21
  std::vector<int32_t> prompt, output; // tokens
  std::vector<int32_t> session;        // interned per replica, first-seen order
  std::vector<std::string> session_names;
  uint64_t arrival_hash = 0;
};

struct TraceRow {
  double arrival_ms = 0.0;
  std::string session;
  int64_t prompt = 1, output = 1;
};
std::vector<TraceRow> synth_rows(const Scenario& sc, int64_t n, uint64_t seed);
std::vector<TraceRow> load_trace_rows(const std::string& path, bool* sorted_warning);
void write_trace_rows(const std::string& path, const std::vector<TraceRow>& rows);
void assign_arrival_times(std::vector<TraceRow>& rows, bool timestamp_mode,
                          double rate, uint64_t seed, double time_scale,
                          bool poisson);
Workload build_workload(const RunCfg& cfg);

inline int64_t to_us(double ms) { return std::llround(ms * 1000.0); }
inline double to_ms(int64_t us) { return static_cast<double>(us) / 1000.0; }
inline uint64_t fnv1a_u64(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 0x100000001b3ULL;
  }
  return h;
}
constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ULL;

}  // namespace nx
