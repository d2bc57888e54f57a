#include "report.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <stdexcept>

#include "json.hpp"

namespace nx {

namespace {
struct PerRequest {
  double ttft, tpot, e2e;
  bool single;
};

PerRequest metrics_of(const RecordRow& r) {  // metrics.cpp:7-26
  if (!(r.arrival_ms <= r.first_token_ms && r.first_token_ms <= r.completed_ms))
    throw std::invalid_argument("RequestRecord timestamps out of order");
  PerRequest m;
  m.ttft = r.first_token_ms - r.arrival_ms;
  m.e2e = r.completed_ms - r.arrival_ms;
  m.single = r.output_tokens < 2;
  m.tpot = m.single ? 0.0
                    : (r.completed_ms - r.first_token_ms) / static_cast<double>(r.output_tokens - 1);
  return m;
}
}  // namespace

double percentile_nearest_rank(std::vector<double> v, double p) {  // metrics.cpp:29-38
  if (v.empty()) throw std::invalid_argument("percentile of empty set");
  if (!(p > 0.0 && p <= 100.0)) throw std::invalid_argument("percentile requires 0 < p <= 100");
  std::sort(v.begin(), v.end());
  const double n = static_cast<double>(v.size());
  const size_t rank = static_cast<size_t>(std::ceil(p / 100.0 * n));
  return v[std::max<size_t>(rank, 1) - 1];
}

Metrics summarize_records(const std::vector<RecordRow>& recs, double ttft_slo,
                          double tpot_slo) {  // metrics.cpp:40-91
  Metrics out;
  out.completed = static_cast<int64_t>(recs.size());
  if (recs.empty()) return out;
  std::vector<double> e2e, ttft, tpot;
  std::map<int, int64_t> per_engine;
  double ttft_sum = 0.0, tpot_sum = 0.0;
  int64_t tpot_n = 0, pass = 0;
  for (const auto& r : recs) {
    const PerRequest m = metrics_of(r);
    e2e.push_back(m.e2e);
    ttft.push_back(m.ttft);
    ttft_sum += m.ttft;
    if (!m.single) {
      tpot.push_back(m.tpot);
      tpot_sum += m.tpot;
      ++tpot_n;
    }
    ++per_engine[r.engine_id];
    if (m.ttft <= ttft_slo && (m.single || m.tpot <= tpot_slo)) ++pass;
  }
  const double n = static_cast<double>(recs.size());
  out.p50_e2e = percentile_nearest_rank(e2e, 50.0);
  out.p90_e2e = percentile_nearest_rank(e2e, 90.0);
  out.p50_ttft = percentile_nearest_rank(ttft, 50.0);
  out.p50_tpot = tpot.empty() ? 0.0 : percentile_nearest_rank(tpot, 50.0);
  out.mean_ttft = ttft_sum / n;
  out.mean_tpot = tpot_n ? tpot_sum / static_cast<double>(tpot_n) : 0.0;
  out.slo_pct = 100.0 * static_cast<double>(pass) / n;
  for (const auto& [e, c] : per_engine)
    out.engine_share.emplace_back(e, static_cast<double>(c) / n);
  return out;
}

std::string build_summary_json(const RunCfg& cfg, int64_t arrived, int64_t completed,
                               int64_t rejected, int64_t unfinished,
                               uint64_t arrival_hash, uint64_t event_hash,
                               const Metrics& m,
                               const std::vector<LearnerRow>& learners) {
  // Key order and formatting follow proj/src/sim.cpp:349-392.
  char hex[32];
  nlohmann::ordered_json j;
  j["seed"] = cfg.seed;
  j["router_policy"] = route_policy_name(cfg.route_policy);
  j["engines"] = cfg.engines.size();
  j["arrived"] = arrived;
  j["completed"] = completed;
  j["rejected"] = rejected;
  j["unfinished"] = unfinished;
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(arrival_hash));
  j["arrival_hash"] = hex;
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(event_hash));
  j["event_hash"] = hex;
  nlohmann::ordered_json mm;
  mm["p50_e2e_ms"] = m.p50_e2e;
  mm["p90_e2e_ms"] = m.p90_e2e;
  mm["p50_ttft_ms"] = m.p50_ttft;
  mm["p50_tpot_ms"] = m.p50_tpot;
  mm["mean_ttft_ms"] = m.mean_ttft;
  mm["mean_tpot_ms"] = m.mean_tpot;
  mm["slo_attainment"] = m.slo_pct;
  j["metrics"] = mm;
  nlohmann::ordered_json share = nlohmann::ordered_json::object();
  for (const auto& [e, f] : m.engine_share) share[std::to_string(e)] = f;
  j["engine_share"] = share;
  nlohmann::ordered_json ls = nlohmann::ordered_json::array();
  for (const auto& l : learners) {
    nlohmann::ordered_json e;
    e["engine_id"] = l.engine_id;
    e["samples"] = l.samples;
    e["p_max"] = l.p_max;
    ls.push_back(e);
  }
  j["learners"] = ls;
  return j.dump(2) + "\n";
}

void write_requests_csv(const std::string& path, const std::vector<RecordRow>& recs) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write csv: " + path);
  out << "request_id,engine_id,arrival_ms,first_token_ms,completed_ms,"
         "prompt_tokens,output_tokens,ttft_ms,tpot_ms,e2e_ms\n";
  char buf[320];
  for (const auto& r : recs) {
    const PerRequest m = metrics_of(r);
    std::snprintf(buf, sizeof buf, "%llu,%d,%.3f,%.3f,%.3f,%lld,%lld,%.3f,%.6f,%.3f\n",
                  static_cast<unsigned long long>(r.request_id), r.engine_id, r.arrival_ms,
                  r.first_token_ms, r.completed_ms, static_cast<long long>(r.prompt_tokens),
                  static_cast<long long>(r.output_tokens), m.ttft, m.tpot, m.e2e);
    out << buf;
  }
}

}  // namespace nx
