// Host post-processing of a finished replica: per-request metrics, the
// summary statistics and the summary.json document. Out of kernel scope
// (SURVEY.md §2 "Metrics"), but byte-identical output is part of parity.
//   request_metrics / percentile / slo_attainment / summarize
//                                  proj/src/metrics.cpp:7-91
//   build_summary                  proj/src/sim.cpp:349-392
//   write_requests_csv             proj/src/metrics.cpp:93-111
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "frontend.hpp"

namespace nx {

struct RecordRow {
  int64_t request_id = 0;
  double arrival_ms = 0.0, first_token_ms = 0.0, completed_ms = 0.0;
  int64_t prompt_tokens = 0, output_tokens = 0;
  int32_t engine_id = 0;
};

struct Metrics {
  int64_t completed = 0;
  double p50_e2e = 0.0, p90_e2e = 0.0, p50_ttft = 0.0, p50_tpot = 0.0;
  double mean_ttft = 0.0, mean_tpot = 0.0, slo_pct = 100.0;
  std::vector<std::pair<int, double>> engine_share;
};

struct LearnerRow {
  int32_t engine_id;
  int64_t samples;
  double p_max;
};

double percentile_nearest_rank(std::vector<double> values, double p);
Metrics summarize_records(const std::vector<RecordRow>& recs, double ttft_slo,
                          double tpot_slo);
std::string build_summary_json(const RunCfg& cfg, int64_t arrived, int64_t completed,
                               int64_t rejected, int64_t unfinished,
                               uint64_t arrival_hash, uint64_t event_hash,
                               const Metrics& m,
                               const std::vector<LearnerRow>& learners);
void write_requests_csv(const std::string& path, const std::vector<RecordRow>& recs);

}  // namespace nx
