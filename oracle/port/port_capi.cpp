// TEST INFRASTRUCTURE — C-ABI for the CPU restatement (oracle/_port).
// Same JSON result layout as oracle/ref_driver.cpp::ref_run_json so tests can
// diff the two field by field.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "report.hpp"
#include "sim_port.hpp"

namespace {
thread_local std::string g_err;

int classify(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::logic_error*>(&e)) return 3;
  if (dynamic_cast<const std::runtime_error*>(&e)) return 2;
  return 9;
}

std::string run_one(const std::string& text, bool with_records, int64_t* decisions,
                    uint64_t* ev_hash) {
  const nx::RunCfg cfg = nx::parse_run_config(text);
  const nx::Workload w = nx::build_workload(cfg);
  const port::Result r = port::simulate(cfg, w);
  std::vector<nx::RecordRow> rows;
  rows.reserve(r.records.size());
  for (const auto& rec : r.records) {
    nx::RecordRow row;
    row.request_id = rec.request;
    row.arrival_ms = w.arrival_ms[rec.request];
    row.first_token_ms = nx::to_ms(rec.first_us);
    row.completed_ms = nx::to_ms(rec.done_us);
    row.prompt_tokens = w.prompt[rec.request];
    row.output_tokens = w.output[rec.request];
    row.engine_id = rec.engine_id;
    rows.push_back(row);
  }
  std::vector<nx::LearnerRow> learners;
  int64_t batches = 0;
  for (const auto& e : r.engines) {
    learners.push_back({e.engine_id, e.samples, e.params.p_max});
    batches += e.samples;
  }
  if (decisions) *decisions = r.arrived + batches;
  if (ev_hash) *ev_hash = r.event_hash;
  const nx::Metrics m = nx::summarize_records(rows, cfg.ttft_slo, cfg.tpot_slo);
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
  j["decisions"] = r.arrived + batches;
  j["events"] = r.events;
  j["summary_json"] = nx::build_summary_json(cfg, r.arrived, r.completed, r.rejected,
                                             r.unfinished, r.arrival_hash, r.event_hash, m,
                                             learners);
  nlohmann::ordered_json params = nlohmann::ordered_json::array();
  for (const auto& e : r.engines) {
    const nx::Params& p = e.params;
    params.push_back({p.tau0, p.w0, p.ws, p.tauB, p.tauS, p.p_max, p.kB, p.kS});
  }
  j["learner_params"] = params;
  if (with_records) {
    std::vector<int64_t> id, eng, pt, ot;
    std::vector<double> arr, ft, done;
    for (const auto& row : rows) {
      id.push_back(row.request_id);
      eng.push_back(row.engine_id);
      pt.push_back(row.prompt_tokens);
      ot.push_back(row.output_tokens);
      arr.push_back(row.arrival_ms);
      ft.push_back(row.first_token_ms);
      done.push_back(row.completed_ms);
    }
    j["rec_id"] = id;
    j["rec_engine"] = eng;
    j["rec_prompt"] = pt;
    j["rec_output"] = ot;
    j["rec_arrival"] = arr;
    j["rec_first"] = ft;
    j["rec_done"] = done;
  }
  return j.dump();
}
}  // namespace

extern "C" {

const char* port_last_error() { return g_err.c_str(); }
void port_free(char* p) { std::free(p); }

int port_run_json(const char* cfg_json, int with_records, char** out) {
  try {
    const std::string s = run_one(cfg_json, with_records != 0, nullptr, nullptr);
    *out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

int port_run_batch(const char* const* cfgs, int n, int threads, int64_t* decisions,
                   uint64_t* event_hash, double* wall) {
  std::atomic<int> next{0}, failed{0};
  const auto t0 = std::chrono::steady_clock::now();
  auto worker = [&]() {
    for (int i = next++; i < n; i = next++) {
      try {
        run_one(cfgs[i], false, &decisions[i], &event_hash[i]);
      } catch (const std::exception& e) {
        g_err = e.what();
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

int port_perf_eval(const double* p8, const int64_t* b, const int64_t* s, int64_t n,
                   double* out_T, double* out_thr) {
  try {
    nx::Params p{p8[0], p8[1], p8[2], p8[3], p8[4], p8[5], p8[6], p8[7]};
    for (int64_t i = 0; i < n; ++i) {
      out_thr[i] = port::throughput(p, b[i], s[i]);
      out_T[i] = port::predict_latency(p, b[i], s[i]);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Writes a JSONL trace (workload.cpp:123-135 format) for `rows` given as arrays.
int port_write_trace(const char* path, const double* arrival, const int64_t* prompt,
                     const int64_t* output, const char* const* session, int64_t n) {
  try {
    std::vector<nx::TraceRow> rows(n);
    for (int64_t i = 0; i < n; ++i) rows[i] = {arrival[i], session[i], prompt[i], output[i]};
    nx::write_trace_rows(path, rows);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

}  // extern "C"
