// TEST INFRASTRUCTURE — CPU restatement ("port") of the NexusSched hot path.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
// The product never links it. It restates, in flat arrays and per-engine event
// slots (the same flattening the device kernel uses), the reference's
//   perf model        proj/src/perf_model.cpp:15-49
//   LENS              proj/src/lens.cpp:10-146, TradeoffEstimator :148-188
//   baseline policies proj/src/engine.cpp:61-108
//   PRISM + baselines proj/src/router.cpp:38-289
//   online learner    proj/src/learner.cpp:24-440
//   engine            proj/src/engine.cpp:110-332
//   event loop        proj/src/sim.cpp:143-347
// Parity of this restatement against the compiled reference (oracle/_ref) is
// checked by tests/test_oracle_parity.py (event_hash, records, summary).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "frontend.hpp"

namespace port {

struct Record {
  int32_t request;
  int32_t engine_id;
  int64_t first_us, done_us;
};

struct EngineOut {
  int32_t engine_id;
  int64_t samples;
  nx::Params params;
  int64_t counters[7];
};

struct Result {
  int64_t arrived = 0, completed = 0, rejected = 0, unfinished = 0;
  uint64_t arrival_hash = 0, event_hash = 0;
  std::vector<Record> records;
  std::vector<EngineOut> engines;
  int64_t events = 0;
};

Result simulate(const nx::RunCfg& cfg, const nx::Workload& w);

// Scalar kernels exposed for unit-level golden checks.
double throughput(const nx::Params& p, int64_t b, int64_t s);
double predict_latency(const nx::Params& p, int64_t b, int64_t s);

}  // namespace port
