// Per-call cost of the scalar drop-in API from C++ (include/nx_servesim.hpp):
// predict_latency, schedule_step, Router::route — each one device round trip.
// Build: g++ -std=gnu++20 -O2 -Iinclude tools/micro/scalar_cpp.cpp -o tools/micro/scalar_cpp \
//   -Lpaper_2509_23384_b200 -l:_nxsched.so -Wl,-rpath,$PWD/paper_2509_23384_b200
#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

#include "nx_servesim.hpp"

using namespace servesim;
using clk = std::chrono::steady_clock;

template <class F>
double us_per_call(int n, F f) {
  for (int i = 0; i < 20; ++i) f(i);
  const auto t0 = clk::now();
  for (int i = 0; i < n; ++i) f(i);
  return std::chrono::duration<double, std::micro>(clk::now() - t0).count() / n;
}

int main() {
  const PerfParams p = perf_profile("fast");
  volatile double sink = 0.0;
  const double t_pred = us_per_call(2000, [&](int i) { sink = sink + predict_latency(p, BatchShape{4, 100 + i}); });
  std::vector<Request> run, wait;
  for (int i = 0; i < 8; ++i) {
    Request r;
    r.id = i;
    r.prompt_len = 64;
    r.prefilled = 64;
    run.push_back(r);
  }
  for (int i = 0; i < 16; ++i) {
    Request r;
    r.id = 100 + i;
    r.prompt_len = 300 + 17 * i;
    wait.push_back(r);
  }
  std::vector<const Request*> wq, rq;
  for (const Request& r : wait) wq.push_back(&r);
  for (const Request& r : run) rq.push_back(&r);
  const double t_lens = us_per_call(500, [&](int) {
    const BatchPlan plan = schedule_step(wq, rq, SLOSpec{}, TradeoffModel{}, p, SchedulerConfig{});
    sink = sink + plan.predicted_ms;
  });
  Router rt(RouterConfig{}, SLOSpec{}, 1);
  for (int e = 0; e < 8; ++e) {
    rt.register_engine(e);
    EngineReport rep;
    rep.state.engine_id = e;
    rep.state.l_hat_ms = 100.0 * e;
    rep.state.w_load_tokens = 1000.0 * e;
    rep.state.m_free_tokens = 50000.0;
    rep.state.p_max = 20.0;
    rep.queue_len = e;
    rt.on_report(rep);
  }
  const double t_route = us_per_call(500, [&](int i) {
    Request r;
    r.id = 1000 + i;
    r.prompt_len = 500 + i;
    r.session_id = "s" + std::to_string(i % 16);
    const RouteDecision d = rt.route(r, 1.0 + i);
    sink = sink + d.score;
  });
  std::printf("C++ drop-in, per call: predict_latency %.1f us, schedule_step %.1f us (8 running + 16 waiting), "
              "Router::route %.1f us (8 engines)\n", t_pred, t_lens, t_route);
  return 0;
}
