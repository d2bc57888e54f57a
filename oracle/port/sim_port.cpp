// TEST INFRASTRUCTURE — flat CPU restatement of the NexusSched hot path.
// See sim_port.hpp. Every block cites the reference lines it restates.
#include "sim_port.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <deque>
#include <limits>
#include <stdexcept>

namespace port {
namespace {

using nx::Params;
using nx::to_ms;
using nx::to_us;

const double kFactorMax = std::nextafter(1.0, 0.0);
constexpr double kInf = std::numeric_limits<double>::infinity();

// perf_model.cpp:17-20
double sat(double k, double x) {
  const double f = -std::expm1(-k * x);
  return f < kFactorMax ? f : kFactorMax;
}

int64_t blocks_for(int64_t tokens, int64_t block) { return (tokens + block - 1) / block; }

// ----------------------------------------------------------------------------
// Online learner (learner.cpp)
// ----------------------------------------------------------------------------
using Mat5 = std::array<std::array<double, 5>, 5>;
using Vec5 = std::array<double, 5>;

// learner.cpp:24-60 — column-scaled partial-pivot elimination.
bool solve5(Mat5 a, Vec5 b, Vec5* x) {
  Vec5 scale{};
  for (int j = 0; j < 5; ++j) {
    double m = 0.0;
    for (int i = 0; i < 5; ++i) m = std::max(m, std::fabs(a[i][j]));
    if (m <= 0.0) return false;
    scale[j] = 1.0 / m;
    for (int i = 0; i < 5; ++i) a[i][j] *= scale[j];
  }
  double norm = 0.0;
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) norm = std::max(norm, std::fabs(a[i][j]));
  for (int col = 0; col < 5; ++col) {
    int piv = col;
    for (int r = col + 1; r < 5; ++r)
      if (std::fabs(a[r][col]) > std::fabs(a[piv][col])) piv = r;
    if (std::fabs(a[piv][col]) < 1e-10 * norm) return false;
    std::swap(a[col], a[piv]);
    std::swap(b[col], b[piv]);
    for (int r = col + 1; r < 5; ++r) {
      const double f = a[r][col] / a[col][col];
      for (int c = col; c < 5; ++c) a[r][c] -= f * a[col][c];
      b[r] -= f * b[col];
    }
  }
  if (!x) return true;
  Vec5& out = *x;
  for (int r = 4; r >= 0; --r) {
    double acc = b[r];
    for (int c = r + 1; c < 5; ++c) acc -= a[r][c] * out[c];
    out[r] = acc / a[r][r];
  }
  for (int j = 0; j < 5; ++j) out[j] *= scale[j];
  return true;
}

struct Normal5 {  // learner.cpp:62-98
  Mat5 ata{};
  Vec5 atb{};
  double y2 = 0.0;
  void add(const Vec5& r) {  // target y = 1 after 1/y row weighting
    for (int i = 0; i < 5; ++i) {
      for (int j = 0; j < 5; ++j) ata[i][j] += r[i] * r[j];
      atb[i] += r[i] * 1.0;
    }
    y2 += 1.0 * 1.0;
  }
  template <class Sse>
  bool solve(const Vec5& prior, Vec5* x, Sse&& sse, double cap) const {
    if (!solve5(ata, atb, x)) return false;
    const double lambda = std::min(cap, sse(*x) / std::max(y2, 1e-30));
    if (lambda > 1e-14) {
      Mat5 a = ata;
      Vec5 b = atb;
      for (int i = 0; i < 5; ++i) {
        const double d = lambda * ata[i][i];
        a[i][i] += d;
        b[i] += d * prior[i];
      }
      if (!solve5(a, b, x)) return false;
    }
    return true;
  }
};

double floor_at(double v, double lo, bool& hit) {
  if (v < lo) {
    hit = true;
    return lo;
  }
  return v;
}

struct Learner {
  int64_t long_w, short_w, s_period, l_period, min_s;
  Params cur;
  std::vector<int32_t> rb, rs;
  std::vector<double> ry;
  int64_t size = 0, head = 0, seen = 0;
  int64_t counters[7] = {0, 0, 0, 0, 0, 0, 0};  // lin, struct, degen, rescale, clamp, failed, lowid

  struct Sample { int64_t b, s; double y; };

  std::vector<Sample> window(int64_t n) const {  // learner.cpp:148-158
    const int64_t count = std::min(n, size);
    std::vector<Sample> out;
    out.reserve(count);
    for (int64_t i = size - count; i < size; ++i) {
      const int64_t k = (head + i) % size;
      out.push_back({rb[k], rs[k], ry[k]});
    }
    return out;
  }

  void record(int64_t b, int64_t s, double y) {  // learner.cpp:130-146
    if (!(y > 0.0) || !(b >= 1 && s >= b)) throw std::invalid_argument("invalid LatencySample");
    if (size < long_w) {
      rb[size] = (int32_t)b; rs[size] = (int32_t)s; ry[size] = y;
      ++size;
    } else {
      rb[head] = (int32_t)b; rs[head] = (int32_t)s; ry[head] = y;
      head = (head + 1) % size;
    }
    ++seen;
    if (seen % l_period == 0) update_linear();
    if (seen >= min_s && seen % s_period == 0) update_structural();
  }

  bool update_linear() {  // learner.cpp:160-207, 300-344
    const auto win = window(short_w);
    if (win.size() < 5) return false;
    Normal5 ols;
    std::vector<Vec5> rows;
    rows.reserve(win.size());
    for (const auto& sm : win) {
      const double thr = throughput(cur, sm.b, sm.s);
      const double s = (double)sm.s, b = (double)sm.b;
      rows.push_back({1.0, 1.0 / thr, s / thr, b, s});
      const double iy = 1.0 / sm.y;
      const Vec5& r = rows.back();
      ols.add({r[0] * iy, r[1] * iy, r[2] * iy, r[3] * iy, r[4] * iy});
    }
    const Vec5 prior{cur.tau0, cur.w0, cur.ws, cur.tauB, cur.tauS};
    auto noise = [&](const Vec5& x) {
      double acc = 0.0;
      for (size_t i = 0; i < rows.size(); ++i) {
        double pred = 0.0;
        for (int j = 0; j < 5; ++j) pred += rows[i][j] * x[j];
        const double r = (win[i].y - pred) / win[i].y;
        acc += r * r;
      }
      return 8.0 * acc;
    };
    Vec5 x{};
    if (!ols.solve(prior, &x, noise, 1e-2)) {
      ++counters[2];
      double num = 0.0, den = 0.0;
      for (const auto& sm : win) {
        const double pred = predict_latency(cur, sm.b, sm.s);
        const double wt = 1.0 / (sm.y * sm.y);
        num += wt * pred * sm.y;
        den += wt * pred * pred;
      }
      const double g = num / den;
      if (std::isfinite(g) && g > 0.0 && g != 1.0) {
        Params nx = cur;
        nx.tau0 *= g;
        nx.w0 *= g;
        nx.ws = std::max(1e-6, nx.ws * g);
        nx.tauB *= g;
        nx.tauS *= g;
        cur = nx;
        ++counters[3];
      }
      return false;
    }
    bool clamped = false;
    Params nx = cur;
    nx.tau0 = floor_at(x[0], 0.0, clamped);
    nx.w0 = floor_at(x[1], 0.0, clamped);
    nx.ws = floor_at(x[2], 1e-6, clamped);
    nx.tauB = floor_at(x[3], 0.0, clamped);
    nx.tauS = floor_at(x[4], 0.0, clamped);
    cur = nx;
    ++counters[0];
    if (clamped) ++counters[4];
    return true;
  }

  double sse_of(const std::vector<Sample>& win, const Params& p) const {  // :209-222
    double sse = 0.0;
    for (const auto& sm : win) {
      const double r = (sm.y - predict_latency(p, sm.b, sm.s)) / sm.y;
      sse += r * r;
    }
    return sse;
  }

  double gauged(const std::vector<Sample>& win, double kB, double kS, Params* out) const {
    // learner.cpp:228-298 — ws = 1 gauge, profiled p_max.
    Normal5 ols;
    std::vector<Vec5> rows;
    rows.reserve(win.size());
    for (const auto& sm : win) {
      const double fb = -std::expm1(-kB * (double)sm.b);
      const double fs = -std::expm1(-kS * (double)sm.s);
      const double f = std::max(fb * fs, 1e-300);
      const double s = (double)sm.s, b = (double)sm.b;
      rows.push_back({1.0, 1.0 / f, s / f, b, s});
      const double iy = 1.0 / sm.y;
      const Vec5& r = rows.back();
      ols.add({r[0] * iy, r[1] * iy, r[2] * iy, r[3] * iy, r[4] * iy});
    }
    const double cur_c = cur.ws / cur.p_max;
    const Vec5 prior{cur.tau0, cur.w0 / cur.p_max, cur_c, cur.tauB, cur.tauS};
    auto sse = [&](const Vec5& x) {
      double acc = 0.0;
      for (size_t i = 0; i < rows.size(); ++i) {
        double pred = 0.0;
        for (int j = 0; j < 5; ++j) pred += rows[i][j] * x[j];
        const double r = (win[i].y - pred) / win[i].y;
        acc += r * r;
      }
      return acc;
    };
    Vec5 x{};
    if (!ols.solve(prior, &x, sse, 1e-7)) return kInf;
    bool clamped = false;
    const double tau0 = floor_at(x[0], 0.0, clamped);
    const double a = floor_at(x[1], 0.0, clamped);
    const double slope = cur.ws / cur.p_max + cur.tauS;
    const double c_lo = std::max(1.0 / 1e4, slope / 16.0);
    const double c_hi = std::max(c_lo, std::min(1.0 / 1e-3, 4.0 * slope));
    const double c = std::clamp(x[2], c_lo, c_hi);
    const double tauB = floor_at(x[3], 0.0, clamped);
    const double tauS = floor_at(x[4], 0.0, clamped);
    Params p = cur;
    p.kB = kB;
    p.kS = kS;
    p.p_max = 1.0 / c;
    p.w0 = a / c;
    p.ws = 1.0;
    p.tau0 = tau0;
    p.tauB = tauB;
    p.tauS = tauS;
    *out = p;
    return sse_of(win, p);
  }

  bool update_structural() {  // learner.cpp:346-440
    const auto all = window(long_w);
    if ((int64_t)all.size() < min_s || all.size() < 5) return false;
    bool saturated = true;
    int64_t shaped = 0;
    for (const auto& sm : all) {
      if (cur.kB * (double)sm.b < 20.0 || cur.kS * (double)sm.s < 20.0) saturated = false;
      if (sm.s >= 64 && sm.s >= 4 * sm.b) ++shaped;
    }
    if (saturated || shaped < 16) {
      ++counters[6];
      return false;
    }
    const double base_err = sse_of(all, cur);
    const double lo = std::log(1e-8), hi = std::log(1e4);
    double th[2] = {std::log(cur.kB), std::log(cur.kS)};
    double step[2] = {0.5, 0.5};
    Params best;
    double best_err = gauged(all, std::exp(th[0]), std::exp(th[1]), &best);
    if (!std::isfinite(best_err)) {
      ++counters[5];
      return false;
    }
    const double kbs[3] = {0.05, 0.7, 8.0}, kss[3] = {0.002, 0.03, 0.4};
    for (double kb : kbs) {
      for (double ks : kss) {
        Params cand;
        const double err = gauged(all, kb, ks, &cand);
        if (std::isfinite(err) && err < best_err * (1.0 - 1e-3)) {
          th[0] = std::log(kb);
          th[1] = std::log(ks);
          best = cand;
          best_err = err;
        }
      }
    }
    for (int sweep = 0; sweep < 50; ++sweep) {
      bool improved = false;
      for (int c = 0; c < 2; ++c) {
        bool hit = false;
        for (double dir : {+1.0, -1.0}) {
          double ct[2] = {th[0], th[1]};
          ct[c] = std::clamp(ct[c] + dir * step[c], lo, hi);
          if (ct[c] == th[c]) continue;
          Params cand;
          const double err = gauged(all, std::exp(ct[0]), std::exp(ct[1]), &cand);
          if (std::isfinite(err) && err < best_err * (1.0 - 1e-3)) {
            th[0] = ct[0];
            th[1] = ct[1];
            best = cand;
            best_err = err;
            hit = true;
            break;
          }
        }
        step[c] *= hit ? 1.6 : 0.5;
        improved |= hit;
      }
      if (!improved && std::max(step[0], step[1]) < 1e-5) break;
    }
    if (!best.valid() || best_err > base_err) {
      ++counters[5];
      return false;
    }
    cur = best;
    ++counters[1];
    update_linear();
    return true;
  }
};

// ----------------------------------------------------------------------------
// Engine-side state (engine.cpp, lens.cpp)
// ----------------------------------------------------------------------------
struct Alloc {
  int32_t req;
  int32_t tokens;
  bool prefill;
};

struct Plan {
  std::vector<Alloc> allocs;
  int64_t b = 0, s = 0;
  double predicted = 0.0, target = 0.0;
  bool overload = false;
};

struct StateVec {
  double l_hat = 0.0, w_load = 0.0, m_free = 0.0, p_max = 1.0, at = 0.0;
  int64_t queue_len = 0;
};

struct Delivery {
  int64_t t;
  uint64_t seq;
  StateVec sv;
};

struct Engine {
  nx::EngineCfg cfg;
  int64_t m_max, q_max;
  Learner learner;
  // tradeoff estimator (lens.cpp:148-188)
  double alpha, beta, l_bar, td_min;
  std::deque<std::pair<double, double>> tw;  // (ttft, tpot)
  int64_t degenerate = 0;
  nx::Xoshiro rng{0};
  // queues: wait = wq[wq_head, wq_head + wq_len), run = rq[0, rq_len)
  std::vector<int32_t> wq, rq;
  int64_t wq_head = 0, wq_len = 0;
  // kv (engine.h:171-177) + prefix LRU keyed by interned session
  int64_t pinned = 0, reserved = 0, cache_blocks = 0;
  std::vector<int32_t> c_tokens, c_prev, c_next;  // per session; c_tokens < 0 = absent
  int32_t c_head = -1, c_tail = -1;
  // in-flight step
  bool busy = false;
  Plan plan;
  int64_t started_us = 0;
  double actual = 0.0;
  // event slots (flattened per-engine queue heads)
  bool step_ev = false, learn_ev = false, report_ev = false;
  int64_t step_t = 0, learn_t = 0, report_t = 0;
  uint64_t step_seq = 0, learn_seq = 0, report_seq = 0;
  int64_t learn_b = 0, learn_s = 0;
  double learn_y = 0.0;
  std::deque<Delivery> deliveries;

  int64_t committed() const { return pinned + reserved; }
  int64_t free_blocks() const { return cfg.kv_blocks - pinned; }
  int64_t bf(int64_t t) const { return blocks_for(t, cfg.block_size); }

  void lru_unlink(int32_t s) {
    const int32_t p = c_prev[s], n = c_next[s];
    if (p >= 0) c_next[p] = n; else c_head = n;
    if (n >= 0) c_prev[n] = p; else c_tail = p;
    c_tokens[s] = -1;
  }
  void lru_push_back(int32_t s, int32_t tokens) {
    c_tokens[s] = tokens;
    c_prev[s] = c_tail;
    c_next[s] = -1;
    if (c_tail >= 0) c_next[c_tail] = s; else c_head = s;
    c_tail = s;
  }
  void evict_to_fit() {  // engine.cpp:298-305
    while (cache_blocks > free_blocks() && c_head >= 0) {
      const int32_t v = c_head;
      cache_blocks -= bf(c_tokens[v]);
      lru_unlink(v);
    }
  }
  void cache_insert(int32_t s, int64_t tokens) {  // engine.cpp:284-296
    if (c_tokens[s] >= 0) {
      cache_blocks -= bf(c_tokens[s]);
      lru_unlink(s);
    }
    lru_push_back(s, (int32_t)tokens);
    cache_blocks += bf(tokens);
    evict_to_fit();
  }
};

struct Req {
  double arr_ms;
  int32_t prompt, target, session;
  int32_t prefilled = 0, decoded = 0;
  int64_t first_us = -1;
  bool admitted_kv = false;
  int32_t remaining() const { return prompt - prefilled; }
};

// lens.cpp:10-31
double target_latency(int64_t wait_count, double ttft, double tpot, double alpha,
                      double beta, double l_bar, double td_min, double q_ref) {
  const double td_tpot = tpot;
  const double td_ttft = (alpha - ttft) / beta;
  double t;
  if (l_bar > beta) t = std::min(td_tpot, std::max(td_min, td_ttft));
  else t = td_tpot;
  if (wait_count > 0) {
    const double relax = std::min(1.0, (double)wait_count / q_ref);
    t += relax * (td_tpot - t);
  }
  return t;
}

// lens.cpp:33-56
int64_t bisect_budget(int64_t b, double target, const Params& p, int64_t m_max,
                      int64_t q_max, int iters, int64_t s_cap) {
  if (b < 1 || b > q_max || !(target > 0.0)) throw std::invalid_argument("binary_search_budget");
  if (s_cap < 0) s_cap = m_max;
  s_cap = std::max(b, std::min(s_cap, m_max));
  int64_t lo = b, hi = s_cap, budget = b;
  for (int it = 0; it < iters; ++it) {
    if (lo > hi) break;
    const int64_t mid = (lo + hi) / 2;
    if (predict_latency(p, b, mid) <= target) {
      budget = mid;
      lo = mid + 1;
    } else {
      hi = mid - 1;
    }
  }
  return budget;
}

struct Sim {
  const nx::RunCfg& cfg;
  const nx::Workload& w;
  std::vector<Req> req;
  std::vector<Engine> eng;
  int E;
  // router
  std::vector<bool> has_rep;
  std::vector<StateVec> rep;
  std::vector<std::deque<std::pair<double, double>>> lat_win;
  std::vector<double> lat_sum;
  std::vector<int32_t> sess_engine;  // session -> engine index, -1 unknown
  uint64_t rr_next = 0;
  double l_bar_ema = 128.0;
  nx::Xoshiro router_rng{0};
  std::vector<double> static_w;
  // loop
  uint64_t next_seq = 0;
  int64_t cursor = 0, arrived = 0, rejected = 0, pending = 0;
  uint64_t ev_hash = nx::kFnvBasis;
  std::vector<Record> records;
  int64_t events = 0;

  Sim(const nx::RunCfg& c, const nx::Workload& wl) : cfg(c), w(wl) {
    const int64_t n = (int64_t)w.prompt.size();
    const int64_t ns = (int64_t)w.session_names.size();
    req.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      req[i].arr_ms = w.arrival_ms[i];
      req[i].prompt = w.prompt[i];
      req[i].target = w.output[i];
      req[i].session = w.session[i];
    }
    E = (int)cfg.engines.size();
    eng.resize(E);
    for (int e = 0; e < E; ++e) {
      Engine& g = eng[e];
      g.cfg = cfg.engines[e];
      g.m_max = g.cfg.m_max;
      g.q_max = g.cfg.q_max;
      Learner& L = g.learner;
      L.long_w = cfg.long_window;
      L.short_w = cfg.short_window;
      L.s_period = cfg.structural_period;
      L.l_period = cfg.linear_period;
      L.min_s = cfg.min_structural;
      L.cur = nx::learner_default_priors();
      L.rb.assign(L.long_w, 0);
      L.rs.assign(L.long_w, 0);
      L.ry.assign(L.long_w, 0.0);
      g.alpha = cfg.alpha;
      g.beta = cfg.beta;
      g.l_bar = cfg.l_bar;
      g.td_min = cfg.td_min;
      g.rng = nx::Xoshiro(nx::substream_seed(cfg.seed, "engine-noise", (uint64_t)g.cfg.engine_id));
      g.wq.assign(n, -1);
      g.rq.reserve(n);
      g.c_tokens.assign(ns, -1);
      g.c_prev.assign(ns, -1);
      g.c_next.assign(ns, -1);
    }
    has_rep.assign(E, false);
    rep.assign(E, {});
    lat_win.resize(E);
    lat_sum.assign(E, 0.0);
    sess_engine.assign(ns, -1);
    router_rng = nx::Xoshiro(nx::substream_seed(cfg.seed, "router"));
    static_w.assign(E, 1.0);
    for (int e = 0; e < E; ++e) {
      auto it = cfg.static_weights.find(cfg.engines[e].engine_id);
      if (it != cfg.static_weights.end()) static_w[e] = it->second;
    }
  }

  int64_t active() const { return arrived - rejected - (int64_t)records.size(); }

  // ---- router (router.cpp) -------------------------------------------------
  double s_latency(const StateVec& sv) const {  // :38-45
    const double knee = cfg.knee * cfg.ttft_slo;
    if (sv.l_hat <= knee) return 1.0;
    const double scale = cfg.scale_ms > 0.0 ? cfg.scale_ms : 0.25 * cfg.ttft_slo;
    return std::exp(-(sv.l_hat - knee) / scale);
  }
  double s_load(const StateVec& sv) const {  // :47-50
    const double rho = sv.w_load / sv.p_max;
    return 1.0 / (1.0 + rho / cfg.load_half);
  }
  double s_capacity(const StateVec& sv, double demand) const {  // :52-60
    if (demand < 1.0) throw std::invalid_argument("score_capacity: demand must be >= 1 token");
    const double r = std::clamp(sv.m_free / (cfg.headroom * demand), 0.0, 1.0);
    return r * r;
  }
  int least_loaded() const {
    int best = 0;
    int64_t best_len = std::numeric_limits<int64_t>::max();
    for (int e = 0; e < E; ++e) {
      const int64_t len = has_rep[e] ? rep[e].queue_len : 0;
      if (len < best_len) {
        best_len = len;
        best = e;
      }
    }
    return best;
  }
  int rr() { return (int)(rr_next++ % (uint64_t)E); }

  int route(int32_t r, double now) {  // :141-289
    const Req& q = req[r];
    int chosen = -1;
    switch (cfg.route_policy) {
      case nx::kRoundRobin: chosen = rr(); break;
      case nx::kSessionAffinity: {
        const int32_t e = sess_engine[q.session];
        chosen = e >= 0 ? e : rr();
        break;
      }
      case nx::kLeastLoaded: chosen = least_loaded(); break;
      case nx::kLatencyBased: {
        chosen = 0;
        double best = kInf;
        for (int e = 0; e < E; ++e) {
          auto& win = lat_win[e];
          while (!win.empty() && win.front().first < now - cfg.latency_window) {
            lat_sum[e] -= win.front().second;
            win.pop_front();
          }
          const double lat = win.empty() ? 0.0 : lat_sum[e] / (double)win.size();
          if (lat < best) {
            best = lat;
            chosen = e;
          }
        }
        break;
      }
      case nx::kWeighted: {
        double total = 0.0;
        for (int e = 0; e < E; ++e) total += static_w[e];
        double draw = router_rng.uniform() * total;
        chosen = E - 1;
        for (int e = 0; e < E; ++e) {
          draw -= static_w[e];
          if (draw <= 0.0) {
            chosen = e;
            break;
          }
        }
        break;
      }
      default: {  // PRISM
        const double demand = std::max(1.0, (double)q.prompt + l_bar_ema);
        bool any_fresh = false;
        double best_score = -1.0, best_rho = kInf;
        int best_id = -1;
        for (int e = 0; e < E; ++e) {
          double f[4] = {1.0, 1.0, 1.0, 1.0};
          double rho = 0.0;
          const double age = has_rep[e] ? now - rep[e].at : kInf;
          if (has_rep[e] && age <= cfg.staleness_limit) {
            any_fresh = true;
            f[0] = s_latency(rep[e]);
            f[1] = s_load(rep[e]);
            f[2] = s_capacity(rep[e], demand);
            rho = rep[e].w_load / rep[e].p_max;
          } else {
            f[0] = 0.5;
            f[2] = 0.5;
            if (has_rep[e]) {
              rho = rep[e].w_load / rep[e].p_max;
              const double blend = std::exp(-(age - cfg.staleness_limit) / cfg.staleness_limit);
              f[1] = 1.0 + (s_load(rep[e]) - 1.0) * blend;
            }
          }
          f[3] = sess_engine[q.session] == e ? cfg.beta_aff : 1.0;
          double score = 1.0;
          for (int i = 0; i < 4; ++i)
            score *= (f[i] == 0.0 && cfg.weights[i] > 0.0) ? 0.0 : std::pow(f[i], cfg.weights[i]);
          const int id = eng[e].cfg.engine_id;
          const bool better = score > best_score ||
                              (score == best_score && (rho < best_rho || (rho == best_rho && id < best_id)));
          if (chosen < 0 || better) {
            best_score = score;
            best_rho = rho;
            best_id = id;
            chosen = e;
          }
        }
        if (!any_fresh) chosen = least_loaded();
        if (has_rep[chosen]) {
          rep[chosen].queue_len += 1;
          rep[chosen].w_load += (double)q.prompt + 32.0;
        }
        break;
      }
    }
    sess_engine[q.session] = chosen;  // remember_session, :107-122
    return chosen;
  }

  // ---- LENS (lens.cpp:96-146) + baselines (engine.cpp:61-108) --------------
  Plan plan_step(int e) {
    Engine& g = eng[e];
    Plan plan;
    const int64_t R = (int64_t)g.rq.size();
    const int64_t W = g.wq_len;
    if (R == 0 && W == 0) return plan;
    const Params& P = g.learner.cur;
    if (g.cfg.policy == nx::kPrefillPriority) {
      if (W > 0) {
        for (int64_t i = 0; i < W; ++i) {
          const int32_t r = g.wq[g.wq_head + i];
          const int64_t need = req[r].remaining();
          if (plan.b >= g.q_max || plan.s + need > g.m_max) {
            if (plan.allocs.empty()) throw std::runtime_error("prefill_priority: prompt exceeds m_max");
            break;
          }
          plan.allocs.push_back({r, (int32_t)need, true});
          plan.b += 1;
          plan.s += need;
        }
      } else {
        for (int32_t r : g.rq) {
          plan.allocs.push_back({r, 1, false});
          plan.b += 1;
          plan.s += 1;
        }
      }
      if (!plan.allocs.empty()) plan.predicted = predict_latency(P, plan.b, plan.s);
      return plan;
    }
    if (g.cfg.policy == nx::kStaticChunked) {
      const int64_t b = std::min<int64_t>(R + W, g.q_max);
      const int64_t s = std::min(g.m_max, std::max(g.cfg.static_budget, b));
      if (b < R || s < b) throw std::invalid_argument("allocate_tokens: budget below queue needs");
      materialize(g, b, s, plan);
      if (!plan.allocs.empty()) plan.predicted = predict_latency(P, plan.b, plan.s);
      return plan;
    }
    const double target = target_latency(W, cfg.ttft_slo, cfg.tpot_slo, g.alpha, g.beta,
                                         g.l_bar, g.td_min, cfg.q_ref);
    if (R > g.q_max) {  // overload: truncated decode plan (:108-117)
      for (int64_t i = 0; i < g.q_max; ++i) plan.allocs.push_back({g.rq[i], 1, false});
      plan.b = g.q_max;
      plan.s = g.q_max;
      plan.predicted = predict_latency(P, plan.b, plan.s);
      plan.target = target;
      plan.overload = true;
      return plan;
    }
    // prefix sums of remaining prompts over the candidate window (:121-124)
    const int64_t b_lo = std::max<int64_t>(R, 1);
    const int64_t b_hi = std::min(R + W, g.q_max);
    const int64_t span = std::max<int64_t>(0, b_hi - R);
    std::vector<int64_t> prefix(span + 1, 0);
    for (int64_t i = 0; i < span; ++i)
      prefix[i + 1] = prefix[i] + req[g.wq[g.wq_head + i]].remaining();
    double min_err = kInf;
    int64_t best_budget = -1, best_b = -1;
    for (int64_t B = b_lo; B <= b_hi; ++B) {
      const int64_t avail = R + prefix[B - R];
      const int64_t s_cap = std::min(g.m_max, avail);
      const int64_t budget = bisect_budget(B, target, P, g.m_max, g.q_max, cfg.n_search_iters, s_cap);
      // realized shape: S = budget, b = R + first j with prefix[j] >= budget - R
      const int64_t need = budget - R;
      int64_t j = 0;
      while (j < B - R && prefix[j] < need) ++j;
      const int64_t b_act = R + j;
      const double err = std::fabs(predict_latency(P, b_act, budget) - target);
      if (err < min_err) {
        min_err = err;
        best_budget = budget;
        best_b = B;
        if (min_err < target * cfg.eps_ratio) break;
      }
    }
    materialize(g, best_b, best_budget, plan);
    plan.predicted = predict_latency(P, plan.b, plan.s);
    plan.target = target;
    return plan;
  }

  // allocate_tokens (lens.cpp:58-79) for the chosen (b, s)
  void materialize(Engine& g, int64_t b, int64_t s, Plan& plan) {
    for (int32_t r : g.rq) plan.allocs.push_back({r, 1, false});
    int64_t slots = b - (int64_t)g.rq.size();
    int64_t budget = s - (int64_t)g.rq.size();
    for (int64_t i = 0; i < g.wq_len; ++i) {
      if (slots <= 0 || budget <= 0) break;
      const int32_t r = g.wq[g.wq_head + i];
      const int64_t take = std::min<int64_t>(req[r].remaining(), budget);
      plan.allocs.push_back({r, (int32_t)take, true});
      --slots;
      budget -= take;
    }
    plan.b = (int64_t)plan.allocs.size();
    plan.s = 0;
    for (const auto& a : plan.allocs) plan.s += a.tokens;
  }

  // engine.cpp:184-214
  void trim_for_kv(Engine& g, Plan& plan) {
    std::vector<Alloc> kept;
    bool trimmed = false;
    for (const auto& a : plan.allocs) {
      Req& r = req[a.req];
      if (!a.prefill || r.admitted_kv) {
        kept.push_back(a);
        continue;
      }
      if (trimmed) continue;
      const int64_t foot = g.bf((int64_t)r.prompt + r.target);
      const int64_t future = foot - g.bf((int64_t)r.prefilled + r.decoded);
      if (g.committed() + future <= g.cfg.kv_blocks) {
        g.reserved += future;
        r.admitted_kv = true;
        kept.push_back(a);
      } else {
        trimmed = true;
      }
    }
    if (kept.size() == plan.allocs.size()) return;
    plan.allocs = std::move(kept);
    plan.b = (int64_t)plan.allocs.size();
    plan.s = 0;
    for (const auto& a : plan.allocs) plan.s += a.tokens;
    plan.predicted = plan.b > 0 ? predict_latency(g.learner.cur, plan.b, plan.s) : 0.0;
  }

  void try_begin_step(int e, int64_t now_us) {  // sim.cpp:143-166, engine.cpp:216-228
    Engine& g = eng[e];
    if (g.busy || (g.wq_len == 0 && g.rq.empty())) return;
    Plan plan = plan_step(e);
    if (plan.allocs.empty()) return;
    trim_for_kv(g, plan);
    if (plan.allocs.empty()) return;
    double actual = predict_latency(g.cfg.true_params, plan.b, plan.s);  // :128-132
    if (g.cfg.noise_sigma != 0.0) actual = actual * std::exp(g.cfg.noise_sigma * g.rng.normal());
    g.busy = true;
    g.plan = std::move(plan);
    g.started_us = now_us;
    g.actual = actual;
    g.step_ev = true;
    g.step_t = now_us + std::max<int64_t>(1, to_us(actual));
    g.step_seq = next_seq++;
  }

  bool admit(int e, int32_t r) {  // engine.cpp:139-169
    Engine& g = eng[e];
    Req& q = req[r];
    if (g.cfg.wait_cap > 0 && g.wq_len >= g.cfg.wait_cap) return false;
    const int32_t cached = g.c_tokens[q.session];
    if (cached >= 0) {
      const int64_t credit = std::min<int64_t>(cached, (int64_t)q.prompt - 1);
      const int64_t cb = g.bf(credit);
      if (credit > 0 && g.committed() + cb <= g.cfg.kv_blocks) {
        g.cache_blocks -= g.bf(cached);
        g.lru_unlink(q.session);
        q.prefilled = (int32_t)credit;
        g.pinned += cb;
      }
    }
    g.wq[g.wq_head + g.wq_len] = r;
    ++g.wq_len;
    return true;
  }

  void tradeoff_update(Engine& g, const std::vector<std::array<double, 3>>& done) {
    for (const auto& c : done) {  // (ttft, tpot, decode_len)
      g.l_bar = std::max(1.0, g.l_bar + 0.05 * (c[2] - g.l_bar));
      if (c[2] >= 2.0) {
        g.tw.emplace_back(c[0], c[1]);
        if (g.tw.size() > 200) g.tw.pop_front();
      }
    }
    if (g.tw.size() < 2) return;
    double mtp = 0.0, mtd = 0.0;
    for (const auto& [tp, td] : g.tw) {
      mtp += tp;
      mtd += td;
    }
    const double n = (double)g.tw.size();
    mtp /= n;
    mtd /= n;
    double var = 0.0, cov = 0.0;
    for (const auto& [tp, td] : g.tw) {
      const double dd = td - mtd;
      var += dd * dd;
      cov += dd * (tp - mtp);
    }
    const double sd = std::sqrt(var / n);
    if (sd <= 0.15 * mtd) {
      ++g.degenerate;
      return;
    }
    const double slope = cov / var;
    g.beta = std::max(1e-3, -slope);
    g.alpha = mtp + g.beta * mtd;
  }

  void step_complete(int e, int64_t now_us) {  // sim.cpp:196-224, engine.cpp:230-282
    Engine& g = eng[e];
    const double now = to_ms(now_us);
    Plan plan = std::move(g.plan);
    g.busy = false;
    std::vector<std::array<double, 3>> done;
    std::vector<int32_t> finished;
    std::vector<int32_t> new_run;
    int64_t wq_removed_span = 0;
    for (const auto& a : plan.allocs) {
      Req& r = req[a.req];
      const int64_t before = g.bf((int64_t)r.prefilled + r.decoded);
      if (a.prefill) r.prefilled += a.tokens;
      else r.decoded += 1;
      const int64_t delta = g.bf((int64_t)r.prefilled + r.decoded) - before;
      g.pinned += delta;
      g.reserved -= delta;
      if (a.prefill && r.prefilled == r.prompt) {
        r.first_us = now_us;
        new_run.push_back(a.req);
        wq_removed_span = 1;
      } else if (!a.prefill && r.decoded == r.target) {
        const double first = to_ms(r.first_us);
        const double ttft = first - r.arr_ms;
        const double tpot = r.target >= 2 ? (now - first) / (double)(r.target - 1) : 0.0;
        done.push_back({ttft, tpot, (double)r.target});
        const int64_t held = g.bf((int64_t)r.prefilled + r.decoded);
        g.pinned -= held;
        g.cache_insert(r.session, (int64_t)r.prefilled + r.decoded);
        finished.push_back(a.req);
      }
    }
    // wait queue: drop requests whose prefill completed (they sit in the
    // scheduled FCFS window at the front; order of survivors preserved)
    if (wq_removed_span) {
      int64_t out = 0;
      std::vector<int32_t> keep;
      for (int64_t i = 0; i < g.wq_len; ++i) {
        const int32_t r = g.wq[g.wq_head + i];
        if (req[r].prefilled == req[r].prompt) continue;
        keep.push_back(r);
      }
      for (int32_t r : keep) g.wq[g.wq_head + out++] = r;
      g.wq_len = out;
    }
    if (!finished.empty()) {
      std::vector<int32_t> keep;
      for (int32_t r : g.rq)
        if (req[r].decoded != req[r].target) keep.push_back(r);
      g.rq = std::move(keep);
    }
    for (int32_t r : new_run) g.rq.push_back(r);
    g.evict_to_fit();
    if (!done.empty()) tradeoff_update(g, done);

    for (int32_t r : finished) {  // records + router.on_completion
      const Req& q = req[r];
      records.push_back({r, g.cfg.engine_id, q.first_us, now_us});
      if (cfg.route_policy == nx::kLatencyBased) {
        lat_win[e].emplace_back(now, now - q.arr_ms);
        lat_sum[e] += now - q.arr_ms;
      }
      l_bar_ema += 0.05 * ((double)q.target - l_bar_ema);
      if (l_bar_ema < 1.0) l_bar_ema = 1.0;
      sess_engine[q.session] = e;
    }
    g.learn_ev = true;
    g.learn_t = now_us;
    g.learn_seq = next_seq++;
    g.learn_b = plan.b;
    g.learn_s = plan.s;
    g.learn_y = g.actual;
    try_begin_step(e, now_us);
  }

  StateVec export_state(int e, int64_t now_us) const {  // engine.cpp:307-332
    const Engine& g = eng[e];
    StateVec sv;
    const double now = to_ms(now_us);
    sv.at = now;
    sv.p_max = g.learner.cur.p_max;
    if (g.busy) {
      const double elapsed = now - to_ms(g.started_us);
      sv.l_hat = std::max(0.0, g.plan.predicted - elapsed);
    }
    double pending_prefill = 0.0, demand = 0.0;
    for (int64_t i = 0; i < g.wq_len; ++i) {
      const double rem = (double)req[g.wq[g.wq_head + i]].remaining();
      pending_prefill += rem;
      demand += rem + g.l_bar;
    }
    sv.w_load = pending_prefill + 32.0 * (double)(g.wq_len + (int64_t)g.rq.size());
    const double free_tokens = (double)(g.free_blocks() * g.cfg.block_size);
    sv.m_free = std::max(0.0, free_tokens - demand);
    sv.queue_len = g.wq_len + (int64_t)g.rq.size();
    return sv;
  }

  Result run() {
    const int64_t n = (int64_t)req.size();
    for (int e = 0; e < E; ++e) {  // initial reports precede arrivals (sim.cpp:272-287)
      eng[e].report_ev = true;
      eng[e].report_t = 0;
      eng[e].report_seq = next_seq++;
    }
    next_seq += (uint64_t)n;  // arrival i carries sequence E + i
    pending = n;
    const int64_t dur_us = to_us(cfg.duration_ms);
    while (true) {
      // pick min (time, seq) over the arrival cursor and the engine slots
      int kind = -1, who = -1;
      int64_t bt = 0;
      uint64_t bs = 0;
      auto consider = [&](int64_t t, uint64_t s, int k, int e) {
        if (kind < 0 || t < bt || (t == bt && s < bs)) {
          bt = t; bs = s; kind = k; who = e;
        }
      };
      if (cursor < n) consider(w.arrival_us[cursor], (uint64_t)(E + cursor), 0, -1);
      for (int e = 0; e < E; ++e) {
        const Engine& g = eng[e];
        if (g.step_ev) consider(g.step_t, g.step_seq, 1, e);
        if (g.report_ev) consider(g.report_t, g.report_seq, 2, e);
        if (g.learn_ev) consider(g.learn_t, g.learn_seq, 3, e);
        if (!g.deliveries.empty()) consider(g.deliveries.front().t, g.deliveries.front().seq, 4, e);
      }
      if (kind < 0) break;
      if (bt > dur_us) break;
      // consume the slot
      int64_t rid = 0;
      if (kind == 0) { rid = cursor; ++cursor; }
      else if (kind == 1) eng[who].step_ev = false;
      else if (kind == 2) eng[who].report_ev = false;
      else if (kind == 3) eng[who].learn_ev = false;
      Delivery dv{};
      if (kind == 4) { dv = eng[who].deliveries.front(); eng[who].deliveries.pop_front(); }
      if (kind == 2 && pending == 0 && active() == 0) continue;  // sim.cpp:297-300
      ++events;
      ev_hash = nx::fnv1a_u64(ev_hash, (uint64_t)bt);
      ev_hash = nx::fnv1a_u64(ev_hash, (uint64_t)kind);
      ev_hash = nx::fnv1a_u64(ev_hash, (uint64_t)(kind == 0 ? 0 : eng[who].cfg.engine_id + 1));
      ev_hash = nx::fnv1a_u64(ev_hash, (uint64_t)rid);
      switch (kind) {
        case 0: {  // sim.cpp:168-194
          ++arrived;
          --pending;
          const int e = route((int32_t)rid, to_ms(bt));
          if (!admit(e, (int32_t)rid)) {
            ++rejected;
            break;
          }
          try_begin_step(e, bt);
          break;
        }
        case 1: step_complete(who, bt); break;
        case 2: {  // sim.cpp:226-243
          Engine& g = eng[who];
          Delivery d;
          d.t = bt + to_us(g.cfg.staleness_ms);
          d.seq = next_seq++;
          d.sv = export_state(who, bt);
          g.deliveries.push_back(d);
          g.report_ev = true;
          g.report_t = bt + to_us(g.cfg.report_period_ms);
          g.report_seq = next_seq++;
          break;
        }
        case 3: {
          Engine& g = eng[who];
          g.learner.record(g.learn_b, g.learn_s, g.learn_y);
          break;
        }
        case 4:
          has_rep[who] = true;
          rep[who] = dv.sv;
          break;
      }
    }
    Result res;
    res.arrived = arrived;
    res.rejected = rejected;
    res.completed = (int64_t)records.size();
    res.unfinished = arrived - rejected - res.completed + pending;
    res.arrival_hash = w.arrival_hash;
    res.event_hash = ev_hash;
    res.records = records;
    res.events = events;
    for (int e = 0; e < E; ++e) {
      EngineOut o;
      o.engine_id = eng[e].cfg.engine_id;
      o.samples = eng[e].learner.seen;
      o.params = eng[e].learner.cur;
      for (int k = 0; k < 7; ++k) o.counters[k] = eng[e].learner.counters[k];
      res.engines.push_back(o);
    }
    return res;
  }
};

}  // namespace

double throughput(const Params& p, int64_t b, int64_t s) {  // perf_model.cpp:22-42
  if (!(b >= 1 && s >= b)) throw std::invalid_argument("BatchShape requires b >= 1 and s >= b");
  if (!p.valid()) throw std::invalid_argument("PerfParams violate invariants");
  return p.p_max * sat(p.kB, (double)b) * sat(p.kS, (double)s);
}

double predict_latency(const Params& p, int64_t b, int64_t s) {  // perf_model.cpp:44-49
  const double thr = throughput(p, b, s);
  const double work = p.w0 + p.ws * (double)s;
  return p.tau0 + work / thr + p.tauB * (double)b + p.tauS * (double)s;
}

Result simulate(const nx::RunCfg& cfg, const nx::Workload& w) {
  Sim sim(cfg, w);
  return sim.run();
}

}  // namespace port
