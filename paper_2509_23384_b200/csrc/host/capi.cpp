// C-ABI implementation (include/nx_sched.h): packs RunConfig batches into the
// SoA image of nx_layout.h, moves it to HBM, launches the device kernels and
// returns reference-shaped results. No simulation logic lives here — every
// scheduling decision is made on the device (csrc/device/*.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../nx_layout.h"
#include "frontend.hpp"
#include "nx_sched.h"
#include <dlfcn.h>
#include <nccl.h>

#include "json.hpp"
#include "report.hpp"

extern "C" cudaError_t nx_launch_sim(const NxPools* d_pools, const int32_t* d_order, int n_rep,
                                     int* d_next, int prefix_cap, int max_eng, int n_ew, int fsm_cap,
                                     int req_cap, size_t smem, int grid, cudaStream_t st);
extern "C" size_t nx_sim_fit_table_doubles(int fsm_cap);
extern "C" cudaError_t nx_launch_summarize(const NxPools* d_pools, int n_rep, double* work, cudaStream_t st);
extern "C" size_t nx_sim_req_smem_bytes(int req_cap);
extern "C" cudaError_t nx_sim_set_debug(unsigned long long* dev_ptr);

namespace {
// NX_DEBUG=1: the simulation kernel's spin-wait watchdog dumps its replica
// CTA's event-loop state into host-mapped memory before it traps.
unsigned long long* g_dbg_host = nullptr;
void arm_debug_dump() {
  const char* v = std::getenv("NX_DEBUG");
  if (!v || v[0] != '1' || g_dbg_host) return;
  void* p = nullptr;
  if (cudaHostAlloc(&p, 4096, cudaHostAllocMapped) != cudaSuccess) return;
  std::memset(p, 0, 4096);
  void* dp = nullptr;
  cudaHostGetDevicePointer(&dp, p, 0);
  g_dbg_host = static_cast<unsigned long long*>(p);
  nx_sim_set_debug(static_cast<unsigned long long*>(dp));
}
void print_debug_dump() {
  if (!g_dbg_host || g_dbg_host[0] == 0) return;
  const unsigned long long* d = g_dbg_host;
  std::fprintf(stderr, "[nx debug] line %llu warp %llu block %llu horizon %llu next_arr %llu final %llu parked %llu "
               "n_done %llu n_fin %llu kd_ready %llu cursor %llu am %llu n_eng %llu stop %llu kd_inf %llu\n",
               d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10], d[11], d[12], d[13], d[14], d[15]);
  for (unsigned long long e = 0; e < d[13] && e < 8; ++e) {
    const unsigned long long* q = d + 16 + 10 * e;
    std::fprintf(stderr, "[nx debug] eng %llu front %llu wpos %llu mpos %llu step %llu report %llu learn %llu dq %llu "
                 "flags %llx log_n %llu wq %llu rq %llu\n",
                 e, q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7], q[8], q[9] & 0xffffffffull, q[9] >> 32);
  }
}
}  // namespace
extern "C" cudaError_t nx_sim_occupancy(int warps_per_block, size_t smem, int* blocks_per_sm);
extern "C" size_t nx_sim_smem_per_warp(int max_engines, int prefix_cap);
extern "C" cudaError_t nx_launch_perf_eval(const double* params, int n_params, const int32_t* idx,
                                           const int32_t* b, const int32_t* s, double* outT,
                                           double* outThr, int64_t n, int fp32, unsigned* bad,
                                           int sms, cudaStream_t st);

extern "C" cudaError_t nx_launch_lens(const nx_lens_problem* probs, int n, const int32_t* rem,
                                      nx_lens_plan* plans, int32_t* alloc, int32_t* gpre, int sms,
                                      int mode, cudaStream_t st);
extern "C" cudaError_t nx_launch_route(nx_route_group* groups, int n, nx_engine_report* reports,
                                       const nx_route_request* reqs, int32_t* smap,
                                       nx_route_decision* dec, int32_t* gstatus, int sms,
                                       int mode, cudaStream_t st);
extern "C" cudaError_t nx_launch_refit(int kind, const nx_refit_problem* probs, int n,
                                       const int32_t* sb, const int32_t* ss, const double* sy,
                                       nx_refit_result* out, double* scratch, int64_t scratch_per,
                                       int grid, int max_long, cudaStream_t st);
extern "C" int64_t nx_refit_scratch_per(int64_t W);
extern "C" cudaError_t nx_launch_scalar_ops(int op, void* recs, int n, const void* aux_in,
                                            void* aux_out, cudaStream_t st);

namespace {

thread_local std::string g_err;

struct NxError : std::runtime_error {
  int code;
  NxError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw NxError(NX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return NX_OK;
  } catch (const NxError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return NX_EINVAL;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return NX_ELOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NX_ERUNTIME;
  }
}

int sm_count(int device) {
  thread_local int cached_dev = -1, cached_n = 0;  // queried once per device (scalar calls)
  if (device == cached_dev) return cached_n;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  cached_dev = device;
  cached_n = n > 0 ? n : 148;
  return cached_n;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Device arena: one allocation, sub-buffers at 256-B aligned offsets.
struct Arena {
  size_t size = 0;
  template <class T>
  size_t take(size_t count) {
    const size_t off = align_up(size, 256);
    size = off + sizeof(T) * std::max<size_t>(count, 1);
    return off;
  }
};

// Replica CTA: a router warp + one warp per engine (engines beyond
// kEngineWarps share warps round-robin); sim_kernel.cu kPdMaxWarps.
constexpr int kEngineWarps = 8;
// Event-log ring entries per engine (power of two): the merger's and the key
// comparisons' window into an engine's past events.
constexpr int64_t kEvLogCap = NX_EVLOG_CAP;


// Stream-ordered scratch (cudaMallocAsync) for the batched operators: keep
// the device's default pool's memory between calls instead of returning it
// at every synchronisation (a re-grow per launch cost milliseconds).
void retain_default_pool() {
  thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done_dev = dev;
}

int current_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  return sm_count(dev);
}

// Device staging for the host-pointer entry points: one grow-only buffer per
// thread and device, so a scalar call (the C++ drop-in's predict_latency,
// route, ...) costs copies + one launch, not a cudaMalloc.
struct Staging {
  Arena A;
  unsigned char* d = nullptr;
  void alloc() {
    struct Buf {
      unsigned char* p = nullptr;
      size_t cap = 0;
      int dev = -1;
    };
    thread_local Buf buf;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (buf.dev != dev || buf.cap < A.size) {
      if (buf.p && buf.dev == dev) cudaFree(buf.p);
      buf.cap = std::max<size_t>(A.size, size_t(1) << 20);
      cuda_check(cudaMalloc(&buf.p, buf.cap), "cudaMalloc");
      buf.dev = dev;
    }
    d = buf.p;
  }
  template <class T>
  T* at(size_t off) { return reinterpret_cast<T*>(d + off); }
};

const char* status_text(int st) {
  switch (st) {
    case NX_EINVAL: return "invalid argument";
    case NX_ERUNTIME: return "runtime error";
    case NX_ELOGIC: return "logic error";
  }
  return "error";
}


}  // namespace

struct nx_sim {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_up = nullptr;  // the last upload's copies out of the pinned inputs
  bool uploaded = false;
  std::vector<nx::RunCfg> cfgs;
  std::vector<nx::Workload> wl;
  int n_rep = 0, max_eng = 1, prefix_cap = 1;
  int n_ew = 1, slots = 1;                 // engine warps per CTA, CTA slots (resident replicas)
  int per_sm = 1;                          // resident replica CTAs per SM
  int64_t max_req = 1, max_long = 1;
  int64_t n_req = 0, n_sess = 0, n_eng = 0;
  // host pinned input image
  std::vector<NxReplicaDesc> rep;
  std::vector<NxEngineDesc> eng;
  std::vector<int32_t> order;
  std::vector<double> cost;  // expected replica cost (longest first)
  int64_t* h_arr_us = nullptr;
  double* h_arr_ms = nullptr;
  NxReqState* h_req0 = nullptr;  // prompt/target + zeroed state
  int32_t* h_session = nullptr;
  // host pinned outputs
  NxReplicaOut* h_rep_out = nullptr;
  NxEngineOut* h_eng_out = nullptr;
  int32_t* h_records = nullptr;
  int64_t* h_first_us = nullptr;
  int64_t* h_done_us = nullptr;
  int32_t* h_req_engine = nullptr;
  // observability logs (allocated only when a replica asks for them)
  int64_t n_plan_log = 0, n_route_log = 0, n_learn_log = 0;
  NxPlanLog* h_plan_log = nullptr;
  NxRouteLog* h_route_log = nullptr;
  NxLearnLog* h_learn_log = nullptr;
  // device
  unsigned char* d_arena = nullptr;
  size_t arena_bytes = 0;
  NxPools pools{};
  NxPools* d_pools = nullptr;
  int32_t* d_order = nullptr;
  int* d_next = nullptr;
  size_t off_rep = 0, off_eng = 0, off_rep_out = 0, off_eng_out = 0, off_metrics = 0, off_sum_work = 0;
  NxReplicaMetrics* h_metrics = nullptr;
  size_t off_state_begin = 0, off_state_end = 0;  // zero-initialised state span
  size_t off_ff_begin = 0, off_ff_end = 0;        // 0xff-initialised span
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  float last_ms = 0.f;
  bool launched = false;

  ~nx_sim() {
    if (d_arena) cudaFree(d_arena);
    if (d_pools) cudaFree(d_pools);
    for (void* p : {(void*)h_arr_us, (void*)h_arr_ms, (void*)h_req0,
                    (void*)h_session, (void*)h_rep_out, (void*)h_eng_out, (void*)h_records,
                    (void*)h_first_us, (void*)h_done_us, (void*)h_req_engine, (void*)h_plan_log,
                    (void*)h_route_log, (void*)h_learn_log, (void*)h_metrics})
      if (p) cudaFreeHost(p);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_up) cudaEventDestroy(ev_up);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

template <class T>
T* pinned(size_t count) {
  void* p = nullptr;
  cuda_check(cudaMallocHost(&p, sizeof(T) * std::max<size_t>(count, 1)), "cudaMallocHost");
  return static_cast<T*>(p);
}

void fill_descriptors(nx_sim& h) {
  h.rep.resize(h.n_rep);
  h.eng.clear();
  int64_t req_off = 0, sess_off = 0, scratch_off = 0;
  // pool element offsets (per engine regions)
  int64_t wq_off = 0, rq_off = 0, plan_off = 0, cache_off = 0, ring_off = 0, tw_off = 0, dq_off = 0,
          lat_off = 0;
  for (int r = 0; r < h.n_rep; ++r) {
    const nx::RunCfg& c = h.cfgs[r];
    const nx::Workload& w = h.wl[r];
    const int n = static_cast<int>(w.prompt.size());
    const int ns = static_cast<int>(w.session_names.size());
    NxReplicaDesc& d = h.rep[r];
    std::memset(&d, 0, sizeof d);
    d.ttft_slo = c.ttft_slo;
    d.tpot_slo = c.tpot_slo;
    d.eps_ratio = c.eps_ratio;
    d.q_ref = c.q_ref;
    d.alpha = c.alpha;
    d.beta = c.beta;
    d.l_bar = c.l_bar;
    d.td_min = c.td_min;
    for (int i = 0; i < 4; ++i) d.weights[i] = c.weights[i];
    d.beta_aff = c.beta_aff;
    d.knee = c.knee;
    d.scale_ms = c.scale_ms;
    d.load_half = c.load_half;
    d.headroom = c.headroom;
    d.stale_limit = c.staleness_limit;
    d.lat_window = c.latency_window;
    nx::Xoshiro rr(nx::substream_seed(c.seed, "router"));
    for (int i = 0; i < 4; ++i) d.router_rng[i] = rr.s[i];
    d.duration_us = nx::to_us(c.duration_ms);
    d.req_off = req_off;
    d.sess_off = sess_off;
    d.scratch_off = scratch_off;
    d.n_eng = static_cast<int32_t>(c.engines.size());
    d.eng_base = static_cast<int32_t>(h.eng.size());
    d.n_req = n;
    d.n_sess = ns;
    d.n_iters = c.n_search_iters;
    d.route_policy = c.route_policy;
    d.long_w = static_cast<int32_t>(c.long_window);
    d.short_w = static_cast<int32_t>(c.short_window);
    d.s_period = static_cast<int32_t>(c.structural_period);
    d.l_period = static_cast<int32_t>(c.linear_period);
    d.min_s = static_cast<int32_t>(std::min<int64_t>(c.min_structural, INT32_MAX));
    // observability: plans / learner snapshots are one per executed step, and
    // every step advances at least one token of some request
    d.log_flags = (c.out_plans_jsonl.empty() ? 0 : NX_LOG_PLANS) |
                  (c.out_routing_jsonl.empty() ? 0 : NX_LOG_ROUTES) |
                  (c.record_learner_history ? NX_LOG_LEARNER : 0);
    int64_t token_bound = 16;
    for (int i = 0; i < n; ++i) token_bound += static_cast<int64_t>(w.prompt[i]) + w.output[i];
    d.plan_log_off = h.n_plan_log;
    d.plan_log_cap = (d.log_flags & NX_LOG_PLANS) ? token_bound : 0;
    h.n_plan_log += d.plan_log_cap;
    d.route_log_off = h.n_route_log;
    h.n_route_log += (d.log_flags & NX_LOG_ROUTES) ? n : 0;
    d.learn_log_off = h.n_learn_log;
    d.learn_log_cap = (d.log_flags & NX_LOG_LEARNER) ? token_bound : 0;
    h.n_learn_log += d.learn_log_cap;
    req_off += n;
    sess_off += ns;
    h.max_req = std::max<int64_t>(h.max_req, n);
    h.max_long = std::max<int64_t>(h.max_long, c.long_window);
    for (const auto& ec : c.engines) {
      NxEngineDesc e;
      std::memset(&e, 0, sizeof e);
      const nx::Params& tp = ec.true_params;
      const double tpv[8] = {tp.tau0, tp.w0, tp.ws, tp.tauB, tp.tauS, tp.p_max, tp.kB, tp.kS};
      for (int i = 0; i < 8; ++i) e.tp[i] = tpv[i];
      e.noise_sigma = ec.noise_sigma;
      auto it = c.static_weights.find(ec.engine_id);
      e.static_w = it != c.static_weights.end() ? it->second : 1.0;
      e.period_us = nx::to_us(ec.report_period_ms);
      e.stale_us = nx::to_us(ec.staleness_ms);
      nx::Xoshiro er(nx::substream_seed(c.seed, "engine-noise", static_cast<uint64_t>(ec.engine_id)));
      for (int i = 0; i < 4; ++i) e.rng[i] = er.s[i];
      e.engine_id = ec.engine_id;
      e.policy = ec.policy;
      e.kv_blocks = static_cast<int32_t>(ec.kv_blocks);
      e.block_size = static_cast<int32_t>(ec.block_size);
      e.m_max = static_cast<int32_t>(ec.m_max);
      e.q_max = static_cast<int32_t>(ec.q_max);
      e.static_budget = static_cast<int32_t>(ec.static_budget);
      e.wait_cap = static_cast<int32_t>(ec.wait_cap);
      // deliveries in flight per engine: ceil(staleness / period) + 1 (+ slack)
      const int64_t per = std::max<int64_t>(1, e.period_us);
      e.dq_cap = static_cast<int32_t>(std::min<int64_t>(e.stale_us / per + 3, 1 << 20));
      e.lat_cap = c.route_policy == nx::kLatencyBased ? std::max(n, 1) : 0;
      e.wq_off = wq_off;
      e.rq_off = rq_off;
      e.plan_off = plan_off;
      e.cache_off = cache_off;
      e.ring_off = ring_off;
      e.tw_off = tw_off;
      e.dq_off = dq_off;
      e.lat_off = lat_off;
      wq_off += n;
      rq_off += n;
      plan_off += std::max(n, 1);
      cache_off += ns;
      ring_off += c.long_window;
      tw_off += NX_TW_CAP;
      dq_off += e.dq_cap;
      lat_off += e.lat_cap;
      h.eng.push_back(e);
    }
    h.max_eng = std::max(h.max_eng, d.n_eng);
    for (const auto& ec : c.engines)
      h.prefix_cap = std::max<int>(h.prefix_cap, static_cast<int>(ec.q_max) + 1);
  }
  h.n_req = req_off;
  h.n_sess = sess_off;
  h.n_eng = static_cast<int64_t>(h.eng.size());
  // per CTA slot (one resident replica per SM): event-log rings, outboxes and
  // learner scratch for every engine warp
  int ew = kEngineWarps;
  if (const char* v = std::getenv("NX_ENGINE_WARPS")) ew = std::max(1, std::min(kEngineWarps, std::atoi(v)));
  h.n_ew = std::min(ew, h.max_eng);
  // resident CTAs per SM: the register file bounds it (occupancy query with
  // the base shared memory; the fit tables then share what is left)
  {
    const size_t base = nx_sim_smem_per_warp(h.max_eng, h.prefix_cap);
    int occ = 0;
    cuda_check(nx_sim_occupancy(1 + h.n_ew, base, &occ), "occupancy");
    if (occ < 1) throw NxError(NX_ECUDA, "simulation kernel does not fit on an SM");
    h.per_sm = occ;
    if (const char* v = std::getenv("NX_SIM_CTAS_PER_SM")) h.per_sm = std::max(1, std::min(occ, std::atoi(v)));
  }
  h.slots = std::max(1, std::min(h.n_rep, h.per_sm * sm_count(h.device)));
  const int64_t scr_stride = nx_refit_scratch_per(h.max_long);
  scratch_off = static_cast<int64_t>(h.slots) * h.n_ew * scr_stride;
  const int64_t n_evlog = static_cast<int64_t>(h.slots) * h.max_eng * kEvLogCap;
  const int64_t n_outbox = static_cast<int64_t>(h.slots) * h.max_eng * h.max_req * 4;

  // device arena layout
  Arena A;
  const size_t o_arr_us = A.take<int64_t>(h.n_req);
  const size_t o_arr_ms = A.take<double>(h.n_req);
  const size_t o_req0 = A.take<NxReqState>(h.n_req);
  const size_t o_session = A.take<int32_t>(h.n_req);
  h.off_rep = A.take<NxReplicaDesc>(h.n_rep);
  h.off_eng = A.take<NxEngineDesc>(h.n_eng);
  const size_t o_order = A.take<int32_t>(h.n_rep);
  // zero-initialised state
  h.off_state_begin = align_up(A.size, 256);

  const size_t o_kv = A.take<uint8_t>(h.n_req);
  const size_t o_began = A.take<uint8_t>(h.n_req);
  const size_t o_next = A.take<int>(3 + 2 * 1024);  // kernel scheduling control (nx_state.cuh kSchedCtlInts)
  h.off_state_end = A.size;
  // 0xff-initialised (-1) state
  h.off_ff_begin = align_up(A.size, 256);
  const size_t o_sess_eng = A.take<int32_t>(h.n_sess);
  const size_t o_ctok = A.take<int32_t>(cache_off);
  h.off_ff_end = A.size;
  // uninitialised state (req is copied from req0 at every launch)
  const size_t o_req = A.take<NxReqState>(h.n_req);
  const size_t o_first = A.take<int64_t>(h.n_req);
  const size_t o_done = A.take<int64_t>(h.n_req);
  const size_t o_reqeng = A.take<int32_t>(h.n_req);
  const size_t o_wq = A.take<int32_t>(wq_off);
  const size_t o_rq = A.take<int32_t>(rq_off);
  const size_t o_preq = A.take<int32_t>(plan_off);
  const size_t o_ptok = A.take<int32_t>(plan_off);
  const size_t o_cprev = A.take<int32_t>(cache_off);
  const size_t o_cnext = A.take<int32_t>(cache_off);
  const size_t o_rb = A.take<int32_t>(ring_off);
  const size_t o_rs = A.take<int32_t>(ring_off);
  const size_t o_ry = A.take<double>(ring_off);
  const size_t o_twt = A.take<double>(tw_off);
  const size_t o_twp = A.take<double>(tw_off);
  const size_t o_dqt = A.take<int64_t>(dq_off);
  const size_t o_dqs = A.take<uint32_t>(dq_off);
  const size_t o_dqv = A.take<double>(5 * dq_off);
  const size_t o_dqq = A.take<int64_t>(dq_off);
  const size_t o_latt = A.take<double>(lat_off);
  const size_t o_late = A.take<double>(lat_off);
  const size_t o_rec = A.take<int32_t>(h.n_req);
  const size_t o_scr = A.take<double>(scratch_off);
  const size_t o_evlog = A.take<NxEvLog>(n_evlog);
  const size_t o_outbox = A.take<int32_t>(n_outbox);
  const size_t o_pstage = A.take<NxPlanLog>(h.n_plan_log * h.max_eng);
  const size_t o_lstage = A.take<NxLearnLog>(h.n_learn_log * h.max_eng);
  const size_t o_plog = A.take<NxPlanLog>(h.n_plan_log);
  const size_t o_rlog = A.take<NxRouteLog>(h.n_route_log);
  const size_t o_llog = A.take<NxLearnLog>(h.n_learn_log);
  h.off_rep_out = A.take<NxReplicaOut>(h.n_rep);
  h.off_metrics = A.take<NxReplicaMetrics>(h.n_rep);
  h.off_sum_work = A.take<double>(4 * h.n_req);  // summary.cu: e2e, ttft, tpot, compacted tpot
  h.off_eng_out = A.take<NxEngineOut>(h.n_eng);
  h.arena_bytes = A.size;

  cuda_check(cudaMalloc(&h.d_arena, h.arena_bytes), "cudaMalloc(arena)");
  unsigned char* B = h.d_arena;
  NxPools& P = h.pools;
  P.arr_us = reinterpret_cast<const int64_t*>(B + o_arr_us);
  P.arr_ms = reinterpret_cast<const double*>(B + o_arr_ms);
  P.req0 = reinterpret_cast<const NxReqState*>(B + o_req0);
  P.session = reinterpret_cast<const int32_t*>(B + o_session);
  P.req = reinterpret_cast<NxReqState*>(B + o_req);
  P.first_us = reinterpret_cast<int64_t*>(B + o_first);
  P.done_us = reinterpret_cast<int64_t*>(B + o_done);
  P.req_engine = reinterpret_cast<int32_t*>(B + o_reqeng);
  P.kv_admitted = reinterpret_cast<uint8_t*>(B + o_kv);
  P.wq = reinterpret_cast<int32_t*>(B + o_wq);
  P.rq = reinterpret_cast<int32_t*>(B + o_rq);
  P.plan_req = reinterpret_cast<int32_t*>(B + o_preq);
  P.plan_tok = reinterpret_cast<int32_t*>(B + o_ptok);
  P.c_tokens = reinterpret_cast<int32_t*>(B + o_ctok);
  P.c_prev = reinterpret_cast<int32_t*>(B + o_cprev);
  P.c_next = reinterpret_cast<int32_t*>(B + o_cnext);
  P.ring_b = reinterpret_cast<int32_t*>(B + o_rb);
  P.ring_s = reinterpret_cast<int32_t*>(B + o_rs);
  P.ring_y = reinterpret_cast<double*>(B + o_ry);
  P.tw_ttft = reinterpret_cast<double*>(B + o_twt);
  P.tw_tpot = reinterpret_cast<double*>(B + o_twp);
  P.dq_t = reinterpret_cast<int64_t*>(B + o_dqt);
  P.dq_seq = reinterpret_cast<uint32_t*>(B + o_dqs);
  P.dq_sv = reinterpret_cast<double*>(B + o_dqv);
  P.dq_qlen = reinterpret_cast<int64_t*>(B + o_dqq);
  P.lat_t = reinterpret_cast<double*>(B + o_latt);
  P.lat_e2e = reinterpret_cast<double*>(B + o_late);
  P.sess_engine = reinterpret_cast<int32_t*>(B + o_sess_eng);
  P.records = reinterpret_cast<int32_t*>(B + o_rec);
  P.scratch = reinterpret_cast<double*>(B + o_scr);
  P.evlog = reinterpret_cast<NxEvLog*>(B + o_evlog);
  P.outbox = reinterpret_cast<int32_t*>(B + o_outbox);
  P.plan_stage = reinterpret_cast<NxPlanLog*>(B + o_pstage);
  P.learn_stage = reinterpret_cast<NxLearnLog*>(B + o_lstage);
  P.began = reinterpret_cast<uint8_t*>(B + o_began);
  P.evlog_cap = kEvLogCap;
  P.outbox_cap = h.max_req;
  P.scratch_stride = scr_stride;
  P.slot_engines = h.max_eng;
  P.slot_warps = h.n_ew;
  P.plan_log = reinterpret_cast<NxPlanLog*>(B + o_plog);
  P.route_log = reinterpret_cast<NxRouteLog*>(B + o_rlog);
  P.learn_log = reinterpret_cast<NxLearnLog*>(B + o_llog);
  P.rep = reinterpret_cast<const NxReplicaDesc*>(B + h.off_rep);
  P.eng = reinterpret_cast<const NxEngineDesc*>(B + h.off_eng);
  P.rep_out = reinterpret_cast<NxReplicaOut*>(B + h.off_rep_out);
  P.eng_out = reinterpret_cast<NxEngineOut*>(B + h.off_eng_out);
  P.metrics = reinterpret_cast<NxReplicaMetrics*>(B + h.off_metrics);
  h.d_order = reinterpret_cast<int32_t*>(B + o_order);
  h.d_next = reinterpret_cast<int*>(B + o_next);
  cuda_check(cudaMalloc(&h.d_pools, sizeof(NxPools)), "cudaMalloc(pools)");
  cuda_check(cudaMemcpy(h.d_pools, &h.pools, sizeof(NxPools), cudaMemcpyHostToDevice),
             "cudaMemcpy(pools)");

  // pinned host image of the inputs
  h.h_arr_us = pinned<int64_t>(h.n_req);
  h.h_arr_ms = pinned<double>(h.n_req);
  h.h_req0 = pinned<NxReqState>(h.n_req);
  h.h_session = pinned<int32_t>(h.n_req);
  for (int r = 0; r < h.n_rep; ++r) {
    const nx::Workload& w = h.wl[r];
    const int64_t o = h.rep[r].req_off;
    const size_t n = w.prompt.size();
    std::memcpy(h.h_arr_us + o, w.arrival_us.data(), n * sizeof(int64_t));
    std::memcpy(h.h_arr_ms + o, w.arrival_ms.data(), n * sizeof(double));
    for (size_t i = 0; i < n; ++i) h.h_req0[o + i] = {0, 0, w.prompt[i], w.output[i]};
    std::memcpy(h.h_session + o, w.session.data(), n * sizeof(int32_t));
  }
  // longest-expected replicas first: more requests and lower rates run longer
  h.order.resize(h.n_rep);
  std::iota(h.order.begin(), h.order.end(), 0);
  std::vector<double>& cost = h.cost;
  cost.assign(h.n_rep, 0.0);
  for (int r = 0; r < h.n_rep; ++r) {
    const auto& w = h.wl[r];
    const double span = w.arrival_ms.empty() ? 0.0 : w.arrival_ms.back();
    cost[r] = static_cast<double>(w.prompt.size()) + span * 0.05;
  }
  std::stable_sort(h.order.begin(), h.order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  h.h_rep_out = pinned<NxReplicaOut>(h.n_rep);
  h.h_metrics = pinned<NxReplicaMetrics>(h.n_rep);
  h.h_eng_out = pinned<NxEngineOut>(h.n_eng);
  h.h_records = pinned<int32_t>(h.n_req);
  h.h_first_us = pinned<int64_t>(h.n_req);
  h.h_done_us = pinned<int64_t>(h.n_req);
  h.h_req_engine = pinned<int32_t>(h.n_req);
  if (h.n_plan_log) h.h_plan_log = pinned<NxPlanLog>(h.n_plan_log);
  if (h.n_route_log) h.h_route_log = pinned<NxRouteLog>(h.n_route_log);
  if (h.n_learn_log) h.h_learn_log = pinned<NxLearnLog>(h.n_learn_log);
}

const char* site_name(int site) {
  switch (site) {
    case NX_SITE_BISECT: return "binary_search_budget: invalid inputs";
    case NX_SITE_ALLOCATE: return "allocate_tokens: budget below queue needs";
    case NX_SITE_PREFILL_CAP: return "prefill_priority: prompt exceeds m_max";
    case NX_SITE_SAMPLE: return "invalid LatencySample";
    case NX_SITE_CAPACITY: return "score_capacity: demand must be >= 1 token";
    case NX_SITE_OVERFLOW: return "device capacity exceeded";
    case NX_SITE_PARAMS: return "PerfParams violate invariants";
  }
  return "error";
}

// The reference's exception text for a failed replica (the throw sites are
// cited in nx_layout.h NX_SITE_*); err_info carries the engine id where the
// reference message names one (engine.cpp:75-78).
std::string replica_message(const NxReplicaOut& o) {
  if (o.err_site == NX_SITE_PREFILL_CAP)
    return "prefill_priority: prompt exceeds m_max; raise m_max for engine " + std::to_string(o.err_info);
  if (o.err_site == NX_SITE_OVERFLOW)
    return std::string(site_name(o.err_site)) + " (code " + std::to_string(o.err_info) + ")";
  return site_name(o.err_site);
}

// Device-path limits the reference does not have: the engine and learner
// knobs travel as int32 in NxEngineDesc / NxReplicaDesc (nx_layout.h), and a
// replica CTA stages q_max + 1 prefix sums per warp in shared memory. Values
// the reference would accept but the device cannot represent are rejected
// here with std::invalid_argument instead of being narrowed silently.
void check_device_limits(const nx::RunCfg& c, size_t smem_optin) {
  auto i32 = [](int64_t v, const std::string& what) {
    if (v < INT32_MIN || v > INT32_MAX)
      throw std::invalid_argument(what + " = " + std::to_string(v) +
                                  ": the device path supports 32-bit values");
  };
  i32(c.long_window, "learner.long_window");
  i32(c.short_window, "learner.short_window");
  i32(c.structural_period, "learner.structural_period");
  i32(c.linear_period, "learner.linear_period");
  for (const auto& e : c.engines) {
    const std::string id = "engine " + std::to_string(e.engine_id) + ": ";
    i32(e.kv_blocks, id + "kv_blocks");
    i32(e.block_size, id + "block_size");
    i32(e.m_max, id + "m_max");
    i32(e.q_max, id + "q_max");
    i32(e.static_budget, id + "static_budget");
    i32(e.wait_cap, id + "wait_cap");
    // KV reservations and token counts are int32 sums of blocks
    if (e.kv_blocks > 0 && e.block_size > 0 && e.kv_blocks > INT32_MAX / 2)
      throw std::invalid_argument(id + "kv_blocks = " + std::to_string(e.kv_blocks) +
                                  ": the device path supports kv_blocks <= 2^30");
    if (smem_optin > 0) {
      const size_t need = nx_sim_smem_per_warp(static_cast<int>(c.engines.size()),
                                               static_cast<int>(e.q_max) + 1);
      if (need > smem_optin) {
        int64_t lim = e.q_max;
        while (lim > 1 && nx_sim_smem_per_warp(static_cast<int>(c.engines.size()),
                                               static_cast<int>(lim) + 1) > smem_optin)
          lim = lim * 7 / 8;
        throw std::invalid_argument(id + "q_max = " + std::to_string(e.q_max) +
                                    ": the device path supports q_max <= " + std::to_string(lim) +
                                    " with " + std::to_string(c.engines.size()) + " engines");
      }
    }
  }
}

}  // namespace

extern "C" {

const char* nx_last_error(void) { return g_err.c_str(); }

int nx_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int nx_sim_create_json(const char* const* configs, int32_t n_replicas, int32_t device,
                       int32_t host_threads, nx_sim_t* out) {
  *out = nullptr;
  return guard([&] {
    if (n_replicas < 1) throw std::invalid_argument("nx_sim_create_json: no replicas");
    auto h = std::make_unique<nx_sim>();
    h->device = device;
    h->n_rep = n_replicas;
    h->cfgs.resize(n_replicas);
    h->wl.resize(n_replicas);
    // shared-memory limit of the replica CTA (0 when no device is visible:
    // the check then happens at launch)
    size_t smem_optin = 0;
    {
      int v = 0;
      if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) == cudaSuccess && v > 0)
        smem_optin = static_cast<size_t>(v);
      else
        cudaGetLastError();
    }
    // parse + synthesise on host threads (reference semantics, host libm)
    std::atomic<int> next{0};
    std::vector<std::string> errs(n_replicas);
    std::vector<int> codes(n_replicas, 0);
    auto work = [&] {
      for (int i = next++; i < n_replicas; i = next++) {
        codes[i] = guard([&] {
          h->cfgs[i] = nx::parse_run_config(configs[i]);
          // one lane per engine in the router warp's merger, lane 31 for arrivals
          if (h->cfgs[i].engines.size() > NX_MAX_ENGINES - 1)
            throw std::invalid_argument("device path supports at most 31 engines per replica");
          check_device_limits(h->cfgs[i], smem_optin);
          h->wl[i] = nx::build_workload(h->cfgs[i]);
          if (h->wl[i].prompt.size() > (1u << 30))
            throw std::invalid_argument("too many requests for one replica");
        });
        if (codes[i]) errs[i] = g_err;
      }
    };
    const int nt = std::max(1, std::min<int>(host_threads > 0 ? host_threads : 1, n_replicas));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (int i = 0; i < n_replicas; ++i)
      if (codes[i]) throw NxError(codes[i], "replica " + std::to_string(i) + ": " + errs[i]);
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreate(&h->ev0), "cudaEventCreate");
    cuda_check(cudaEventCreate(&h->ev1), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&h->ev_up, cudaEventDisableTiming), "cudaEventCreate");
    fill_descriptors(*h);
    *out = h.release();
  });
}

int nx_sim_rebuild_workloads(nx_sim_t h, int32_t host_threads) {
  return guard([&] {
    // build_workload (sim.cpp:101-141) again for every replica on host
    // threads, then the pinned input image; configs stay parsed (the
    // reference's own clock also starts after RunConfig parsing). Safe to
    // call while the previous launch runs: the pinned image is rewritten
    // only after the previous upload's copies out of it have completed.
    std::atomic<int> next{0};
    std::vector<std::string> errs(h->n_rep);
    std::vector<int> codes(h->n_rep, 0);
    auto work = [&] {
      for (int i = next++; i < h->n_rep; i = next++) {
        codes[i] = guard([&] {
          nx::Workload w = nx::build_workload(h->cfgs[i]);
          if (w.prompt.size() != h->wl[i].prompt.size() || w.session_names.size() != h->wl[i].session_names.size())
            throw std::logic_error("nx_sim_rebuild_workloads: workload shape changed");
          h->wl[i] = std::move(w);
        });
        if (codes[i]) errs[i] = g_err;
      }
    };
    const int nt = std::max(1, std::min<int>(host_threads > 0 ? host_threads : 1, h->n_rep));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (int i = 0; i < h->n_rep; ++i)
      if (codes[i]) throw NxError(codes[i], "replica " + std::to_string(i) + ": " + errs[i]);
    if (h->uploaded) cuda_check(cudaEventSynchronize(h->ev_up), "upload event");
    for (int r = 0; r < h->n_rep; ++r) {
      const nx::Workload& w = h->wl[r];
      const int64_t o = h->rep[r].req_off;
      const size_t n = w.prompt.size();
      std::memcpy(h->h_arr_us + o, w.arrival_us.data(), n * sizeof(int64_t));
      std::memcpy(h->h_arr_ms + o, w.arrival_ms.data(), n * sizeof(double));
      for (size_t i = 0; i < n; ++i) h->h_req0[o + i] = {0, 0, w.prompt[i], w.output[i]};
      std::memcpy(h->h_session + o, w.session.data(), n * sizeof(int32_t));
    }
  });
}

int nx_sim_upload(nx_sim_t h) {
  return guard([&] {
    cuda_check(cudaSetDevice(h->device), "cudaSetDevice");
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream), "H2D");
      h->h2d_bytes += static_cast<int64_t>(bytes);
    };
    h->h2d_bytes = 0;
    NxPools& P = h->pools;
    cp(const_cast<int64_t*>(P.arr_us), h->h_arr_us, h->n_req * sizeof(int64_t));
    cp(const_cast<double*>(P.arr_ms), h->h_arr_ms, h->n_req * sizeof(double));
    cp(const_cast<NxReqState*>(P.req0), h->h_req0, h->n_req * sizeof(NxReqState));
    cp(const_cast<int32_t*>(P.session), h->h_session, h->n_req * sizeof(int32_t));
    cp(h->d_arena + h->off_rep, h->rep.data(), h->rep.size() * sizeof(NxReplicaDesc));
    cp(h->d_arena + h->off_eng, h->eng.data(), h->eng.size() * sizeof(NxEngineDesc));
    cp(h->d_order, h->order.data(), h->order.size() * sizeof(int32_t));
    cuda_check(cudaEventRecord(h->ev_up, h->stream), "event");
    h->uploaded = true;
  });
}

int nx_sim_launch(nx_sim_t h) {
  return guard([&] {
    cuda_check(cudaSetDevice(h->device), "cudaSetDevice");
    cudaStream_t st = h->stream;
    // the launch's device time covers the per-launch state reset too
    cuda_check(cudaEventRecord(h->ev0, st), "event");
    cuda_check(cudaMemsetAsync(h->d_arena + h->off_state_begin, 0,
                               h->off_state_end - h->off_state_begin, st), "memset state");
    cuda_check(cudaMemsetAsync(h->d_arena + h->off_ff_begin, 0xff,
                               h->off_ff_end - h->off_ff_begin, st), "memset state");
    cuda_check(cudaMemcpyAsync(h->pools.req, h->pools.req0, h->n_req * sizeof(NxReqState),
                               cudaMemcpyDeviceToDevice, st), "request state image");
    // one replica CTA per SM (router warp + engine warps use the register
    // file); the engine warps' fit tables take the shared memory left over
    size_t base = nx_sim_smem_per_warp(h->max_eng, h->prefix_cap);
    int optin = 0, per_sm_smem = 0;
    cuda_check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device), "attr");
    cuda_check(cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device), "attr");
    int fsm_cap = -1;
    // per CTA: its share of the SM's shared memory (1 KB reserved per CTA),
    // minus the kernel's static shared memory
    size_t room = std::min<size_t>(static_cast<size_t>(optin), static_cast<size_t>(per_sm_smem) / h->per_sm - 1024);
    room = room > 1024 ? room - 1024 : 0;
    // request state in shared memory when the largest replica's fits in a
    // quarter of the room (17 B per request); else it stays in HBM
    int req_cap = 0;
    if (const size_t need = nx_sim_req_smem_bytes(static_cast<int>(h->max_req)); base + need <= room / 4 + base &&
        need <= room / 4)
      req_cap = static_cast<int>(h->max_req);
    if (const char* v = std::getenv("NX_REQ_SMEM")) if (v[0] == '0') req_cap = 0;
    base += nx_sim_req_smem_bytes(req_cap);
    // The fit tables stay in each warp's global scratch by default: every KB
    // of shared memory comes out of the SM's L1, and the event loop's global
    // accesses (queues, logs, request SoA) need it more than the refit's
    // table reads need shared memory (bench shard: 30.4-30.8 vs 29.4-29.6 M
    // decisions/s, 5 interleaved A/B pairs; profiles/r02_l1_ab.txt).
    // NX_FIT_SMEM=auto: tables in the shared memory left over; =N: N entries.
    if (const char* fc = std::getenv("NX_FIT_SMEM")) {
      if (std::string(fc) == "auto") {
        if (room > base) {
          const int64_t per = static_cast<int64_t>((room - base) / h->n_ew / sizeof(double)) -
                              static_cast<int64_t>(nx_sim_fit_table_doubles(0));
          if (per >= 256) fsm_cap = static_cast<int>(std::min<int64_t>(per, 4096));
        }
      } else {
        fsm_cap = std::atoi(fc) < 0 ? -1 : std::min(std::atoi(fc), 4096);
      }
    }
    const size_t smem = base + (fsm_cap >= 0 ? static_cast<size_t>(h->n_ew) * nx_sim_fit_table_doubles(fsm_cap) *
                                                   sizeof(double)
                                             : 0);
    int per_sm = 0;
    cuda_check(nx_sim_occupancy(1 + h->n_ew, smem, &per_sm), "occupancy");
    if (per_sm < 1) throw NxError(NX_ECUDA, "simulation kernel does not fit on an SM");
    // (the slots were planned without the request state's shared memory: a
    // launch that fits fewer CTAs per SM uses fewer of them)
    const int grid = std::max(1, std::min({h->n_rep, h->slots, std::min(per_sm, h->per_sm) * sm_count(h->device)}));
    arm_debug_dump();
    cuda_check(nx_launch_sim(h->d_pools, h->d_order, h->n_rep, h->d_next, h->prefix_cap, h->max_eng, h->n_ew,
                             fsm_cap, req_cap, smem, grid, st), "nx_sim_kernel launch");
    // K7: the metrics summaries on the device, same stream (summary.cu)
    cuda_check(nx_launch_summarize(h->d_pools, h->n_rep, reinterpret_cast<double*>(h->d_arena + h->off_sum_work), st),
               "nx_summarize_kernel launch");
    cuda_check(cudaEventRecord(h->ev1, st), "event");
    h->launched = true;
  });
}

int nx_sim_download(nx_sim_t h) {
  return guard([&] {
    cuda_check(cudaSetDevice(h->device), "cudaSetDevice");
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream), "D2H");
      h->d2h_bytes += static_cast<int64_t>(bytes);
    };
    h->d2h_bytes = 0;
    const NxPools& P = h->pools;
    cp(h->h_rep_out, P.rep_out, h->n_rep * sizeof(NxReplicaOut));
    cp(h->h_metrics, P.metrics, h->n_rep * sizeof(NxReplicaMetrics));
    cp(h->h_eng_out, P.eng_out, h->n_eng * sizeof(NxEngineOut));
    cp(h->h_records, P.records, h->n_req * sizeof(int32_t));
    cp(h->h_first_us, P.first_us, h->n_req * sizeof(int64_t));
    cp(h->h_done_us, P.done_us, h->n_req * sizeof(int64_t));
    cp(h->h_req_engine, P.req_engine, h->n_req * sizeof(int32_t));
    if (h->n_plan_log) cp(h->h_plan_log, P.plan_log, h->n_plan_log * sizeof(NxPlanLog));
    if (h->n_route_log) cp(h->h_route_log, P.route_log, h->n_route_log * sizeof(NxRouteLog));
    if (h->n_learn_log) cp(h->h_learn_log, P.learn_log, h->n_learn_log * sizeof(NxLearnLog));
  });
}

int nx_sim_synchronize(nx_sim_t h) {
  return guard([&] {
    const cudaError_t se = cudaStreamSynchronize(h->stream);
    if (se != cudaSuccess) print_debug_dump();
    cuda_check(se, "nx_sim stream");
    if (h->launched) {
      cuda_check(cudaEventElapsedTime(&h->last_ms, h->ev0, h->ev1), "event time");
      h->launched = false;
    }
  });
}

int nx_sim_run(nx_sim_t h) {
  int rc = nx_sim_upload(h);
  if (!rc) rc = nx_sim_launch(h);
  if (!rc) rc = nx_sim_download(h);
  if (!rc) rc = nx_sim_synchronize(h);
  return rc;
}

int nx_sim_last_kernel_ms(nx_sim_t h, float* ms) {
  *ms = h->last_ms;
  return NX_OK;
}

int nx_sim_io_bytes(nx_sim_t h, int64_t* h2d, int64_t* d2h) {
  *h2d = h->h2d_bytes;
  *d2h = h->d2h_bytes;
  return NX_OK;
}

int nx_sim_replica_count(nx_sim_t h) { return h->n_rep; }

int nx_sim_summaries(nx_sim_t h, nx_replica_summary* out) {
  return guard([&] {
    for (int r = 0; r < h->n_rep; ++r) {
      const NxReplicaOut& o = h->h_rep_out[r];
      const NxReplicaDesc& d = h->rep[r];
      nx_replica_summary& s = out[r];
      s.arrived = o.arrived;
      s.completed = o.completed;
      s.rejected = o.rejected;
      s.unfinished = o.arrived - o.rejected - o.completed + o.pending;
      s.events = o.events;
      int64_t batches = 0;
      for (int e = 0; e < d.n_eng; ++e) batches += h->h_eng_out[d.eng_base + e].samples;
      s.decisions = o.arrived + batches;
      s.arrival_hash = h->wl[r].arrival_hash;
      s.event_hash = o.event_hash;
      s.status = o.status;
      s.err_site = o.err_site;
    }
  });
}

int nx_sim_error(nx_sim_t h, int32_t replica, char* buf, int64_t cap) {
  if (!h || replica < 0 || replica >= h->n_rep) {
    g_err = "nx_sim_error: replica out of range";
    return NX_EINVAL;
  }
  const NxReplicaOut& o = h->h_rep_out[replica];
  const std::string msg = o.status ? replica_message(o) : std::string();
  if (buf && cap > 0) {
    const size_t k = std::min<size_t>(msg.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, msg.data(), k);
    buf[k] = 0;
  }
  return o.status;
}

int nx_sim_records(nx_sim_t h, int32_t replica, nx_request_record* out, int64_t cap, int64_t* n) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const NxReplicaDesc& d = h->rep[replica];
    const NxReplicaOut& o = h->h_rep_out[replica];
    const nx::Workload& w = h->wl[replica];
    *n = o.completed;
    const int64_t m = std::min<int64_t>(cap, o.completed);
    for (int64_t k = 0; k < m; ++k) {
      const int r = h->h_records[d.req_off + k];
      nx_request_record& rec = out[k];
      rec.request_id = r;
      rec.arrival_ms = w.arrival_ms[r];
      rec.first_token_ms = nx::to_ms(h->h_first_us[d.req_off + r]);
      rec.completed_ms = nx::to_ms(h->h_done_us[d.req_off + r]);
      rec.prompt_tokens = w.prompt[r];
      rec.output_tokens = w.output[r];
      rec.engine_id = h->eng[d.eng_base + h->h_req_engine[d.req_off + r]].engine_id;
      rec.pad_ = 0;
    }
  });
}

namespace {
// The device's summary (summary.cu) as the report's Metrics: engine counts by
// index become shares ordered by engine id (std::map in metrics.cpp:60-88).
nx::Metrics device_metrics(const nx_sim& h, int32_t replica) {
  const NxReplicaMetrics& dm = h.h_metrics[replica];
  const NxReplicaDesc& d = h.rep[replica];
  if (!dm.valid) throw std::invalid_argument("RequestRecord timestamps out of order");
  nx::Metrics m;
  m.completed = dm.completed;
  if (dm.completed == 0) return m;
  m.p50_e2e = dm.p50_e2e;
  m.p90_e2e = dm.p90_e2e;
  m.p50_ttft = dm.p50_ttft;
  m.p50_tpot = dm.p50_tpot;
  m.mean_ttft = dm.mean_ttft;
  m.mean_tpot = dm.mean_tpot;
  m.slo_pct = dm.slo_pct;
  std::map<int, int64_t> per_engine;
  for (int e = 0; e < d.n_eng; ++e)
    if (dm.engine_count[e]) per_engine[h.eng[d.eng_base + e].engine_id] += dm.engine_count[e];
  for (const auto& [id, cnt] : per_engine)
    m.engine_share.emplace_back(id, static_cast<double>(cnt) / static_cast<double>(dm.completed));
  return m;
}
}  // namespace

extern "C" int nx_sim_metrics(nx_sim_t h, int32_t replica, nx_replica_metrics* out) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const NxReplicaOut& o = h->h_rep_out[replica];
    if (o.status != 0) throw std::runtime_error(replica_message(o));
    const nx::Metrics m = device_metrics(*h, replica);
    out->completed = m.completed;
    out->p50_e2e_ms = m.p50_e2e;
    out->p90_e2e_ms = m.p90_e2e;
    out->p50_ttft_ms = m.p50_ttft;
    out->p50_tpot_ms = m.p50_tpot;
    out->mean_ttft_ms = m.mean_ttft;
    out->mean_tpot_ms = m.mean_tpot;
    out->slo_attainment_pct = m.slo_pct;
  });
}

int nx_sim_summary_json(nx_sim_t h, int32_t replica, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const NxReplicaOut& o = h->h_rep_out[replica];
    if (o.status != 0) {
      const std::string msg = replica_message(o);
      if (o.status == 1) throw std::invalid_argument(msg);
      if (o.status == 3) throw std::logic_error(msg);
      throw std::runtime_error(msg);
    }
    const NxReplicaDesc& d = h->rep[replica];
    const nx::RunCfg& c = h->cfgs[replica];
    std::vector<nx::LearnerRow> learners;
    for (int e = 0; e < d.n_eng; ++e) {
      const NxEngineOut& eo = h->h_eng_out[d.eng_base + e];
      learners.push_back({h->eng[d.eng_base + e].engine_id, eo.samples, eo.params[5]});
    }
    const nx::Metrics m = device_metrics(*h, replica);
    const std::string s = nx::build_summary_json(
        c, o.arrived, o.completed, o.rejected, o.arrived - o.rejected - o.completed + o.pending,
        h->wl[replica].arrival_hash, o.event_hash, m, learners);
    *len = static_cast<int64_t>(s.size());
    if (cap > 0) {
      const size_t k = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, s.data(), k);
      buf[k] = 0;
    }
  });
}

int nx_sim_plan_log(nx_sim_t h, int32_t replica, nx_plan_log_row* out, int64_t cap, int64_t* n) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const NxReplicaDesc& d = h->rep[replica];
    const int64_t m = (d.log_flags & NX_LOG_PLANS) ? h->h_rep_out[replica].n_plan_log : 0;
    *n = m;
    for (int64_t k = 0; k < std::min(cap, m); ++k) {
      const NxPlanLog& L = h->h_plan_log[d.plan_log_off + k];
      out[k] = {nx::to_ms(L.t_us), L.engine_id, 0, L.b, L.s, L.predicted_ms, L.target_ms};
    }
  });
}

int nx_sim_route_log(nx_sim_t h, int32_t replica, nx_route_log_row* out, int64_t cap, int64_t* n) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const NxReplicaDesc& d = h->rep[replica];
    const int64_t m = (d.log_flags & NX_LOG_ROUTES) ? h->h_rep_out[replica].n_route_log : 0;
    *n = m;
    for (int64_t k = 0; k < std::min(cap, m); ++k) {
      const NxRouteLog& L = h->h_route_log[d.route_log_off + k];
      out[k] = {nx::to_ms(L.t_us), L.request, L.engine_id, 0, L.factors[0], L.factors[1],
                L.factors[2], L.factors[3], L.score};
    }
  });
}

int nx_sim_learner_history(nx_sim_t h, int32_t replica, nx_learner_snapshot* out, int64_t cap,
                           int64_t* n) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const NxReplicaDesc& d = h->rep[replica];
    const int64_t m = (d.log_flags & NX_LOG_LEARNER) ? h->h_rep_out[replica].n_learn_log : 0;
    *n = m;
    for (int64_t k = 0; k < std::min(cap, m); ++k) {
      const NxLearnLog& L = h->h_learn_log[d.learn_log_off + k];
      nx_learner_snapshot& o = out[k];
      o.engine_id = L.engine_id;
      o.pad_ = 0;
      o.sim_time_ms = nx::to_ms(L.t_us);
      o.samples_seen = L.samples;
      for (int i = 0; i < 8; ++i) o.params[i] = L.params[i];
    }
  });
}

// Simulation::write_outputs (sim.cpp:393-413): summary.json, requests.csv and
// the two JSONL logs (rows as sim.cpp:149-158, 176-186 format them).
int nx_sim_write_outputs(nx_sim_t h, int32_t replica) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const nx::RunCfg& c = h->cfgs[replica];
    if (c.out_dir.empty()) return;
    namespace fs = std::filesystem;
    const fs::path dir(c.out_dir);
    fs::create_directories(dir);
    if (!c.out_summary.empty()) {
      int64_t len = 0;
      if (nx_sim_summary_json(h, replica, nullptr, 0, &len) != NX_OK) throw std::runtime_error(g_err);
      std::string s(static_cast<size_t>(len) + 1, '\0');
      nx_sim_summary_json(h, replica, s.data(), len + 1, &len);
      s.resize(static_cast<size_t>(len));
      std::ofstream out(dir / c.out_summary);
      out << s;
    }
    if (!c.out_requests_csv.empty()) {
      const NxReplicaOut& o = h->h_rep_out[replica];
      std::vector<nx_request_record> recs(static_cast<size_t>(o.completed));
      int64_t n = 0;
      if (nx_sim_records(h, replica, recs.data(), o.completed, &n) != NX_OK) throw std::runtime_error(g_err);
      std::vector<nx::RecordRow> rows(recs.size());
      for (size_t i = 0; i < recs.size(); ++i)
        rows[i] = {recs[i].request_id, recs[i].arrival_ms, recs[i].first_token_ms, recs[i].completed_ms,
                   recs[i].prompt_tokens, recs[i].output_tokens, recs[i].engine_id};
      nx::write_requests_csv((dir / c.out_requests_csv).string(), rows);
    }
    if (!c.out_plans_jsonl.empty()) {
      int64_t n = 0;
      nx_sim_plan_log(h, replica, nullptr, 0, &n);
      std::vector<nx_plan_log_row> rows(static_cast<size_t>(n));
      nx_sim_plan_log(h, replica, rows.data(), n, &n);
      std::ofstream out(dir / c.out_plans_jsonl);
      for (const auto& r : rows) {
        nlohmann::ordered_json j;
        j["sim_time"] = r.sim_time_ms;
        j["engine_id"] = r.engine_id;
        j["b"] = r.b;
        j["s"] = r.s;
        j["predicted_ms"] = r.predicted_ms;
        j["target_ms"] = r.target_ms;
        out << j.dump() << '\n';
      }
    }
    if (!c.out_routing_jsonl.empty()) {
      int64_t n = 0;
      nx_sim_route_log(h, replica, nullptr, 0, &n);
      std::vector<nx_route_log_row> rows(static_cast<size_t>(n));
      nx_sim_route_log(h, replica, rows.data(), n, &n);
      std::ofstream out(dir / c.out_routing_jsonl);
      for (const auto& r : rows) {
        nlohmann::ordered_json j;
        j["sim_time"] = r.sim_time_ms;
        j["request_id"] = static_cast<uint64_t>(r.request_id);
        j["chosen_engine"] = r.chosen_engine;
        j["s_latency"] = r.s_latency;
        j["s_load"] = r.s_load;
        j["s_capacity"] = r.s_capacity;
        j["s_affinity"] = r.s_affinity;
        j["score"] = r.score;
        out << j.dump() << '\n';
      }
    }
  });
}

int nx_sim_learner(nx_sim_t h, int32_t replica, int32_t engine, double* params8, int64_t* samples,
                   int64_t* counters7) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    const NxReplicaDesc& d = h->rep[replica];
    if (engine < 0 || engine >= d.n_eng) throw std::invalid_argument("engine out of range");
    const NxEngineOut& eo = h->h_eng_out[d.eng_base + engine];
    for (int i = 0; i < 8; ++i) params8[i] = eo.params[i];
    *samples = eo.samples;
    for (int i = 0; i < 7; ++i) counters7[i] = eo.counters[i];
  });
}

int nx_sim_work(nx_sim_t h, int32_t replica, int64_t* out6) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    for (int i = 0; i < 6; ++i) out6[i] = h->h_rep_out[replica].work[i];
  });
}

int nx_sim_timeline(nx_sim_t h, int32_t replica, int64_t* begin_end_ns) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    begin_end_ns[0] = h->h_rep_out[replica].t_begin_ns;
    begin_end_ns[1] = h->h_rep_out[replica].t_end_ns;
  });
}

int nx_sim_phase_cycles(nx_sim_t h, int32_t replica, int64_t* out10) {
  return guard([&] {
    if (replica < 0 || replica >= h->n_rep) throw std::invalid_argument("replica out of range");
    for (int i = 0; i < 16; ++i) out10[i] = h->h_rep_out[replica].cycles[i];
  });
}

int nx_sim_copy_summaries(nx_sim_t h, void* dst_dev) {
  return guard([&] {
    cuda_check(cudaMemcpyAsync(dst_dev, h->pools.rep_out,
                               static_cast<size_t>(h->n_rep) * sizeof(NxReplicaOut),
                               cudaMemcpyDeviceToDevice, h->stream), "D2D summaries");
    cuda_check(cudaStreamSynchronize(h->stream), "sync");
  });
}

int nx_sim_summaries_dev(nx_sim_t h, void** dev_ptr, int64_t* bytes) {
  *dev_ptr = h->pools.rep_out;
  *bytes = static_cast<int64_t>(h->n_rep) * static_cast<int64_t>(sizeof(NxReplicaOut));
  return NX_OK;
}

void nx_sim_destroy(nx_sim_t h) { delete h; }

// ---- K1 --------------------------------------------------------------------------
int nx_perf_eval_async(const double* params, int32_t n_params, const int32_t* idx, const int32_t* b,
                       const int32_t* s, double* out_T, double* out_thr, int64_t n, int32_t mode,
                       uint32_t* dev_status, void* stream) {
  return guard([&] {
    if (n < 0 || n_params < 1) throw std::invalid_argument("nx_perf_eval: empty parameter table");
    for (const void* p : {(const void*)idx, (const void*)b, (const void*)s, (const void*)out_T})
      if (reinterpret_cast<uintptr_t>(p) % 16) throw std::invalid_argument("nx_perf_eval: buffers must be 16-byte aligned");
    if (out_thr && reinterpret_cast<uintptr_t>(out_thr) % 16)
      throw std::invalid_argument("nx_perf_eval: buffers must be 16-byte aligned");
    if (n == 0) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cuda_check(nx_launch_perf_eval(params, n_params, idx, b, s, out_T, out_thr, n,
                                   mode == NX_FAST_FP32, dev_status, sm_count(dev),
                                   static_cast<cudaStream_t>(stream)),
               "perf_eval launch");
  });
}

int nx_perf_eval_dev(const double* params, int32_t n_params, const int32_t* idx, const int32_t* b,
                     const int32_t* s, double* out_T, double* out_thr, int64_t n, int32_t mode,
                     void* stream) {
  return guard([&] {
    static thread_local unsigned* flag = nullptr;
    if (!flag) cuda_check(cudaMalloc(&flag, sizeof(unsigned)), "cudaMalloc(flag)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cuda_check(cudaMemsetAsync(flag, 0, sizeof(unsigned), st), "memset");
    const int rc = nx_perf_eval_async(params, n_params, idx, b, s, out_T, out_thr, n, mode, flag, stream);
    if (rc) throw NxError(rc, g_err);
    unsigned bad = 0;
    cuda_check(cudaMemcpyAsync(&bad, flag, sizeof bad, cudaMemcpyDeviceToHost, st), "D2H flag");
    cuda_check(cudaStreamSynchronize(st), "perf_eval sync");
    if (bad) throw std::invalid_argument("BatchShape requires b >= 1 and s >= b, valid params");
  });
}

// Small host batches (the scalar drop-in calls: predict_latency,
// throughput): one packed copy each way through a pinned per-thread buffer —
// parameters, inputs and a zeroed status word in, status + outputs out —
// instead of four pageable copies, a memset, a status read and one or two
// result reads (8 API calls → 3 and one synchronize).
constexpr int64_t kPackedEvalMax = 1 << 16;

// Grow-only pinned host buffer per thread for the packed host-pointer calls.
static unsigned char* pinned_stage(size_t bytes) {
  struct Pinned {
    unsigned char* p = nullptr;
    size_t cap = 0;
  };
  thread_local Pinned h;
  if (h.cap < bytes) {
    if (h.p) cudaFreeHost(h.p);
    h.p = nullptr;
    h.cap = 0;
    const size_t cap = std::max<size_t>(bytes, size_t(1) << 16);
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&h.p), cap, cudaHostAllocDefault), "cudaHostAlloc");
    h.cap = cap;
  }
  return h.p;
}

static int perf_eval_packed(const double* params, int32_t n_params, const int32_t* idx, const int32_t* b,
                     const int32_t* s, double* out_T, double* out_thr, int64_t n, int32_t mode) {
  Arena A;
  const size_t op = A.take<double>(8 * static_cast<size_t>(n_params));
  const size_t oi = A.take<int32_t>(n), ob = A.take<int32_t>(n), os = A.take<int32_t>(n);
  const size_t of = A.take<uint32_t>(4);  // status word (the end of the inbound copy)
  const size_t oT = A.take<double>(n), oh = A.take<double>(out_thr ? n : 0);
  const size_t in_bytes = of + 16, total = A.size;
  struct {
    unsigned char* p;
  } h{pinned_stage(total)};
  Staging S;
  S.A = A;
  S.alloc();
  std::memcpy(h.p + op, params, 8 * sizeof(double) * static_cast<size_t>(n_params));
  std::memcpy(h.p + oi, idx, sizeof(int32_t) * static_cast<size_t>(n));
  std::memcpy(h.p + ob, b, sizeof(int32_t) * static_cast<size_t>(n));
  std::memcpy(h.p + os, s, sizeof(int32_t) * static_cast<size_t>(n));
  std::memset(h.p + of, 0, 16);
  unsigned char* d = S.d;
  cudaStream_t st = nullptr;
  cuda_check(cudaMemcpyAsync(d, h.p, in_bytes, cudaMemcpyHostToDevice, st), "H2D");
  const int rc = nx_perf_eval_async(reinterpret_cast<double*>(d + op), n_params, reinterpret_cast<int32_t*>(d + oi),
                                    reinterpret_cast<int32_t*>(d + ob), reinterpret_cast<int32_t*>(d + os),
                                    reinterpret_cast<double*>(d + oT),
                                    out_thr ? reinterpret_cast<double*>(d + oh) : nullptr, n, mode,
                                    reinterpret_cast<uint32_t*>(d + of), st);
  if (rc) return rc;
  cuda_check(cudaMemcpyAsync(h.p + of, d + of, total - of, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "perf_eval sync");
  uint32_t bad = 0;
  std::memcpy(&bad, h.p + of, sizeof bad);
  if (bad) throw std::invalid_argument("BatchShape requires b >= 1 and s >= b, valid params");
  std::memcpy(out_T, h.p + oT, sizeof(double) * static_cast<size_t>(n));
  if (out_thr) std::memcpy(out_thr, h.p + oh, sizeof(double) * static_cast<size_t>(n));
  return NX_OK;
}

int nx_perf_eval_host(const double* params, int32_t n_params, const int32_t* idx, const int32_t* b,
                      const int32_t* s, double* out_T, double* out_thr, int64_t n, int32_t mode) {
  return guard([&] {
    if (n < 0 || n_params < 1) throw std::invalid_argument("nx_perf_eval: empty parameter table");
    if (n <= kPackedEvalMax) {
      const int rc = perf_eval_packed(params, n_params, idx, b, s, out_T, out_thr, n, mode);
      if (rc) throw NxError(rc, g_err);
      return;
    }
    Staging S;
    Arena& A = S.A;
    const size_t op = A.take<double>(8 * static_cast<size_t>(n_params));
    const size_t oi = A.take<int32_t>(n), ob = A.take<int32_t>(n), os = A.take<int32_t>(n);
    const size_t oT = A.take<double>(n), oh = A.take<double>(n);
    S.alloc();
    unsigned char* d = S.d;
    cuda_check(cudaMemcpy(d + op, params, 8 * sizeof(double) * n_params, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d + oi, idx, sizeof(int32_t) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d + ob, b, sizeof(int32_t) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d + os, s, sizeof(int32_t) * n, cudaMemcpyHostToDevice), "H2D");
    const int rc = nx_perf_eval_dev(reinterpret_cast<double*>(d + op), n_params,
                                    reinterpret_cast<int32_t*>(d + oi), reinterpret_cast<int32_t*>(d + ob),
                                    reinterpret_cast<int32_t*>(d + os), reinterpret_cast<double*>(d + oT),
                                    out_thr ? reinterpret_cast<double*>(d + oh) : nullptr, n, mode, nullptr);
    if (rc) throw NxError(rc, g_err);
    cuda_check(cudaMemcpy(out_T, d + oT, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H");
    if (out_thr) cuda_check(cudaMemcpy(out_thr, d + oh, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H");
  });
}

// ---- K2 / K3 / K4 batched operators ------------------------------------------------
}  // extern "C"

namespace {
}  // namespace

extern "C" {

int nx_abi_sizes(int64_t* out, int32_t n) {
  const int64_t sz[] = {sizeof(nx_lens_problem), sizeof(nx_lens_plan), sizeof(nx_route_group),
                        sizeof(nx_engine_report), sizeof(nx_route_request), sizeof(nx_route_decision),
                        sizeof(nx_refit_problem), sizeof(nx_refit_result), sizeof(nx_replica_summary),
                        sizeof(nx_request_record), sizeof(nx_baseline_problem)};
  for (int32_t i = 0; i < n && i < static_cast<int32_t>(sizeof sz / sizeof sz[0]); ++i) out[i] = sz[i];
  return NX_OK;
}

int nx_lens_schedule_mode_dev(const nx_lens_problem* problems, int32_t n_problems,
                              const int32_t* wait_remaining, int64_t n_wait_total, nx_lens_plan* plans,
                              int32_t* alloc_tokens, int32_t mode, void* stream) {
  return guard([&] {
    if (n_problems < 0 || n_wait_total < 0) throw std::invalid_argument("nx_lens_schedule: negative sizes");
    if (mode != NX_DETERMINISTIC_FP64 && mode != NX_FAST_FP32) throw std::invalid_argument("nx_lens_schedule: unknown mode");
    if (n_problems == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    retain_default_pool();
    int32_t* gpre = nullptr;  // prefix scratch for spans beyond the shared-memory stage
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&gpre),
                               sizeof(int32_t) * static_cast<size_t>(n_wait_total + n_problems), st),
               "cudaMallocAsync");
    cudaError_t e = nx_launch_lens(problems, n_problems, wait_remaining, plans, alloc_tokens, gpre,
                                   current_sms(), mode, st);
    const cudaError_t e2 = cudaFreeAsync(gpre, st);
    cuda_check(e, "nx_lens_kernel launch");
    cuda_check(e2, "cudaFreeAsync");
  });
}

int nx_lens_schedule_dev(const nx_lens_problem* problems, int32_t n_problems,
                         const int32_t* wait_remaining, int64_t n_wait_total, nx_lens_plan* plans,
                         int32_t* alloc_tokens, void* stream) {
  return nx_lens_schedule_mode_dev(problems, n_problems, wait_remaining, n_wait_total, plans, alloc_tokens,
                                   NX_DETERMINISTIC_FP64, stream);
}

int nx_lens_schedule_mode_host(const nx_lens_problem* problems, int32_t n_problems,
                               const int32_t* wait_remaining, int64_t n_wait_total, nx_lens_plan* plans,
                               int32_t* alloc_tokens, int32_t mode) {
  return guard([&] {
    if (n_problems < 0 || n_wait_total < 0) throw std::invalid_argument("nx_lens_schedule: negative sizes");
    if (mode != NX_DETERMINISTIC_FP64 && mode != NX_FAST_FP32) throw std::invalid_argument("nx_lens_schedule: unknown mode");
    if (n_problems == 0) return;
    for (int32_t i = 0; i < n_problems; ++i)
      if (problems[i].n_wait < 0 || problems[i].wait_off < 0 ||
          problems[i].wait_off + problems[i].n_wait > n_wait_total)
        throw std::invalid_argument("nx_lens_schedule: waiter range out of bounds");
    // one packed copy each way through pinned memory (problems + waiters in;
    // plans + allocations out), the prefix scratch in the same staging
    // buffer: the scalar schedule_step pays 3 API calls and one synchronize
    Staging S;
    const size_t op = S.A.take<nx_lens_problem>(n_problems), orm = S.A.take<int32_t>(n_wait_total),
                 opl = S.A.take<nx_lens_plan>(n_problems), oal = S.A.take<int32_t>(n_wait_total),
                 ogp = S.A.take<int32_t>(static_cast<size_t>(n_wait_total) + n_problems);
    S.alloc();
    unsigned char* h = pinned_stage(ogp);
    std::memcpy(h + op, problems, sizeof(nx_lens_problem) * n_problems);
    if (n_wait_total) std::memcpy(h + orm, wait_remaining, sizeof(int32_t) * n_wait_total);
    cudaStream_t st = nullptr;
    cuda_check(cudaMemcpyAsync(S.d, h, opl, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(nx_launch_lens(S.at<nx_lens_problem>(op), n_problems, S.at<int32_t>(orm), S.at<nx_lens_plan>(opl),
                              S.at<int32_t>(oal), S.at<int32_t>(ogp), current_sms(), mode, st),
               "nx_lens_kernel launch");
    cuda_check(cudaMemcpyAsync(h + opl, S.d + opl, ogp - opl, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "nx_lens_schedule sync");
    std::memcpy(plans, h + opl, sizeof(nx_lens_plan) * n_problems);
    if (n_wait_total) std::memcpy(alloc_tokens, h + oal, sizeof(int32_t) * n_wait_total);
    for (int32_t i = 0; i < n_problems; ++i)
      if (plans[i].status != NX_OK)
        throw NxError(plans[i].status, "schedule_step: problem " + std::to_string(i) + ": " +
                                           status_text(plans[i].status));
  });
}

int nx_lens_schedule_host(const nx_lens_problem* problems, int32_t n_problems,
                          const int32_t* wait_remaining, int64_t n_wait_total, nx_lens_plan* plans,
                          int32_t* alloc_tokens) {
  return nx_lens_schedule_mode_host(problems, n_problems, wait_remaining, n_wait_total, plans, alloc_tokens,
                                    NX_DETERMINISTIC_FP64);
}

int nx_prism_route_mode_dev(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                            const nx_route_request* requests, int32_t* session_map,
                            nx_route_decision* decisions, int32_t* group_status, int32_t mode,
                            void* stream) {
  return guard([&] {
    if (n_groups < 0) throw std::invalid_argument("nx_prism_route: negative sizes");
    if (mode != NX_DETERMINISTIC_FP64 && mode != NX_FAST_FP32) throw std::invalid_argument("nx_prism_route: unknown mode");
    if (n_groups == 0) return;
    cuda_check(nx_launch_route(groups, n_groups, reports, requests, session_map, decisions, group_status,
                               current_sms(), mode, static_cast<cudaStream_t>(stream)),
               "nx_route_kernel launch");
  });
}

int nx_prism_route_dev(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                       const nx_route_request* requests, int32_t* session_map,
                       nx_route_decision* decisions, int32_t* group_status, void* stream) {
  return nx_prism_route_mode_dev(groups, n_groups, reports, requests, session_map, decisions, group_status,
                                 NX_DETERMINISTIC_FP64, stream);
}

int nx_prism_route_mode_host(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                             int64_t n_reports, const nx_route_request* requests, int64_t n_requests,
                             int32_t* session_map, int64_t n_session_entries,
                             nx_route_decision* decisions, int32_t* group_status, int32_t mode) {
  return guard([&] {
    if (n_groups < 0 || n_reports < 0 || n_requests < 0 || n_session_entries < 0)
      throw std::invalid_argument("nx_prism_route: negative sizes");
    if (mode != NX_DETERMINISTIC_FP64 && mode != NX_FAST_FP32) throw std::invalid_argument("nx_prism_route: unknown mode");
    if (n_groups == 0) return;
    for (int32_t i = 0; i < n_groups; ++i) {
      const nx_route_group& g = groups[i];
      if (g.n_engines < 0 || g.n_requests < 0 || g.n_sessions < 0 || g.engine_off < 0 ||
          g.request_off < 0 || g.session_off < 0 || g.engine_off + g.n_engines > n_reports ||
          g.request_off + g.n_requests > n_requests || g.session_off + g.n_sessions > n_session_entries)
        throw std::invalid_argument("nx_prism_route: group ranges out of bounds");
    }
    // one packed copy each way through pinned memory (the routers' state,
    // requests and session maps in; state, maps, decisions and statuses out)
    Staging S;
    const size_t og = S.A.take<nx_route_group>(n_groups), orp = S.A.take<nx_engine_report>(n_reports),
                 orq = S.A.take<nx_route_request>(n_requests), osm = S.A.take<int32_t>(n_session_entries),
                 odc = S.A.take<nx_route_decision>(n_requests), ost = S.A.take<int32_t>(n_groups);
    const size_t total = S.A.size;
    S.alloc();
    unsigned char* h = pinned_stage(total);
    std::memcpy(h + og, groups, sizeof(nx_route_group) * n_groups);
    if (n_reports) std::memcpy(h + orp, reports, sizeof(nx_engine_report) * n_reports);
    if (n_requests) std::memcpy(h + orq, requests, sizeof(nx_route_request) * n_requests);
    if (n_session_entries) std::memcpy(h + osm, session_map, sizeof(int32_t) * n_session_entries);
    cudaStream_t st = nullptr;
    cuda_check(cudaMemcpyAsync(S.d, h, odc, cudaMemcpyHostToDevice, st), "H2D");
    const int rc = nx_prism_route_mode_dev(S.at<nx_route_group>(og), n_groups, S.at<nx_engine_report>(orp),
                                           S.at<nx_route_request>(orq), S.at<int32_t>(osm),
                                           S.at<nx_route_decision>(odc), S.at<int32_t>(ost), mode, st);
    if (rc) throw NxError(rc, g_err);
    cuda_check(cudaMemcpyAsync(h, S.d, total, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "nx_prism_route sync");
    std::memcpy(groups, h + og, sizeof(nx_route_group) * n_groups);
    if (n_reports) std::memcpy(reports, h + orp, sizeof(nx_engine_report) * n_reports);
    if (n_session_entries) std::memcpy(session_map, h + osm, sizeof(int32_t) * n_session_entries);
    if (n_requests) std::memcpy(decisions, h + odc, sizeof(nx_route_decision) * n_requests);
    std::memcpy(group_status, h + ost, sizeof(int32_t) * n_groups);
    for (int32_t i = 0; i < n_groups; ++i)
      if (group_status[i] != NX_OK)
        throw NxError(group_status[i], "Router::route: group " + std::to_string(i) + ": " +
                                           status_text(group_status[i]));
  });
}

int nx_prism_route_host(nx_route_group* groups, int32_t n_groups, nx_engine_report* reports,
                        int64_t n_reports, const nx_route_request* requests, int64_t n_requests,
                        int32_t* session_map, int64_t n_session_entries,
                        nx_route_decision* decisions, int32_t* group_status) {
  return nx_prism_route_mode_host(groups, n_groups, reports, n_reports, requests, n_requests, session_map,
                                  n_session_entries, decisions, group_status, NX_DETERMINISTIC_FP64);
}

int nx_refit_dev(int32_t kind, const nx_refit_problem* problems, int32_t n_problems,
                 const int32_t* sample_b, const int32_t* sample_s, const double* sample_y,
                 int64_t max_long_window, nx_refit_result* results, void* stream) {
  return guard([&] {
    if (kind != NX_REFIT_LINEAR && kind != NX_REFIT_STRUCTURAL)
      throw std::invalid_argument("nx_refit: unknown kind");
    if (n_problems < 0 || max_long_window < 1 || max_long_window > (1 << 24))
      throw std::invalid_argument("nx_refit: bad sizes");
    if (n_problems == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    retain_default_pool();
    const int64_t per = nx_refit_scratch_per(max_long_window);
    // one scratch slice per resident warp: bounded by the device, not the batch
    int grid = std::min<int64_t>(n_problems, static_cast<int64_t>(current_sms()) * 16);
    const int64_t budget = int64_t(1) << 31;  // bytes of scratch at most
    while (grid > 1 && per * 8 * grid > budget) grid /= 2;
    double* scratch = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(double) * per * grid, st),
               "cudaMallocAsync");
    const cudaError_t e = nx_launch_refit(kind, problems, n_problems, sample_b, sample_s, sample_y,
                                          results, scratch, per, grid, static_cast<int>(max_long_window), st);
    const cudaError_t e2 = cudaFreeAsync(scratch, st);
    cuda_check(e, "nx_refit_kernel launch");
    cuda_check(e2, "cudaFreeAsync");
  });
}

int nx_refit_host(int32_t kind, const nx_refit_problem* problems, int32_t n_problems,
                  const int32_t* sample_b, const int32_t* sample_s, const double* sample_y,
                  int64_t n_samples_total, nx_refit_result* results) {
  return guard([&] {
    if (n_problems < 0 || n_samples_total < 0) throw std::invalid_argument("nx_refit: negative sizes");
    if (n_problems == 0) return;
    int64_t max_w = 1;
    for (int32_t i = 0; i < n_problems; ++i) {
      const nx_refit_problem& p = problems[i];
      if (p.n_samples < 0 || p.sample_off < 0 || p.sample_off + p.n_samples > n_samples_total)
        throw std::invalid_argument("nx_refit: sample range out of bounds");
      max_w = std::max<int64_t>(max_w, std::min<int64_t>(p.long_window, 1 << 24));
    }
    Staging S;
    const size_t op = S.A.take<nx_refit_problem>(n_problems), ob = S.A.take<int32_t>(n_samples_total),
                 os = S.A.take<int32_t>(n_samples_total), oy = S.A.take<double>(n_samples_total),
                 orr = S.A.take<nx_refit_result>(n_problems);
    S.alloc();
    cuda_check(cudaMemcpy(S.at<void>(op), problems, sizeof(nx_refit_problem) * n_problems, cudaMemcpyHostToDevice), "H2D");
    if (n_samples_total) {
      cuda_check(cudaMemcpy(S.at<void>(ob), sample_b, sizeof(int32_t) * n_samples_total, cudaMemcpyHostToDevice), "H2D");
      cuda_check(cudaMemcpy(S.at<void>(os), sample_s, sizeof(int32_t) * n_samples_total, cudaMemcpyHostToDevice), "H2D");
      cuda_check(cudaMemcpy(S.at<void>(oy), sample_y, sizeof(double) * n_samples_total, cudaMemcpyHostToDevice), "H2D");
    }
    const int rc = nx_refit_dev(kind, S.at<nx_refit_problem>(op), n_problems, S.at<int32_t>(ob),
                                S.at<int32_t>(os), S.at<double>(oy), max_w, S.at<nx_refit_result>(orr), nullptr);
    if (rc) throw NxError(rc, g_err);
    cuda_check(cudaMemcpy(results, S.at<void>(orr), sizeof(nx_refit_result) * n_problems, cudaMemcpyDeviceToHost), "D2H");
    for (int32_t i = 0; i < n_problems; ++i)
      if (results[i].status != NX_OK)
        throw NxError(results[i].status, "OnlineLearner refit: problem " + std::to_string(i) + ": " +
                                             status_text(results[i].status));
  });
}

// ---- scheduling building blocks --------------------------------------------------
}  // extern "C"

namespace {

// Stage records (+ optional aux arrays) on the device, run one scalar-ops
// kernel, copy records (+ aux out) back. Returns after synchronising.
void run_scalar_op(int op, void* recs, size_t rec_bytes, int n, const void* aux_in,
                   size_t aux_in_bytes, void* aux_out, size_t aux_out_bytes) {
  Staging S;
  const size_t orc = S.A.take<unsigned char>(rec_bytes * n), oi = S.A.take<unsigned char>(aux_in_bytes),
               oo = S.A.take<unsigned char>(aux_out_bytes);
  S.alloc();
  cuda_check(cudaMemcpy(S.at<void>(orc), recs, rec_bytes * n, cudaMemcpyHostToDevice), "H2D");
  if (aux_in_bytes) cuda_check(cudaMemcpy(S.at<void>(oi), aux_in, aux_in_bytes, cudaMemcpyHostToDevice), "H2D");
  if (aux_out_bytes) cuda_check(cudaMemcpy(S.at<void>(oo), aux_out, aux_out_bytes, cudaMemcpyHostToDevice), "H2D");
  cuda_check(nx_launch_scalar_ops(op, S.at<void>(orc), n, S.at<void>(oi), S.at<void>(oo), nullptr), "launch");
  cuda_check(cudaMemcpy(recs, S.at<void>(orc), rec_bytes * n, cudaMemcpyDeviceToHost), "D2H");
  if (aux_out_bytes) cuda_check(cudaMemcpy(aux_out, S.at<void>(oo), aux_out_bytes, cudaMemcpyDeviceToHost), "D2H");
}

template <class R>
void first_status(const R* r, int32_t n, const char* what) {
  for (int32_t i = 0; i < n; ++i)
    if (r[i].status != NX_OK)
      throw NxError(r[i].status, std::string(what) + ": record " + std::to_string(i) + ": " +
                                     status_text(r[i].status));
}

}  // namespace

extern "C" {

int nx_target_latency_host(nx_target_query* q, int32_t n) {
  return guard([&] {
    if (n <= 0) return;
    run_scalar_op(0, q, sizeof *q, n, nullptr, 0, nullptr, 0);
    first_status(q, n, "target_latency");
  });
}

int nx_budget_search_host(nx_budget_query* q, int32_t n) {
  return guard([&] {
    if (n <= 0) return;
    run_scalar_op(1, q, sizeof *q, n, nullptr, 0, nullptr, 0);
    first_status(q, n, "binary_search_budget");
  });
}

int nx_allocate_tokens_host(nx_allocate_problem* p, int32_t n, const int32_t* wait_remaining,
                            int64_t n_wait_total, int32_t* tokens) {
  return guard([&] {
    if (n <= 0) return;
    for (int32_t i = 0; i < n; ++i)
      if (p[i].n_wait < 0 || p[i].wait_off < 0 || p[i].wait_off + p[i].n_wait > n_wait_total)
        throw std::invalid_argument("allocate_tokens: waiter range out of bounds");
    run_scalar_op(2, p, sizeof *p, n, wait_remaining, sizeof(int32_t) * n_wait_total, tokens,
                  sizeof(int32_t) * n_wait_total);
    first_status(p, n, "allocate_tokens");
  });
}

int nx_baseline_schedule_host(nx_baseline_problem* p, int32_t n, const int32_t* wait_remaining,
                              int64_t n_wait_total, int32_t* tokens) {
  return guard([&] {
    if (n <= 0) return;
    for (int32_t i = 0; i < n; ++i)
      if (p[i].n_run < 0 || p[i].n_wait < 0 || p[i].wait_off < 0 || p[i].wait_off + p[i].n_wait > n_wait_total)
        throw std::invalid_argument("schedule_baseline: queue range out of bounds");
    run_scalar_op(5, p, sizeof *p, n, wait_remaining, sizeof(int32_t) * n_wait_total, tokens,
                  sizeof(int32_t) * n_wait_total);
    first_status(p, n, "schedule_baseline");
  });
}

int nx_router_scores_host(nx_score_query* q, int32_t n) {
  return guard([&] {
    if (n <= 0) return;
    run_scalar_op(3, q, sizeof *q, n, nullptr, 0, nullptr, 0);
    first_status(q, n, "router scores");
  });
}

int nx_tradeoff_update_host(nx_tradeoff_state* st, int32_t n, const nx_completion* completions,
                            int64_t n_completions) {
  return guard([&] {
    if (n <= 0) return;
    for (int32_t i = 0; i < n; ++i)
      if (st[i].n_new < 0 || st[i].comp_off < 0 || st[i].comp_off + st[i].n_new > n_completions ||
          st[i].win_len < 0 || st[i].win_len > NX_TRADEOFF_WINDOW || st[i].win_head < 0 ||
          st[i].win_head >= NX_TRADEOFF_WINDOW)
        throw std::invalid_argument("TradeoffEstimator: state out of range");
    run_scalar_op(4, st, sizeof *st, n, completions, sizeof(nx_completion) * n_completions, nullptr, 0);
  });
}

// ---- K6: NCCL gather --------------------------------------------------------------
}  // extern "C"

namespace {
// libnccl resolved at run time (the one torch already loaded, else the
// system's): the product library has no link-time NCCL dependency.
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw NxError(NX_ERUNTIME, "libnccl.so.2 not found");
    x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    x.all_gather = reinterpret_cast<decltype(x.all_gather)>(dlsym(h, "ncclAllGather"));
    x.error_string = reinterpret_cast<decltype(x.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!x.get_unique_id || !x.comm_init_rank || !x.comm_destroy || !x.all_gather || !x.error_string)
      throw NxError(NX_ERUNTIME, "libnccl.so.2 lacks the collective entry points");
    return x;
  }();
  return n;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NxError(NX_ECUDA, std::string(what) + ": " + nccl().error_string(r));
}
}  // namespace

extern "C" {

int nx_nccl_unique_id(char* id128) {
  return guard([&] {
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == NX_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id128, &id, sizeof id);
  });
}

int nx_nccl_comm_init(const char* id128, int32_t nranks, int32_t rank, int32_t device, void** comm) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("nx_nccl_comm_init: bad rank");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t c = nullptr;
    nccl_check(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
    *comm = c;
  });
}

int nx_nccl_comm_destroy(void* comm) {
  return guard([&] {
    if (comm) nccl_check(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

int nx_sim_gather_summaries(nx_sim_t h, void* comm, void* recv_dev) {
  return guard([&] {
    if (!comm || !recv_dev) throw std::invalid_argument("nx_sim_gather_summaries: null communicator or buffer");
    cuda_check(cudaSetDevice(h->device), "cudaSetDevice");
    const size_t bytes = static_cast<size_t>(h->n_rep) * sizeof(NxReplicaOut);
    nccl_check(nccl().all_gather(h->pools.rep_out, recv_dev, bytes, ncclUint8, static_cast<ncclComm_t>(comm),
                                 h->stream),
               "ncclAllGather");
  });
}

// ---- host utilities -------------------------------------------------------------
int nx_workload_info(const char* config_json, uint64_t* arrival_hash, int64_t* n_requests,
                     int64_t* n_sessions) {
  return guard([&] {
    const nx::RunCfg c = nx::parse_run_config(config_json);
    const nx::Workload w = nx::build_workload(c);
    *arrival_hash = w.arrival_hash;
    *n_requests = static_cast<int64_t>(w.prompt.size());
    *n_sessions = static_cast<int64_t>(w.session_names.size());
  });
}

int nx_rng_state(uint64_t root_seed, const char* tag, uint64_t index, uint64_t* state4) {
  return guard([&] {
    nx::Xoshiro x(nx::substream_seed(root_seed, tag ? tag : "", index));
    for (int i = 0; i < 4; ++i) state4[i] = x.s[i];
  });
}

int nx_synth_generate(const char* scenario, int64_t n, uint64_t seed, int64_t* prompts,
                      int64_t* outputs, char* session_ids16) {
  return guard([&] {
    const auto rows = nx::synth_rows(nx::scenario_named(scenario), n, seed);
    for (int64_t i = 0; i < n; ++i) {
      prompts[i] = rows[i].prompt;
      outputs[i] = rows[i].output;
      std::snprintf(session_ids16 + 16 * i, 16, "%s", rows[i].session.c_str());
    }
  });
}

}  // extern "C"
