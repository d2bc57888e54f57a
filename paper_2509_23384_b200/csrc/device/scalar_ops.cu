// Batched forms of the LENS / router / tradeoff building blocks that the
// reference exposes as free functions (proj/include/servesim/lens.h:93-124,
// router.h:57-66, lens.h:127-151). They let the C++ drop-in layer
// (include/nx_servesim.hpp) answer every scheduling call on the device; the
// arithmetic is the shared core the simulator and nx_lens_schedule use.
#include "../../../include/nx_sched.h"
#include "nx_lens.cuh"
#include "nx_router.cuh"

namespace nxd {

// target_latency (lens.cpp:10-31), one thread per query.
__global__ void nx_target_kernel(nx_target_query* __restrict__ q, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  nx_target_query& r = q[i];
  if (!(r.ttft_slo_ms > 0.0 && r.tpot_slo_ms > 0.0) ||
      !(r.beta > 0.0 && r.l_bar >= 1.0 && r.td_min_ms > 0.0) || !(r.q_ref > 0.0)) {
    r.status = NX_EINVAL;
    return;
  }
  bool risk = false;
  r.target_ms = lens_target(r.ttft_slo_ms, r.tpot_slo_ms, r.alpha_ms, r.beta, r.l_bar, r.td_min_ms,
                            r.q_ref, r.wait_count, &risk);
  r.slo_risk = risk;
  r.status = NX_OK;
}

// binary_search_budget (lens.cpp:33-56), one thread per query.
__global__ void nx_budget_kernel(nx_budget_query* __restrict__ q, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  nx_budget_query& r = q[i];
  const Params P = params_from(r.params);
  if (r.b < 1 || r.b > r.q_max || !(r.target_ms > 0.0) || !params_valid(P)) {
    r.status = NX_EINVAL;
    return;
  }
  int64_t s_cap = r.s_cap < 0 ? r.m_max : r.s_cap;
  s_cap = (r.m_max < s_cap) ? r.m_max : s_cap;
  s_cap = (r.b < s_cap) ? s_cap : r.b;
  const double bd = static_cast<double>(r.b);
  const double fb = sat(P.kB, bd);
  int64_t lo = r.b, hi = s_cap, budget = r.b;
  for (int it = 0; it < r.n_search_iters; ++it) {
    if (lo > hi) break;
    const int64_t mid = lo + (hi - lo) / 2;
    if (latency_fb(P, fb, bd, static_cast<double>(mid)) <= r.target_ms) {
      budget = mid;
      lo = mid + 1;
    } else {
      hi = mid - 1;
    }
  }
  r.budget = budget;
  r.status = NX_OK;
}

// Saturating inclusive prefix of the first `slots` waiters' remaining prompts:
// pr[0] = 0, pr[k + 1] = min(2^30, sum_{i<=k} wr[i]); one warp.
__device__ void waiter_prefix(const int32_t* wr, int slots, int32_t* pr, int lane) {
  __syncwarp();
  if (lane == 0) pr[0] = 0;
  long long carry = 0;
  for (int base = 0; base < slots; base += 32) {
    const int i = base + lane;
    long long s = i < slots ? wr[i] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(NX_FULL, s, o);
      if (lane >= o) s += u;
    }
    const long long tot = carry + s;
    if (i < slots) pr[i + 1] = static_cast<int32_t>(tot < (1 << 30) ? tot : (1 << 30));
    carry += __shfl_sync(NX_FULL, s, 31);
    if (carry > (1 << 30)) carry = 1 << 30;
  }
  __syncwarp();
}

// allocate_tokens (lens.cpp:58-79), one warp per problem: every waiter takes
// min(remaining, budget left) while slots remain (the prefix-sum form).
__global__ void nx_allocate_kernel(nx_allocate_problem* __restrict__ probs, int n,
                                   const int32_t* __restrict__ rem, int32_t* __restrict__ tokens) {
  __shared__ int32_t pre[4][1025];
  const int lane = lane_id(), w = threadIdx.x >> 5;
  const int pi = blockIdx.x * 4 + w;
  if (pi >= n) return;
  nx_allocate_problem& p = probs[pi];
  if (p.b < p.n_run || p.s < p.b || p.n_run < 0 || p.n_wait < 0) {
    if (lane == 0) p.status = NX_EINVAL;  // allocate_tokens: budget below queue needs
    return;
  }
  const int64_t slots64 = p.b - p.n_run;
  const int slots = static_cast<int>(slots64 < p.n_wait ? slots64 : p.n_wait);
  const int64_t budget64 = p.s - p.n_run;
  if (slots > 1024 || budget64 >= (int64_t(1) << 30)) {
    if (lane == 0) p.status = NX_EINVAL;  // device limit
    return;
  }
  const int budget = static_cast<int>(budget64);
  const int32_t* wr = rem + p.wait_off;
  bool bad = false;
  for (int i = lane; i < slots; i += 32) bad |= wr[i] < 1;
  if (__any_sync(NX_FULL, bad)) {
    if (lane == 0) p.status = NX_EINVAL;  // device limit: remaining prompt >= 1
    return;
  }
  // saturating prefix (only compared against budgets < 2^30)
  int32_t* pr = pre[w];
  waiter_prefix(wr, slots, pr, lane);
  const int j = budget > 0 ? lens_lower_bound(pr, slots, budget) : 0;
  for (int k = lane; k < j; k += 32) {
    const int rr = pr[k + 1] - pr[k];
    const int left = budget - pr[k];
    tokens[p.wait_off + k] = rr < left ? rr : left;
  }
  if (lane == 0) {
    p.n_prefill = j;
    p.status = NX_OK;
  }
}

// schedule_baseline (engine.cpp:61-108), one warp per problem.
//  prefill_priority: whole remaining prompts, FCFS, while the batch stays
//    within q_max requests and m_max tokens (k waiters fit iff k <= q_max and
//    prefix[k] <= m_max); with nobody waiting, every runner decodes.
//  static_chunked: allocate_tokens(run, wait, b, s) with b = min(|run| +
//    |wait|, q_max), s = min(m_max, max(static_budget, b)).
__global__ void nx_baseline_kernel(nx_baseline_problem* __restrict__ probs, int n,
                                   const int32_t* __restrict__ rem, int32_t* __restrict__ tokens) {
  __shared__ int32_t pre[4][1025];
  const int lane = lane_id(), w = threadIdx.x >> 5;
  const int pi = blockIdx.x * 4 + w;
  if (pi >= n) return;
  nx_baseline_problem& p = probs[pi];
  auto finish = [&](int status) {
    if (lane == 0) p.status = status;
  };
  if (lane == 0) {
    p.b = 0;
    p.s = 0;
    p.predicted_ms = 0.0;
    p.n_decode = 0;
    p.n_prefill = 0;
  }
  if (p.policy != NX_SCHED_PREFILL_PRIORITY && p.policy != NX_SCHED_STATIC_CHUNKED) {
    finish(p.policy == NX_SCHED_LENS ? NX_ELOGIC : NX_EINVAL);
    return;
  }
  const int R = p.n_run, W = p.n_wait;
  if (R == 0 && W == 0) {
    finish(NX_OK);  // empty plan, no prediction
    return;
  }
  const int32_t* wr = rem + p.wait_off;
  int32_t* pr = pre[w];
  int64_t b = 0, s = 0;
  int n_dec = 0, j = 0;
  if (p.policy == NX_SCHED_PREFILL_PRIORITY) {
    if (W > 0) {
      const int64_t cap = p.q_max < W ? p.q_max : W;
      if (cap > 1024 || p.m_max >= (int64_t(1) << 30)) {
        finish(NX_EINVAL);  // device limit
        return;
      }
      const int slots = static_cast<int>(cap);
      bool bad = false;
      for (int i = lane; i < slots; i += 32) bad |= wr[i] < 1;
      if (__any_sync(NX_FULL, bad)) {
        finish(NX_EINVAL);  // device limit: remaining prompt >= 1
        return;
      }
      waiter_prefix(wr, slots, pr, lane);
      j = lens_lower_bound(pr + 1, slots, static_cast<int>(p.m_max) + 1);
      if (j == 0) {
        finish(NX_ERUNTIME);  // prompt exceeds m_max
        return;
      }
      b = j;
      s = pr[j];
      for (int k = lane; k < j; k += 32) tokens[p.wait_off + k] = wr[k];
    } else {
      n_dec = R;
      b = R;
      s = R;
    }
  } else {
    const int64_t tot = static_cast<int64_t>(R) + W;
    const int64_t bb = tot < p.q_max ? tot : p.q_max;
    const int64_t sb = p.static_budget < bb ? bb : p.static_budget;
    const int64_t ss = p.m_max < sb ? p.m_max : sb;
    if (bb < R || ss < bb) {
      finish(NX_EINVAL);  // allocate_tokens: budget below queue needs
      return;
    }
    const int64_t slots64 = bb - R < W ? bb - R : W;
    const int64_t budget64 = ss - R;
    if (slots64 > 1024 || budget64 >= (int64_t(1) << 30)) {
      finish(NX_EINVAL);  // device limit
      return;
    }
    const int slots = static_cast<int>(slots64), budget = static_cast<int>(budget64);
    bool bad = false;
    for (int i = lane; i < slots; i += 32) bad |= wr[i] < 1;
    if (__any_sync(NX_FULL, bad)) {
      finish(NX_EINVAL);
      return;
    }
    waiter_prefix(wr, slots, pr, lane);
    j = budget > 0 ? lens_lower_bound(pr, slots, budget) : 0;
    int64_t got = 0;
    for (int k = lane; k < j; k += 32) {
      const int rr = pr[k + 1] - pr[k];
      const int left = budget - pr[k];
      const int t = rr < left ? rr : left;
      tokens[p.wait_off + k] = t;
      got += t;
    }
    for (int o = 16; o > 0; o >>= 1) got += __shfl_xor_sync(NX_FULL, got, o);
    n_dec = R;
    b = static_cast<int64_t>(R) + j;
    s = static_cast<int64_t>(R) + got;
  }
  // predict_latency(params, {b, s}) (perf_model.cpp:22-49)
  const Params P = params_from(p.params);
  if (!params_valid(P)) {
    finish(NX_EINVAL);
    return;
  }
  if (lane == 0) {
    p.b = b;
    p.s = s;
    p.n_decode = n_dec;
    p.n_prefill = j;
    p.predicted_ms = predict(P, static_cast<double>(b), static_cast<double>(s));
    p.status = NX_OK;
  }
}

// score_latency / score_load / score_capacity (router.cpp:38-60), one thread
// per (state, demand) query.
__global__ void nx_router_scores_kernel(nx_score_query* __restrict__ q, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  nx_score_query& r = q[i];
  const double knee = r.latency_knee * r.ttft_slo_ms;
  if (r.l_hat_ms <= knee) {
    r.latency = 1.0;
  } else {
    const double scale = r.latency_scale_ms > 0.0 ? r.latency_scale_ms : 0.25 * r.ttft_slo_ms;
    r.latency = exp(-(r.l_hat_ms - knee) / scale);
  }
  r.load = prism_load(r.w_load_tokens, r.p_max, r.load_half_ms);
  if (r.demand_tokens < 1.0) {
    r.status = NX_EINVAL;  // score_capacity: demand must be >= 1 token
    return;
  }
  const double c = r.m_free_tokens / (r.capacity_headroom * r.demand_tokens);
  const double cl = (c < 0.0) ? 0.0 : ((1.0 < c) ? 1.0 : c);
  r.capacity = cl * cl;
  r.status = NX_OK;
}

// TradeoffEstimator::update (lens.cpp:148-188), one warp per estimator: the
// decode-length EMA in completion order, the 200-deep window, and the line
// refit with the reference's left folds (lane 0 folds TTFT, lane 1 TPOT).
__global__ void nx_tradeoff_kernel(nx_tradeoff_state* __restrict__ st, int n,
                                   const nx_completion* __restrict__ comp) {
  const int lane = lane_id();
  const int ei = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (ei >= n) return;
  nx_tradeoff_state& E = st[ei];
  if (lane == 0) {
    for (int k = 0; k < E.n_new; ++k) {
      const nx_completion& c = comp[E.comp_off + k];
      const double lb = E.l_bar + 0.05 * (static_cast<double>(c.decode_len) - E.l_bar);
      E.l_bar = (1.0 < lb) ? lb : 1.0;
      if (c.decode_len >= 2) {
        const int cap = NX_TRADEOFF_WINDOW;
        if (E.win_len < cap) {
          const int slot = (E.win_head + E.win_len) % cap;
          E.win_ttft[slot] = c.ttft_ms;
          E.win_tpot[slot] = c.tpot_ms;
          E.win_len += 1;
        } else {
          E.win_ttft[E.win_head] = c.ttft_ms;
          E.win_tpot[E.win_head] = c.tpot_ms;
          E.win_head = (E.win_head + 1) % cap;
        }
      }
    }
  }
  __syncwarp();
  const int len = E.win_len, head = E.win_head;
  if (len < 2) return;
  double m = 0.0;
  if (lane < 2) {
    const double* src = lane == 0 ? E.win_ttft : E.win_tpot;
    for (int i = 0; i < len; ++i) m += src[(head + i) % NX_TRADEOFF_WINDOW];
  }
  const double dn = static_cast<double>(len);
  const double mtp = __shfl_sync(NX_FULL, m, 0) / dn;
  const double mtd = __shfl_sync(NX_FULL, m, 1) / dn;
  double acc = 0.0;
  if (lane < 2) {
    for (int i = 0; i < len; ++i) {
      const int k = (head + i) % NX_TRADEOFF_WINDOW;
      const double dd = E.win_tpot[k] - mtd;
      acc += lane == 0 ? dd * dd : dd * (E.win_ttft[k] - mtp);
    }
  }
  const double var = __shfl_sync(NX_FULL, acc, 0);
  const double cov = __shfl_sync(NX_FULL, acc, 1);
  if (lane == 0) {
    const double sd = sqrt(var / dn);
    if (sd <= 0.15 * mtd) {
      E.degenerate_updates += 1;
    } else {
      const double slope = cov / var;
      const double nb = -slope;
      E.beta = (1e-3 < nb) ? nb : 1e-3;
      E.alpha_ms = mtp + E.beta * mtd;
    }
  }
}

}  // namespace nxd

extern "C" cudaError_t nx_launch_scalar_ops(int op, void* recs, int n, const void* aux_in,
                                            void* aux_out, cudaStream_t st) {
  using namespace nxd;
  if (n <= 0) return cudaSuccess;
  switch (op) {
    case 0:
      nx_target_kernel<<<(n + 127) / 128, 128, 0, st>>>(static_cast<nx_target_query*>(recs), n);
      break;
    case 1:
      nx_budget_kernel<<<(n + 127) / 128, 128, 0, st>>>(static_cast<nx_budget_query*>(recs), n);
      break;
    case 2:
      nx_allocate_kernel<<<(n + 3) / 4, 128, 0, st>>>(static_cast<nx_allocate_problem*>(recs), n,
                                                      static_cast<const int32_t*>(aux_in),
                                                      static_cast<int32_t*>(aux_out));
      break;
    case 3:
      nx_router_scores_kernel<<<(n + 127) / 128, 128, 0, st>>>(static_cast<nx_score_query*>(recs), n);
      break;
    case 4:
      nx_tradeoff_kernel<<<(n + 3) / 4, 128, 0, st>>>(static_cast<nx_tradeoff_state*>(recs), n,
                                                      static_cast<const nx_completion*>(aux_in));
      break;
    case 5:
      nx_baseline_kernel<<<(n + 3) / 4, 128, 0, st>>>(static_cast<nx_baseline_problem*>(recs), n,
                                                      static_cast<const int32_t*>(aux_in),
                                                      static_cast<int32_t*>(aux_out));
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
