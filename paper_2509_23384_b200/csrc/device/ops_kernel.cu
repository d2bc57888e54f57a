// Batched entry points for the three per-decision operators of the hot path,
// each one warp per independent problem (include/nx_sched.h):
//   K2 nx_lens_kernel   — servesim::schedule_step       (proj/src/lens.cpp:96-146)
//   K3 nx_route_kernel  — servesim::Router::route        (proj/src/router.cpp:141-289)
//   K4 nx_refit_kernel  — OnlineLearner::update_linear / update_structural
//                                                         (proj/src/learner.cpp:300-440)
// They run the same device code as the lockstep simulator (nx_lens.cuh,
// nx_router.cuh, nx_learner.cuh), so the simulator's end-to-end parity and
// these per-operator parity tests pin one implementation.
#include "../../../include/nx_sched.h"
#include "nx_learner.cuh"
#include "nx_lens.cuh"
#include "nx_router.cuh"

namespace nxd {

// ---- K2 ---------------------------------------------------------------------------
constexpr int kLensWarps = 4;      // warps per block
constexpr int kLensPre = 1025;     // shared prefix entries per warp (span <= 1024)
constexpr int kLensMax = 1 << 30;  // device limit on q_max / m_max; prefix saturates here

__device__ __forceinline__ bool lens_cfg_valid(const nx_lens_problem& p) {  // lens.h:70-74
  return p.m_max >= p.q_max && p.q_max >= 1 && p.n_search_iters >= 1 && p.eps_ratio > 0.0 &&
         p.eps_ratio < 1.0 && p.q_ref > 0.0;
}

// kF32: NX_FAST_FP32 (lens_sweep_f32); validation, prefix and allocation are
// the deterministic mode's.
template <bool kF32>
__global__ void __launch_bounds__(32 * kLensWarps) nx_lens_kernel(
    const nx_lens_problem* __restrict__ probs, int n_prob, const int32_t* __restrict__ rem,
    nx_lens_plan* __restrict__ plans, int32_t* __restrict__ alloc, int32_t* __restrict__ gpre) {
  __shared__ int32_t spre[kLensWarps][kLensPre];
  const int lane = lane_id(), wib = threadIdx.x >> 5;
  for (int pi = blockIdx.x * kLensWarps + wib; pi < n_prob; pi += gridDim.x * kLensWarps) {
    const nx_lens_problem& pr = probs[pi];
    nx_lens_plan out;
    out.b = 0; out.s = 0; out.predicted_ms = 0.0; out.target_ms = 0.0;
    out.overload = 0; out.slo_risk = 0; out.n_decode = 0; out.n_prefill = 0;
    out.status = NX_OK; out.pad_ = 0;
    const int R = pr.n_run, W = pr.n_wait;
    const Params P = params_from(pr.params);
    bool risk = false;
    double target = 0.0;
    if (!lens_cfg_valid(pr) || R < 0 || W < 0) {
      out.status = NX_EINVAL;
    } else if (R == 0 && W == 0) {
      // empty queues: empty plan (lens.cpp:101)
    } else if (!(pr.ttft_slo_ms > 0.0 && pr.tpot_slo_ms > 0.0) ||
               !(pr.beta > 0.0 && pr.l_bar >= 1.0 && pr.td_min_ms > 0.0)) {
      out.status = NX_EINVAL;  // target_latency: invalid inputs (lens.cpp:12-14)
    } else if (pr.q_max >= kLensMax || pr.m_max >= kLensMax || !params_valid(P)) {
      out.status = NX_EINVAL;  // device limit / predict_latency's require_valid
    } else {
      target = lens_target(pr.ttft_slo_ms, pr.tpot_slo_ms, pr.alpha_ms, pr.beta, pr.l_bar,
                           pr.td_min_ms, pr.q_ref, W, &risk);
      const int qmax = static_cast<int>(pr.q_max), mmax = static_cast<int>(pr.m_max);
      out.target_ms = target;
      out.slo_risk = risk;
      if (R > qmax) {  // transient overload (lens.cpp:107-117)
        out.b = qmax;
        out.s = qmax;
        if constexpr (kF32) {
          const ParamsF F = params_f32(P);
          const float q = static_cast<float>(qmax);
          out.predicted_ms = latency_fb_f32(F, sat_f32(F.kB, q), q, q);
        } else {
          out.predicted_ms = predict(P, qmax, qmax);
        }
        out.overload = 1;
        out.n_decode = qmax;
      } else if (!(target > 0.0)) {
        out.status = NX_EINVAL;  // binary_search_budget (lens.cpp:36-38)
      } else {
        const int span = ((R + W < qmax) ? R + W : qmax) - R;
        int32_t* pre = span + 1 <= kLensPre ? spre[wib] : gpre + pr.wait_off + pi;
        const int32_t* wr = rem + pr.wait_off;
        // saturating prefix (exact: only comparisons against budgets <= m_max
        // and min(remaining, left) read it)
        __syncwarp();
        if (lane == 0) pre[0] = 0;
        long long carry = 0;
        bool bad = false;
        for (int base = 0; base < span; base += 32) {
          const int i = base + lane;
          const int v = i < span ? wr[i] : 1;
          bad |= v < 1;
          long long s = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long u = __shfl_up_sync(NX_FULL, s, o);
            if (lane >= o) s += u;
          }
          const long long tot = carry + s;
          if (i < span) pre[i + 1] = static_cast<int32_t>(tot < kLensMax ? tot : kLensMax);
          carry += __shfl_sync(NX_FULL, s, 31);
          if (carry > kLensMax) carry = kLensMax;
        }
        __syncwarp();
        if (__any_sync(NX_FULL, bad)) {
          out.status = NX_EINVAL;
        } else {
          const LensPick pick =
              kF32 ? lens_sweep_f32(lane, P, R, span, mmax, pr.n_search_iters, target, pr.eps_ratio, pre)
                   : lens_sweep(lane, P, R, span, mmax, pr.n_search_iters, target, pr.eps_ratio, pre);
          if (pick.budget < 0) {  // every error NaN: the default (empty) BatchPlan
            out.target_ms = 0.0;
          } else {
            const int need = pick.budget - R;
            for (int k = lane; k < pick.j; k += 32) {  // allocate_tokens (lens.cpp:71-77)
              const int rr = pre[k + 1] - pre[k];
              const int left = need - pre[k];
              alloc[pr.wait_off + k] = rr < left ? rr : left;
            }
            out.b = R + pick.j;
            out.s = pick.budget;
            out.predicted_ms = pick.T;
            out.n_decode = R;
            out.n_prefill = pick.j;
          }
        }
      }
    }
    if (out.status != NX_OK) {
      out.b = 0; out.s = 0; out.predicted_ms = 0.0; out.target_ms = 0.0;
      out.overload = 0; out.n_decode = 0; out.n_prefill = 0;
    }
    __syncwarp();
    if (lane == 0) plans[pi] = out;
  }
}

// ---- K3 ---------------------------------------------------------------------------
constexpr int kRouteWarps = 4;
constexpr int kSessionCapacity = 100000;  // Router::kSessionCapacity (router.h:107)

template <bool kF32>  // NX_FAST_FP32: prism_choose_f32 for the PRISM policy
__global__ void __launch_bounds__(32 * kRouteWarps) nx_route_kernel(
    nx_route_group* __restrict__ groups, int n_groups, nx_engine_report* __restrict__ reports,
    const nx_route_request* __restrict__ reqs, int32_t* __restrict__ smap,
    nx_route_decision* __restrict__ dec, int32_t* __restrict__ gstatus) {
  const int lane = lane_id();
  for (int gi = blockIdx.x * kRouteWarps + (threadIdx.x >> 5); gi < n_groups;
       gi += gridDim.x * kRouteWarps) {
    nx_route_group& G = groups[gi];
    const int n = G.n_engines, pol = G.policy;
    int status = NX_OK;
    bool cfg_ok = G.beta_aff > 1.0 && G.latency_knee >= 0.0 && G.latency_scale_ms >= 0.0 &&
                  G.load_half_ms > 0.0 && G.capacity_headroom >= 1.0 && G.staleness_limit_ms > 0.0;
    for (int i = 0; i < 4; ++i) cfg_ok = cfg_ok && G.weights[i] >= 0.0;
    if (n < 1) status = NX_ERUNTIME;  // route: no engines registered (router.cpp:142)
    else if (!cfg_ok || n > 32 || G.n_sessions < 0 || G.n_sessions > kSessionCapacity ||
             !(pol >= 0 && pol <= 5) || (pol == 4 && G.n_requests > 1))
      status = NX_EINVAL;
    if (status != NX_OK) {
      if (lane == 0) gstatus[gi] = status;
      continue;
    }
    nx_engine_report* rows = reports + G.engine_off;
    int32_t* sm = smap + G.session_off;
    EngineView v;
    v.on = lane < n;
    v.has_rep = false;
    v.lhat = v.wload = v.mfree = v.at = 0.0;
    v.pmax = 1.0;
    v.qlen = 0;
    v.id = 0x7fffffff;
    v.affine = false;
    double sw = 0.0, lat = 0.0;
    if (v.on) {
      const nx_engine_report& r = rows[lane];
      v.has_rep = r.has_report != 0;
      v.lhat = r.l_hat_ms;
      v.wload = r.w_load_tokens;
      v.mfree = r.m_free_tokens;
      v.pmax = r.p_max;
      v.at = r.reported_at_ms;
      v.qlen = r.queue_len;
      v.id = r.engine_id;
      sw = r.static_weight;
      lat = r.rolling_latency_ms;
    }
    RouterCfgD rc;
    for (int i = 0; i < 4; ++i) rc.w[i] = G.weights[i];
    rc.beta_aff = G.beta_aff;
    rc.knee = G.latency_knee;
    rc.scale_ms = G.latency_scale_ms;
    rc.load_half = G.load_half_ms;
    rc.headroom = G.capacity_headroom;
    rc.stale_limit = G.staleness_limit_ms;
    rc.ttft_slo = G.ttft_slo_ms;
    const double lbar = G.l_bar_ema;
    uint64_t rr_next = G.rr_next;
    Rng rng;
    for (int i = 0; i < 4; ++i) rng.s[i] = G.rng[i];
    const nx_route_request* q = reqs + G.request_off;
    nx_route_decision* d = dec + G.request_off;
    for (int k = 0; k < G.n_requests; ++k) {
      const nx_route_request rq = q[k];
      if (rq.session < 0 || rq.session >= G.n_sessions) {
        status = NX_EINVAL;
        break;
      }
      const int se = sm[rq.session];
      int chosen = 0;
      nx_route_decision o;
      o.score = 0.0;
      for (int i = 0; i < 4; ++i) o.factors[i] = 1.0;
      o.degraded = 0;
      switch (pol) {
        case 1:  // round_robin (router.cpp:146-148, 126-128)
          chosen = static_cast<int>(rr_next % static_cast<uint64_t>(n));
          ++rr_next;
          break;
        case 2:  // session_affinity (:150-155)
          if (se >= 0 && se < n) {
            chosen = se;
          } else {
            chosen = static_cast<int>(rr_next % static_cast<uint64_t>(n));
            ++rr_next;
          }
          break;
        case 3:  // least_loaded (:157-170)
          chosen = prism_least_loaded(v);
          break;
        case 4: {  // latency_based (:172-184): first strict minimum, NaN never wins
          double best = __builtin_huge_val();
          chosen = 0;
          for (int e = 0; e < n; ++e) {
            const double l = __shfl_sync(NX_FULL, lat, e);
            if (l < best) {
              best = l;
              chosen = e;
            }
          }
          break;
        }
        case 5: {  // weighted draw (:186-203), sequential over lanes on every lane
          double total = 0.0;
          for (int e = 0; e < n; ++e) total += __shfl_sync(NX_FULL, sw, e);
          double draw = rng.uniform() * total;
          chosen = n - 1;
          for (int e = 0; e < n; ++e) {
            draw -= __shfl_sync(NX_FULL, sw, e);
            if (draw <= 0.0) {
              chosen = e;
              break;
            }
          }
          break;
        }
        default: {  // PRISM (:205-284)
          const double dem = static_cast<double>(rq.prompt_len) + lbar;
          const double demand = (1.0 < dem) ? dem : 1.0;
          v.affine = v.on && se == lane;
          const PrismPick pk = kF32 ? prism_choose_f32(rc, v, demand, rq.now_ms, n)
                                    : prism_choose(rc, v, demand, rq.now_ms, n);
          chosen = pk.who;
          o.score = pk.score;
          for (int i = 0; i < 4; ++i) o.factors[i] = pk.f[i];
          o.degraded = pk.degraded;
          if (lane == chosen && v.has_rep) {  // dispatch echo (:275-282)
            v.qlen += 1;
            v.wload += static_cast<double>(rq.prompt_len) + 32.0;
          }
          break;
        }
      }
      o.engine_id = __shfl_sync(NX_FULL, v.id, chosen);
      __syncwarp();
      if (lane == 0) {
        d[k] = o;
        sm[rq.session] = chosen;  // remember_session (router.cpp:107-122)
      }
      __syncwarp();
    }
    if (v.on) {  // the router's report view after the echoes
      rows[lane].queue_len = v.qlen;
      rows[lane].w_load_tokens = v.wload;
    }
    if (lane == 0) {
      G.rr_next = rr_next;
      for (int i = 0; i < 4; ++i) G.rng[i] = rng.s[i];
      gstatus[gi] = status;
    }
    __syncwarp();
  }
}

// ---- K4 ---------------------------------------------------------------------------
// One warp per learner: the simulator's refit code (nx_learner.cuh) runs on a
// one-engine context whose ring is the problem's sample window.
struct RefitSm {
  RepSm rs;
  EngSm eng;
  NxPools pools;
  NxReplicaDesc rep;
  NxEngineDesc ed;
  double chunk[32 * 5];
};

__global__ void __launch_bounds__(32) nx_refit_kernel(int kind, const nx_refit_problem* __restrict__ probs,
                                                      int n_prob, const int32_t* __restrict__ sb,
                                                      const int32_t* __restrict__ ss,
                                                      const double* __restrict__ sy,
                                                      nx_refit_result* __restrict__ out,
                                                      double* __restrict__ scratch, int64_t scratch_per,
                                                      int max_long) {
  __shared__ RefitSm sm;
  const int lane = lane_id();
  double* my_scratch = scratch + static_cast<int64_t>(blockIdx.x) * scratch_per;
  for (int pi = blockIdx.x; pi < n_prob; pi += gridDim.x) {
    const nx_refit_problem& pr = probs[pi];
    nx_refit_result res;
    const Params prior = params_from(pr.params);
    for (int i = 0; i < 8; ++i) res.params[i] = pr.params[i];
    for (int i = 0; i < 7; ++i) res.counters[i] = 0;
    res.updated = 0;
    res.status = NX_OK;
    // LearnerConfig::valid with the periods out of play (learner.h:19-23)
    const bool cfg_ok = pr.long_window > 0 && pr.short_window > 0 && pr.min_structural_samples > 0 &&
                        pr.short_window < pr.long_window && pr.long_window <= max_long &&
                        pr.n_samples >= 0;
    if (!cfg_ok || !params_valid(prior)) {
      res.status = NX_EINVAL;
    } else {
      bool bad = false;  // record_sample's validation (learner.cpp:131-133)
      for (int i = lane; i < pr.n_samples; i += 32) {
        const int b = sb[pr.sample_off + i], s = ss[pr.sample_off + i];
        const double y = sy[pr.sample_off + i];
        bad |= !(y > 0.0) || !(b >= 1 && s >= b);
      }
      if (__any_sync(NX_FULL, bad)) res.status = NX_EINVAL;
    }
    if (res.status == NX_OK) {
      const int W = static_cast<int>(pr.long_window);
      const int n = pr.n_samples;
      const int keep = n < W ? n : W;  // the ring holds the last long_window samples
      __syncwarp();
      if (lane == 0) {
        sm.pools.ring_b = const_cast<int32_t*>(sb);
        sm.pools.ring_s = const_cast<int32_t*>(ss);
        sm.pools.ring_y = const_cast<double*>(sy);
        sm.rep.long_w = W;
        sm.rep.short_w = static_cast<int32_t>(pr.short_window);
        sm.rep.min_s = static_cast<int32_t>(pr.min_structural_samples < 0x7fffffff
                                                ? pr.min_structural_samples : 0x7fffffff);
        sm.ed.ring_off = pr.sample_off + (n - keep);
        for (int i = 0; i < 6; ++i) sm.rs.work[i] = 0;
        for (int i = 0; i < 16; ++i) sm.rs.cycles[i] = 0;
        sm.rs.err[0].status = 0;
        sm.eng.lp = prior;
        sm.eng.ring_size = keep;
        sm.eng.ring_head = 0;
        sm.eng.lp_ver = 0;
        for (int i = 0; i < 7; ++i) sm.eng.cnt[i] = 0;
      }
      __syncwarp();
      Ctx c;
      c.P = &sm.pools;
      c.d = &sm.rep;
      c.ed = &sm.ed;
      c.rs = &sm.rs;
      c.err = &sm.rs.err[0];
      c.inline_refit = 1;
      c.eng = &sm.eng;
      c.chunk = sm.chunk;
      c.prefix = reinterpret_cast<int32_t*>(sm.chunk);
      c.scratch = my_scratch;
      c.lin_rows = my_scratch + 6 * static_cast<int64_t>(W) + kFbTable;
      c.roff = 0;
      c.soff = 0;
      c.n_eng = 1;
      c.n_req = 0;
      c.n_sess = 0;
      c.lane = lane;
      c.prefix_cap = 0;
      c.worker = 0;
      c.log_flags = 0;
      c.team = 1;
      c.fsm = nullptr;  // fit tables in the warp's global scratch
      c.fsm_cap = 0;
      if (kind == NX_REFIT_LINEAR) {
        const bool ok = update_linear(c, 0);
        res.updated = ok;
      } else {
        update_structural(c, 0);
        res.updated = sm.eng.cnt[1] > 0;
      }
      __syncwarp();
      params_to(sm.eng.lp, res.params);
      for (int i = 0; i < 7; ++i) res.counters[i] = sm.eng.cnt[i];
    }
    __syncwarp();
    if (lane == 0) out[pi] = res;
    __syncwarp();
  }
}

}  // namespace nxd

// Scratch doubles one refit warp needs for long_window W (nx_learner.cuh layout).
extern "C" int64_t nx_refit_scratch_per(int64_t W) {
  return nxd::refit_scratch_stride(W);
}

extern "C" cudaError_t nx_launch_lens(const nx_lens_problem* probs, int n, const int32_t* rem,
                                      nx_lens_plan* plans, int32_t* alloc, int32_t* gpre, int sms,
                                      int mode, cudaStream_t st) {
  using namespace nxd;
  int grid = (n + kLensWarps - 1) / kLensWarps;
  const int cap = sms * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (mode == NX_FAST_FP32) nx_lens_kernel<true><<<grid, 32 * kLensWarps, 0, st>>>(probs, n, rem, plans, alloc, gpre);
  else nx_lens_kernel<false><<<grid, 32 * kLensWarps, 0, st>>>(probs, n, rem, plans, alloc, gpre);
  return cudaGetLastError();
}

extern "C" cudaError_t nx_launch_route(nx_route_group* groups, int n, nx_engine_report* reports,
                                       const nx_route_request* reqs, int32_t* smap,
                                       nx_route_decision* dec, int32_t* gstatus, int sms,
                                       int mode, cudaStream_t st) {
  using namespace nxd;
  int grid = (n + kRouteWarps - 1) / kRouteWarps;
  const int cap = sms * 16;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (mode == NX_FAST_FP32) nx_route_kernel<true><<<grid, 32 * kRouteWarps, 0, st>>>(groups, n, reports, reqs, smap, dec, gstatus);
  else nx_route_kernel<false><<<grid, 32 * kRouteWarps, 0, st>>>(groups, n, reports, reqs, smap, dec, gstatus);
  return cudaGetLastError();
}

extern "C" cudaError_t nx_launch_refit(int kind, const nx_refit_problem* probs, int n,
                                       const int32_t* sb, const int32_t* ss, const double* sy,
                                       nx_refit_result* out, double* scratch, int64_t scratch_per,
                                       int grid, int max_long, cudaStream_t st) {
  using namespace nxd;
  nx_refit_kernel<<<grid, 32, 0, st>>>(kind, probs, n, sb, ss, sy, out, scratch, scratch_per, max_long);
  return cudaGetLastError();
}
