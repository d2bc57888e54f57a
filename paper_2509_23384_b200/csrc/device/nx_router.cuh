// K3 core — PRISM multiplicative score (proj/src/router.cpp:38-60, 205-273),
// one warp per routing decision, lane e = the e-th registered engine.
// Shared by the lockstep simulator (sim_kernel.cu) and the batched
// nx_prism_route entry point (ops_kernel.cu).
#pragma once
#include "nx_math.cuh"

namespace nxd {

struct RouterCfgD {  // RouterConfig (router.h:31-52) + SLOSpec::ttft_slo_ms
  double w[4], beta_aff, knee, scale_ms, load_half, headroom, stale_limit, ttft_slo;
};

struct EngineView {  // the router's copy of one engine's latest report
  bool on;           // lane holds a registered engine
  bool has_rep;
  double lhat, wload, mfree, pmax, at;
  int64_t qlen;
  int id;            // engine id (registration order = lane order)
  bool affine;       // the request's session was last routed here
};

struct PrismPick {
  int who;           // chosen lane
  double score, f[4];
  bool degraded;
};

// score_load (router.cpp:47-50)
__device__ __forceinline__ double prism_load(double w_load, double p_max, double half) {
  const double rho = w_load / p_max;
  return 1.0 / (1.0 + rho / half);
}

// Least known load (router.cpp:158-170, 259-271): first minimum of the
// reported queue length in registration order (no report counts as 0).
__device__ __forceinline__ int prism_least_loaded(const EngineView& v) {
  int64_t len = v.on ? (v.has_rep ? v.qlen : 0) : INT64_MAX;
  int who = v.on ? lane_id() : 64;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t ol = __shfl_xor_sync(NX_FULL, len, o);
    const int ow = __shfl_xor_sync(NX_FULL, who, o);
    if (ol < len || (ol == len && ow < who)) {
      len = ol;
      who = ow;
    }
  }
  return who;
}

// Router::route, kPrism (router.cpp:205-273) without the echo: each lane
// scores its engine, then the sequential scan's "better" fold runs over the
// lanes in registration order (exactly the reference's order, NaN included).
__device__ __forceinline__ PrismPick prism_choose(const RouterCfgD& cfg, const EngineView& v,
                                                  double demand, double now, int n) {
  double f[4] = {1.0, 1.0, 1.0, 1.0};
  double rho = 0.0, score = 0.0;
  bool fresh = false;
  if (v.on) {
    const double age = v.has_rep ? now - v.at : __builtin_huge_val();
    if (v.has_rep && age <= cfg.stale_limit) {
      fresh = true;
      const double knee = cfg.knee * cfg.ttft_slo;  // score_latency (router.cpp:38-45)
      if (v.lhat <= knee) {
        f[0] = 1.0;
      } else {
        const double scale = cfg.scale_ms > 0.0 ? cfg.scale_ms : 0.25 * cfg.ttft_slo;
        f[0] = exp(-(v.lhat - knee) / scale);
      }
      f[1] = prism_load(v.wload, v.pmax, cfg.load_half);
      const double r = v.mfree / (cfg.headroom * demand);  // score_capacity (:52-60)
      const double cl = (r < 0.0) ? 0.0 : ((1.0 < r) ? 1.0 : r);
      f[2] = cl * cl;
      rho = v.wload / v.pmax;
    } else {  // graceful degradation (router.cpp:226-236)
      f[0] = 0.5;
      f[2] = 0.5;
      if (v.has_rep) {
        rho = v.wload / v.pmax;
        const double blend = exp(-(age - cfg.stale_limit) / cfg.stale_limit);
        f[1] = 1.0 + (prism_load(v.wload, v.pmax, cfg.load_half) - 1.0) * blend;
      }
    }
    f[3] = v.affine ? cfg.beta_aff : 1.0;  // score_affinity (router.cpp:94-101)
    score = 1.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double w = cfg.w[i];
      double term;
      if (f[i] == 0.0 && w > 0.0) term = 0.0;
      else if (w == 1.0) term = f[i];  // pow(x, 1) == x exactly
      else if (w == 0.0) term = 1.0;   // pow(x, 0) == 1, NaN included
      else term = pow(f[i], w);
      score *= term;
    }
  }
  // sequential "better" scan (router.cpp:246-257)
  double best_s = -1.0, best_rho = __builtin_huge_val();
  int best = -1, best_id = -1;
  for (int e = 0; e < n; ++e) {
    const double s = __shfl_sync(NX_FULL, score, e);
    const double r = __shfl_sync(NX_FULL, rho, e);
    const int id = __shfl_sync(NX_FULL, v.id, e);
    const bool better = s > best_s || (s == best_s && (r < best_rho || (r == best_rho && id < best_id)));
    if (best < 0 || better) {
      best_s = s;
      best_rho = r;
      best = e;
      best_id = id;
    }
  }
  PrismPick p;
  p.who = best;
  p.score = best_s;
#pragma unroll
  for (int i = 0; i < 4; ++i) p.f[i] = __shfl_sync(NX_FULL, f[i], best);
  p.degraded = !__any_sync(NX_FULL, fresh);
  if (p.degraded) p.who = prism_least_loaded(v);
  return p;
}

// NX_FAST_FP32 (include/nx_sched.h): prism_choose with the per-engine score,
// its factors and the load ratio in float (expf / powf), and the "better"
// scan over the float scores. Choices can differ from the deterministic mode
// where two engines' scores lie within float rounding; scores and factors are
// within ~1e-6 relative of the fp64 ones. Batched K3 entry point only.
__device__ __forceinline__ PrismPick prism_choose_f32(const RouterCfgD& cfg, const EngineView& v,
                                                      double demand, double now, int n) {
  float f[4] = {1.0f, 1.0f, 1.0f, 1.0f};
  float rho = 0.0f, score = 0.0f;
  bool fresh = false;
  if (v.on) {
    const float age = v.has_rep ? static_cast<float>(now - v.at) : __builtin_huge_valf();
    const float stale = static_cast<float>(cfg.stale_limit), ttft = static_cast<float>(cfg.ttft_slo);
    const float wl = static_cast<float>(v.wload), pm = static_cast<float>(v.pmax);
    const float half = static_cast<float>(cfg.load_half);
    if (v.has_rep && age <= stale) {
      fresh = true;
      const float knee = static_cast<float>(cfg.knee) * ttft;
      const float lh = static_cast<float>(v.lhat);
      if (lh <= knee) {
        f[0] = 1.0f;
      } else {
        const float scale = cfg.scale_ms > 0.0 ? static_cast<float>(cfg.scale_ms) : 0.25f * ttft;
        f[0] = expf(-(lh - knee) / scale);
      }
      f[1] = 1.0f / (1.0f + (wl / pm) / half);
      const float r = static_cast<float>(v.mfree) / (static_cast<float>(cfg.headroom) * static_cast<float>(demand));
      const float cl = (r < 0.0f) ? 0.0f : ((1.0f < r) ? 1.0f : r);
      f[2] = cl * cl;
      rho = wl / pm;
    } else {
      f[0] = 0.5f;
      f[2] = 0.5f;
      if (v.has_rep) {
        rho = wl / pm;
        const float blend = expf(-(age - stale) / stale);
        f[1] = 1.0f + (1.0f / (1.0f + rho / half) - 1.0f) * blend;
      }
    }
    f[3] = v.affine ? static_cast<float>(cfg.beta_aff) : 1.0f;
    score = 1.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float w = static_cast<float>(cfg.w[i]);
      float term;
      if (f[i] == 0.0f && w > 0.0f) term = 0.0f;
      else if (w == 1.0f) term = f[i];
      else if (w == 0.0f) term = 1.0f;
      else term = powf(f[i], w);
      score *= term;
    }
  }
  float best_s = -1.0f, best_rho = __builtin_huge_valf();
  int best = -1, best_id = -1;
  for (int e = 0; e < n; ++e) {
    const float s = __shfl_sync(NX_FULL, score, e);
    const float r = __shfl_sync(NX_FULL, rho, e);
    const int id = __shfl_sync(NX_FULL, v.id, e);
    const bool better = s > best_s || (s == best_s && (r < best_rho || (r == best_rho && id < best_id)));
    if (best < 0 || better) {
      best_s = s;
      best_rho = r;
      best = e;
      best_id = id;
    }
  }
  PrismPick p;
  p.who = best;
  p.score = best_s;
#pragma unroll
  for (int i = 0; i < 4; ++i) p.f[i] = __shfl_sync(NX_FULL, f[i], best);
  p.degraded = !__any_sync(NX_FULL, fresh);
  if (p.degraded) p.who = prism_least_loaded(v);
  return p;
}

}  // namespace nxd
