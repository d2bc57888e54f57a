// K2 core — LENS budget search (proj/src/lens.cpp:10-146), one warp per
// scheduling decision. Shared by the lockstep simulator (sim_kernel.cu) and
// the batched nx_lens_schedule entry point (ops_kernel.cu).
#pragma once
#include "nx_math.cuh"

namespace nxd {

// target_latency (lens.cpp:10-31). Callers validate SLOSpec / TradeoffModel.
__device__ __forceinline__ double lens_target(double ttft_slo, double tpot_slo, double alpha,
                                              double beta, double l_bar, double td_min, double q_ref,
                                              int64_t wait_count, bool* risk = nullptr) {
  const double td_tpot = tpot_slo;
  const double td_ttft = (alpha - ttft_slo) / beta;
  if (risk) *risk = td_ttft > td_tpot;
  double t;
  if (l_bar > beta) {
    const double lo = (td_min < td_ttft) ? td_ttft : td_min;  // max(td_min, td_ttft)
    t = (lo < td_tpot) ? lo : td_tpot;                        // min(td_tpot, .)
  } else {
    t = td_tpot;
  }
  if (wait_count > 0) {
    const double q = static_cast<double>(wait_count) / q_ref;
    const double relax = (q < 1.0) ? q : 1.0;
    t += relax * (td_tpot - t);
  }
  return t;
}

// Inclusive prefix sums of the remaining prompts of the first `count`
// waiters into pre[0..count] (pre[0] = 0; lens.cpp:121-124). rem(i) yields
// waiter i's remaining prompt.
template <class Rem>
__device__ __forceinline__ void lens_prefix(int lane, int32_t* pre, int count, Rem rem) {
  __syncwarp();
  if (lane == 0) pre[0] = 0;
  int carry = 0;
  for (int base = 0; base < count; base += 32) {
    const int i = base + lane;
    const int v = i < count ? rem(i) : 0;
    const int s = warp_incl_scan(v);
    if (i < count) pre[i + 1] = carry + s;
    carry += __shfl_sync(NX_FULL, s, 31);
  }
  __syncwarp();
}

// first j in [0, hi] with pre[j] >= need (pre non-decreasing)
__device__ __forceinline__ int lens_lower_bound(const int32_t* pre, int hi, int need) {
  int lo = 0;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (pre[m] >= need) hi = m;
    else lo = m + 1;
  }
  return lo;
}

struct LensPick {
  int budget;   // chosen token budget S (-1: every candidate error was NaN)
  int j;        // waiters admitted (allocate_tokens prefix length)
  double T;     // predicted latency of the realized plan
};

// The candidate sweep of schedule_step (lens.cpp:126-145) for R running and
// `span` = min(R + W, q_max) - R schedulable waiters with prefix sums `pre`.
// Each lane owns one candidate batch size B and runs binary_search_budget's
// probe sequence (lens.cpp:33-56) with f_B hoisted; the realized plan of a
// budget is S = budget, b = R + first j with pre[j] >= budget - R (every
// waiter takes min(remaining, budget left)). Selection is
// the sequential loop's: the first B with error < eps*target, else the
// first strict minimum (NaN never wins).
__device__ __forceinline__ LensPick lens_sweep(int lane, const Params& P, int R, int span, int mmax,
                                               int iters, double target, double eps_ratio,
                                               const int32_t* pre) {
  const int b_lo = R > 1 ? R : 1;
  const int b_hi = R + span;
  const double thr_eps = target * eps_ratio;
  double best_err = __builtin_huge_val(), best_T = 0.0;
  int best_budget = -1;
  for (int B0 = b_lo; B0 <= b_hi; B0 += 32) {
    const int B = B0 + lane;
    const bool act = B <= b_hi;
    double err = __builtin_huge_val(), T = 0.0;
    int budget = 0;
    if (act) {
      const int avail = R + pre[B - R];
      int s_cap = (mmax < avail) ? mmax : avail;
      s_cap = (B < s_cap) ? s_cap : B;  // max(b, min(s_cap, m_max))
      const double bd = static_cast<double>(B);
      const double fb = sat(P.kB, bd);
      int lo = B, hi = s_cap;
      budget = B;
      for (int it = 0; it < iters; ++it) {  // binary_search_budget (lens.cpp:46-55)
        if (lo > hi) break;
        const int mid = lo + (hi - lo) / 2;
        if (latency_fb(P, fb, bd, static_cast<double>(mid)) <= target) {
          budget = mid;
          lo = mid + 1;
        } else {
          hi = mid - 1;
        }
      }
      const int j = lens_lower_bound(pre, B - R, budget - R);
      T = predict(P, static_cast<double>(R + j), static_cast<double>(budget));
      err = fabs(T - target);
    }
    const unsigned hit = __ballot_sync(NX_FULL, act && err < thr_eps);
    if (hit) {
      best_budget = __shfl_sync(NX_FULL, budget, __ffs(hit) - 1);
      best_T = __shfl_sync(NX_FULL, T, __ffs(hit) - 1);
      break;
    }
    double v = (act && !isnan(err)) ? err : __builtin_huge_val();
    int who = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(NX_FULL, v, o);
      const int ow = __shfl_xor_sync(NX_FULL, who, o);
      if (ov < v || (ov == v && ow < who)) {
        v = ov;
        who = ow;
      }
    }
    const int wb = __shfl_sync(NX_FULL, budget, who & 31);
    const double wT = __shfl_sync(NX_FULL, T, who & 31);
    if (v < best_err) {
      best_err = v;
      best_budget = wb;
      best_T = wT;
    }
  }
  LensPick pick;
  pick.budget = best_budget;
  pick.T = best_T;
  pick.j = best_budget >= 0 ? lens_lower_bound(pre, span, best_budget - R) : 0;
  return pick;
}

// ---- NX_FAST_FP32 (include/nx_sched.h) --------------------------------------
// The same sweep with every probe in float: f_B, f_S, the predicted latency
// and the error. Decisions follow the fp32 arithmetic (they can differ from
// the deterministic mode where two candidates or a probe and the target lie
// within float rounding of each other); predicted latencies are within 1e-4
// relative of the fp64 model for the plan chosen. Used by the batched K2
// entry point only; the simulator always runs the deterministic sweep.
struct ParamsF {
  float tau0, w0, ws, tauB, tauS, p_max, kB, kS;
};
__device__ __forceinline__ ParamsF params_f32(const Params& p) {
  ParamsF f;
  f.tau0 = static_cast<float>(p.tau0); f.w0 = static_cast<float>(p.w0); f.ws = static_cast<float>(p.ws);
  f.tauB = static_cast<float>(p.tauB); f.tauS = static_cast<float>(p.tauS);
  f.p_max = static_cast<float>(p.p_max); f.kB = static_cast<float>(p.kB); f.kS = static_cast<float>(p.kS);
  return f;
}
__device__ __forceinline__ float sat_f32(float k, float x) {
  return fminf(-expm1f(-k * x), 0x1.fffffep-1f);
}
__device__ __forceinline__ float latency_fb_f32(const ParamsF& p, float fb, float b, float s) {
  const float thr = p.p_max * fb * sat_f32(p.kS, s);
  return p.tau0 + (p.w0 + p.ws * s) / thr + p.tauB * b + p.tauS * s;
}

__device__ __forceinline__ LensPick lens_sweep_f32(int lane, const Params& P64, int R, int span, int mmax,
                                                   int iters, double target64, double eps_ratio,
                                                   const int32_t* pre) {
  const ParamsF P = params_f32(P64);
  const float target = static_cast<float>(target64);
  const int b_lo = R > 1 ? R : 1;
  const int b_hi = R + span;
  const float thr_eps = static_cast<float>(target64 * eps_ratio);
  float best_err = __builtin_huge_valf(), best_T = 0.0f;
  int best_budget = -1;
  for (int B0 = b_lo; B0 <= b_hi; B0 += 32) {
    const int B = B0 + lane;
    const bool act = B <= b_hi;
    float err = __builtin_huge_valf(), T = 0.0f;
    int budget = 0;
    if (act) {
      const int avail = R + pre[B - R];
      int s_cap = (mmax < avail) ? mmax : avail;
      s_cap = (B < s_cap) ? s_cap : B;
      const float bd = static_cast<float>(B);
      const float fb = sat_f32(P.kB, bd);
      int lo = B, hi = s_cap;
      budget = B;
      for (int it = 0; it < iters; ++it) {
        if (lo > hi) break;
        const int mid = lo + (hi - lo) / 2;
        if (latency_fb_f32(P, fb, bd, static_cast<float>(mid)) <= target) {
          budget = mid;
          lo = mid + 1;
        } else {
          hi = mid - 1;
        }
      }
      const int j = lens_lower_bound(pre, B - R, budget - R);
      const float bj = static_cast<float>(R + j);
      T = latency_fb_f32(P, sat_f32(P.kB, bj), bj, static_cast<float>(budget));
      err = fabsf(T - target);
    }
    const unsigned hit = __ballot_sync(NX_FULL, act && err < thr_eps);
    if (hit) {
      best_budget = __shfl_sync(NX_FULL, budget, __ffs(hit) - 1);
      best_T = __shfl_sync(NX_FULL, T, __ffs(hit) - 1);
      break;
    }
    float v = (act && !isnan(err)) ? err : __builtin_huge_valf();
    int who = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(NX_FULL, v, o);
      const int ow = __shfl_xor_sync(NX_FULL, who, o);
      if (ov < v || (ov == v && ow < who)) {
        v = ov;
        who = ow;
      }
    }
    const int wb = __shfl_sync(NX_FULL, budget, who & 31);
    const float wT = __shfl_sync(NX_FULL, T, who & 31);
    if (v < best_err) {
      best_err = v;
      best_budget = wb;
      best_T = wT;
    }
  }
  LensPick pick;
  pick.budget = best_budget;
  pick.T = static_cast<double>(best_T);
  pick.j = best_budget >= 0 ? lens_lower_bound(pre, span, best_budget - R) : 0;
  return pick;
}

}  // namespace nxd
