// K7 — device-side metrics summary of every replica's completion records
// (servesim::summarize, proj/src/metrics.cpp:40-91; the "metrics" and
// "engine_share" blocks of sim.cpp:349-392's summary JSON).
//
// One CTA per replica, after the simulation kernel on the same stream:
//   * per record (in completion order, the reference's records_ order):
//     ttft = first - arrival, e2e = done - arrival, tpot = (done - first) /
//     (output - 1) for multi-token requests (metrics.cpp:7-26), the SLO pass
//     test, per-engine counts — the same double operations as the host code;
//   * the two means are the reference's left folds in record order (one
//     thread: they are order-sensitive);
//   * the nearest-rank percentiles (metrics.cpp:29-38) are order statistics:
//     an 8-pass radix select on the values' bit patterns (non-negative
//     doubles order like their bits) — no sort, O(n) per percentile.
// Results are bitwise the host restatement's (csrc/host/report.cpp), which is
// the reference's; tests/test_summary_gpu.py compares them.
#include <stdint.h>

#include "../nx_layout.h"

namespace nxs {

constexpr int kThreads = 256;

__device__ __forceinline__ double to_ms(int64_t us) { return static_cast<double>(us) / 1000.0; }

// k-th smallest (0-based) of v[0, n) by the bit patterns (all v >= 0).
__device__ double select_kth(const double* v, int n, int k, unsigned* hist) {
  unsigned long long prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v[i]));
      if ((b & mask) == prefix) atomicAdd(&hist[(b >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    // the bin holding rank k (every thread scans the 256 counts)
    unsigned below = 0;
    int bin = 255;
    for (int d = 0; d < 256; ++d) {
      if (static_cast<int>(below + hist[d]) > k) {
        bin = d;
        break;
      }
      below += hist[d];
    }
    k -= static_cast<int>(below);
    prefix |= static_cast<unsigned long long>(bin) << shift;
    mask |= 0xffull << shift;
    __syncthreads();
  }
  return __longlong_as_double(static_cast<long long>(prefix));
}

// nearest-rank index of percentile p over n values (metrics.cpp:35-37)
__device__ __forceinline__ int rank_index(double p, int n) {
  const double r = ceil(p / 100.0 * static_cast<double>(n));
  const long long k = static_cast<long long>(r);
  return static_cast<int>((k < 1 ? 1 : k) - 1);
}

__global__ void __launch_bounds__(kThreads) nx_summarize_kernel(const NxPools* __restrict__ pools,
                                                                double* __restrict__ work) {
  const int r = blockIdx.x;
  const NxPools& P = *pools;
  const NxReplicaDesc& d = P.rep[r];
  NxReplicaMetrics& out = P.metrics[r];
  const NxReplicaOut& ro = P.rep_out[r];
  __shared__ unsigned hist[256];
  __shared__ int s_pass, s_bad, s_ntpot;
  __shared__ int s_cnt[NX_MAX_ENGINES];
  const int n = static_cast<int>(ro.completed);
  if (threadIdx.x == 0) {
    s_pass = 0;
    s_bad = 0;
    s_ntpot = 0;
  }
  for (int e = threadIdx.x; e < NX_MAX_ENGINES; e += blockDim.x) s_cnt[e] = 0;
  __syncthreads();
  if (ro.status != 0 || n == 0) {  // no summary (failed) / empty (metrics.cpp:45-46)
    if (threadIdx.x == 0) {
      out.completed = n;
      out.valid = ro.status == 0;
      out.p50_e2e = out.p90_e2e = out.p50_ttft = out.p50_tpot = 0.0;
      out.mean_ttft = out.mean_tpot = 0.0;
      out.slo_pct = 100.0;
      out.n_tpot = 0;
      for (int e = 0; e < NX_MAX_ENGINES; ++e) out.engine_count[e] = 0;
    }
    return;
  }
  double* e2e = work + 4 * d.req_off;  // record order (4 doubles per request of the replica)
  double* ttft = e2e + n;
  double* tpot = ttft + n;       // record order, single-token requests excluded later
  double* tpot_c = tpot + n;     // compacted multi-token tpot values (selection input)
  const int64_t ro_off = d.req_off;
  int pass = 0, bad = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int rid = P.records[ro_off + k];
    const double arr = P.arr_ms[ro_off + rid];
    const double first = to_ms(P.first_us[ro_off + rid]);
    const double done = to_ms(P.done_us[ro_off + rid]);
    const int out_tok = P.req0[ro_off + rid].target;
    if (!(arr <= first && first <= done)) bad = 1;  // metrics.cpp:13-16
    const double t = first - arr;
    const double e = done - arr;
    const bool single = out_tok < 2;
    const double tp = single ? 0.0 : (done - first) / static_cast<double>(out_tok - 1);
    e2e[k] = e;
    ttft[k] = t;
    tpot[k] = single ? -1.0 : tp;  // -1: excluded (all real values are >= 0)
    if (t <= d.ttft_slo && (single || tp <= d.tpot_slo)) ++pass;
    atomicAdd(&s_cnt[P.req_engine[ro_off + rid]], 1);
  }
  if (pass) atomicAdd(&s_pass, pass);
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  // left folds in record order, and the compacted tpot values (same order)
  __shared__ double s_mean_ttft, s_mean_tpot;
  if (threadIdx.x == 0) {
    double ts = 0.0, ps = 0.0;
    int m = 0;
    for (int k = 0; k < n; ++k) {
      ts += ttft[k];
      if (tpot[k] >= 0.0) {
        ps += tpot[k];
        tpot_c[m++] = tpot[k];
      }
    }
    s_mean_ttft = ts / static_cast<double>(n);
    s_mean_tpot = m ? ps / static_cast<double>(m) : 0.0;
    s_ntpot = m;
  }
  __syncthreads();
  const int m = s_ntpot;
  const double p50_e2e = select_kth(e2e, n, rank_index(50.0, n), hist);
  const double p90_e2e = select_kth(e2e, n, rank_index(90.0, n), hist);
  const double p50_ttft = select_kth(ttft, n, rank_index(50.0, n), hist);
  const double p50_tpot = m ? select_kth(tpot_c, m, rank_index(50.0, m), hist) : 0.0;
  if (threadIdx.x == 0) {
    out.completed = n;
    out.valid = s_bad ? 0 : 1;
    out.p50_e2e = p50_e2e;
    out.p90_e2e = p90_e2e;
    out.p50_ttft = p50_ttft;
    out.p50_tpot = p50_tpot;
    out.mean_ttft = s_mean_ttft;
    out.mean_tpot = s_mean_tpot;
    out.slo_pct = 100.0 * static_cast<double>(s_pass) / static_cast<double>(n);
    out.n_tpot = m;
    for (int e = 0; e < NX_MAX_ENGINES; ++e) out.engine_count[e] = s_cnt[e];
  }
}

}  // namespace nxs

extern "C" cudaError_t nx_launch_summarize(const NxPools* d_pools, int n_rep, double* work, cudaStream_t st) {
  nxs::nx_summarize_kernel<<<n_rep, nxs::kThreads, 0, st>>>(d_pools, work);
  return cudaGetLastError();
}
