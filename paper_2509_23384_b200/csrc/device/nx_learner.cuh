// K4 — online coefficient refit, one warp per engine update.
//
// Replaces OnlineLearner (proj/src/learner.cpp:130-440). Reduction orders:
//  * coefficients a learner adopts come from normal equations (15 unique
//    A^T A entries + 5 A^T b) folded in the reference's left-to-right sample
//    order, one accumulator per lane over 32-sample chunks staged in shared
//    memory — the linear tier always, the structural tier for its winning
//    (kB, kS) (exact_elem) — so they are the reference's bit for bit (modulo
//    libm ulps);
//  * the structural search ranks its ~50-100 candidate fits on fast sums
//    (team passes, grouped per-batch-size / per-token-count aggregates), and
//    the squared-error sums (ridge scale, windowed SSE) are fixed-order warp
//    trees; every decision they drive (lambda cap, accept/reject, rank test)
//    is certified against an explicit rounding bound and, if it falls inside,
//    re-taken on the exact left fold. Decisions therefore equal the
//    reference's left-fold decisions.
#pragma once
#include "nx_state.cuh"
#ifdef NX_TRACE_FIT
#include <cstdio>
#endif

namespace nxd {


// ---- 5x5 elimination (learner.cpp:24-60) -------------------------------------
__device__ __forceinline__ double dmax(double m, double v) { return (m < v) ? v : m; }

// Warp-parallel form of solve5: lane 5i+j (< 25) holds a[i][j], lane 25+i holds
// b[i]. Every element sees exactly the serial algorithm's operations in the
// same order (scaling, pivot choice, row swap, elimination, back
// substitution), so the result is bitwise identical — without the serial
// version's 5x5 register arrays (which spilled) or its dependent loops.
__device__ __forceinline__ double pick5(const double v[5], int k) {
  double r = v[0];
#pragma unroll
  for (int q = 1; q < 5; ++q)
    if (k == q) r = v[q];
  return r;
}

// K independent systems in lockstep: their shuffle and division latencies
// overlap. ok[k] reports each system's rank test separately.
// Inline, with the column loop rolled (a ~4k-instruction fully unrolled body
// streamed through the instruction cache once per fit). Out of line it cost
// 10k cycles per call: shuffles in a non-inlined function compile to
// WARPSYNC/ENDCOLLECTIVE sequences, and the array arguments go to the stack.
// amb[k]: some pivot the rank test looked at lies within [0.5, 2] x its
// threshold 1e-10 * norm — a decision that rounding in the inputs could flip
// (entries accurate to ~n u relative move a pivot by ~1e-11 norm at most).
template <int K>
__device__ __forceinline__ void solve5_warp_k(double (&v)[K], double (&x)[K][5], bool (&ok)[K], bool (&amb)[K]) {
  const int lane = lane_id();
  const bool isA = lane < 25;
  const int i = isA ? lane / 5 : (lane < 30 ? lane - 25 : 0);
  const int j = isA ? lane % 5 : 5;
  double sc[K][5], norm[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double m = 0.0;
#pragma unroll
    for (int r = 0; r < 5; ++r)
      m = dmax(m, fabs(__shfl_sync(NX_FULL, v[k], r * 5 + (j < 5 ? j : 0))));
    ok[k] = !__any_sync(NX_FULL, isA && i == 0 && m <= 0.0);
    amb[k] = false;
    const double scale = (isA && m > 0.0) ? 1.0 / m : 1.0;
    if (isA) v[k] *= scale;
#pragma unroll
    for (int q = 0; q < 5; ++q) sc[k][q] = __shfl_sync(NX_FULL, scale, q);
    double nm = isA ? fabs(v[k]) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nm = dmax(nm, __shfl_xor_sync(NX_FULL, nm, o));
    norm[k] = nm;
  }
#pragma unroll 1
  for (int col = 0; col < 5; ++col) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double cv[5];
#pragma unroll
      for (int r = 0; r < 5; ++r) cv[r] = fabs(__shfl_sync(NX_FULL, v[k], r * 5 + col));
      int piv = col;
      double pv = 0.0;
#pragma unroll
      for (int r = 0; r < 5; ++r)
        if (r == col) pv = cv[r];
#pragma unroll
      for (int r = 1; r < 5; ++r)  // first strict maximum below the diagonal
        if (r > col && cv[r] > pv) {
          piv = r;
          pv = cv[r];
        }
      if (ok[k] && pv < 2e-10 * norm[k] && !(pv < 5e-11 * norm[k])) amb[k] = true;
      if (pv < 1e-10 * norm[k]) ok[k] = false;
      int src = lane;
      if (lane < 30) {
        const int base = isA ? 0 : 25, stride = isA ? 5 : 1, off = isA ? j : 0;
        if (i == col) src = base + piv * stride + off;
        else if (i == piv) src = base + col * stride + off;
      }
      v[k] = __shfl_sync(NX_FULL, v[k], src);
      const double diag = __shfl_sync(NX_FULL, v[k], col * 5 + col);
      const double pivrow = __shfl_sync(NX_FULL, v[k], isA ? col * 5 + j : 25 + col);
      const double arc = __shfl_sync(NX_FULL, v[k], i * 5 + col);
      if (lane < 30 && i > col && j >= col) {
        const double f = arc / diag;
        v[k] -= f * pivrow;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double u[5][5], bb[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
#pragma unroll
      for (int q = r; q < 5; ++q) u[r][q] = __shfl_sync(NX_FULL, v[k], r * 5 + q);
      bb[r] = __shfl_sync(NX_FULL, v[k], 25 + r);
    }
#pragma unroll
    for (int r = 4; r >= 0; --r) {
      double acc = bb[r];
#pragma unroll
      for (int q = r + 1; q < 5; ++q) acc -= u[r][q] * x[k][q];
      x[k][r] = acc / u[r][r];
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) x[k][q] *= sc[k][q];
  }
}

template <int K>
__device__ __forceinline__ void solve5_warp_k(double (&v)[K], double (&x)[K][5], bool (&ok)[K]) {
  bool amb[K];
  solve5_warp_k<K>(v, x, ok, amb);
}

__device__ __forceinline__ bool solve5_warp(double v, double x[5], bool* ambiguous = nullptr) {
  double vv[1] = {v};
  double xx[1][5];
  bool ok[1], amb[1];
  solve5_warp_k<1>(vv, xx, ok, amb);
#pragma unroll
  for (int q = 0; q < 5; ++q) x[q] = xx[0][q];
  if (ambiguous && amb[0]) *ambiguous = true;
  return ok[0];
}

// lane -> (i, j) of the 15 unique A^T A entries; lanes 15..19 own A^T b[i].
// (3-bit fields of two constants: a local-array table here was stored to and
// reloaded from local memory on every call.)
__device__ __forceinline__ void acc_slot(int lane, int& i, int& j) {
  constexpr unsigned long long kTi = 0ull | 0ull << 3 | 0ull << 6 | 0ull << 9 | 0ull << 12 | 1ull << 15 |
                                     1ull << 18 | 1ull << 21 | 1ull << 24 | 2ull << 27 | 2ull << 30 |
                                     2ull << 33 | 3ull << 36 | 3ull << 39 | 4ull << 42;
  constexpr unsigned long long kTj = 0ull | 1ull << 3 | 2ull << 6 | 3ull << 9 | 4ull << 12 | 1ull << 15 |
                                     2ull << 18 | 3ull << 21 | 4ull << 24 | 2ull << 27 | 3ull << 30 |
                                     4ull << 33 | 3ull << 36 | 4ull << 39 | 4ull << 42;
  if (lane < 15) {
    i = static_cast<int>((kTi >> (3 * lane)) & 7ull);
    j = static_cast<int>((kTj >> (3 * lane)) & 7ull);
  } else {
    i = lane - 15;
    j = -1;
  }
}
__device__ __forceinline__ int slot_of(int i, int j) {
  if (i > j) { const int t = i; i = j; j = t; }
  // row-major upper triangle: offset(i) = 5i - i(i-1)/2
  return 5 * i - (i * (i - 1)) / 2 + (j - i);
}

// Folds the 32-sample chunk staged in c.chunk (cnt rows of 5 scaled values)
// into this lane's accumulator, in sample order.
__device__ __forceinline__ void fold_chunk(const Ctx& c, int cnt, double& acc) {
  int i, j;
  acc_slot(c.lane, i, j);
  if (c.lane < 15) {
    for (int k = 0; k < cnt; ++k) acc += c.chunk[k * 5 + i] * c.chunk[k * 5 + j];
  } else if (c.lane < 20) {
    for (int k = 0; k < cnt; ++k) acc += c.chunk[k * 5 + i] * 1.0;
  }
}


// Lane element of the normal equations from the 15 unique A^T A entries
// (slot_of order) and the 5 A^T b entries.
__device__ __forceinline__ double normal_elem(const double u15[15], const double t5[5]) {
  const int lane = lane_id();
  double e = 0.0;
  if (lane < 25) {
    const int k = slot_of(lane / 5, lane % 5);
#pragma unroll
    for (int q = 0; q < 15; ++q)
      if (k == q) e = u15[q];
  } else if (lane < 30) {
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (lane - 25 == q) e = t5[q];
  }
  return e;
}

// Ridge anchored at `prior` (learner.cpp:86-93): a[i][i] += lambda a[i][i],
// b[i] += (lambda a[i][i]) prior[i].
__device__ __forceinline__ double ridge_elem(double e, double lambda, const double prior[5]) {
  const int lane = lane_id();
  const int src = (lane >= 25 && lane < 30) ? (lane - 25) * 6 : lane;
  const double diag = __shfl_sync(NX_FULL, e, src);
  if (lane < 25 && lane % 6 == 0) return e + lambda * e;
  if (lane >= 25 && lane < 30) return e + (lambda * diag) * pick5(prior, lane - 25);
  return e;
}

// Exact left fold of per-lane values v (valid where `on`) in index order,
// called once per 32-sample chunk; running total lives in lane 0's `run`.
__device__ __forceinline__ void fold_exact_chunk(Ctx& c, double v, int cnt, double& run) {
  __syncwarp();
  c.chunk[c.lane] = v;
  __syncwarp();
  if (c.lane == 0)
    for (int k = 0; k < cnt; ++k) run += c.chunk[k];
  __syncwarp();
}

struct Window {
  const int32_t* rb;
  const int32_t* rs;
  const double* ry;
  int size, head, n;
  __device__ __forceinline__ int slot(int i) const {
    const int k = head + size - n + i;  // < 2 * size
    return k >= size ? k - size : k;
  }
};

__device__ __forceinline__ Window window_of(const Ctx& c, int e, int n_want) {
  const NxEngineDesc& ed = c.ed[e];
  const EngSm& g = c.eng[e];
  Window w;
  w.rb = c.P->ring_b + ed.ring_off;
  w.rs = c.P->ring_s + ed.ring_off;
  w.ry = c.P->ring_y + ed.ring_off;
  w.size = g.ring_size;
  w.head = g.ring_head;
  w.n = n_want < w.size ? n_want : w.size;
  return w;
}

// ---- linear tier (learner.cpp:160-207, 300-344) ------------------------------
static __device__ NX_COLD bool update_linear(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const Window w = window_of(c, e, c.d->short_w);
  const int n = w.n;
  if (n < 5) return false;
  const Params cur = g.lp;
  if (c.lane == 0) count(c.rs->work[3], n);
  double* rows = c.lin_rows;  // (1/thr, s/thr) per sample; one buffer per warp
  double acc = 0.0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + c.lane;
    __syncwarp();
    if (i < n) {
      const int k = w.slot(i);
      const double b = w.rb[k], s = w.rs[k], y = w.ry[k];
      const double thr = throughput(cur, b, s);
      const double r1 = 1.0 / thr, r2 = s / thr;
      rows[2 * i] = r1;
      rows[2 * i + 1] = r2;
      const double iy = 1.0 / y;
      double* row = c.chunk + c.lane * 5;
      row[0] = 1.0 * iy;
      row[1] = r1 * iy;
      row[2] = r2 * iy;
      row[3] = b * iy;
      row[4] = s * iy;
    }
    __syncwarp();
    fold_chunk(c, min(32, n - base), acc);
  }
  // lane element: A^T A slot (lanes < 25) or A^T b (lanes 25..29) from the fold lanes
  const int src = c.lane < 25 ? slot_of(c.lane / 5, c.lane % 5) : (c.lane < 30 ? 15 + c.lane - 25 : 0);
  const double ne = __shfl_sync(NX_FULL, acc, src);
  const double y2 = static_cast<double>(n);
  const double prior[5] = {cur.tau0, cur.w0, cur.ws, cur.tauB, cur.tauS};
  double x[5];
  bool ok = solve5_warp(ne, x);
  if (ok) {
    // noise_level = 8 * rel_sse(x), exact left fold over <= short_window rows
    double run = 0.0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + c.lane;
      double rr = 0.0;
      if (i < n) {
        const int k = w.slot(i);
        const double b = w.rb[k], s = w.rs[k], y = w.ry[k];
        double pred = 0.0;
        pred += 1.0 * x[0];
        pred += rows[2 * i] * x[1];
        pred += rows[2 * i + 1] * x[2];
        pred += b * x[3];
        pred += s * x[4];
        const double r = (y - pred) / y;
        rr = r * r;
      }
      fold_exact_chunk(c, rr, min(32, n - base), run);
    }
    const double noise = 8.0 * __shfl_sync(NX_FULL, run, 0);
    const double den = (y2 < 1e-30) ? 1e-30 : y2;
    const double v = noise / den;
    const double lambda = (v < 1e-2) ? v : 1e-2;
    if (lambda > 1e-14) ok = solve5_warp(ridge_elem(ne, lambda, prior), x);
  }
  if (!ok) {
    // Degenerate design: rescale the linear tier (learner.cpp:304-333).
    double num = 0.0, den = 0.0;  // exact left folds: lane 0 -> num, lane 1 -> den
    for (int base = 0; base < n; base += 32) {
      const int i = base + c.lane;
      __syncwarp();
      if (i < n) {
        const int k = w.slot(i);
        const double y = w.ry[k];
        const double pred = predict(cur, w.rb[k], w.rs[k]);
        const double wt = 1.0 / (y * y);
        c.chunk[2 * c.lane] = wt * pred * y;
        c.chunk[2 * c.lane + 1] = wt * pred * pred;
      }
      __syncwarp();
      const int cnt = min(32, n - base);
      if (c.lane == 0)
        for (int k = 0; k < cnt; ++k) num += c.chunk[2 * k];
      if (c.lane == 1)
        for (int k = 0; k < cnt; ++k) den += c.chunk[2 * k + 1];
    }
    num = __shfl_sync(NX_FULL, num, 0);
    den = __shfl_sync(NX_FULL, den, 1);
    const double gm = num / den;
    __syncwarp();
    if (c.lane == 0) {
      g.cnt[2] += 1;
      if (isfinite(gm) && gm > 0.0 && gm != 1.0) {
        Params nx = cur;
        nx.tau0 *= gm;
        nx.w0 *= gm;
        const double ws = nx.ws * gm;
        nx.ws = (1e-6 < ws) ? ws : 1e-6;  // std::max(kWsMin, ws)
        nx.tauB *= gm;
        nx.tauS *= gm;
        g.lp = nx;
        g.lp_ver += 1;
        g.cnt[3] += 1;
      }
    }
    __syncwarp();
    return false;
  }
  bool clamped = false;
  auto floor_at = [&](double v, double lo) {
    if (v < lo) {
      clamped = true;
      return lo;
    }
    return v;
  };
  Params nx = cur;
  nx.tau0 = floor_at(x[0], 0.0);
  nx.w0 = floor_at(x[1], 0.0);
  nx.ws = floor_at(x[2], 1e-6);
  nx.tauB = floor_at(x[3], 0.0);
  nx.tauS = floor_at(x[4], 0.0);
  __syncwarp();
  if (c.lane == 0) {
    g.lp = nx;
    g.lp_ver += 1;
    g.cnt[0] += 1;
    if (clamped) g.cnt[4] += 1;
  }
  __syncwarp();
  return true;
}

// ---- structural tier (learner.cpp:209-298, 346-440) --------------------------
//
// One structural update evaluates ~76 profiled fits (learner.cpp:373-430) over
// the same <= long_window samples. Per update the window is staged once in
// chronological order (b, s, y, 1/y); per fit only the (kB, kS)-dependent
// quantities are rebuilt: a 1/f_B table over batch sizes and a per-sample
// 1/f_S cache, reused while kS is unchanged (every other coordinate move).
// The scaled design row is r = (1, 1/f, s/f, b, s) / y, so of the 15 unique
// A^T A entries and 5 A^T b entries, the 9 + 3 built only from {1, b, s}/y are
// fit-invariant and accumulated once per update; each fit accumulates the
// other 11 in one pass.
//
// Both squared-error sums a fit needs have closed forms in those normal
// equations — with the target y = 1 after 1/y weighting,
//   SSE(x) = y2 - 2 x.t + x^T A x
// — for the ridge scale (sse(x), learner.cpp:251-260) and for the windowed
// SSE of the clamped fit (windowed_sse(p), :209-222; T(p) is exactly x'.row
// for x' = (tau0, a, c, tauB, tauS)). Each closed form carries an explicit
// rounding-error bound; any decision inside the bound is re-taken on the
// reference's direct left-fold evaluation (wsse_exact / sse_x_exact).

constexpr double kU = 1.1102230246251565e-16;  // 2^-53

// Replica scratch layout (doubles), W = long_window:
//   [0,W) b  [W,2W) s  [2W,3W) y  [3W,5W) packed {1/y, b | s<<32} records
//   [5W,6W) 1/f_S per sample (only when s exceeds the token-count table)
//   [6W, 6W+1024) 1/f_B by batch size   [6W+1024, 8W+1024) linear-tier rows
//   [8W+1024, 9W+1024) distinct token counts (int32)
//   [9W+1024, 10W+1024) 1/f_S by distinct-count index (dense)
//   [10W+1024, 10W+1024+kSTab/2) token count -> dense index (int32)
//   then (group_base(W), nx_state.cuh) the grouped-sum arrays: sample indices
//   by batch size and by distinct token count, their group offsets, and the
//   per-group aggregates (8 per batch size, 4 per distinct token count)
constexpr int kSTab = 10240;  // token-count table (bitmap fits the 1280 B stage)

struct Stage {          // chronological window staged in the replica scratch
  const double* sb;     // b
  const double* ss;     // s
  const double* sy;     // observed_ms
  const double2* rec;   // {1 / observed_ms, b | s << 32}: one 16-byte load per sample
  double* ifs;          // 1 / f_S(s_i) for kS == ifs_k (when s exceeds the table)
  double* ifb;          // 1 / f_B(b) for kB == ifb_k, b in [1, tab]
  int* us;              // distinct s values of the window
  double* stab;         // 1 / f_S(us[k]) for kS == ifs_k, dense in k
  int* s2id;            // s -> k with us[k] == s
  int n, tab, U;
  bool use_tab;
  double ifs_k, ifb_k;
  // fit-invariant normal-equation entries: A00 A03 A04 A33 A34 A44, t0 t3 t4
  double A00, A03, A04, A33, A34, A44, t0, t3, t4;
  // Grouped sums (see gauged_fit_impl): samples grouped by batch size (pb, ob)
  // and by distinct token count (ps, os); ab holds 8 aggregates per batch
  // size for kS == ab_k, as 4 per distinct token count for kB == as_k.
  int *pb, *ps, *ob, *os;
  double *ab, *as, *part;
  double ab_k, as_k, last_kB, last_kS;
  bool grouped;
};

__device__ __forceinline__ Stage stage_of(const Ctx& c) {
  const int W = c.d->long_w;
  Stage s;
  s.sb = c.scratch;
  s.ss = c.scratch + W;
  s.sy = c.scratch + 2 * W;
  s.rec = reinterpret_cast<const double2*>(c.scratch + 3 * W);
  s.ifs = c.scratch + 5 * W;
  // 1/f_B and 1/f_S are gathered per sample in every fit pass: served from
  // shared memory when the CTA has the stage (latency ~30 cycles instead of
  // an L2 round trip on each of the pass's dependent gathers)
  s.ifb = c.fsm ? c.fsm : c.scratch + 6 * W;
  s.us = reinterpret_cast<int*>(c.scratch + 8 * W + kFbTable);
  s.stab = c.scratch + 9 * W + kFbTable;
  s.s2id = reinterpret_cast<int*>(c.scratch + 10 * W + kFbTable);
  const int64_t g = group_base(W), h = half_up(W);
  s.pb = reinterpret_cast<int*>(c.scratch + g);
  s.ps = reinterpret_cast<int*>(c.scratch + g + h);
  s.ob = reinterpret_cast<int*>(c.scratch + g + 2 * h);
  s.os = reinterpret_cast<int*>(c.scratch + g + 2 * h + half_up(kFbTable + 3));
  s.ab = c.scratch + g + 2 * h + half_up(kFbTable + 3) + half_up(W + 2);
  s.as = s.ab + 8 * kFbTable;
  s.part = s.as + 4 * W;
  s.n = 0;
  s.tab = 0;
  s.U = 0;
  s.use_tab = false;
  s.grouped = false;
  s.ifs_k = -1.0;
  s.ifb_k = -1.0;
  s.ab_k = s.as_k = s.last_kB = s.last_kS = -1.0;
  return s;
}

// Stable grouping of samples [0, n) by key(i) in [0, nkeys): afterwards group
// k is perm[off[k], off[k+1]) in ascending sample order (off: nkeys + 2 ints).
// One warp, chunks of 32 samples in order; ranks within a chunk come from
// __match_any_sync, so the placement is deterministic. The counters live in
// `work` (shared memory, >= nkeys + 2 ints) when given, else in `off`.
template <class Key>
__device__ void group_samples(int lane, int n, int nkeys, int* off, int* perm, Key key, int* work) {
  int* cnt = work ? work : off;
  __syncwarp();
  for (int k = lane; k < nkeys + 2; k += 32) cnt[k] = 0;
  __syncwarp();
  for (int i = lane; i < n; i += 32) atomicAdd(&cnt[key(i) + 2], 1);
  __syncwarp();
  int carry = 0;  // inclusive scan: cnt[k + 1] = first slot of group k
  for (int base = 0; base < nkeys + 2; base += 32) {
    const int k = base + lane;
    int v = k < nkeys + 2 ? cnt[k] : 0;
    v = warp_incl_scan(v) + carry;
    if (k < nkeys + 2) cnt[k] = v;
    carry = __shfl_sync(NX_FULL, v, 31);
  }
  __syncwarp();
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int k = i < n ? key(i) : -1;
    const unsigned peers = __match_any_sync(NX_FULL, k);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (i < n) perm[cnt[k + 1] + rank] = i;
    __syncwarp();
    if (i < n && rank == 0) cnt[k + 1] += __popc(peers);
    __syncwarp();
  }
  if (work)
    for (int k = lane; k < nkeys + 2; k += 32) off[k] = cnt[k];
  __syncwarp();
}

// windowed_sse (learner.cpp:209-222), direct model evaluation, tree order
static __device__ NX_COLD double wsse_tree(Ctx& c, const Stage& S, const Params& p) {
  double part = 0.0;
  for (int i = c.lane; i < S.n; i += 32) {
    const double y = S.sy[i];
    const double r = (y - predict(p, S.sb[i], S.ss[i])) / y;
    part += r * r;
  }
  return warp_sum(part);
}
// the same sum in the reference's left-to-right order
static __device__ NX_COLD double wsse_exact(Ctx& c, const Stage& S, const Params& p) {
  double run = 0.0;
  for (int base = 0; base < S.n; base += 32) {
    const int i = base + c.lane;
    double rr = 0.0;
    if (i < S.n) {
      const double y = S.sy[i];
      const double r = (y - predict(p, S.sb[i], S.ss[i])) / y;
      rr = r * r;
    }
    fold_exact_chunk(c, rr, min(32, S.n - base), run);
  }
  return __shfl_sync(NX_FULL, run, 0);
}
// gauged_fit's ridge-scale sse(x) exactly as the reference forms it
// (rows (1, 1/f, s/f, b, s), f = max(fB fS, 1e-300); learner.cpp:234-260)
static __device__ NX_COLD double sse_x_exact(Ctx& c, const Stage& S, double kB, double kS, const double x[5]) {
  double run = 0.0;
  for (int base = 0; base < S.n; base += 32) {
    const int i = base + c.lane;
    double rr = 0.0;
    if (i < S.n) {
      const double b = S.sb[i], s = S.ss[i], y = S.sy[i];
      double f = raw_factor(kB, b) * raw_factor(kS, s);
      f = (f < 1e-300) ? 1e-300 : f;
      double pred = 0.0;
      pred += 1.0 * x[0];
      pred += (1.0 / f) * x[1];
      pred += (s / f) * x[2];
      pred += b * x[3];
      pred += s * x[4];
      const double r = (y - pred) / y;
      rr = r * r;
    }
    fold_exact_chunk(c, rr, min(32, S.n - base), run);
  }
  return __shfl_sync(NX_FULL, run, 0);
}


// SSE(x) = y2 - 2 x.t + x^T A x with its absolute rounding bound: accumulation
// error of every entry (all terms positive) plus the closed-form arithmetic,
// plus the per-term gap between x.row and the reference's model evaluation.
static __device__ NX_COLD void closed_sse(double e, const double x[5], int n, double y2, double& val,
                           double& bound) {
  const int lane = lane_id();
  double q = 0.0, qa = 0.0, l = 0.0, la = 0.0;
  if (lane < 25) {
    const double xi = pick5(x, lane / 5), xj = pick5(x, lane % 5);
    q = xi * xj * e;
    qa = fabs(xi) * fabs(xj) * e;
  } else if (lane < 30) {
    const double xi = pick5(x, lane - 25);
    l = xi * e;
    la = fabs(xi) * e;
  }
  const double quad = warp_sum(q), quad_abs = warp_sum(qa), lin = warp_sum(l), lin_abs = warp_sum(la);
  val = y2 - 2.0 * lin + quad;
  const double M = y2 + 2.0 * lin_abs + quad_abs;
  const double sv = val > 0.0 ? val : 0.0;
  bound = 2.0 * (static_cast<double>(n) + 64.0) * kU * M +
          32.0 * kU * (sqrt(static_cast<double>(n) * (sv + 1.0)) + sv) + 1e-300;
}

// Per-update staging: chronological copy, gate statistics, invariant sums.
static __device__ NX_COLD void stage_window(Ctx& c, const Window& w, const Params& cur, Stage& S, bool& saturated,
                             int& shaped, int& bmax) {
  double* sb = const_cast<double*>(S.sb);
  double* ss = const_cast<double*>(S.ss);
  double* sy = const_cast<double*>(S.sy);
  double2* rec = const_cast<double2*>(S.rec);
  S.n = w.n;
  bool unsat = false;
  int shp = 0, bm = 1, smx = 1;
  double a00 = 0, a03 = 0, a04 = 0, a33 = 0, a34 = 0, a44 = 0, t0 = 0, t3 = 0, t4 = 0;
  for (int i = c.lane; i < w.n; i += 32) {
    const int k = w.slot(i);
    const int bi = w.rb[k], si = w.rs[k];
    const double b = bi, s = si, y = w.ry[k];
    const double iy = 1.0 / y;
    sb[i] = b;
    ss[i] = s;
    sy[i] = y;
    // {1/y, b | (distinct-s index << 16) | s << 32}; the index is filled in below
    rec[i] = make_double2(iy, __longlong_as_double(static_cast<long long>(
                                  (static_cast<unsigned long long>(si) << 32) |
                                  static_cast<unsigned>(bi & 0xffff))));
    if (cur.kB * b < 20.0 || cur.kS * s < 20.0) unsat = true;
    if (si >= 64 && si >= 4 * bi) ++shp;
    bm = max(bm, bi);
    smx = max(smx, si);
    const double r3 = b * iy, r4 = s * iy;
    a00 += iy * iy; a03 += iy * r3; a04 += iy * r4;
    a33 += r3 * r3; a34 += r3 * r4; a44 += r4 * r4;
    t0 += iy; t3 += r3; t4 += r4;
  }
  saturated = !__any_sync(NX_FULL, unsat);
  shaped = static_cast<int>(__reduce_add_sync(NX_FULL, static_cast<unsigned>(shp)));
  bmax = warp_max_int(bm);
  S.A00 = warp_sum(a00); S.A03 = warp_sum(a03); S.A04 = warp_sum(a04);
  S.A33 = warp_sum(a33); S.A34 = warp_sum(a34); S.A44 = warp_sum(a44);
  S.t0 = warp_sum(t0); S.t3 = warp_sum(t3); S.t4 = warp_sum(t4);
  S.tab = bmax < kFbTable ? bmax : kFbTable - 1;
  // distinct token counts: a presence bitmap in the shared stage, compacted
  // into S.us so each new kS costs one expm1 per distinct s, not per sample
  const int smax = warp_max_int(smx);
  S.use_tab = smax < kSTab && bmax < 65536 && w.n <= 65536;
  if (S.use_tab) {
    uint32_t* bits = reinterpret_cast<uint32_t*>(c.chunk);
    const int words = (smax >> 5) + 1;
    __syncwarp();
    for (int wd = c.lane; wd < words; wd += 32) bits[wd] = 0u;
    __syncwarp();
    for (int i = c.lane; i < w.n; i += 32) {
      const int si = static_cast<int>(ss[i]);
      atomicOr(&bits[si >> 5], 1u << (si & 31));
    }
    __syncwarp();
    int base = 0;
    for (int w0 = 0; w0 < words; w0 += 32) {
      const int wd = w0 + c.lane;
      unsigned m = wd < words ? bits[wd] : 0u;
      const int cnt = __popc(m);
      const int incl = warp_incl_scan(cnt);
      int off = base + incl - cnt;
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        S.us[off++] = wd * 32 + bit;
      }
      base += __shfl_sync(NX_FULL, incl, 31);
    }
    S.U = base;
    if (c.fsm && S.U <= c.fsm_cap) S.stab = c.fsm + kFbTable;
    __syncwarp();
    for (int k = c.lane; k < S.U; k += 32) S.s2id[S.us[k]] = k;
    __syncwarp();
    for (int i = c.lane; i < w.n; i += 32) {
      const unsigned long long bits64 = static_cast<unsigned long long>(__double_as_longlong(rec[i].y));
      const int si = static_cast<int>(bits64 >> 32);
      rec[i].y = __longlong_as_double(static_cast<long long>(
          bits64 | (static_cast<unsigned long long>(S.s2id[si]) << 16)));
    }
    __syncwarp();
    // grouped sums need every batch size inside the 1/f_B table
    S.grouped = bmax < kFbTable;
    if (S.grouped) {
      const double2* rc = S.rec;
      // counters in the (not yet built) shared 1/f_S table when it is there
      int* work = c.fsm && S.U + 2 <= 2 * c.fsm_cap ? reinterpret_cast<int*>(c.fsm + kFbTable) : nullptr;
      group_samples(c.lane, w.n, S.tab + 1, S.ob, S.pb, [rc](int i) {
        return static_cast<int>(static_cast<unsigned long long>(__double_as_longlong(rc[i].y)) & 0xffffull);
      }, work);
      group_samples(c.lane, w.n, S.U, S.os, S.ps, [rc](int i) {
        return static_cast<int>((static_cast<unsigned long long>(__double_as_longlong(rc[i].y)) >> 16) & 0xffffull);
      }, work);
#ifdef NX_TRACE_FIT
      __syncwarp();
      if (c.lane == 0 && w.n == 1024) {
        int bad = 0, badk = 0;
        for (int g = 0; g <= S.tab; ++g)
          for (int j = S.ob[g]; j < S.ob[g + 1]; ++j)
            if ((static_cast<unsigned long long>(__double_as_longlong(rc[S.pb[j]].y)) & 0xffffull) != (unsigned)g) ++bad;
        for (int k = 0; k < S.U; ++k)
          for (int j = S.os[k]; j < S.os[k + 1]; ++j)
            if (((static_cast<unsigned long long>(__double_as_longlong(rc[S.ps[j]].y)) >> 16) & 0xffffull) != (unsigned)k) ++badk;
        printf("GROUPCHECK n %d tab %d U %d ob_end %d os_end %d bad_b %d bad_s %d\n", w.n, S.tab, S.U, S.ob[S.tab + 1], S.os[S.U], bad, badk);
      }
      __syncwarp();
#endif
    }
  }
  __syncwarp();
}

struct FitOut {
  Params p;
  double err, bound;  // closed-form windowed SSE and its rounding bound; err=inf on failure
};

// gauged_fit (learner.cpp:228-298) for fixed (kB, kS).
// ---- the fit pass, optionally split across the refit team ---------------------
// Accumulates the 11 (kB,kS)-dependent normal-equation entries over samples
// [lo, hi) of the staged window (table path); lanes stride 32, 8 samples in
// flight per lane. Returns this warp's totals (warp_sum) in out[11].
static __device__ __forceinline__ void pass_range(const double2* rec, const double* stab, const double* ifb_t,
                                                  int tab, double kB, int lo, int hi, int lane, double out[11]) {
  double a01 = 0, a02 = 0, a11 = 0, a12 = 0, a22 = 0, a13 = 0, a14 = 0, a23 = 0, a24 = 0;
  double t1 = 0, t2 = 0;
  auto accumulate = [&](double iy, int bi, int si, double ifs) {
    const double b = bi, s = si;
    const double ifb = bi <= tab ? ifb_t[bi] : 1.0 / raw_factor(kB, b);
    double q = ifb * ifs;  // 1 / max(fB fS, 1e-300)
    q = q > 1e300 ? 1e300 : q;
    const double u1 = q * iy, u2 = (s * q) * iy, r3 = b * iy, r4 = s * iy;
    a01 += iy * u1; a02 += iy * u2; a11 += u1 * u1; a12 += u1 * u2; a22 += u2 * u2;
    a13 += u1 * r3; a14 += u1 * r4; a23 += u2 * r3; a24 += u2 * r4;
    t1 += u1; t2 += u2;
  };
  auto unpack = [](double y, int& bi, int& id, int& si) {
    const unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(y));
    bi = static_cast<int>(v & 0xffffull);
    id = static_cast<int>((v >> 16) & 0xffffull);
    si = static_cast<int>(v >> 32);
  };
  int i = lo + lane;
  for (; i + 224 < hi; i += 256) {
    double2 r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) r[u] = rec[i + 32 * u];
    double fs[8];
    int bi[8], si[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int id;
      unpack(r[u].y, bi[u], id, si[u]);
      fs[u] = stab[id];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) accumulate(r[u].x, bi[u], si[u], fs[u]);
  }
  for (; i < hi; i += 32) {
    const double2 r = rec[i];
    int bi, id, si;
    unpack(r.y, bi, id, si);
    accumulate(r.x, bi, si, stab[id]);
  }
  out[0] = warp_sum(a01); out[1] = warp_sum(a02); out[2] = warp_sum(a11); out[3] = warp_sum(a12);
  out[4] = warp_sum(a22); out[5] = warp_sum(a13); out[6] = warp_sum(a14); out[7] = warp_sum(a23);
  out[8] = warp_sum(a24); out[9] = warp_sum(t1); out[10] = warp_sum(t2);
}

// Totals of 11 per-lane partials in every lane: a reduce-scatter (each
// butterfly level keeps half of the slots, 16 double shuffles for 16 padded
// slots instead of 55 for 11 separate trees), then one broadcast per slot.
// Fixed pattern, so the result never depends on timing.
__device__ __forceinline__ void warp_sum11(const double a[11], double tot[11]) {
  const int lane = lane_id();
  const int h4 = (lane >> 4) & 1, h3 = (lane >> 3) & 1, h2 = (lane >> 2) & 1, h1 = (lane >> 1) & 1;
  double v8[8], v4[4], v2[2];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double lo = a[j], hi = j + 8 < 11 ? a[j + 8] : 0.0;
    v8[j] = (h4 ? hi : lo) + __shfl_xor_sync(NX_FULL, h4 ? lo : hi, 16);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) v4[j] = (h3 ? v8[j + 4] : v8[j]) + __shfl_xor_sync(NX_FULL, h3 ? v8[j] : v8[j + 4], 8);
#pragma unroll
  for (int j = 0; j < 2; ++j) v2[j] = (h2 ? v4[j + 2] : v4[j]) + __shfl_xor_sync(NX_FULL, h2 ? v4[j] : v4[j + 2], 4);
  double v = (h1 ? v2[1] : v2[0]) + __shfl_xor_sync(NX_FULL, h1 ? v2[0] : v2[1], 2);
  v = v + __shfl_xor_sync(NX_FULL, v, 1);  // lane holds slot 8 h4 + 4 h3 + 2 h2 + h1
#pragma unroll
  for (int q = 0; q < 11; ++q)
    tot[q] = __shfl_sync(NX_FULL, v, (((q >> 3) & 1) << 4) | (((q >> 2) & 1) << 3) | (((q >> 1) & 1) << 2) | ((q & 1) << 1));
}

// Named barrier of the refit team (warps 1..kRefitWarps of the replica CTA).
__device__ __forceinline__ void team_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kRefitWarps) : "memory");
}

// ---- grouped sums ------------------------------------------------------------
// Every (kB,kS)-dependent entry is a sum of positive per-sample terms
// g(1/f_B(b)) * h(1/f_S(s)) * m(b, s, 1/y). While kS stays fixed (a move of kB
// alone) each entry is a sum over batch sizes b of 1/f_B(b) (or its square)
// times one of 8 per-b aggregates that depend on kS only (ab); while kB stays
// fixed, a sum over the distinct token counts of 1/f_S (or its square) times
// one of 4 per-count aggregates that depend on kB only (as). The coordinate
// search moves one coordinate at a time and mostly misses, so ~85% of its
// fits become sums over <= 1024 batch sizes / the distinct token counts
// instead of passes over the window; the aggregates are rebuilt only after a
// move is accepted. Terms stay positive, so the closed-form SSE bound holds.

// Aggregate rebuilds. The grouped sample order is cut into one contiguous
// chunk per team lane (balanced however skewed the groups are: a low-load
// replica has few batch sizes, each with hundreds of samples). A lane writes
// the groups that lie inside its chunk; a group cut by a chunk boundary
// leaves per-lane partials (tail: the group it ends its chunk in, head: the
// group it starts its chunk in) that a second phase adds in lane order.
// Deterministic for a given team size.
//   ab[8b + .] (kS of the stab table), over the samples with batch size b:
//     F w, s F w, F^2 w, s F^2 w, s^2 F^2 w, s^2 F w, F v, s F v
//   as[4k + .] (kB of the ifb table), over the samples with token count us[k]:
//     G w, G^2 w, b G w, G v
//   (F = 1/f_S(s), G = 1/f_B(b), v = 1/y, w = v^2)
template <int NV>
__device__ __forceinline__ void agg_terms(const TeamTask& t, const double2 r, double (&a)[8]) {
  const unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(r.y));
  if (NV == 8) {
    const double sv = static_cast<double>(static_cast<int>(v >> 32));
    const double F = t.stab[(v >> 16) & 0xffffull];
    const double Fy = F * r.x, Fw = Fy * r.x, F2w = F * Fw;
    a[0] += Fw; a[1] += sv * Fw; a[2] += F2w; a[3] += sv * F2w;
    a[4] += sv * (sv * F2w); a[5] += sv * (sv * Fw); a[6] += Fy; a[7] += sv * Fy;
  } else {
    const int bi = static_cast<int>(v & 0xffffull);
    const double G = t.ifb[bi];
    const double Gy = G * r.x, Gw = Gy * r.x;
    a[0] += Gw; a[1] += G * Gw; a[2] += static_cast<double>(bi) * Gw; a[3] += Gy;
  }
}
template <int NV>
__device__ __forceinline__ int agg_key(const double2 r) {
  const unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(r.y));
  return NV == 8 ? static_cast<int>(v & 0xffffull) : static_cast<int>((v >> 16) & 0xffffull);
}
template <int NV>
static __device__ void rebuild_groups(const TeamTask& t, int gl, int nl, int team) {
  const int* perm = NV == 8 ? t.pb : t.ps;
  const int* off = NV == 8 ? t.ob : t.os;
  const int ng = NV == 8 ? t.tab + 1 : t.U;
  double* out = NV == 8 ? t.ab : t.as;
  double* head = t.part;            // [nl][8]
  double* tail = t.part + 8 * nl;   // [nl][8]
  const int per = (t.n + nl - 1) / nl;
  const int lo = min(t.n, gl * per), hi = min(t.n, lo + per);
  if (lo < hi) {
    double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int g = agg_key<NV>(t.rec[perm[lo]]);
    auto flush = [&](int gg) {
      const int g0 = off[gg], g1 = off[gg + 1];
      double* o = g0 >= lo && g1 <= hi ? out + NV * gg : (g0 < lo ? head : tail) + 8 * gl;
#pragma unroll
      for (int q = 0; q < NV; ++q) o[q] = a[q];
    };
    for (int j = lo; j < hi; ++j) {
      const double2 r = t.rec[perm[j]];
      const int k = agg_key<NV>(r);
      if (k != g) {
        flush(g);
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = 0.0;
        g = k;
      }
      agg_terms<NV>(t, r, a);
    }
    flush(g);
  }
  if (team > 1) team_sync();
  else __syncwarp();
  // empty groups, and groups cut by chunk boundaries: tail of the first lane
  // + heads of the rest
  for (int gg = gl; gg < ng; gg += nl) {
    const int g0 = off[gg], g1 = off[gg + 1];
    if (g0 >= g1) {  // no samples: the sums over groups read every slot
#pragma unroll
      for (int q = 0; q < NV; ++q) out[NV * gg + q] = 0.0;
      continue;
    }
    const int l0 = g0 / per, l1 = (g1 - 1) / per;
    if (l0 == l1) continue;
    double a[8];
#pragma unroll
    for (int q = 0; q < NV; ++q) a[q] = tail[8 * l0 + q];  // the group starts in l0's chunk
    for (int l = l0 + 1; l <= l1; ++l)
#pragma unroll
      for (int q = 0; q < NV; ++q) a[q] += head[8 * l + q];
#pragma unroll
    for (int q = 0; q < NV; ++q) out[NV * gg + q] = a[q];
  }
}
// The 11 entries (pass_range order) from ab and the ifb table (kB move).
static __device__ void sum_over_b(const TeamTask& t, int g0, int gstep, double a[11]) {
  for (int b = 1 + g0; b <= t.tab; b += gstep) {
    const double g = t.ifb[b], bb = static_cast<double>(b);
    const double* P = t.ab + 8 * b;
    const double gP0 = g * P[0], gP1 = g * P[1], g2 = g * g;
    a[0] += gP0; a[1] += gP1; a[2] += g2 * P[2]; a[3] += g2 * P[3]; a[4] += g2 * P[4];
    a[5] += bb * gP0; a[6] += gP1; a[7] += bb * gP1; a[8] += g * P[5]; a[9] += g * P[6]; a[10] += g * P[7];
  }
}
// The 11 entries from as and the stab table (kS move).
static __device__ void sum_over_s(const TeamTask& t, int g0, int gstep, double a[11]) {
  for (int k = g0; k < t.U; k += gstep) {
    const double h = t.stab[k], sv = static_cast<double>(t.us[k]);
    const double* Q = t.as + 4 * k;
    const double hQ0 = h * Q[0], h2Q1 = h * (h * Q[1]), hQ2 = h * Q[2], hQ3 = h * Q[3];
    a[0] += hQ0; a[1] += sv * hQ0; a[2] += h2Q1; a[3] += sv * h2Q1; a[4] += sv * (sv * h2Q1);
    a[5] += hQ2; a[6] += sv * hQ0; a[7] += sv * hQ2; a[8] += sv * (sv * hQ0); a[9] += hQ3; a[10] += sv * hQ3;
  }
}

// Contiguous, 256-aligned share of [0, n) for team member k of `team`.
__device__ __forceinline__ void team_range(int n, int k, int team, int& lo, int& hi) {
  const int per = ((n + 255) / 256 + team - 1) / team * 256;
  lo = min(n, k * per);
  hi = min(n, lo + per);
}

// Member k's share of task t; ops 1-3 return this warp's totals in out[11]
// (warp_sum), ops 4-5 write aggregates.
__device__ __forceinline__ void team_work(const TeamTask& t, int k, int team, int lane, double out[11]) {
  if (t.op == 1) {
    int lo, hi;
    team_range(t.n, k, team, lo, hi);
    pass_range(t.rec, t.stab, t.ifb, t.tab, t.kB, lo, hi, lane, out);
  } else if (t.op == 4) {
    rebuild_groups<8>(t, 32 * k + lane, 32 * team, team);
  } else if (t.op == 5) {
    rebuild_groups<4>(t, 32 * k + lane, 32 * team, team);
  } else {
    double a[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (t.op == 2) sum_over_b(t, 32 * k + lane, 32 * team, a);
    else sum_over_s(t, 32 * k + lane, 32 * team, a);
#pragma unroll
    for (int q = 0; q < 11; ++q) out[q] = warp_sum(a[q]);
  }
}

// Helper warps of the refit team: run their share of each task the leader
// (warp 1) publishes, until it publishes op -1.
static __device__ NX_COLD void team_helper(Ctx& c) {
  const int k = c.worker - 1;
  while (true) {
    team_sync();  // task published
    const TeamTask t = c.rs->team;
    if (t.op < 0) break;
    double part[11];
    team_work(t, k, kRefitWarps, c.lane, part);
    if (c.lane == 0 && t.op <= 3)
      for (int q = 0; q < 11; ++q) c.rs->team_part[k][q] = part[q];
    team_sync();  // partial totals / aggregates written
  }
}

// Leader side: run t over the team (or alone) and combine the members'
// totals in member order.
static __device__ void run_task(Ctx& c, const TeamTask& t, double tot[11]) {
  if (c.team > 1) {
    if (c.lane == 0) c.rs->team = t;
    team_sync();  // publish
    team_work(t, 0, c.team, c.lane, tot);
    team_sync();  // members done
    if (t.op <= 3)
      for (int k = 1; k < c.team; ++k)
#pragma unroll
        for (int q = 0; q < 11; ++q) tot[q] += c.rs->team_part[k][q];
  } else {
    team_work(t, 0, 1, c.lane, tot);
  }
  __syncwarp();
}

static __device__ FitOut gauged_fit_impl(Ctx& c, Stage& S, const Params& cur, double kB, double kS, bool exact);
static __device__ FitOut finish_fit(Ctx& c, const Stage& S, const Params& cur, double kB, double kS, double e,
                                   bool* ambiguous);
static __device__ double exact_elem(Ctx& c, Stage& S, double kB, double kS);
static __device__ FitOut gauged_fit(Ctx& c, Stage& S, const Params& cur, double kB, double kS, bool exact = false) {
  const long long t0 = nx_clock();
  FitOut o = gauged_fit_impl(c, S, cur, kB, kS, exact);
  if (c.lane == 0) count(c.rs->lcycles[10], nx_clock() - t0);
  return o;
}
static __device__ NX_COLD FitOut gauged_fit_impl(Ctx& c, Stage& S, const Params& cur, double kB, double kS,
                                                 bool exact) {
  const int n = S.n;
  double e;
  if (exact) {
    e = exact_elem(c, S, kB, kS);
  } else {
  if (c.lane == 0) count(c.rs->work[5], 1);
  const long long tf0 = nx_clock();
  // Which sum: over b (kS unchanged since ab was built), over the distinct
  // token counts (kB unchanged since as was built), either after rebuilding
  // its aggregates when the previous fit shared the other coordinate, or a
  // pass over the samples. 1/f >= 1e100 never occurs under the guard, so the
  // reference's max(fB fS, 1e-300) floor (= a 1e300 cap on the product of
  // the inverses) cannot bind there.
  int op = 1;
  bool rebuild = false;
  if (S.grouped && kB >= 1e-100 && kS >= 1e-100) {
    if (kS == S.ab_k) op = 2;
    else if (kB == S.as_k) op = 3;
    else if (kB == S.last_kB) op = 3, rebuild = true;
    else if (kS == S.last_kS) op = 2, rebuild = true;
  }
  S.last_kB = kB;
  S.last_kS = kS;
  const bool need_fb = op != 3 || rebuild, need_fs = op != 2 || rebuild;
  if (need_fb && kB != S.ifb_k) {
    __syncwarp();
#pragma unroll 4
    for (int b = 1 + c.lane; b <= S.tab; b += 32)
      S.ifb[b] = 1.0 / raw_factor(kB, static_cast<double>(b));
    S.ifb_k = kB;
    __syncwarp();
  }
  const bool new_s = kS != S.ifs_k;
  if (need_fs && new_s && S.use_tab) {
    __syncwarp();
#pragma unroll 4
    for (int k = c.lane; k < S.U; k += 32)
      S.stab[k] = 1.0 / raw_factor(kS, static_cast<double>(S.us[k]));
    __syncwarp();
  }
  const long long tf1 = nx_clock();
  if (c.lane == 0) count(c.rs->lcycles[7], tf1 - tf0);
  // per-entry totals (fixed combination order across the team; every term is
  // positive, so the closed-form SSE bound covers any order)
  double tot[11];
  if (S.use_tab) {
    TeamTask t;
    t.rec = S.rec;
    t.stab = S.stab;
    t.ifb = S.ifb;
    t.pb = S.pb;
    t.ps = S.ps;
    t.ob = S.ob;
    t.os = S.os;
    t.us = S.us;
    t.ab = S.ab;
    t.as = S.as;
    t.part = S.part;
    t.kB = kB;
    t.n = n;
    t.tab = S.tab;
    t.U = S.U;
    if (rebuild) {
      t.op = op == 2 ? 4 : 5;
      run_task(c, t, tot);
      if (op == 2) S.ab_k = kS;
      else S.as_k = kB;
#ifdef NX_TRACE_FIT
      if (op == 2 && n == 1024 && c.lane == 0) {
        const int per = (n + 95) / 96;
        for (int g = 1; g <= S.tab; ++g) {
          double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          for (int j = S.ob[g]; j < S.ob[g + 1]; ++j) agg_terms<8>(t, S.rec[S.pb[j]], d);
          for (int q = 0; q < 8; ++q)
            if (fabs(d[q] - S.ab[8 * g + q]) > 1e-9 * fabs(d[q])) {
              printf("    AB g %d q %d direct %.17g ab %.17g span [%d,%d) lanes %d..%d\n", g, q, d[q], S.ab[8 * g + q],
                     S.ob[g], S.ob[g + 1], S.ob[g] / per, (S.ob[g + 1] - 1) / per);
              break;
            }
        }
      }
#endif
    }
    t.op = op;
    const long long tq = nx_clock();
    if (op == 1) {
      run_task(c, t, tot);
    } else {  // a few hundred groups at most: the leader alone, no team round trip
      double a[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      if (op == 2) sum_over_b(t, c.lane, 32, a);
      else sum_over_s(t, c.lane, 32, a);
      warp_sum11(a, tot);
    }
    if (c.lane == 0 && op != 1) count(c.rs->lcycles[11], nx_clock() - tq);
#ifdef NX_TRACE_FIT
    if (op != 1 && S.n == 1024) {
      if (kS != S.ifs_k) {
        for (int k = c.lane; k < S.U; k += 32) S.stab[k] = 1.0 / raw_factor(kS, static_cast<double>(S.us[k]));
        S.ifs_k = kS;
      }
      if (kB != S.ifb_k) {
        for (int b = 1 + c.lane; b <= S.tab; b += 32) S.ifb[b] = 1.0 / raw_factor(kB, static_cast<double>(b));
        S.ifb_k = kB;
      }
      __syncwarp();
      double chk[11];
      t.op = 1;
      run_task(c, t, chk);
      for (int q = 0; q < 11; ++q)
        if (c.lane == 0 && fabs(chk[q] - tot[q]) > 1e-9 * fabs(chk[q]))
          printf("    op %d kB %.6g kS %.6g entry %d grouped %.17g pass %.17g\n", op, kB, kS, q, tot[q], chk[q]);
    }
#endif
  } else {
    double a01 = 0, a02 = 0, a11 = 0, a12 = 0, a22 = 0, a13 = 0, a14 = 0, a23 = 0, a24 = 0;
    double t1 = 0, t2 = 0;
    for (int i = c.lane; i < n; i += 32) {
      const double2 r = S.rec[i];
      const long long bs = __double_as_longlong(r.y);
      const int bi = static_cast<int>(S.sb[i]), si = static_cast<int>(bs >> 32);
      double ifs;
      if (new_s) {
        ifs = 1.0 / raw_factor(kS, static_cast<double>(si));
        S.ifs[i] = ifs;  // lane-private slot: read back only by this lane
      } else {
        ifs = S.ifs[i];
      }
      const double iy = r.x, b = bi, s = si;
      const double ifb = bi <= S.tab ? S.ifb[bi] : 1.0 / raw_factor(kB, b);
      double q = ifb * ifs;  // 1 / max(fB fS, 1e-300)
      q = q > 1e300 ? 1e300 : q;
      const double u1 = q * iy, u2 = (s * q) * iy, r3 = b * iy, r4 = s * iy;
      a01 += iy * u1; a02 += iy * u2; a11 += u1 * u1; a12 += u1 * u2; a22 += u2 * u2;
      a13 += u1 * r3; a14 += u1 * r4; a23 += u2 * r3; a24 += u2 * r4;
      t1 += u1; t2 += u2;
    }
    tot[0] = warp_sum(a01); tot[1] = warp_sum(a02); tot[2] = warp_sum(a11); tot[3] = warp_sum(a12);
    tot[4] = warp_sum(a22); tot[5] = warp_sum(a13); tot[6] = warp_sum(a14); tot[7] = warp_sum(a23);
    tot[8] = warp_sum(a24); tot[9] = warp_sum(t1); tot[10] = warp_sum(t2);
  }
  if (need_fs) S.ifs_k = kS;
  if (c.lane == 0) count(c.rs->lcycles[9], nx_clock() - tf1);
  const long long tf2 = nx_clock();
  const double u15[15] = {S.A00, tot[0], tot[1], S.A03, S.A04, tot[2], tot[3], tot[5], tot[6],
                          tot[4], tot[7], tot[8], S.A33, S.A34, S.A44};
  const double t5[5] = {S.t0, tot[9], tot[10], S.t3, S.t4};
  e = normal_elem(u15, t5);
  (void)tf2;
  }
  const long long ts = nx_clock();
  // one call site of the solve (it is large): a rank test too close to call
  // on the fast sums goes round once more on the reference's exact ones
  bool ambiguous = false;
  FitOut out;
#pragma unroll 1
  for (int pass = exact ? 1 : 0;; ++pass) {
    out = finish_fit(c, S, cur, kB, kS, e, pass == 0 ? &ambiguous : nullptr);
    if (pass > 0 || !ambiguous) break;
    e = exact_elem(c, S, kB, kS);
  }
  if (c.lane == 0) count(c.rs->lcycles[13], nx_clock() - ts);
  return out;
}

// The reference's exact normal equations for (kB, kS): rows (1, 1/f, s/f, b,
// s) / y with f = max(fB fS, 1e-300), accumulated left to right in window
// order (Ols5::add, learner.cpp:62-75, 228-245) — one fold lane per entry.
// The coordinate search ranks candidates on the fast sums (every ranking
// certified); the winner's coefficients are recomputed here so the learner
// adopts the reference's values, not values a few ulps of the window sums
// away (the 5x5 solve amplifies those by the system's condition number).
static __device__ NX_COLD double exact_elem(Ctx& c, Stage& S, double kB, double kS) {
  const int n = S.n;
  // f_B by batch size and f_S by distinct token count (the reference's
  // per-sample expm1 values) in the fit tables' storage, which the next fit
  // then rebuilds
  const bool tab = S.use_tab && S.grouped;
  if (tab) {
    __syncwarp();
    for (int b = 1 + c.lane; b <= S.tab; b += 32) S.ifb[b] = raw_factor(kB, static_cast<double>(b));
    for (int k = c.lane; k < S.U; k += 32) S.stab[k] = raw_factor(kS, static_cast<double>(S.us[k]));
    S.ifb_k = S.ifs_k = -1.0;
    __syncwarp();
  }
  double acc = 0.0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + c.lane;
    __syncwarp();
    if (i < n) {
      const double b = S.sb[i], sv = S.ss[i];
      double f;
      if (tab) {
        const unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(S.rec[i].y));
        f = S.ifb[v & 0xffffull] * S.stab[(v >> 16) & 0xffffull];
      } else {
        f = raw_factor(kB, b) * raw_factor(kS, sv);
      }
      f = (f < 1e-300) ? 1e-300 : f;
      const double iy = S.rec[i].x;  // == 1.0 / S.sy[i]
      double* row = c.chunk + c.lane * 5;
      row[0] = 1.0 * iy;
      row[1] = (1.0 / f) * iy;
      row[2] = (sv / f) * iy;
      row[3] = b * iy;
      row[4] = sv * iy;
    }
    __syncwarp();
    const int cnt = min(32, n - base);
    if (cnt == 32) {  // unrolled: the loads run ahead of the add chain
      int ei, ej;
      acc_slot(c.lane, ei, ej);
      if (c.lane < 15) {
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += c.chunk[k * 5 + ei] * c.chunk[k * 5 + ej];
      } else if (c.lane < 20) {
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += c.chunk[k * 5 + ei] * 1.0;
      }
    } else {
      fold_chunk(c, cnt, acc);
    }
  }
  const int src = c.lane < 25 ? slot_of(c.lane / 5, c.lane % 5) : (c.lane < 30 ? 15 + c.lane - 25 : 0);
  return __shfl_sync(NX_FULL, acc, src);
}

// Solve, ridge and trust region of gauged_fit (learner.cpp:246-297) from the
// normal equations e (lane element: A^T A slot or A^T b).
static __device__ NX_COLD FitOut finish_fit(Ctx& c, const Stage& S, const Params& cur, double kB, double kS,
                                            double e, bool* ambiguous) {
  const int n = S.n;
  const double y2 = static_cast<double>(n);  // sum of 1.0 * 1.0 (learner.cpp:73)
  const double prior[5] = {cur.tau0, cur.w0 / cur.p_max, cur.ws / cur.p_max, cur.tauB, cur.tauS};
  FitOut out;
  out.err = __longlong_as_double(0x7ff0000000000000LL);
  out.bound = 0.0;
  // unridged solve and the ridge at the cap (lambda = 1e-7, the value
  // certified below in all but near-noise-free windows) run in lockstep
  double x[5];
  double vk[2] = {e, ridge_elem(e, 1e-7, prior)};
  double xk[2][5];
  bool okk[2], amb[2];
  const long long ts5 = nx_clock();
  solve5_warp_k<2>(vk, xk, okk, amb);
  if (c.lane == 0) count(c.rs->lcycles[15], nx_clock() - ts5);
  if (ambiguous && amb[0]) *ambiguous = true;
  if (!okk[0]) return out;
#pragma unroll
  for (int q = 0; q < 5; ++q) x[q] = xk[0][q];
  // lambda = min(1e-7, sse(x) / max(y2, 1e-30))  (learner.cpp:84-85, cap 1e-7)
  const double den = (y2 < 1e-30) ? 1e-30 : y2;
  // Certify sse(x) / den >= 1e-7 (=> lambda = cap): first by the closed
  // form (four warp sums; it clears the threshold by more than its rounding
  // bound in nearly every fit), else by a lower bound — the sum has
  // non-negative terms, so 32 of them evaluated directly (one per lane, the
  // reference's per-term formula) bound the left-fold total from below —
  // and the exact fold decides the rest.
  const double thr = 1e-7 * (1.0 + 8.0 * kU);
  double sv = 0.0, sb = 0.0;
  closed_sse(e, x, n, y2, sv, sb);
  bool at_cap = (sv - sb) / den > thr;
  if (!at_cap) {
    const int i = c.lane * (n / 32);
    double rr = 0.0;
    if (i < n) {
      const double b = S.sb[i], s = S.ss[i], y = S.sy[i];
      double f = raw_factor(kB, b) * raw_factor(kS, s);
      f = (f < 1e-300) ? 1e-300 : f;
      double pred = 0.0;
      pred += 1.0 * x[0];
      pred += (1.0 / f) * x[1];
      pred += (s / f) * x[2];
      pred += b * x[3];
      pred += s * x[4];
      const double r = (y - pred) / y;
      rr = r * r;
    }
    const double lb = warp_sum(rr) * (1.0 - 1e-6);
    at_cap = lb / den > thr;
  }
  double lambda = 1e-7;
  if (!at_cap) {
    const double v = sse_x_exact(c, S, kB, kS, x) / den;
    lambda = (v < 1e-7) ? v : 1e-7;
  }
  if (lambda == 1e-7) {
    if (ambiguous && amb[1]) *ambiguous = true;
    if (!okk[1]) return out;
#pragma unroll
    for (int q = 0; q < 5; ++q) x[q] = xk[1][q];
  } else if (lambda > 1e-14 && !solve5_warp(ridge_elem(e, lambda, prior), x, ambiguous)) {
    return out;
  }
  const double tau0 = x[0] < 0.0 ? 0.0 : x[0];
  const double aa = x[1] < 0.0 ? 0.0 : x[1];
  const double slope = cur.ws / cur.p_max + cur.tauS;
  const double s16 = slope / 16.0;
  const double c_lo = (1.0 / 1e4 < s16) ? s16 : 1.0 / 1e4;
  const double s4 = 4.0 * slope;
  const double cap_hi = (s4 < 1.0 / 1e-3) ? s4 : 1.0 / 1e-3;
  const double c_hi = (c_lo < cap_hi) ? cap_hi : c_lo;
  const double cc = (x[2] < c_lo) ? c_lo : ((c_hi < x[2]) ? c_hi : x[2]);  // std::clamp
  Params p = cur;
  p.kB = kB;
  p.kS = kS;
  p.p_max = 1.0 / cc;
  p.w0 = aa / cc;
  p.ws = 1.0;
  p.tau0 = tau0;
  p.tauB = x[3] < 0.0 ? 0.0 : x[3];
  p.tauS = x[4] < 0.0 ? 0.0 : x[4];
  out.p = p;
  const double xp[5] = {p.tau0, aa, cc, p.tauB, p.tauS};  // T(p) == xp . row
  closed_sse(e, xp, n, y2, out.err, out.bound);
  return out;
}

// Certified "exact(a) < exact(b) * f" for two windowed-SSE intervals; exact
// re-evaluation only when the intervals cannot decide.
static __device__ bool less_scaled_impl(Ctx& c, const Stage& S, const FitOut& a, const FitOut& b, double f);
static __device__ bool less_scaled(Ctx& c, const Stage& S, const FitOut& a, const FitOut& b, double f) {
  const long long t0 = nx_clock();
  const bool r = less_scaled_impl(c, S, a, b, f);
  (void)t0;
  return r;
}
static __device__ NX_COLD bool less_scaled_impl(Ctx& c, const Stage& S, const FitOut& a, const FitOut& b, double f) {
  const double a_hi = a.err + a.bound, a_lo = a.err - a.bound;
  const double b_hi = (b.err + b.bound) * f, b_lo = (b.err - b.bound) * f;
  if (a_hi < b_lo * (1.0 - 4.0 * kU)) return true;
  if (a_lo > b_hi * (1.0 + 4.0 * kU)) return false;
  return wsse_exact(c, S, a.p) < wsse_exact(c, S, b.p) * f;
}

static __device__ NX_COLD void update_structural(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const Window w = window_of(c, e, c.d->long_w);
  const int n = w.n;
  if (n < c.d->min_s || n < 5) return;
  const Params cur = g.lp;
  Stage S = stage_of(c);
  bool saturated;
  int shaped, bmax;
  const long long ts0 = nx_clock();
  stage_window(c, w, cur, S, saturated, shaped, bmax);
  if (c.lane == 0) count(c.rs->lcycles[12], nx_clock() - ts0);
  if (saturated || shaped < 16) {
    __syncwarp();
    if (c.lane == 0) g.cnt[6] += 1;
    __syncwarp();
    return;
  }
  if (c.lane == 0) count(c.rs->work[4], n);
  // base_err: direct evaluation, tree order; tree vs left fold of n positive
  // terms differ by at most 2(n-1)u of the sum
  FitOut base;
  base.p = cur;
  const long long tb0 = nx_clock();
  base.err = wsse_tree(c, S, cur);
  (void)tb0;
  base.bound = 2.0 * (static_cast<double>(n) + 2.0) * kU * base.err;
  const double lo = log(1e-8), hi = log(1e4);
  const double shrink = 1.0 - 1e-3;
  double th0 = log(cur.kB), th1 = log(cur.kS);
  double st0 = 0.5, st1 = 0.5;
  const double kbs[3] = {0.05, 0.7, 8.0}, kss[3] = {0.002, 0.03, 0.4};
  // learner.cpp:389-430 as a candidate generator around ONE gauged_fit call
  // site: the start point, the 3x3 grid seed, the coordinate sweeps (+1 then
  // -1 per coordinate, step x1.6 on a hit, x0.5 otherwise, stop when a sweep
  // misses with both steps < 1e-5, at most 50 sweeps) and the winner's exact
  // refit. Written as nested loops the fit was inlined four times (~0.8 MB
  // of the kernel's code); one copy halves the kernel (96 k -> 50 k SASS
  // instructions) at equal speed (profiles/r02_l1_ab.txt).
  enum { kPhStart, kPhGrid, kPhSweep, kPhExact };
  int ph = kPhStart, gi = 0, sweep = 0, cdim = 0, dir = 0;
  bool hit = false, improved = false;
  double t0 = th0, t1 = th1;
  FitOut best;
#pragma unroll 1
  while (true) {
    double kB, kS;
    if (ph == kPhSweep) {  // the next candidate that moves its coordinate
#pragma unroll 1
      while (true) {
        if (sweep >= 50) {
          ph = kPhExact;
          break;
        }
        if (cdim == 2) {  // end of a sweep
          const double smax = (st0 < st1) ? st1 : st0;
          if (!improved && smax < 1e-5) {
            ph = kPhExact;
            break;
          }
          ++sweep;
          cdim = 0;
          dir = 0;
          hit = false;
          improved = false;
          continue;
        }
        if (hit || dir == 2) {  // this coordinate is done
          if (cdim == 0) st0 *= hit ? 1.6 : 0.5;
          else st1 *= hit ? 1.6 : 0.5;
          improved |= hit;
          ++cdim;
          dir = 0;
          hit = false;
          continue;
        }
        const double sgn = dir == 0 ? 1.0 : -1.0;
        t0 = th0;
        t1 = th1;
        double& tc = cdim == 0 ? t0 : t1;
        const double v = tc + sgn * (cdim == 0 ? st0 : st1);
        tc = (v < lo) ? lo : ((hi < v) ? hi : v);
        if (tc == (cdim == 0 ? th0 : th1)) {
          ++dir;
          continue;
        }
        break;
      }
    }
    if (ph == kPhStart) {
      kB = exp(th0);
      kS = exp(th1);
    } else if (ph == kPhGrid) {
      kB = kbs[gi / 3];
      kS = kss[gi % 3];
    } else if (ph == kPhSweep) {
      kB = exp(t0);
      kS = exp(t1);
    } else {
      kB = best.p.kB;
      kS = best.p.kS;
    }
    const long long tx = nx_clock();
    const FitOut cand = gauged_fit(c, S, cur, kB, kS, ph == kPhExact);
    if (ph == kPhStart) {
      best = cand;
      if (!isfinite(best.err)) {
        __syncwarp();
        if (c.lane == 0) g.cnt[5] += 1;
        __syncwarp();
        return;
      }
      ph = kPhGrid;
    } else if (ph == kPhExact) {
      // the winner's coefficients from the reference's exact normal equations
      if (c.lane == 0) count(c.rs->lcycles[14], nx_clock() - tx);
      if (isfinite(cand.err)) best = cand;
      else best.err = cand.err;  // the exact system is singular: the reference fails this fit too
      break;
    } else {
      if (isfinite(cand.err) && less_scaled(c, S, cand, best, shrink)) {
        best = cand;
        if (ph == kPhGrid) {
          th0 = log(kB);
          th1 = log(kS);
        } else {
          th0 = t0;
          th1 = t1;
          hit = true;
        }
      }
      if (ph == kPhGrid) {
        if (++gi == 9) ph = kPhSweep;
      } else {
        ++dir;
      }
    }
  }
  // reject if invalid or worse than the current model (learner.cpp:432-435)
  bool worse;
  if (best.err - best.bound > (base.err + base.bound) * (1.0 + 4.0 * kU)) worse = true;
  else if (best.err + best.bound < (base.err - base.bound) * (1.0 - 4.0 * kU)) worse = false;
  else worse = wsse_exact(c, S, best.p) > wsse_exact(c, S, cur);
  if (!params_valid(best.p) || worse) {
    __syncwarp();
    if (c.lane == 0) g.cnt[5] += 1;
    __syncwarp();
    return;
  }
  __syncwarp();
  if (c.lane == 0) {
    g.lp = best.p;
    g.lp_ver += 1;
    g.cnt[1] += 1;
  }
  __syncwarp();
  update_linear(c, e);
}

// Queue a structural refit of engine e for the refit warp. The engine's
// learner state (params, ring, counters) is frozen until the refit clears
// refit_pending: the event loop waits (wait_refit) before its next read.
static __device__ void post_refit(Ctx& c, int e) {
  __syncwarp();
  if (c.lane == 0) {
    vstore(c.eng[e].refit_pending, 1);
    const int t = vload(c.rs->jq_tail);
    c.rs->jq_eng[t & 63] = e;
    __threadfence_block();
    vstore(c.rs->jq_tail, t + 1);
  }
  __syncwarp();
}

// Tells the refit leader the replica is done (job id -1).
static __device__ void post_exit(Ctx& c) {
  __syncwarp();
  if (c.lane == 0) {
    const int t = vload(c.rs->jq_tail);
    c.rs->jq_eng[t & 63] = -1;
    __threadfence_block();
    vstore(c.rs->jq_tail, t + 1);
  }
  __syncwarp();
}

static __device__ void wait_refit(Ctx& c, int e) {
  if (!vload(c.eng[e].refit_pending)) return;
  const long long t0 = nx_clock();
  // exponential backoff: a structural update runs ~1-2 ms, so microsecond
  // polling granularity costs nothing while tight polling burned issue slots
  // and instruction fetch of the co-resident replicas (ncu: ~1/4 of all
  // executed instructions were wait loops)
  unsigned ns = 64;
  while (vload(c.eng[e].refit_pending)) {
    __nanosleep(ns);
    ns = ns < 1024 ? 2 * ns : 1024;
  }
  __threadfence_block();
  __syncwarp();
  if (c.lane == 0) count(c.rs->lcycles[8], nx_clock() - t0);
}

// The refit leader (warp 1): claims the next job (engine id) and runs
// update_structural — its fit passes split across the team's helper warps —
// until it claims -1, then releases the helpers. At most one job per engine
// is outstanding (record_sample waits before posting the next), so the
// 64-slot ring never wraps onto an unclaimed job. (Measured: refits of
// different engines rarely overlap, so one team per refit beats one worker
// per refit.)
static __device__ NX_COLD void refit_worker(Ctx& c) {
  while (true) {
    int e = -2;
    if (c.lane == 0) {
      const int h = atomicAdd(&c.rs->jq_head, 1);
      unsigned ns = 128;
      while (vload(c.rs->jq_tail) <= h) {
        __nanosleep(ns);
        ns = ns < 2048 ? 2 * ns : 2048;
      }
      __threadfence_block();
      e = *reinterpret_cast<const volatile int32_t*>(&c.rs->jq_eng[h & 63]);
    }
    e = __shfl_sync(NX_FULL, e, 0);
    if (e < 0) {
      if (c.team > 1) {
        if (c.lane == 0) c.rs->team.op = -1;
        team_sync();  // helpers leave
      }
      __syncwarp();
      return;
    }
    {
      PhaseTimer pt(c.rs, 6);
      update_structural(c, e);
    }
    __threadfence_block();
    __syncwarp();
    if (c.lane == 0) vstore(c.eng[e].refit_pending, 0);
    __syncwarp();
  }
}

// record_sample (learner.cpp:130-146): ring push + periodic refits.
static __device__ NX_COLD void record_sample(Ctx& c, int e, int b, int s, double y) {
  EngSm& g = c.eng[e];
  wait_refit(c, e);
  if (!(y > 0.0) || !(b >= 1 && s >= b)) {
    fail(c, 1, NX_SITE_SAMPLE, b);
    return;
  }
  const NxEngineDesc& ed = c.ed[e];
  const int W = c.d->long_w;
  __syncwarp();
  if (c.lane == 0) {
    int slot;
    if (g.ring_size < W) {
      slot = g.ring_size;
      g.ring_size += 1;
    } else {
      slot = g.ring_head;
      g.ring_head = g.ring_head + 1 == g.ring_size ? 0 : g.ring_head + 1;
    }
    c.P->ring_b[ed.ring_off + slot] = b;
    c.P->ring_s[ed.ring_off + slot] = s;
    c.P->ring_y[ed.ring_off + slot] = y;
    g.seen += 1;
    // seen % period == 0 as countdowns (a 64-bit remainder by a runtime
    // divisor is a long software sequence on the event loop)
    if (--g.lin_left == 0) g.lin_left = c.d->l_period;
    if (--g.str_left == 0) g.str_left = c.d->s_period;
  }
  __syncwarp();
  const int64_t seen = g.seen;
  if (g.lin_left == c.d->l_period) {
    PhaseTimer pt(c.rs, 5);
    update_linear(c, e);
  }
  if (seen >= c.d->min_s && g.str_left == c.d->s_period) {
    // engine-parallel loop: the engine's own warp refits (its timeline waits
    // for the new params anyway; other engines' warps keep running)
#ifdef NX_INLINE_REFIT
    if (nx_timers_on && c.lane == 0) c.rs->lcycles[3] = 1;  // window attribution (tools/merge_probe.py)
    PhaseTimer pt(c.rs, 6);
    update_structural(c, e);
#else
    post_refit(c, e);
#endif
  }
}

}  // namespace nxd
