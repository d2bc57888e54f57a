// K4 — online coefficient refit, one warp per engine update.
//
// Replaces OnlineLearner (proj/src/learner.cpp:130-440). Reduction orders:
//  * the normal-equation accumulators (15 unique A^T A entries + 5 A^T b) are
//    folded in the reference's left-to-right sample order, one accumulator
//    per lane over 32-sample chunks staged in shared memory — so the fitted
//    coefficients are the reference's bit for bit (modulo libm ulps);
//  * the squared-error sums (ridge scale, windowed SSE) are fixed-order warp
//    trees; every decision they drive (lambda cap, accept/reject) is
//    certified against the summation error bound and, if the tree value sits
//    inside it, recomputed as an exact left fold. Decisions therefore equal
//    the reference's left-fold decisions.
#pragma once
#include "nx_state.cuh"

namespace nxd {

constexpr double kCertMargin = 1e-9;  // >> 2*(n-1)*2^-53 for n <= 2^20

// ---- 5x5 elimination (learner.cpp:24-60), fully unrolled in registers -----
__device__ __forceinline__ double dmax(double m, double v) { return (m < v) ? v : m; }

__device__ bool solve5(double a[5][5], double b[5], double x[5]) {
  double scale[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) m = dmax(m, fabs(a[i][j]));
    if (m <= 0.0) return false;
    scale[j] = 1.0 / m;
#pragma unroll
    for (int i = 0; i < 5; ++i) a[i][j] *= scale[j];
  }
  double norm = 0.0;
#pragma unroll
  for (int i = 0; i < 5; ++i)
#pragma unroll
    for (int j = 0; j < 5; ++j) norm = dmax(norm, fabs(a[i][j]));
#pragma unroll
  for (int col = 0; col < 5; ++col) {
    int piv = col;
    double pv = fabs(a[col][col]);
#pragma unroll
    for (int r = col + 1; r < 5; ++r) {
      const double v = fabs(a[r][col]);
      if (v > pv) {
        piv = r;
        pv = v;
      }
    }
    if (pv < 1e-10 * norm) return false;
#pragma unroll
    for (int r = col + 1; r < 5; ++r) {
      if (piv == r) {
#pragma unroll
        for (int cc = 0; cc < 5; ++cc) {
          const double t = a[col][cc];
          a[col][cc] = a[r][cc];
          a[r][cc] = t;
        }
        const double t = b[col];
        b[col] = b[r];
        b[r] = t;
      }
    }
#pragma unroll
    for (int r = col + 1; r < 5; ++r) {
      const double f = a[r][col] / a[col][col];
#pragma unroll
      for (int cc = col; cc < 5; ++cc) a[r][cc] -= f * a[col][cc];
      b[r] -= f * b[col];
    }
  }
#pragma unroll
  for (int r = 4; r >= 0; --r) {
    double acc = b[r];
#pragma unroll
    for (int cc = r + 1; cc < 5; ++cc) acc -= a[r][cc] * x[cc];
    x[r] = acc / a[r][r];
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) x[j] *= scale[j];
  return true;
}

// lane -> (i, j) of the 15 unique A^T A entries; lanes 15..19 own A^T b[i].
__device__ __forceinline__ void acc_slot(int lane, int& i, int& j) {
  const int ti[15] = {0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 3, 3, 4};
  const int tj[15] = {0, 1, 2, 3, 4, 1, 2, 3, 4, 2, 3, 4, 3, 4, 4};
  if (lane < 15) {
    i = ti[lane];
    j = tj[lane];
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

__device__ __forceinline__ void gather_normal(double acc, double ata[5][5], double atb[5]) {
#pragma unroll
  for (int i = 0; i < 5; ++i) {
#pragma unroll
    for (int j = 0; j < 5; ++j) ata[i][j] = __shfl_sync(NX_FULL, acc, slot_of(i, j));
    atb[i] = __shfl_sync(NX_FULL, acc, 15 + i);
  }
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
  __device__ __forceinline__ int slot(int i) const { return (head + size - n + i) % size; }
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
__device__ bool update_linear(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const Window w = window_of(c, e, c.d->short_w);
  const int n = w.n;
  if (n < 5) return false;
  const Params cur = g.lp;
  double* rows = c.scratch + c.d->long_w + kFbTable;  // (1/thr, s/thr) per sample
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
  double ata[5][5], atb[5];
  gather_normal(acc, ata, atb);
  const double y2 = static_cast<double>(n);
  const double prior[5] = {cur.tau0, cur.w0, cur.ws, cur.tauB, cur.tauS};
  double x[5];
  bool ok;
  {
    double a[5][5], bb[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      bb[i] = atb[i];
#pragma unroll
      for (int j = 0; j < 5; ++j) a[i][j] = ata[i][j];
    }
    ok = solve5(a, bb, x);
  }
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
    if (lambda > 1e-14) {
      double a[5][5], bb[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        bb[i] = atb[i];
#pragma unroll
        for (int j = 0; j < 5; ++j) a[i][j] = ata[i][j];
      }
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const double d = lambda * ata[i][i];
        a[i][i] += d;
        bb[i] += d * prior[i];
      }
      ok = solve5(a, bb, x);
    }
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
    g.cnt[0] += 1;
    if (clamped) g.cnt[4] += 1;
  }
  __syncwarp();
  return true;
}

// ---- structural tier (learner.cpp:209-298, 346-440) --------------------------

// windowed_sse (learner.cpp:209-222) with direct model evaluation.
__device__ double wsse_tree(Ctx& c, const Window& w, const Params& p) {
  double part = 0.0;
  for (int i = c.lane; i < w.n; i += 32) {
    const int k = w.slot(i);
    const double y = w.ry[k];
    const double r = (y - predict(p, w.rb[k], w.rs[k])) / y;
    part += r * r;
  }
  return warp_sum(part);
}
__device__ double wsse_exact(Ctx& c, const Window& w, const Params& p) {
  double run = 0.0;
  for (int base = 0; base < w.n; base += 32) {
    const int i = base + c.lane;
    double rr = 0.0;
    if (i < w.n) {
      const int k = w.slot(i);
      const double y = w.ry[k];
      const double r = (y - predict(p, w.rb[k], w.rs[k])) / y;
      rr = r * r;
    }
    fold_exact_chunk(c, rr, min(32, w.n - base), run);
  }
  return __shfl_sync(NX_FULL, run, 0);
}

// Certified "a < b * f" between two windowed SSE values whose tree sums are
// a_t, b_t; falls back to exact folds when the tree cannot decide.
__device__ bool less_scaled(Ctx& c, const Window& w, double a_t, const Params& pa, double b_t,
                            const Params& pb, double f) {
  const double rhs = b_t * f;
  if (a_t < rhs * (1.0 - kCertMargin)) return true;
  if (a_t > rhs * (1.0 + kCertMargin)) return false;
  const double a = wsse_exact(c, w, pa);
  const double b = wsse_exact(c, w, pb);
  return a < b * f;
}

struct FitOut {
  Params p;
  double err;  // tree value; +inf when the solve failed
};

// gauged_fit (learner.cpp:228-298) for fixed (kB, kS).
__device__ FitOut gauged_fit(Ctx& c, const Window& w, const Params& cur, double kB, double kS,
                             int bmax) {
  const int n = w.n;
  double* fs_cache = c.scratch;
  double* fbt = c.scratch + c.d->long_w;  // raw batch factors, index b
  const int tab = bmax < kFbTable ? bmax : kFbTable - 1;
  __syncwarp();
  for (int b = 1 + c.lane; b <= tab; b += 32) fbt[b] = raw_factor(kB, static_cast<double>(b));
  __syncwarp();
  double acc = 0.0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + c.lane;
    __syncwarp();
    if (i < n) {
      const int k = w.slot(i);
      const int bi = w.rb[k];
      const double b = bi, s = w.rs[k], y = w.ry[k];
      const double fb = bi <= tab ? fbt[bi] : raw_factor(kB, b);
      const double fs = raw_factor(kS, s);
      fs_cache[i] = fs;
      double f = fb * fs;
      f = (f < 1e-300) ? 1e-300 : f;
      const double iy = 1.0 / y;
      double* row = c.chunk + c.lane * 5;
      row[0] = 1.0 * iy;
      row[1] = (1.0 / f) * iy;
      row[2] = (s / f) * iy;
      row[3] = b * iy;
      row[4] = s * iy;
    }
    __syncwarp();
    fold_chunk(c, min(32, n - base), acc);
  }
  double ata[5][5], atb[5];
  gather_normal(acc, ata, atb);
  const double y2 = static_cast<double>(n);
  const double prior[5] = {cur.tau0, cur.w0 / cur.p_max, cur.ws / cur.p_max, cur.tauB, cur.tauS};
  FitOut out;
  out.err = __longlong_as_double(0x7ff0000000000000LL);
  double x[5];
  {
    double a[5][5], bb[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      bb[i] = atb[i];
#pragma unroll
      for (int j = 0; j < 5; ++j) a[i][j] = ata[i][j];
    }
    if (!solve5(a, bb, x)) return out;
  }
  // residual of the unweighted rows under x (lambda scale)
  auto resid = [&](int i) {
    const int k = w.slot(i);
    const int bi = w.rb[k];
    const double b = bi, s = w.rs[k], y = w.ry[k];
    const double fb = bi <= tab ? fbt[bi] : raw_factor(kB, b);
    double f = fb * fs_cache[i];
    f = (f < 1e-300) ? 1e-300 : f;
    double pred = 0.0;
    pred += 1.0 * x[0];
    pred += (1.0 / f) * x[1];
    pred += (s / f) * x[2];
    pred += b * x[3];
    pred += s * x[4];
    const double r = (y - pred) / y;
    return r * r;
  };
  double part = 0.0;
  for (int i = c.lane; i < n; i += 32) part += resid(i);
  const double sse_t = warp_sum(part);
  const double den = (y2 < 1e-30) ? 1e-30 : y2;
  double lambda = 1e-7;
  if (!(sse_t / den > 1e-7 * (1.0 + kCertMargin))) {
    double run = 0.0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + c.lane;
      fold_exact_chunk(c, i < n ? resid(i) : 0.0, min(32, n - base), run);
    }
    const double v = __shfl_sync(NX_FULL, run, 0) / den;
    lambda = (v < 1e-7) ? v : 1e-7;
  }
  if (lambda > 1e-14) {
    double a[5][5], bb[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      bb[i] = atb[i];
#pragma unroll
      for (int j = 0; j < 5; ++j) a[i][j] = ata[i][j];
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const double d = lambda * ata[i][i];
      a[i][i] += d;
      bb[i] += d * prior[i];
    }
    if (!solve5(a, bb, x)) return out;
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
  // windowed_sse(samples, p) reusing this fit's factors (same kB, kS)
  part = 0.0;
  for (int i = c.lane; i < n; i += 32) {
    const int k = w.slot(i);
    const int bi = w.rb[k];
    const double b = bi, s = w.rs[k], y = w.ry[k];
    const double fb = clamp_factor(bi <= tab ? fbt[bi] : raw_factor(kB, b));
    const double thr = p.p_max * fb * clamp_factor(fs_cache[i]);
    const double work = p.w0 + p.ws * s;
    const double T = p.tau0 + work / thr + p.tauB * b + p.tauS * s;
    const double r = (y - T) / y;
    part += r * r;
  }
  out.err = warp_sum(part);
  return out;
}

__device__ void update_structural(Ctx& c, int e) {
  EngSm& g = c.eng[e];
  const Window w = window_of(c, e, c.d->long_w);
  const int n = w.n;
  if (n < c.d->min_s || n < 5) return;
  const Params cur = g.lp;
  bool unsat = false;
  int shaped = 0, bmax = 1;
  for (int i = c.lane; i < n; i += 32) {
    const int k = w.slot(i);
    const int b = w.rb[k], s = w.rs[k];
    if (cur.kB * static_cast<double>(b) < 20.0 || cur.kS * static_cast<double>(s) < 20.0) unsat = true;
    if (s >= 64 && s >= 4 * b) ++shaped;
    bmax = max(bmax, b);
  }
  const bool saturated = !__any_sync(NX_FULL, unsat);
  shaped = static_cast<int>(__reduce_add_sync(NX_FULL, static_cast<unsigned>(shaped)));
  bmax = warp_max_int(bmax);
  if (saturated || shaped < 16) {
    __syncwarp();
    if (c.lane == 0) g.cnt[6] += 1;
    __syncwarp();
    return;
  }
  const double base_t = wsse_tree(c, w, cur);
  const double lo = log(1e-8), hi = log(1e4);
  const double shrink = 1.0 - 1e-3;
  double th0 = log(cur.kB), th1 = log(cur.kS);
  double st0 = 0.5, st1 = 0.5;
  FitOut best = gauged_fit(c, w, cur, exp(th0), exp(th1), bmax);
  if (!isfinite(best.err)) {
    __syncwarp();
    if (c.lane == 0) g.cnt[5] += 1;
    __syncwarp();
    return;
  }
  const double kbs[3] = {0.05, 0.7, 8.0}, kss[3] = {0.002, 0.03, 0.4};
  for (int a = 0; a < 3; ++a) {
    for (int bq = 0; bq < 3; ++bq) {
      const FitOut cand = gauged_fit(c, w, cur, kbs[a], kss[bq], bmax);
      if (isfinite(cand.err) && less_scaled(c, w, cand.err, cand.p, best.err, best.p, shrink)) {
        th0 = log(kbs[a]);
        th1 = log(kss[bq]);
        best = cand;
      }
    }
  }
  for (int sweep = 0; sweep < 50; ++sweep) {
    bool improved = false;
    for (int cdim = 0; cdim < 2; ++cdim) {
      bool hit = false;
      for (int dir = 0; dir < 2 && !hit; ++dir) {
        const double sgn = dir == 0 ? 1.0 : -1.0;
        double t0 = th0, t1 = th1;
        double& tc = cdim == 0 ? t0 : t1;
        const double v = tc + sgn * (cdim == 0 ? st0 : st1);
        tc = (v < lo) ? lo : ((hi < v) ? hi : v);
        if (tc == (cdim == 0 ? th0 : th1)) continue;
        const FitOut cand = gauged_fit(c, w, cur, exp(t0), exp(t1), bmax);
        if (isfinite(cand.err) && less_scaled(c, w, cand.err, cand.p, best.err, best.p, shrink)) {
          th0 = t0;
          th1 = t1;
          best = cand;
          hit = true;
        }
      }
      if (cdim == 0) st0 *= hit ? 1.6 : 0.5;
      else st1 *= hit ? 1.6 : 0.5;
      improved |= hit;
    }
    const double smax = (st0 < st1) ? st1 : st0;
    if (!improved && smax < 1e-5) break;
  }
  // reject if invalid or worse than the current model (learner.cpp:432-435)
  bool worse;
  if (best.err > base_t * (1.0 + kCertMargin)) worse = true;
  else if (best.err < base_t * (1.0 - kCertMargin)) worse = false;
  else worse = wsse_exact(c, w, best.p) > wsse_exact(c, w, cur);
  if (!params_valid(best.p) || worse) {
    __syncwarp();
    if (c.lane == 0) g.cnt[5] += 1;
    __syncwarp();
    return;
  }
  __syncwarp();
  if (c.lane == 0) {
    g.lp = best.p;
    g.cnt[1] += 1;
  }
  __syncwarp();
  update_linear(c, e);
}

// record_sample (learner.cpp:130-146): ring push + periodic refits.
__device__ void record_sample(Ctx& c, int e, int b, int s, double y) {
  EngSm& g = c.eng[e];
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
      g.ring_head = (g.ring_head + 1) % g.ring_size;
    }
    c.P->ring_b[ed.ring_off + slot] = b;
    c.P->ring_s[ed.ring_off + slot] = s;
    c.P->ring_y[ed.ring_off + slot] = y;
    g.seen += 1;
  }
  __syncwarp();
  const int64_t seen = g.seen;
  if (seen % c.d->l_period == 0) update_linear(c, e);
  if (seen >= c.d->min_s && seen % c.d->s_period == 0) update_structural(c, e);
}

}  // namespace nxd
