// Device math shared by every kernel: the perf model (Eq. 1-2), xoshiro256++,
// warp helpers. Compiled with --fmad=false: the reference build has no FMA
// contraction (proj/CMakeLists.txt:1-8, x86-64 baseline), so every a*b+c here
// rounds twice exactly like the host code it replaces.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define NX_FULL 0xffffffffu

namespace nxd {

struct Params {  // PerfParams field order (proj/include/servesim/perf_model.h:14-27)
  double tau0, w0, ws, tauB, tauS, p_max, kB, kS;
};

__device__ __forceinline__ Params params_from(const double* p) {
  Params q;
  q.tau0 = p[0]; q.w0 = p[1]; q.ws = p[2]; q.tauB = p[3];
  q.tauS = p[4]; q.p_max = p[5]; q.kB = p[6]; q.kS = p[7];
  return q;
}
__device__ __forceinline__ void params_to(const Params& q, double* p) {
  p[0] = q.tau0; p[1] = q.w0; p[2] = q.ws; p[3] = q.tauB;
  p[4] = q.tauS; p[5] = q.p_max; p[6] = q.kB; p[7] = q.kS;
}
__device__ __forceinline__ bool params_valid(const Params& p) {  // perf_model.cpp:33-36
  return p.p_max > 0.0 && p.kB > 0.0 && p.kS > 0.0 && p.tau0 >= 0.0 && p.tauB >= 0.0 &&
         p.tauS >= 0.0 && p.ws > 0.0 && p.w0 >= 0.0;
}

// nextafter(1.0, 0.0): saturation factors are clamped just below one
// (perf_model.cpp:12-20).
constexpr double kFactorMax = 0x1.fffffffffffffp-1;

// -expm1(-kx) for kx >= 45: e^-45 < 2^-64, so the exact value 1 - e^-kx
// rounds to 1.0 in double (any expm1 within 1 ulp returns -1 there); the
// transcendental is skipped. Most LENS probes (S in the thousands) and
// large-batch f_B arguments sit in this saturated range.
constexpr double kSatArg = 45.0;

// The simulation kernel can call one out-of-line copy of expm1
// (NX_COMPACT_MATH); streaming kernels (K1) keep it inline.
#ifdef NX_COMPACT_MATH
static __device__ __noinline__ double expm1_neg(double kx) { return -expm1(-kx); }
#else
__device__ __forceinline__ double expm1_neg(double kx) { return -expm1(-kx); }
#endif
// 1 - e^-x for x in [0, kSatArg): a branch-free expm1 for the streaming
// evaluator (K1), ~22 instructions instead of libm's general expm1. With
// y = -x = k ln2 + r, |r| <= ln2/2: expm1(y) = 2^k expm1(r) + (2^k - 1), and
// expm1(r) = r + r^2 P(r) with the degree-13 Taylor polynomial (truncation
// below 1e-17 relative). Within ~1 ulp of the correctly rounded value; K1's
// contract is 1e-9 relative in fp64 mode, and the simulator keeps libm's
// expm1 (bit-for-bit decisions are certified against it).
// Coefficients in the constant bank: a DFMA reads a c[bank][offset] operand
// directly, while an inline FP64 immediate costs two UMOVs per use (the K1
// loop issued more UMOVs than DFMAs before).
static __constant__ double kOmeC[16] = {
    1.4426950408889634,          // 1 / ln2
    6.93147180369123816490e-01,  // ln2 hi
    1.90821492927058770002e-10,  // ln2 lo
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0,
    1.0 / 40320.0, 1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0};
__device__ __forceinline__ double one_minus_exp_neg(double x) {
  const double y = -x;
  const double kd = rint(y * kOmeC[0]);                    // y / ln2
  const double r0 = fma(-kd, kOmeC[1], y);                 // ln2 hi
  const double r = fma(-kd, kOmeC[2], r0);                 // ln2 lo
  double p = kOmeC[3];                                     // 1/13!
#pragma unroll
  for (int i = 4; i < 15; ++i) p = fma(p, r, kOmeC[i]);    // ... 1/3!, 1/2
  const double em = fma(r * r, p, r);                      // expm1(r)
  const double s = __longlong_as_double(static_cast<long long>(1023 + static_cast<int>(kd)) << 52);  // 2^k
  return fma(-s, em, kOmeC[15] - s);                       // -(2^k em + 2^k - 1)
}
__device__ __forceinline__ double sat_fast(double k, double x) {
  const double kx = k * x;
  const double f = one_minus_exp_neg(kx);
  return kx >= kSatArg ? kFactorMax : (f < kFactorMax ? f : kFactorMax);
}

__device__ __forceinline__ double raw_factor(double k, double x) {
  const double kx = k * x;
  return kx >= kSatArg ? 1.0 : expm1_neg(kx);
}
__device__ __forceinline__ double clamp_factor(double f) { return f < kFactorMax ? f : kFactorMax; }
__device__ __forceinline__ double sat(double k, double x) { return clamp_factor(raw_factor(k, x)); }

// T(B,S) given the (clamped) batch factor fb — lets callers that sweep S at a
// fixed B reuse fb; bitwise identical to predict_latency (perf_model.cpp:44-49).
__device__ __forceinline__ double latency_fb(const Params& p, double fb, double b, double s) {
  const double thr = p.p_max * fb * sat(p.kS, s);
  const double work = p.w0 + p.ws * s;
  return p.tau0 + work / thr + p.tauB * b + p.tauS * s;
}
__device__ __forceinline__ double predict(const Params& p, double b, double s) {
  return latency_fb(p, sat(p.kB, b), b, s);
}
__device__ __forceinline__ double throughput(const Params& p, double b, double s) {
  return p.p_max * sat(p.kB, b) * sat(p.kS, s);
}

__device__ __forceinline__ int64_t to_us(double ms) { return llround(ms * 1000.0); }
__device__ __forceinline__ double to_ms(int64_t us) { return static_cast<double>(us) / 1000.0; }

// FNV-1a over the 8 little-endian bytes of v (sim.cpp:24-30).
__device__ __forceinline__ uint64_t fnv1a(uint64_t h, uint64_t v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 0x100000001b3ULL;
  }
  return h;
}

// P^k for the FNV prime P: a zero byte leaves h ^ 0 = h, so k trailing zero
// bytes of a field collapse into one multiply by P^k.
constexpr uint64_t kFnvP1 = 0x00000100000001b3ull, kFnvP3 = 0x08a97b0004e7feabull,
                   kFnvP4 = 0x9ffaac085635bc91ull, kFnvP7 = 0xc5527b8a51d3d2dbull;

__device__ __forceinline__ uint64_t fnv_bytes(uint64_t h, uint64_t v, int nbytes) {
#pragma unroll
  for (int i = 0; i < nbytes; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= kFnvP1;
  }
  return h;
}

// The event fingerprint of sim.cpp:302-305 — fnv1a over (time_us, kind,
// engine_id + 1, request_id). Straight-line fast path for the common widths
// (time < 2^40 us, engine id + 1 < 256, request id < 2^32): 11 byte rounds +
// 4 power multiplies instead of 32 rounds; identical value.
__device__ __forceinline__ uint64_t fnv_event(uint64_t h, uint64_t t, uint64_t kind, uint64_t eid1,
                                              uint64_t rid) {
  if ((t >> 40) == 0 && (eid1 >> 8) == 0 && (rid >> 32) == 0 && (kind >> 8) == 0) {
    h = fnv_bytes(h, t, 5) * kFnvP3;
    h = ((h ^ kind) * kFnvP1) * kFnvP7;
    h = ((h ^ eid1) * kFnvP1) * kFnvP7;
    return fnv_bytes(h, rid, 4) * kFnvP4;
  }
  return fnv1a(fnv1a(fnv1a(fnv1a(h, t), kind), eid1), rid);
}

// xoshiro256++ (proj/include/servesim/rng.h:19-45)
struct Rng {
  uint64_t s[4];
  __device__ __forceinline__ static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t out = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
  }
  __device__ __forceinline__ double uniform() {
    return (static_cast<double>(next() >> 11) + 1.0) * 0x1.0p-53;
  }
  __device__ __forceinline__ double normal() {
    const double u1 = uniform();
    const double u2 = uniform();
    return sqrt(-2.0 * log(u1)) * cos((2.0 * 3.141592653589793) * u2);
  }
};

// ---- warp helpers -----------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(NX_FULL, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Fixed-order butterfly sum: every lane ends with the bitwise-same value
// (each level adds commuting pairs), and the order never depends on timing.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(NX_FULL, v, o);
  return v;
}
__device__ __forceinline__ int warp_max_int(int v) {
  return static_cast<int>(__reduce_max_sync(NX_FULL, static_cast<unsigned>(v)));
}

}  // namespace nxd
