// Microbenchmark: cycles per solve5_warp_k<K> call on one warp (diagnostic).
#include <cstdio>
#include "../../paper_2509_23384_b200/csrc/device/nx_learner.cuh"
using namespace nxd;


// serial per-lane variant (reference op order), lane k solves system k
template <int K>
__device__ __forceinline__ void solve5_lanes(const double (&v)[K], double (&x)[K][5], bool (&ok)[K]) {
  const int lane = lane_id();
  double a[5][5], b[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) { const double g = __shfl_sync(NX_FULL, v[k], 5 * i + j); if (lane == k) t = g; }
      a[i][j] = t;
    }
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) { const double g = __shfl_sync(NX_FULL, v[k], 25 + i); if (lane == k) t = g; }
    b[i] = t;
  }
  bool good = true;
  double scale[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) m = dmax(m, fabs(a[i][j]));
    good = good && m > 0.0;
    scale[j] = m > 0.0 ? 1.0 / m : 1.0;
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
    int pivot = col;
    double pv = fabs(a[col][col]);
#pragma unroll
    for (int r = col + 1; r < 5; ++r) if (fabs(a[r][col]) > pv) { pivot = r; pv = fabs(a[r][col]); }
    good = good && !(pv < 1e-10 * norm);
#pragma unroll
    for (int r = col + 1; r < 5; ++r) {
      const bool sw = pivot == r;
#pragma unroll
      for (int c2 = 0; c2 < 5; ++c2) { const double t0 = a[col][c2], t1 = a[r][c2]; a[col][c2] = sw ? t1 : t0; a[r][c2] = sw ? t0 : t1; }
      const double u0 = b[col], u1 = b[r]; b[col] = sw ? u1 : u0; b[r] = sw ? u0 : u1;
    }
#pragma unroll
    for (int r = col + 1; r < 5; ++r) {
      const double f = a[r][col] / a[col][col];
#pragma unroll
      for (int c2 = col; c2 < 5; ++c2) a[r][c2] -= f * a[col][c2];
      b[r] -= f * b[col];
    }
  }
  double out[5];
#pragma unroll
  for (int r = 4; r >= 0; --r) {
    double acc = b[r];
#pragma unroll
    for (int c2 = r + 1; c2 < 5; ++c2) acc -= a[r][c2] * out[c2];
    out[r] = acc / a[r][r];
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) out[j] *= scale[j];
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int q = 0; q < 5; ++q) x[k][q] = __shfl_sync(NX_FULL, out[q], k);
    ok[k] = __shfl_sync(NX_FULL, good ? 1 : 0, k) != 0;
  }
}

template <int K, bool kSerial>
__global__ void bench(double* out, long long* cyc, int iters) {
  const int lane = threadIdx.x & 31;
  // a well-conditioned SPD-ish normal matrix per system
  double v[K];
  for (int k = 0; k < K; ++k) {
    const int i = lane / 5, j = lane % 5;
    v[k] = lane < 25 ? (i == j ? 10.0 + i + k : 1.0 / (1 + i + j)) : (lane < 30 ? 1.0 + lane - 25 : 0.0);
  }
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double vv[K], x[K][5];
    bool ok[K];
    for (int k = 0; k < K; ++k) vv[k] = v[k] * (1.0 + 1e-9 * it);
    if (kSerial) solve5_lanes<K>(vv, x, ok); else solve5_warp_k<K>(vv, x, ok);
    acc += x[0][0] + (ok[0] ? 1.0 : 0.0);
  }
  long long t1 = clock64();
  if (lane == 0) { out[blockIdx.x] = acc; cyc[blockIdx.x] = (t1 - t0) / iters; }
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 8 * 64); cudaMalloc(&c, 8 * 64);
  long long h[1];
  bench<1, false><<<1, 32>>>(d, c, 200); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost); printf("warp   K=1: %lld cycles/call\n", h[0]);
  bench<2, false><<<1, 32>>>(d, c, 200); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost); printf("warp   K=2: %lld cycles/call\n", h[0]);
  bench<1, true><<<1, 32>>>(d, c, 200); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost); printf("serial K=1: %lld cycles/call\n", h[0]);
  bench<2, true><<<1, 32>>>(d, c, 200); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost); printf("serial K=2: %lld cycles/call\n", h[0]);
  return 0;
}
