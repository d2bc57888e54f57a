// Microbenchmark: cycles per solve5_warp_k<K> call on one warp (diagnostic).
#include <cstdio>
#include "../../paper_2509_23384_b200/csrc/device/nx_learner.cuh"
using namespace nxd;

template <int K>
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
    solve5_warp_k<K>(vv, x, ok);
    acc += x[0][0] + (ok[0] ? 1.0 : 0.0);
  }
  long long t1 = clock64();
  if (lane == 0) { out[blockIdx.x] = acc; cyc[blockIdx.x] = (t1 - t0) / iters; }
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 8 * 64); cudaMalloc(&c, 8 * 64);
  long long h[1];
  bench<1><<<1, 32>>>(d, c, 200); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost); printf("K=1: %lld cycles/call\n", h[0]);
  bench<2><<<1, 32>>>(d, c, 200); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost); printf("K=2: %lld cycles/call\n", h[0]);
  return 0;
}
