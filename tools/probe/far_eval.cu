// Throughput ceiling of the far-field evaluation's instruction mix on this B200:
// per evaluation r2 = fma(ax, sx, fma(ay, sy, fma(az, sz, nt + ns))), MUFU.RSQ64H
// + one Newton step, two accumulating FMAs (9 FP64 + 1 MUFU), with K independent
// evaluations per thread in flight; reports evaluations / s and FP64 instr / s
// (one extra DADD per 8 K evaluations keeps the rows loop-variant).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rs(double x) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  return y0 * fma(-x * y0, y0, 3.0);
}
template <int K>
__global__ void evals(double* out, int iters) {
  double sx[K], sy[K], sz[K], ns[K], xs[K], ps[K];
  for (int k = 0; k < K; ++k) {
    sx[k] = 1.0 + 1e-3 * (threadIdx.x + k); sy[k] = 0.5; sz[k] = 0.25; ns[k] = sx[k] * sx[k] + 0.3125;
    xs[k] = 1.0; ps[k] = 0.0;
  }
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double drift = 1e-3 * threadIdx.x;  // changes every iteration: nothing is loop-invariant
  for (int i = 0; i < iters; ++i) {
    drift = drift + 1e-12;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double ax = drift - 0.1 * r, ay = 0.02 * r, az = 0.01, nt = 0.005 * r + 0.01, xt = 1.0 + r;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double r2 = fma(ax, sx[k], fma(ay, sy[k], fma(az, sz[k], nt + ns[k])));
        const double g = rs(r2);
        acc[r] = fma(g, xs[k], acc[r]);
        ps[k] = fma(g, xt, ps[k]);
      }
    }
  }
  double t = 0;
  for (int r = 0; r < 8; ++r) t += acc[r];
  for (int k = 0; k < K; ++k) t += ps[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int K>
void run(double* out, int nsm, int warps_per_sm) {
  const int threads = 256, blocks = nsm * warps_per_sm / 8, iters = 2000;
  evals<K><<<blocks, threads>>>(out, 10);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); evals<K><<<blocks, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double ev = (double)blocks * threads * iters * 8 * K;
  printf("K=%d warps/SM=%d: %.3f T evals/s, %.2f T FP64 instr/s (%.3f ms)\n", K, warps_per_sm, ev / ms / 1e9,
         9 * ev / ms / 1e9, ms);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * nsm * 64 * 32 * 4);
  for (int w : {16, 24, 32, 48}) { run<2>(out, nsm, w); run<4>(out, nsm, w); }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
