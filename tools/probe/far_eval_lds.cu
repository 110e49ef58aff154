// The column-stream far-field inner loop in isolation (synthetic data, no
// global traffic): R target rows broadcast from shared memory (two 16 B + one
// 8 B load per row), C source columns per lane, per-row accumulators in
// registers.  Reports evaluations / s for (R, C, CTAs per SM).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rs(double x) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  return y0 * fma(-x * y0, y0, 3.0);
}
template <int R, int C, int MINB>
__global__ void __launch_bounds__(256, MINB) evals(double* out, int iters) {
  __shared__ __align__(16) double sh[8][5 * 32];
  double* rw = sh[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < R; i += 32) {
    rw[4 * i] = -0.1 * i; rw[4 * i + 1] = 0.02 * i; rw[4 * i + 2] = 0.01; rw[4 * i + 3] = 0.005 * i + 0.01;
    rw[4 * R + i] = 1.0 + i;
  }
  __syncwarp();
  double acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.0;
  double sx[C], sy[C], sz[C], ns[C], xs[C], ps[C];
#pragma unroll
  for (int k = 0; k < C; ++k) { sx[k] = 1.0 + 1e-3 * (lane + k); sy[k] = 0.5; sz[k] = 0.25; xs[k] = 1.0; ps[k] = 0.0; }
  for (int it = 0; it < iters; ++it) {
    asm volatile("" ::: "memory");  // the row loads stay in the loop (as in the kernel, per column chunk)
#pragma unroll
    for (int k = 0; k < C; ++k) { sx[k] = sx[k] + 1e-12; ns[k] = sx[k] * sx[k] + 0.3125; }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 a01 = *reinterpret_cast<const double2*>(rw + 4 * r);
      const double2 a23 = *reinterpret_cast<const double2*>(rw + 4 * r + 2);
      const double xt = rw[4 * R + r];
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const double r2 = fma(a01.x, sx[k], fma(a01.y, sy[k], fma(a23.x, sz[k], a23.y + ns[k])));
        const double g = rs(r2);
        acc[r] = fma(g, xs[k], acc[r]);
        ps[k] = fma(g, xt, ps[k]);
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) t += acc[r];
#pragma unroll
  for (int k = 0; k < C; ++k) t += ps[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int R, int C, int MINB>
void run(double* out, int nsm) {
  const int threads = 256, blocks = nsm * MINB * 4, iters = 400;
  evals<R, C, MINB><<<blocks, threads>>>(out, 5);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); evals<R, C, MINB><<<blocks, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, evals<R, C, MINB>);
  const double ev = (double)blocks * threads * iters * R * C;
  printf("R=%2d C=%d MINB=%d regs=%3d local=%zu: %.3f T evals/s (%.3f ms)\n", R, C, MINB, fa.numRegs,
         fa.localSizeBytes, ev / ms / 1e9, ms);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * nsm * 16 * 256);
  run<25, 1, 2>(out, nsm); run<25, 2, 2>(out, nsm); run<25, 2, 3>(out, nsm); run<25, 3, 2>(out, nsm);
  run<25, 4, 2>(out, nsm); run<25, 4, 1>(out, nsm);
  run<13, 2, 3>(out, nsm); run<13, 4, 2>(out, nsm); run<13, 4, 3>(out, nsm); run<13, 6, 2>(out, nsm);
  run<8, 4, 3>(out, nsm); run<8, 8, 2>(out, nsm);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
