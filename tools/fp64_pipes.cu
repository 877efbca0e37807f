// Do DMMA (mma.sync m8n8k4 f64) and DFMA share one issue resource on sm_100a?
// Each warp runs ITERS iterations of D independent DMMAs plus F independent DFMAs
// (8 accumulator chains each); WPS warps per SM sub-partition.  If the pipes are
// separate, time(D, F) ~ max(time(D, 0), time(0, F)); if shared, ~ the sum.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_pipes tools/fp64_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int D, int F>
__global__ void mix(double* out, int iters) {
  double d[4][2];
  double f[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k][0] = d[k][1] = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = 1e-3 * k;
  const double a = 1e-3 * threadIdx.x, b = 0.5, c = 0.999;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < (D > F ? D : F); ++k) {
      if (k < D)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[k & 3][0]), "+d"(d[k & 3][1]) : "d"(a), "d"(b));
      if (k < F) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k & 7]) : "d"(c), "d"(a));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int D, int F>
void run(int sms, double* o, int wps) {
  const int threads = 128 * wps, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<D, F><<<sms, threads>>>(o, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) mix<D, F><<<sms, threads>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz (max)
  // SMSP cycles per iteration per warp at the max clock
  const double cyc = (ms * 1e-3 / 5.0) * clk * 1e3 / ((double)iters * wps);
  printf("{\"wps\": %d, \"dmma\": %d, \"dfma\": %d, \"ms\": %.4f, \"smsp_cycles_per_warp_iter\": %.2f}\n", wps, D, F,
         ms / 5.0, cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, (size_t)sms * 1024 * 8);
  for (int wps : {2, 4}) {
    run<4, 0>(sms, o, wps);
    run<0, 8>(sms, o, wps);
    run<0, 16>(sms, o, wps);
    run<0, 32>(sms, o, wps);
    run<4, 4>(sms, o, wps);
    run<4, 8>(sms, o, wps);
    run<4, 16>(sms, o, wps);
    run<4, 32>(sms, o, wps);
  }
  return 0;
}
