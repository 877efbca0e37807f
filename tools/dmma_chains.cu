// DMMA (mma.sync m8n8k4 f64) throughput vs independent accumulator chains in flight per SM
// sub-partition: WPS warps per SMSP (one CTA of 4*WPS warps per SM) x CH chains per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_chains tools/dmma_chains.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chains(double* out, int iters) {
  double d[CH][2];
#pragma unroll
  for (int k = 0; k < CH; ++k) d[k][0] = d[k][1] = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
void run(int sms, double* o, int wps) {
  const int threads = 128 * wps, iters = 8192 / CH;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chains<CH><<<sms, threads>>>(o, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) chains<CH><<<sms, threads>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = 5.0 * iters * CH * (threads / 32) * (double)sms;
  printf("{\"warps_per_smsp\": %d, \"chains_per_warp\": %d, \"TFLOPs\": %.2f}\n", wps, CH,
         mmas * 512 / (ms * 1e-3) / 1e12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, (size_t)sms * 1024 * 8);
  for (int wps : {1, 2, 3, 4, 8}) {
    run<1>(sms, o, wps);
    run<2>(sms, o, wps);
    run<4>(sms, o, wps);
    run<8>(sms, o, wps);
  }
  return 0;
}
