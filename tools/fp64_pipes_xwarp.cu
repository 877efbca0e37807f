// Cross-warp mixing of DMMA and DFMA on one SM sub-partition (sm_100a).  WPS warps per
// sub-partition; the first NV of them run only DFMA (F independent chains per iteration), the
// others only DMMA (4 independent chains per iteration).  Does a vector-FP64 warp running next
// to a DMMA warp cost the 2 cycles per DFMA it costs alone, or more?  Reports the time of the
// mixed launch, of the DMMA warps alone and of the DFMA warps alone (same iteration counts).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_pipes_xwarp tools/fp64_pipes_xwarp.cu
#include <cstdio>
#include <cuda_runtime.h>

// mode: 0 mixed, 1 only the DMMA warps work, 2 only the DFMA warps work
template <int F>
__global__ void xmix(double* out, int iters_d, int iters_f, int nv, int mode) {
  const int warp = threadIdx.x >> 5;
  const int wslot = warp >> 2;                 // index of the warp on its sub-partition (warp % 4 = SMSP)
  const bool vec = wslot < nv;
  double d[4][2], f[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k][0] = d[k][1] = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = 1e-3 * k;
  const double a = 1e-3 * threadIdx.x, b = 0.5, c = 0.999;
  if (vec) {
    if (mode != 1)
      for (int i = 0; i < iters_f; ++i) {
#pragma unroll
        for (int k = 0; k < F; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k & 7]) : "d"(c), "d"(a));
      }
  } else if (mode != 2) {
    for (int i = 0; i < iters_d; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int F>
float timed(int sms, double* o, int wps, int nv, int id, int iff, int mode) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  xmix<F><<<sms, 128 * wps>>>(o, id, iff, nv, mode);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) xmix<F><<<sms, 128 * wps>>>(o, id, iff, nv, mode);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5.0f;
}

template <int F>
void run(int sms, double* o, int wps, int nv, double ratio) {
  // DMMA warps: 4096 iterations of 4 DMMAs (64 pipe cycles each); DFMA warps: iterations chosen
  // so that their stand-alone pipe time is `ratio` of the DMMA warps' total
  const int id = 4096;
  const int nd = wps - nv;
  const int iff = (int)(ratio * id * 64.0 * nd / (2.0 * F * nv));
  const float tm = timed<F>(sms, o, wps, nv, id, iff, 0), td = timed<F>(sms, o, wps, nv, id, iff, 1),
              tf = timed<F>(sms, o, wps, nv, id, iff, 2);
  printf("{\"warps_per_smsp\": %d, \"dfma_warps\": %d, \"dfma_per_iter\": %d, \"dfma_iters\": %d, "
         "\"dfma_share_of_dmma_time\": %.2f, \"ms_mixed\": %.4f, \"ms_dmma_only\": %.4f, \"ms_dfma_only\": %.4f, "
         "\"mixed_over_sum\": %.3f}\n", wps, nv, F, iff, ratio, tm, td, tf, tm / (td + tf));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, (size_t)sms * 1024 * 8);
  for (double ratio : {0.1, 0.25, 0.5}) {
    run<8>(sms, o, 2, 1, ratio);
    run<8>(sms, o, 3, 1, ratio);
    run<8>(sms, o, 4, 1, ratio);
    run<8>(sms, o, 4, 2, ratio);
    run<1>(sms, o, 2, 1, ratio);    // one dependent chain: latency-bound vector warp
  }
  return 0;
}
