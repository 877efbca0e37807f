// membench.cu -- B200 ceilings for the 1D SEM hot path's data-movement skeleton
// and FP64 pipes (not part of the product; results go to profiles/).
//   copy_ldg   : grid-stride double2 load/store copy (the STREAM-style ceiling)
//   copy_tma   : persistent CTAs, 1D bulk-tensor loads into a smem ring
//                (mbarrier complete_tx), bulk stores back out -- the skeleton of
//                the operator kernels without any arithmetic
//   dfma_peak  : dependent-chain-free DFMA throughput
//   dmma_peak  : mma.sync m8n8k4 f64 throughput
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void copy_ldg(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int TILE>  // TILE in doubles
__global__ void copy_tma(const double* __restrict__ a, double* __restrict__ b, int ntiles) {
  extern __shared__ __align__(16) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * TILE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto issue = [&](int t, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(TILE * 8));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(sm + s * TILE)), "l"(a + (size_t)t * TILE), "r"(TILE * 8), "r"(sa(&full[s])) : "memory");
  };
  int it = 0;
  for (int p = 0; p < STAGES - 1; ++p) {
    int t = blockIdx.x + p * gridDim.x;
    if (t < ntiles) issue(t, p);
  }
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % STAGES;
    const int tn = t + (STAGES - 1) * gridDim.x;
    if (tn < ntiles) {
      // stage (it+STAGES-1)%STAGES was stored out last iteration: wait for the read
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(tn, (it + STAGES - 1) % STAGES);
    }
    uint32_t ok = 0, par = (it / STAGES) & 1;
    while (!ok) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(sa(&full[s])), "r"(par) : "memory");
    }
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(b + (size_t)t * TILE),
                 "r"(sa(sm + s * TILE)), "r"(TILE * 8) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_peak(double* out, int iters) {
  double d[8][2] = {};
  double a = 1e-3 * threadIdx.x, bb = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(bb));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n = (size_t)29360128;  // config-2 DOF
  double *a, *b;
  CK(cudaMalloc(&a, n * 8));
  CK(cudaMalloc(&b, n * 8));
  CK(cudaMemset(a, 0, n * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto fn, int reps) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
  };
  float ms = timeit([&] { copy_ldg<<<sms * 8, 256>>>((const double2*)a, (double2*)b, n / 2); }, 20);
  printf("{\"kernel\":\"copy_ldg\",\"us\":%.2f,\"GBs\":%.1f}\n", ms * 1e3, 2.0 * n * 8 / (ms * 1e-3) / 1e9);
  {
    constexpr int TILE = 1792, ST = 6;
    const int ntiles = (int)(n / TILE);
    const size_t smem = ST * TILE * 8 + 64;
    CK(cudaFuncSetAttribute(copy_tma<ST, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int per = 1; per <= 3; ++per) {
      ms = timeit([&] { copy_tma<ST, TILE><<<sms * per, 32, smem>>>(a, b, ntiles); }, 20);
      printf("{\"kernel\":\"copy_tma_14KB_x%d_stages%d_ctas_per_sm%d\",\"us\":%.2f,\"GBs\":%.1f}\n", ST, ST, per,
             ms * 1e3, 2.0 * ntiles * TILE * 8 / (ms * 1e-3) / 1e9);
    }
  }
  {
    double* o;
    CK(cudaMalloc(&o, (size_t)sms * 8 * 256 * 8));
    const int it = 4096;
    ms = timeit([&] { dfma_peak<<<sms * 8, 256>>>(o, it); }, 5);
    const double fl = 2.0 * 8 * it * (double)sms * 8 * 256;
    printf("{\"kernel\":\"dfma_peak\",\"TFLOPs\":%.2f}\n", fl / (ms * 1e-3) / 1e12);
    ms = timeit([&] { dmma_peak<<<sms * 8, 256>>>(o, it / 4); }, 5);
    const double fm = 2.0 * 256 * 8 * (it / 4) * (double)sms * 8 * 256 / 32;
    printf("{\"kernel\":\"dmma_peak\",\"TFLOPs\":%.2f}\n", fm / (ms * 1e-3) / 1e12);
  }
  return 0;
}
