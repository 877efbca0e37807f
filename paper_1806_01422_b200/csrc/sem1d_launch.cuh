// sem1d_launch.cuh -- host-side launchers for the templated operator kernels.
// One translation unit per degree N instantiates launch_apply<N> (see
// sem1d_inst.cu + Makefile), so the 32 degrees compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "sem1d_device.cuh"

namespace sem1d {

struct PlanView {
  const void* consts;  // Consts<N>, packed by the plan
  Geo geo;
  int64_t batch;
};

template <int N, int OP, int PRO, int EPI>
static cudaError_t launch_one(const PlanView& p, const Args& a, cudaStream_t s) {
  auto kern = apply_kernel<N, OP, PRO, EPI>;
  constexpr size_t smem = apply_smem_bytes<N, OP>();
  static bool attr_done = false;  // benign race: idempotent attribute set
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int64_t nblk = (p.geo.E + Tile<N>::TPB - 1) / Tile<N>::TPB;
  dim3 grid((unsigned)nblk, (unsigned)p.batch);
  kern<<<grid, Tile<N>::TPB, smem, s>>>(*static_cast<const Consts<N>*>(p.consts), p.geo, a);
  return cudaGetLastError();
}

// kind: 0 F, 1 J, 2 J^T, 3 RK stage (F + combine), 4 adjoint stage (J^T + recurrence)
template <int N>
cudaError_t launch_apply(const PlanView& p, int kind, const Args& a, cudaStream_t s) {
  switch (kind) {
    case 0: return launch_one<N, OP_RHS, PRO_PLAIN, EPI_STORE>(p, a, s);
    case 1: return launch_one<N, OP_JAC, PRO_PLAIN, EPI_STORE>(p, a, s);
    case 2: return launch_one<N, OP_JACT, PRO_PLAIN, EPI_STORE>(p, a, s);
    case 3: return launch_one<N, OP_RHS, PRO_PLAIN, EPI_RK>(p, a, s);
    case 4: return launch_one<N, OP_JACT, PRO_ADJ, EPI_ADJ>(p, a, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int N>
constexpr size_t consts_size() { return sizeof(Consts<N>); }

}  // namespace sem1d
