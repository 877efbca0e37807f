// sem1d_launch.cuh -- host-side launchers for the templated operator kernels.
// One translation unit per degree N instantiates launch_apply<N> (see
// sem1d_inst.cu + Makefile), so the 32 degrees compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>

#include "sem1d_devguard.cuh"
#include "sem1d_device.cuh"
#include "sem1d_ensemble.cuh"
#include "sem1d_smallring.cuh"
#include "sem1d_tilerf.cuh"
#include "sem1d_ensrf.cuh"

namespace sem1d {

// Kernel-path override for A/B measurements and tests: 0 = auto (warp-specialised
// tensor-core kernel, else TMA/DFMA, else plain), 1 = no tensor-core path,
// 2 = plain kernel only, 3 = the first (CTA-synchronous) tensor-core kernel.
int sem1d_path_override();
// Tile-step kernel variant for A/B measurements and tests: 0 = auto (register-resident
// N = 7 kernels), 1 = the shared-memory tile kernels for every degree
int sem1d_tile_variant();

#ifndef WS_PDL
#define WS_PDL 1
#endif

struct PlanView {
  const void* consts;  // Consts<N>, packed by the plan
  const double* frag;  // n % 8 == 0: device B-fragment table (bfrag_perm order), or null
  Geo geo;
  int64_t batch;
};

template <int N, int OP, int PRO, int EPI>
static cudaError_t launch_one(const PlanView& p, const Args& a, cudaStream_t s) {
  auto kern = apply_kernel<N, OP, PRO, EPI>;
  constexpr size_t smem = apply_smem_bytes<N, OP>();
  static DevCache attr;            // benign race: idempotent attribute set
  int& attr_done = attr.here();
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_done = 1;
  }
  const int64_t nblk = (p.geo.E + Tile<N>::TPB - 1) / Tile<N>::TPB;
  dim3 grid((unsigned)nblk, (unsigned)p.batch);
  kern<<<grid, Tile<N>::TPB, smem, s>>>(*static_cast<const Consts<N>*>(p.consts), p.geo, a);
  return cudaGetLastError();
}

constexpr int kTmaStages = 2;

template <int N, int OP, int EPI>
static cudaError_t launch_tma(const PlanView& p, const Args& a, cudaStream_t s) {
  auto kern = apply_tma_kernel<N, OP, EPI, kTmaStages>;
  constexpr size_t smem = tma_smem_bytes<N, OP, kTmaStages>();
  static DevCache resident;       // resident CTAs for this instantiation, per device
  int& max_resident = resident.here();
  if (max_resident == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Tile<N>::TPB, smem);
    if (e != cudaSuccess) return e;
    max_resident = (per_sm > 0 ? per_sm : 1) * device_sms();
  }
  const int64_t per_ring = (p.geo.E + Tile<N>::TPB - 1) / Tile<N>::TPB;
  const int64_t total = per_ring * p.batch;
  if (total > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)(total < max_resident ? total : max_resident);
  kern<<<grid, Tile<N>::TPB, smem, s>>>(*static_cast<const Consts<N>*>(p.consts), p.geo, a,
                                        (int)per_ring, (int)total);
  return cudaGetLastError();
}

template <int N, int OP, int EPI>
static cudaError_t launch_mma(const PlanView& p, const Args& a, cudaStream_t s) {
  if constexpr ((N + 1) % 8 != 0) {
    return cudaErrorInvalidValue;
  } else {
    auto kern = apply_mma_kernel<N, OP, EPI, kTmaStages>;
    constexpr size_t smem = mma_smem_bytes<N, OP, kTmaStages>();
    static DevCache resident;
    int& max_resident = resident.here();
    if (max_resident == 0) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      int per_sm = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, MmaTile<N>::THREADS, smem);
      if (e != cudaSuccess) return e;
      max_resident = (per_sm > 0 ? per_sm : 1) * device_sms();
    }
    const int64_t per_ring = (p.geo.E + MmaTile<N>::ELEMS - 1) / MmaTile<N>::ELEMS;
    const int64_t total = per_ring * p.batch;
    if (total > 0x7fffffffLL) return cudaErrorInvalidValue;
    const int grid = (int)(total < max_resident ? total : max_resident);
    kern<<<grid, MmaTile<N>::THREADS, smem, s>>>(*static_cast<const Consts<N>*>(p.consts), p.geo, a,
                                                 (int)per_ring, (int)total);
    return cudaGetLastError();
  }
}


template <int N, int OP, int EPI, int NZ = -1>
static cudaError_t launch_ws(const PlanView& p, const Args& a, cudaStream_t s) {
  if constexpr ((N + 1) % 8 != 0) {
    return cudaErrorInvalidValue;
  } else {
    constexpr bool EO = ws_eo<N, EPI, NZ>();
    using W = WsTile<N, OP, NZ, EO>;
    constexpr int ST = ws_stages<N, OP, NZ, EO>();
    auto kern = apply_ws_kernel<N, OP, EPI, ST, NZ>;
    constexpr size_t smem = ws_smem_bytes<N, OP, ST, NZ, EO>();
    static DevCache resident;
    int& max_resident = resident.here();
    if (max_resident == 0) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      int per_sm = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W::THREADS, smem);
      if (e != cudaSuccess) return e;
      max_resident = (per_sm > 0 ? per_sm : 1) * device_sms();
    }
    const int64_t per_ring = (p.geo.E + W::ELEMS - 1) / W::ELEMS;
    const int64_t total = per_ring * p.batch;
    if (total > 0x7fffffffLL) return cudaErrorInvalidValue;
    const int grid = (int)(total < max_resident ? total : max_resident);
    // programmatic dependent launch: the prologue (barrier init, fragment table) overlaps the
    // previous kernel's drain; the producer's griddep_wait() orders the data path after it
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(W::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = WS_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, *static_cast<const Consts<N>*>(p.consts), p.geo, a, (int)per_ring,
                              (int)total, p.frag);
  }
}

// FP64 tensor-core path: n = N+1 a multiple of 8 (N = 7, 15, 23, 31), >= 3 tiles per ring.
template <int N>
static bool use_mma(const PlanView& p) {
  if constexpr ((N + 1) % 8 != 0) {
    return false;
  } else {
    return p.geo.E >= 3 * (int64_t)MmaTile<N>::ELEMS;
  }
}

// The TMA path needs odd N (contiguous, conflict-free element stride) and at
// least three tiles per ring (first and last tile take the synchronous path).
template <int N>
static bool use_tma(const PlanView& p) {
  return (N % 2 == 1) && p.geo.E >= 3 * (int64_t)Tile<N>::TPB;
}

// kind: 0 F, 1 J, 2 J^T, 3 RK stage (F + combine), 4 adjoint stage (J^T + recurrence)
template <int N>
cudaError_t launch_apply(const PlanView& p, int kind, const Args& a, cudaStream_t s) {
  const bool tma = use_tma<N>(p) && sem1d_path_override() != 2;
  if constexpr ((N + 1) % 8 == 0) {
    // warp-specialised DMMA kernel handles every ring size (wrap / ragged pieces in-kernel)
    if (kind <= 3 && sem1d_path_override() == 0) {
      switch (kind) {
        case 0: return launch_ws<N, OP_RHS, EPI_STORE>(p, a, s);
        case 1: return launch_ws<N, OP_JAC, EPI_STORE>(p, a, s);
        case 2: return launch_ws<N, OP_JACT, EPI_STORE>(p, a, s);
        default: return launch_ws<N, OP_RHS, EPI_RK>(p, a, s);
      }
    }
    // adjoint stage: z = b lam + up to two a_j l_j terms (RK4 needs one, Kutta-3 two)
    if (kind == 4 && sem1d_path_override() == 0 && a.zin.n <= 2) {
      switch (a.zin.n) {
        case 0: return launch_ws<N, OP_JACT, EPI_ADJ, 0>(p, a, s);
        case 1: return launch_ws<N, OP_JACT, EPI_ADJ, 1>(p, a, s);
        default: return launch_ws<N, OP_JACT, EPI_ADJ, 2>(p, a, s);
      }
    }
    if (kind <= 3 && use_mma<N>(p) && sem1d_path_override() == 3) {
      switch (kind) {
        case 0: return launch_mma<N, OP_RHS, EPI_STORE>(p, a, s);
        case 1: return launch_mma<N, OP_JAC, EPI_STORE>(p, a, s);
        case 2: return launch_mma<N, OP_JACT, EPI_STORE>(p, a, s);
        default: return launch_mma<N, OP_RHS, EPI_RK>(p, a, s);
      }
    }
  }
  switch (kind) {
    case 0: return tma ? launch_tma<N, OP_RHS, EPI_STORE>(p, a, s)
                       : launch_one<N, OP_RHS, PRO_PLAIN, EPI_STORE>(p, a, s);
    case 1: return tma ? launch_tma<N, OP_JAC, EPI_STORE>(p, a, s)
                       : launch_one<N, OP_JAC, PRO_PLAIN, EPI_STORE>(p, a, s);
    case 2: return tma ? launch_tma<N, OP_JACT, EPI_STORE>(p, a, s)
                       : launch_one<N, OP_JACT, PRO_PLAIN, EPI_STORE>(p, a, s);
    case 3: return tma ? launch_tma<N, OP_RHS, EPI_RK>(p, a, s)
                       : launch_one<N, OP_RHS, PRO_PLAIN, EPI_RK>(p, a, s);
    case 4: return launch_one<N, OP_JACT, PRO_ADJ, EPI_ADJ>(p, a, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int N>
constexpr size_t consts_size() { return sizeof(Consts<N>); }

// the stored-stage adjoint step fits shared memory for this degree
template <int N>
constexpr bool stages_fit() {
  if constexpr ((N + 1) % 8 != 0) return false;
  else return TileCfg<N>::adj_smem_ld <= 227 * 1024;
}

// Small rings (E*(N+1) <= 1024): one thread per (element, row), any degree and
// boundary kind, whole sweep per launch.
template <int N>
static cudaError_t launch_small(const PlanView& p, const EnsArgs* fa, const EnsAdjArgs* aa,
                                cudaStream_t s) {
  const int n = N + 1;
  const int64_t threads = ((p.geo.E * n + 31) / 32) * 32;
  if (threads > 1024) return cudaErrorNotSupported;
  SmallGeo sg;
  sg.E = (int)p.geo.E; sg.N = N; sg.ndof = (int)p.geo.ndof; sg.periodic = p.geo.periodic;
  const Consts<N>& C = *static_cast<const Consts<N>*>(p.consts);
  const int ts = fa ? fa->tab.s : aa->tab.s;     // compile-time tableau (TabC) per scheme
  if (ts != 1 && ts != 3 && ts != 4) return cudaErrorInvalidValue;
  if (fa) {
    const size_t smem = small_fwd_smem(N, sg.ndof, sg.E);
    if (smem > 220 * 1024) return cudaErrorNotSupported;
    auto kern = ts == 4 ? small_forward_kernel<N, 2> : (ts == 3 ? small_forward_kernel<N, 1> : small_forward_kernel<N, 0>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)p.batch, (unsigned)threads, smem, s>>>(C, sg, *fa);
  } else {
    const size_t smem = small_adj_smem(N, sg.ndof, sg.E);
    if (smem > 220 * 1024) return cudaErrorNotSupported;
    auto kern = ts == 4 ? small_adjoint_kernel<N, 2> : (ts == 3 ? small_adjoint_kernel<N, 1> : small_adjoint_kernel<N, 0>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)p.batch, (unsigned)threads, smem, s>>>(C, sg, *aa);
  }
  return cudaGetLastError();
}

// Ring-resident backward sweep: DMMA ring kernel for n % 8 == 0 periodic rings of
// <= 256 elements, else the small-ring kernel when E*(N+1) <= 1024.
template <int N>
cudaError_t launch_ens_adjoint(const PlanView& p, const EnsAdjArgs& a, cudaStream_t s) {
  if constexpr ((N + 1) % 8 == 0) {
    constexpr int W = ens_adj_warps<N>();
    constexpr int WMT = 32 / W;
    const size_t smem = ens_adj_smem_bytes<N>((int)p.geo.ndof);
    if (p.geo.periodic && p.geo.E % 8 == 0 && p.geo.E / 8 <= W * WMT && smem <= 227 * 1024 &&
        p.geo.E * (N + 1) > 1024) {
      const bool ilv = ENS_ILV && p.geo.E % (8 * WMT) == 0;
      // a.check = 0: outputs-only form (the caller re-runs a flagged sweep with check = 1)
      auto pick = [&](auto chk) {
        constexpr bool K = decltype(chk)::value;
        return a.tab.s == 4 ? (ilv ? ens_adjoint_kernel<N, WMT, true, 2, K> : ens_adjoint_kernel<N, WMT, false, 2, K>)
             : a.tab.s == 3 ? (ilv ? ens_adjoint_kernel<N, WMT, true, 1, K> : ens_adjoint_kernel<N, WMT, false, 1, K>)
                            : (ilv ? ens_adjoint_kernel<N, WMT, true, 0, K> : ens_adjoint_kernel<N, WMT, false, 0, K>);
      };
      auto kern = a.check ? pick(std::true_type{}) : pick(std::false_type{});
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<(unsigned)p.batch, EnsCfg<N, W>::THREADS, smem, s>>>(
          *static_cast<const Consts<N>*>(p.consts), p.geo, a);
      return cudaGetLastError();
    }
  }
  return launch_small<N>(p, nullptr, &a, s);
}

// Ring-resident forward sweep (same selection as the backward sweep).
template <int N>
cudaError_t launch_ens_forward(const PlanView& p, const EnsArgs& a, cudaStream_t s) {
  if constexpr ((N + 1) % 8 == 0) {
    constexpr int W = ens_fwd_warps<N>();
    constexpr int WMT = 32 / W;
    const size_t smem = ens_smem_bytes<N>((int)p.geo.ndof);
    if (p.geo.periodic && p.geo.E % 8 == 0 && p.geo.E / 8 <= W * WMT && smem <= 220 * 1024 &&
        p.geo.E * (N + 1) > 1024) {
      if constexpr (N == 15) {
        // register-resident sweep (sem1d_ensrf.cuh): rings of 32..256 elements, 32 | E
        if (ENS_RF && p.geo.E % 32 == 0 && sem1d_tile_variant() != 1) {
          const size_t sm = EnsRf::smem((int)p.geo.ndof, a.tab.s == 3);
          auto kr = a.tab.s == 4 ? ens_forward_rf_kernel<2> : a.tab.s == 3 ? ens_forward_rf_kernel<1>
                                                                           : ens_forward_rf_kernel<0>;
          cudaError_t e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          if (e != cudaSuccess) return e;
          kr<<<(unsigned)p.batch, EnsRf::THREADS, sm, s>>>(*static_cast<const Consts<N>*>(p.consts), p.geo, a);
          return cudaGetLastError();
        }
      }
      const bool ilv = ENS_ILV && p.geo.E % (8 * WMT) == 0;
      auto kern = a.tab.s == 4 ? (ilv ? ens_forward_kernel<N, WMT, true, 2> : ens_forward_kernel<N, WMT, false, 2>)
                : a.tab.s == 3 ? (ilv ? ens_forward_kernel<N, WMT, true, 1> : ens_forward_kernel<N, WMT, false, 1>)
                               : (ilv ? ens_forward_kernel<N, WMT, true, 0> : ens_forward_kernel<N, WMT, false, 0>);
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<(unsigned)p.batch, EnsCfg<N, W>::THREADS, smem, s>>>(
          *static_cast<const Consts<N>*>(p.consts), p.geo, a);
      return cudaGetLastError();
    }
  }
  return launch_small<N>(p, &a, nullptr, s);
}

// One tile-step kernel instantiation: occupancy queried once per device,
// grid = min(tiles, resident CTAs).
template <int N, auto KERN>
cudaError_t launch_tile_one(const PlanView& p, const TileStepArgs& a, int threads, size_t smem,
                            size_t smem_limit, cudaStream_t s) {
  static DevCache occ;             // per device
  int& per_sm = occ.here();
  const int sms = device_sms();
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_limit);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, KERN, threads, smem);
    if (per_sm < 1) per_sm = 1;
  }
  const int grid = (int)std::min<int64_t>(a.tile_cnt > 0 ? a.tile_cnt : a.ntiles, (int64_t)per_sm * sms);
  // programmatic dependent launch (consecutive steps of a sweep): the prologue overlaps the
  // previous step's drain; the kernel's griddep_wait() precedes its data path
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = WS_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, KERN, *static_cast<const Consts<N>*>(p.consts), p.geo, a);
}

// register-resident N = 7 forward step (sem1d_tilerf.cuh); variant 3: 192-element tiles
#ifndef TILE_RF3_MINB
#define TILE_RF3_MINB 3
#endif
template <int SCH, int WMT, int MINB>
cudaError_t launch_tile_rf(const PlanView& p, const TileStepArgs& a, cudaStream_t s) {
  constexpr size_t sm = RfCfg<WMT>::smem;
  constexpr int th = 32 * RfCfg<WMT>::W;
  if (a.stages[0])
    return a.check ? launch_tile_one<7, tile_step_rf_kernel<SCH, true, true, WMT, MINB>>(p, a, th, sm, sm, s)
                   : launch_tile_one<7, tile_step_rf_kernel<SCH, true, false, WMT, MINB>>(p, a, th, sm, sm, s);
  return a.check ? launch_tile_one<7, tile_step_rf_kernel<SCH, false, true, WMT, MINB>>(p, a, th, sm, sm, s)
                 : launch_tile_one<7, tile_step_rf_kernel<SCH, false, false, WMT, MINB>>(p, a, th, sm, sm, s);
}

template <int SCH, bool LD, int WMT, int MINB, bool DR = false>
cudaError_t launch_tile_adj_rf(const PlanView& p, const TileStepArgs& a, cudaStream_t s) {
  constexpr size_t sm = RfAdjCfg<WMT>::template smem<LD, DR>();
  if (!a.check)   // run-ahead form: outputs-only check (classifying re-run by the caller)
    return launch_tile_one<7, tile_adj_rf_kernel<SCH, LD, WMT, MINB, DR, false>>(p, a, 32 * RfAdjCfg<WMT>::W, sm, sm, s);
  return launch_tile_one<7, tile_adj_rf_kernel<SCH, LD, WMT, MINB, DR, true>>(p, a, 32 * RfAdjCfg<WMT>::W, sm, sm, s);
}

// elements per tile of the kernel launch_tile_sch picks (kind 0 forward, 1 adjoint)
template <int N>
int tile_elems(int kind, bool ld) {
  using TC = TileCfg<N>;
  if constexpr (N == 7) {
    const int var = sem1d_tile_variant();
    if (var != 1) {
      if (kind == 0) return var == 2 ? RfCfg<2>::TE : (var == 3 ? RfCfg<3>::TE : RfCfg<4>::TE);
      if (ld) return var == 2 ? RfAdjCfg<2>::TE : RfAdjCfg<3>::TE;
      return var == 2 ? RfAdjCfg<4>::TE : RfAdjCfg<3>::TE;
    }
  }
  return kind == 0 ? TC::TE_F : (ld ? TC::TE_L : TC::TE_A);
}

// tiling of a step launch: tiles, owned elements per tile, ghost elements per side
template <int N>
cudaError_t tile_layout(const PlanView& p, int kind, bool ld, int s, int* ntiles, int* owned, int* ghost) {
  if constexpr ((N + 1) % 8 != 0) {
    return cudaErrorNotSupported;
  } else {
    const int H = (kind == 0 || ld) ? s : 2 * s - 1;
    const int T = tile_elems<N>(kind, ld) - 2 * H;
    *ntiles = (int)((p.geo.E + T - 1) / T);
    *owned = T;
    *ghost = H;
    return cudaSuccess;
  }
}

template <int N, int SCH>
cudaError_t launch_tile_sch(const PlanView& p, int kind, const TileStepArgs& a, cudaStream_t s) {
  using TC = TileCfg<N>;
  if constexpr (N == 7) {
    const int var = sem1d_tile_variant();
    if (kind == 0 && var != 1) {
      if (var == 2) return launch_tile_rf<SCH, 2, 3>(p, a, s);
      if (var == 3) return launch_tile_rf<SCH, 3, TILE_RF3_MINB>(p, a, s);
      return launch_tile_rf<SCH, 4, 2>(p, a, s);
    }
    if (kind == 1 && var != 1) {
      if (a.stin[0]) {
        if constexpr (SCH == 0) return cudaErrorNotSupported;
        else if (var == 2) return launch_tile_adj_rf<SCH, true, 2, 3>(p, a, s);
        else return launch_tile_adj_rf<SCH, true, 3, 2>(p, a, s);
      }
      if (var == 2) return launch_tile_adj_rf<SCH, false, 4, 2>(p, a, s);
      return launch_tile_adj_rf<SCH, false, 3, 2, true>(p, a, s);
    }
  }
  if (kind == 0) {
    if (a.stages[0]) return launch_tile_one<N, tile_step_kernel<N, TC::W, TC::WMT_F, SCH, 1>>(p, a, 32 * TC::W, TC::fwd_smem, TC::fwd_smem, s);
    return launch_tile_one<N, tile_step_kernel<N, TC::W, TC::WMT_F, SCH, 0>>(p, a, 32 * TC::W, TC::fwd_smem, TC::fwd_smem, s);
  }
  if (a.stin[0]) {
    if constexpr (SCH == 0 || TC::adj_smem_ld > 227 * 1024) {
      return cudaErrorNotSupported;
    } else {
      constexpr size_t sm = TC::template adj_smem_ld_s<SCH>();
      return launch_tile_one<N, tile_adj_kernel<N, TC::W_L, TC::WMT_L, SCH, 1>>(p, a, 32 * TC::W_L, sm, sm, s);
    }
  }
  constexpr size_t sma = TC::template adj_smem_s<SCH>();
  return launch_tile_one<N, tile_adj_kernel<N, TC::W_A, TC::WMT_A, SCH, 0>>(p, a, 32 * TC::W_A, sma, sma, s);
}

// Temporally blocked RK step / adjoint step for large periodic rings (batch 1).
// kind 0: forward step (H = s), 1: adjoint step (H = 2s - 1, or s from stored stage states).
// The tableau (euler / Kutta-3 / RK4) is a template parameter of the kernels.
template <int N>
cudaError_t launch_tile_step(const PlanView& p, int kind, TileStepArgs a, cudaStream_t s) {
  if constexpr ((N + 1) % 8 != 0) {
    return cudaErrorNotSupported;
  } else {
    using TC = TileCfg<N>;
    if (!p.geo.periodic || p.batch != 1 || p.geo.E < 2 * TC::TE_MAX) return cudaErrorNotSupported;
    // ghost elements: s per side for a step (one per stage), 2s-1 for an adjoint step that
    // recomputes its stages, s when the forward stored them
    a.H = (kind == 0 || a.stin[0]) ? a.tab.s : 2 * a.tab.s - 1;
    const int T = tile_elems<N>(kind, a.stin[0] != nullptr) - 2 * a.H;
    a.ntiles = (int)((p.geo.E + T - 1) / T);
    bool rf = false;
    if constexpr (N == 7) rf = sem1d_tile_variant() != 1;
    if (a.tile_cnt != 0 && (!rf || a.tile_lo < 0 || a.tile_lo >= a.ntiles || a.tile_cnt < 0 || a.tile_cnt > a.ntiles))
      return cudaErrorInvalidValue;
    switch (a.tab.s) {
      case 1: return launch_tile_sch<N, 0>(p, kind, a, s);
      case 3: return launch_tile_sch<N, 1>(p, kind, a, s);
      case 4: return launch_tile_sch<N, 2>(p, kind, a, s);
      default: return cudaErrorInvalidValue;
    }
  }
}

}  // namespace sem1d
