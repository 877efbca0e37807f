// sem1d_device.cuh -- sm_100a device code for the 1D GLL spectral-element
// Burgers operator: F(u), J(u)v, J(u)^T z, fused with their gather-scatter,
// M^-1 scaling, Dirichlet mask, non-finite detection and (optionally) the
// RK / discrete-adjoint stage arithmetic that surrounds them.
//
// Reference semantics (all fp64):
//   element kernels   ops.py:161-212   F_e = -nu K u - u o (Dw u)
//                                      J_e v = -nu K v - v o (Dw u) - u o (Dw v)
//                                      J_e^T z = -nu K z - z o (Dw u) - Dw^T (u o z)
//   scatter Q         grid.py:165-169  (element e reads global nodes e*N .. e*N+N, mod ndof)
//   gather Q^T        grid.py:157-161  (<= 2 terms per node in 1D; IEEE-commutative)
//   M^-1, mask        ops.py:226-230, 252-257
//
// Data layout in HBM: a field is `batch` contiguous fp64 vectors of ndof
// global nodes (grid.py:61-63); no index table and no (ndof,) M^-1 array is
// ever read -- element e's slab is the contiguous node range [e*N, e*N+N].
//
// Tiling: one CTA owns TPB consecutive elements, one thread per element.
// The CTA stages the node range of its elements plus ONE halo element on the
// left into shared memory with coalesced loads, every thread contracts its
// element in registers (D/K/Dw live in kernel-parameter constant space, so
// the DFMAs take them as constant-bank operands), the shared interface node
// between neighbouring elements is summed in shared memory (no atomics, the
// two-term sum is order-free), and the CTA writes its node range back with
// coalesced stores.  The halo element's last row is recomputed by thread 0,
// so CTAs never communicate and results are bitwise reproducible.
#pragma once
#include <cmath>

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/sem1d.h"

namespace sem1d {

enum { OP_RHS = 0, OP_JAC = 1, OP_JACT = 2 };
enum { PRO_PLAIN = 0, PRO_ADJ = 1 };
enum { EPI_STORE = 0, EPI_RK = 1, EPI_ADJ = 2 };

// Per-plan constants, passed by value in kernel-parameter space.
template <int N>
struct Consts {
  static constexpr int n = N + 1;
  double K[n * n];    // symmetrised stiffness, row-major (ops.py:105-106)
  double Dw[n * n];   // diag(rho) D (ops.py:104)
  double minv[N + 2]; // see sem1d.h: [0] interface, [i] interior, [N] first, [N+1] last (Dirichlet)
  double mass[N + 2];
  double nu;
};

struct Geo {
  int64_t E;        // elements per batch member
  int64_t ndof;     // global nodes per batch member
  int periodic;
};

struct Combo {
  const double* ptr[SEM1D_MAX_TERMS];
  double coef[SEM1D_MAX_TERMS];
  int n;
};

struct Args {
  const double* u;   // state / linearisation point
  const double* w;   // PRO_PLAIN: v or z; PRO_ADJ: lam
  double* out;       // EPI_STORE: result; EPI_RK: k_out; EPI_ADJ: l_out (both nullable)
  int* flag;
  double b;          // PRO_ADJ: z = b*lam + sum zin
  Combo zin;
  const double* base;  // EPI_RK: base state; EPI_ADJ: lam (accumulation start)
  Combo epi;
  double dt;
  double* Y;         // EPI_RK: new stage state; EPI_ADJ: lam_out (nullable)
  int check;
};

template <int N>
struct Tile {
  static constexpr int n = N + 1;
  static constexpr int TPB = (N <= 8) ? 256 : 128;
  // register cap: <=80 regs for N<=8 (3 CTAs of 256), <=128 for N<=16, else 255
  static constexpr int MINB = (N <= 8) ? 3 : (N <= 16 ? 4 : 1);
  // even element strides would put a half-warp on one bank: skew by one
  // double every N nodes so the per-thread element stride is N+1 (odd).
  static constexpr bool PAD = (N % 2 == 0);
  static constexpr int SLAB = (TPB + 1) * N + 1;
  static constexpr int SLAB_ALLOC = PAD ? SLAB + SLAB / N + 1 : SLAB;
  __device__ static __forceinline__ int sidx(int k) { return PAD ? k + k / N : k; }
};

// non-finite test without a DFMA dependency chain: exponent field all ones (Inf / NaN).
// Integer pipe, so it does not compete with DMMA for the FP64 pipe.
__device__ __forceinline__ unsigned nonfinite_bit(double x) {
  return ((unsigned)__double2hiint(x) & 0x7ff00000u) == 0x7ff00000u ? 1u : 0u;
}
#ifndef SEM1D_NONFINITE_INT
#define SEM1D_NONFINITE_INT 1
#endif
#if SEM1D_NONFINITE_INT
__device__ __forceinline__ bool nonfinite(double v) { return nonfinite_bit(v) != 0u; }
#else
__device__ __forceinline__ bool nonfinite(double v) { return !isfinite(v); }
#endif

// One output row i of the element operator.  x = u, y = v or zm, t = u o zm.
template <int N, int OP>
__device__ __forceinline__ double elem_row(const Consts<N>& C, const double* x, const double* y,
                                           const double* t, const int i) {
  constexpr int n = N + 1;
  const double mnu = -C.nu;
  if (OP == OP_RHS) {
    double ku = 0.0, du = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      ku = fma(C.K[i * n + j], x[j], ku);
      du = fma(C.Dw[i * n + j], x[j], du);
    }
    // acc = K u; acc *= -nu; acc -= u o (Dw u)      (ops.py:166-172)
    return __dsub_rn(__dmul_rn(ku, mnu), __dmul_rn(x[i], du));
  } else if (OP == OP_JAC) {
    double kv = 0.0, du = 0.0, dv = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      kv = fma(C.K[i * n + j], y[j], kv);
      du = fma(C.Dw[i * n + j], x[j], du);
      dv = fma(C.Dw[i * n + j], y[j], dv);
    }
    // acc = K v; *= -nu; -= v o Dw u; -= u o Dw v    (ops.py:181-188)
    double acc = __dmul_rn(kv, mnu);
    acc = __dsub_rn(acc, __dmul_rn(y[i], du));
    return __dsub_rn(acc, __dmul_rn(x[i], dv));
  } else {
    double kz = 0.0, du = 0.0, dtr = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      kz = fma(C.K[i * n + j], y[j], kz);
      du = fma(C.Dw[i * n + j], x[j], du);
      dtr = fma(C.Dw[j * n + i], t[j], dtr);
    }
    // acc = K z; *= -nu; -= z o Dw u; -= Dw^T (u o z)  (ops.py:200-207)
    double acc = __dmul_rn(kz, mnu);
    acc = __dsub_rn(acc, __dmul_rn(y[i], du));
    return __dsub_rn(acc, dtr);
  }
}

template <int N, int OP>
__device__ __forceinline__ void load_elem(const double* su, const double* sw, int base, double* x,
                                          double* y, double* t) {
  using T = Tile<N>;
  constexpr int n = N + 1;
#pragma unroll
  for (int j = 0; j < n; ++j) {
    x[j] = su[T::sidx(base + j)];
    if (OP != OP_RHS) y[j] = sw[T::sidx(base + j)];
  }
  if (OP == OP_JACT) {
#pragma unroll
    for (int j = 0; j < n; ++j) t[j] = __dmul_rn(x[j], y[j]);
  }
}

// Position-dependent mass-pattern lookup (see sem1d.h).
template <int N>
__device__ __forceinline__ double pattern(const double* pat, int64_t g, int local, bool periodic,
                                          int64_t last_node) {
  if (!periodic) {
    if (g == 0) return pat[N];
    if (g == last_node) return pat[N + 1];
  }
  return pat[local];
}

template <int N, int OP, int PRO, int EPI>
__global__ void __launch_bounds__(Tile<N>::TPB, Tile<N>::MINB)
    apply_kernel(const __grid_constant__ Consts<N> C, const Geo G, const Args A) {
  using T = Tile<N>;
  constexpr int n = N + 1;
  constexpr int TPB = T::TPB;
  extern __shared__ double smem[];
  double* su = smem;                                        // u slab (+ halo element)
  double* sw = smem + T::SLAB_ALLOC;                        // v / zm slab
  double* so = smem + (OP == OP_RHS ? 1 : 2) * T::SLAB_ALLOC;  // assembled outputs
  double* slast = so + T::SLAB_ALLOC;                       // row N of each element

  const int64_t bofs = (int64_t)blockIdx.y * G.ndof;
  const int64_t e0 = (int64_t)blockIdx.x * TPB;
  const int nel = (int)min((int64_t)TPB, G.E - e0);
  const bool periodic = G.periodic != 0;
  const int64_t g0 = (e0 - 1) * N;  // first node of the halo element
  const int cnt = (nel + 1) * N + 1;
  const int64_t last_node = G.E * N;
  const int tid = threadIdx.x;

  // ---- stage the node slab (coalesced), forming the second input on the fly
  bool bad_u = false, bad_w = false;
  const double* __restrict__ pu = A.u + bofs;
  const double* __restrict__ pw = (OP != OP_RHS) ? A.w + bofs : nullptr;
  for (int k = tid; k < cnt; k += TPB) {
    int64_t g = g0 + k;
    bool valid = true;
    if (g < 0) {
      if (periodic) g += G.ndof; else valid = false;
    } else if (g >= G.ndof) {
      g -= G.ndof;
    }
    double uv = 0.0, wv = 0.0;
    if (valid) {
      uv = __ldg(pu + g);
      bad_u |= nonfinite(uv);
      if (OP != OP_RHS) {
        if (PRO == PRO_PLAIN) {
          wv = __ldg(pw + g);
        } else {
          // z = b*lam + a_0 l_0 + a_1 l_1 + ...        (adjoint.py:58-60)
          wv = __dmul_rn(A.b, __ldg(pw + g));
          for (int j = 0; j < A.zin.n; ++j)
            wv = __dadd_rn(wv, __dmul_rn(A.zin.coef[j], __ldg(A.zin.ptr[j] + bofs + g)));
        }
        bad_w |= nonfinite(wv);
        if (OP == OP_JACT) {
          // zm = mask(z * M^-1)                          (ops.py:252-254)
          wv = __dmul_rn(wv, pattern<N>(C.minv, g, k % N, periodic, last_node));
          if (!periodic && (g == 0 || g == last_node)) wv = __dmul_rn(wv, 0.0);
        }
      }
    }
    su[T::sidx(k)] = uv;
    if (OP != OP_RHS) sw[T::sidx(k)] = wv;
  }
  if (bad_u || bad_w)
    atomicOr(A.flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) |
                         (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0));
  __syncthreads();

  // ---- element contraction, one thread per element; rows stream to `so`
  //      (row 0 waits in `so` for the left neighbour's row N, kept in slast)
  {
    double x[n], y[(OP != OP_RHS) ? n : 1], t[(OP == OP_JACT) ? n : 1];
    if (tid < nel) {
      load_elem<N, OP>(su, sw, (tid + 1) * N, x, y, t);
#pragma unroll
      for (int i = 0; i < N; ++i) so[T::sidx(tid * N + i)] = elem_row<N, OP>(C, x, y, t, i);
      slast[tid + 1] = elem_row<N, OP>(C, x, y, t, N);
    }
    if (tid == 0) {
      double hl = 0.0;
      if (periodic || e0 > 0) {
        load_elem<N, OP>(su, sw, 0, x, y, t);
        hl = elem_row<N, OP>(C, x, y, t, N);
      }
      slast[0] = hl;
    }
  }
  __syncthreads();
  const bool last_cta = (e0 + nel == G.E);

  // ---- epilogue: M^-1, mask, stage arithmetic, coalesced stores
  const int nout = nel * N + ((!periodic && last_cta) ? 1 : 0);
  const int64_t gbase = e0 * N;
  bool bad_y = false;
  for (int k = tid; k < nout; k += TPB) {
    const int64_t g = gbase + k;
    const int loc = k % N;
    double v;
    if (loc != 0) {
      v = so[T::sidx(k)];
    } else {
      // node e*N receives element e-1's row N and element e's row 0 (grid.py:157-161);
      // the Dirichlet end node E*N only the last element's row N
      const int te = k / N;
      v = (te < nel) ? __dadd_rn(slast[te], so[T::sidx(k)]) : slast[te];
    }
    if (OP != OP_JACT) v = __dmul_rn(v, pattern<N>(C.minv, g, loc, periodic, last_node));
    if (!periodic && (g == 0 || g == last_node)) v = __dmul_rn(v, 0.0);
    const int64_t ga = bofs + g;
    if (EPI == EPI_STORE) {
      A.out[ga] = v;
    } else if (EPI == EPI_RK) {
      if (A.out) A.out[ga] = v;
      double y;
      if (A.epi.n == 1) {
        // base + (dt * a) * k                            (timeloop.py:114,123)
        const double kk = A.epi.ptr[0] ? __ldg(A.epi.ptr[0] + ga) : v;
        y = __dadd_rn(__ldg(A.base + ga), __dmul_rn(__dmul_rn(A.dt, A.epi.coef[0]), kk));
      } else {
        // base + dt * ((a0 k0 + a1 k1) + ...)            (timeloop.py:116,125,127)
        double s = 0.0;
        for (int j = 0; j < A.epi.n; ++j) {
          const double kk = A.epi.ptr[j] ? __ldg(A.epi.ptr[j] + ga) : v;
          const double term = __dmul_rn(A.epi.coef[j], kk);
          s = (j == 0) ? term : __dadd_rn(s, term);
        }
        y = __dadd_rn(__ldg(A.base + ga), __dmul_rn(A.dt, s));
      }
      if (A.check) bad_y |= nonfinite(y);
      A.Y[ga] = y;
    } else {  // EPI_ADJ
      const double l = __dmul_rn(A.dt, v);  // l = dt * J^T(U) z   (adjoint.py:58-60)
      if (A.out) A.out[ga] = l;
      if (A.Y) {
        // lam + l_0 + l_1 + ...                          (adjoint.py:61)
        double acc = __ldg(A.base + ga);
        for (int j = 0; j < A.epi.n; ++j)
          acc = __dadd_rn(acc, A.epi.ptr[j] ? __ldg(A.epi.ptr[j] + ga) : l);
        A.Y[ga] = acc;
      }
    }
  }
  if (EPI == EPI_RK && bad_y) atomicOr(A.flag, SEM1D_FLAG_STEP_NONFINITE);
}

// ============================================================================
// Persistent, TMA-pipelined variant (odd N; the BASELINE degrees 7/9/15/31).
//
// One CTA per SM slot loops over tiles of TPB elements.  Thread 0 issues the
// slab loads of the tile STAGES-1 iterations ahead as 1D bulk-tensor copies
// (cp.async.bulk global->shared, completion counted on an mbarrier), so HBM
// streams continuously while the CTA contracts the current tile; the
// non-finite checks and the J^T input scaling move into registers.  The
// first and last tile of every ring (periodic wrap / Dirichlet ends / ragged
// tail) take a synchronous per-thread load path.
// ============================================================================

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int N>
struct TmaTile {
  static constexpr int TPB = Tile<N>::TPB;
  static constexpr int SLAB = (TPB + 1) * N + 1;
  // +1 double for the 16-byte alignment shift, rounded to a 16-byte multiple
  static constexpr int SLAB_ALLOC = ((SLAB + 1) + 1) & ~1;
};

// zm = mask(z * M^-1) for local node j of element e (ops.py:252-254), in registers
template <int N>
__device__ __forceinline__ double jt_scale(const Consts<N>& C, double z, int j, int64_t e,
                                           const Geo& G) {
  int pos = (j == 0 || j == N) ? 0 : j;
  bool zero = false;
  if (!G.periodic) {
    if (j == 0 && e == 0) { pos = N; zero = true; }
    if (j == N && e == G.E - 1) { pos = N + 1; zero = true; }
  }
  double v = __dmul_rn(z, C.minv[pos]);
  return zero ? __dmul_rn(v, 0.0) : v;
}

template <int N, int OP, int EPI, int STAGES>
__global__ void __launch_bounds__(Tile<N>::TPB, Tile<N>::MINB)
    apply_tma_kernel(const __grid_constant__ Consts<N> C, const Geo G, const Args A,
                     const int tiles_per_ring, const int total_tiles) {
  using TT = TmaTile<N>;
  constexpr int n = N + 1;
  constexpr int TPB = TT::TPB;
  constexpr int NIN = (OP == OP_RHS) ? 1 : 2;
  constexpr int SA = TT::SLAB_ALLOC;
  extern __shared__ __align__(16) double smem[];
  double* stage_buf = smem;                          // [STAGES][NIN][SA]
  double* so = smem + STAGES * NIN * SA;             // [SA]
  double* slast = so + SA;                           // [TPB + 2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(slast + TPB + 2);
  const int tid = threadIdx.x;
  const bool periodic = G.periodic != 0;
  const int64_t last_node = G.E * N;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto tile_of = [&](int T, int64_t& bofs, int64_t& e0, int& nel, bool& boundary) {
    const int b = T / tiles_per_ring;
    const int tl = T - b * tiles_per_ring;
    bofs = (int64_t)b * G.ndof;
    e0 = (int64_t)tl * TPB;
    nel = (int)min((int64_t)TPB, G.E - e0);
    boundary = (tl == 0) || (tl == tiles_per_ring - 1);
  };
  auto issue = [&](int T, int s) {  // thread 0
    int64_t bofs, e0;
    int nel;
    bool boundary;
    tile_of(T, bofs, e0, nel, boundary);
    if (boundary) return;
    const int64_t gg0 = bofs + (e0 - 1) * N;
    const int64_t a0 = gg0 & ~(int64_t)1;
    const int shift = (int)(gg0 - a0);
    const int cnt = (nel + 1) * N + 1;
    const uint32_t bytes = (uint32_t)(((cnt + shift) * 8 + 15) & ~15);
    mbar_expect_tx(&bars[s], NIN * bytes);
    bulk_g2s(stage_buf + (s * NIN + 0) * SA, A.u + a0, bytes, &bars[s]);
    if (NIN == 2) bulk_g2s(stage_buf + (s * NIN + 1) * SA, A.w + a0, bytes, &bars[s]);
  };

  if (tid == 0) {
    for (int p = 0; p < STAGES - 1; ++p) {
      const int T = blockIdx.x + p * gridDim.x;
      if (T < total_tiles) issue(T, p);
    }
  }

  bool bad_u = false, bad_w = false, bad_y = false;
  uint32_t phases = 0;
  int iter = 0;
  for (int T = blockIdx.x; T < total_tiles; T += gridDim.x, ++iter) {
    const int s = iter % STAGES;
    if (tid == 0) {
      const int Tn = T + (STAGES - 1) * gridDim.x;
      if (Tn < total_tiles) issue(Tn, (iter + STAGES - 1) % STAGES);
    }
    int64_t bofs, e0;
    int nel;
    bool boundary;
    tile_of(T, bofs, e0, nel, boundary);
    double* su = stage_buf + (s * NIN + 0) * SA;
    double* sw = stage_buf + (s * NIN + 1) * SA;
    int shift;
    const int64_t g0 = (e0 - 1) * N;
    if (boundary) {
      shift = 0;
      const int cnt = (nel + 1) * N + 1;
      for (int k = tid; k < cnt; k += TPB) {
        int64_t g = g0 + k;
        bool valid = true;
        if (g < 0) {
          if (periodic) g += G.ndof; else valid = false;
        } else if (g >= G.ndof) {
          g -= G.ndof;
        }
        su[k] = valid ? __ldg(A.u + bofs + g) : 0.0;
        if (NIN == 2) sw[k] = valid ? __ldg(A.w + bofs + g) : 0.0;
      }
      __syncthreads();
    } else {
      const int64_t gg0 = bofs + g0;
      shift = (int)(gg0 & 1);
      while (!mbar_try_wait(&bars[s], (phases >> s) & 1u)) {
      }
      phases ^= (1u << s);
    }

    // ---- contraction (one element per thread) ----
    {
      double x[n], y[(OP != OP_RHS) ? n : 1], t[(OP == OP_JACT) ? n : 1];
      auto load = [&](int base, int64_t e) {
#pragma unroll
        for (int j = 0; j < n; ++j) {
          x[j] = su[shift + base + j];
          bad_u |= nonfinite(x[j]);
          if (OP != OP_RHS) {
            y[j] = sw[shift + base + j];
            bad_w |= nonfinite(y[j]);
            if (OP == OP_JACT) y[j] = jt_scale<N>(C, y[j], j, e, G);
          }
        }
        if (OP == OP_JACT) {
#pragma unroll
          for (int j = 0; j < n; ++j) t[j] = __dmul_rn(x[j], y[j]);
        }
      };
      if (tid < nel) {
        load((tid + 1) * N, e0 + tid);
#pragma unroll
        for (int i = 0; i < N; ++i) so[tid * N + i] = elem_row<N, OP>(C, x, y, t, i);
        slast[tid + 1] = elem_row<N, OP>(C, x, y, t, N);
      }
      if (tid == 0) {
        double hl = 0.0;
        if (periodic || e0 > 0) {
          load(0, (e0 == 0) ? G.E - 1 : e0 - 1);
          hl = elem_row<N, OP>(C, x, y, t, N);
        }
        slast[0] = hl;
      }
    }
    __syncthreads();

    // ---- gather, M^-1, mask, stage arithmetic; coalesced stores ----
    const bool last_tile = (e0 + nel == G.E);
    const int nout = nel * N + ((!periodic && last_tile) ? 1 : 0);
    const int64_t gbase = e0 * N;
    for (int k = tid; k < nout; k += TPB) {
      const int64_t g = gbase + k;
      const int loc = k % N;
      double v;
      if (loc != 0) {
        v = so[k];
      } else {
        const int te = k / N;
        v = (te < nel) ? __dadd_rn(slast[te], so[k]) : slast[te];
      }
      if (OP != OP_JACT) v = __dmul_rn(v, pattern<N>(C.minv, g, loc, periodic, last_node));
      if (!periodic && (g == 0 || g == last_node)) v = __dmul_rn(v, 0.0);
      const int64_t ga = bofs + g;
      if (EPI == EPI_STORE) {
        A.out[ga] = v;
      } else {  // EPI_RK
        if (A.out) A.out[ga] = v;
        double yv;
        if (A.epi.n == 1) {
          const double kk = A.epi.ptr[0] ? __ldg(A.epi.ptr[0] + ga) : v;
          yv = __dadd_rn(__ldg(A.base + ga), __dmul_rn(__dmul_rn(A.dt, A.epi.coef[0]), kk));
        } else {
          double sacc = 0.0;
          for (int j = 0; j < A.epi.n; ++j) {
            const double kk = A.epi.ptr[j] ? __ldg(A.epi.ptr[j] + ga) : v;
            const double term = __dmul_rn(A.epi.coef[j], kk);
            sacc = (j == 0) ? term : __dadd_rn(sacc, term);
          }
          yv = __dadd_rn(__ldg(A.base + ga), __dmul_rn(A.dt, sacc));
        }
        if (A.check) bad_y |= nonfinite(yv);
        A.Y[ga] = yv;
      }
    }
    __syncthreads();
  }
  if (bad_u || bad_w || bad_y)
    atomicOr(A.flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) |
                         (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0) |
                         (bad_y ? SEM1D_FLAG_STEP_NONFINITE : 0));
}

// ============================================================================
// FP64 tensor-core variant (n = N+1 in {8, 16, 32}: BASELINE degrees 7, 15, 31).
//
// The per-element contractions of a tile are small GEMMs: Out[e][i] =
// sum_j A[e][j] M[i][j] with A = u, v or zm and M = K, Dw (or Dw^T for the
// J^T advection term).  A warp handles 8 elements at a time with
// mma.sync.m8n8k4.f64 (SASS DMMA): one instruction does 8 elements x 8 rows x
// 4 columns, replacing 32 DFMA + 32 constant loads per thread.  A-fragments
// come straight from the staged slab (element e's nodes are contiguous), the
// B-fragments of K / Dw are built once per CTA, interior nodes are finalised
// (M^-1) in place, the shared interface node is fixed up after one barrier,
// and full tiles leave through a TMA bulk store (cp.async.bulk shared->global).
// ============================================================================

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int N>
struct MmaTile {
  static constexpr int n = N + 1;
  static_assert(n % 8 == 0, "tensor-core path needs n = N+1 divisible by 8");
  static constexpr int THREADS = 256;
  static constexpr int ELEMS = (n == 8) ? 256 : (n == 16 ? 128 : 64);   // elements per tile
  static constexpr int MT = ELEMS / 8;                                  // 8-element m-tiles
  static constexpr int NT = n / 8;                                      // 8-row n-tiles
  static constexpr int KC = n / 4;                                      // 4-column k-chunks
  static constexpr int SLAB = (ELEMS + 1) * N + 1;
  static constexpr int SLAB_ALLOC = ((SLAB + 1) + 1) & ~1;
  static constexpr bool B_IN_SMEM = (n > 16);
  static constexpr int MINB = (n == 32) ? 1 : 2;
};

// fragment matrices: 0 = K (used as M^T), 1 = Dw (as M^T: Dw u), 2 = Dw (as M: Dw^T t)
template <int N>
__device__ __forceinline__ double bfrag_value(const Consts<N>& C, int mat, int nt, int kc, int lane) {
  constexpr int n = N + 1;
  const int i = 8 * nt + (lane >> 2);
  const int j = 4 * kc + (lane & 3);
  if (mat == 0) return C.K[i * n + j];
  if (mat == 1) return C.Dw[i * n + j];
  return C.Dw[j * n + i];
}

template <int N, int OP, int EPI, int STAGES>
__global__ void __launch_bounds__(MmaTile<N>::THREADS, MmaTile<N>::MINB)
    apply_mma_kernel(const __grid_constant__ Consts<N> C, const Geo G, const Args A,
                     const int tiles_per_ring, const int total_tiles) {
  using MT_ = MmaTile<N>;
  constexpr int n = N + 1;
  constexpr int THREADS = MT_::THREADS;
  constexpr int ELEMS = MT_::ELEMS;
  constexpr int NT = MT_::NT;
  constexpr int KC = MT_::KC;
  constexpr int NIN = (OP == OP_RHS) ? 1 : 2;
  constexpr int NMAT = (OP == OP_JACT) ? 3 : 2;
  constexpr int SA = MT_::SLAB_ALLOC;
  extern __shared__ __align__(16) double smem[];
  double* stage_buf = smem;                               // [STAGES][NIN][SA]
  double* so = smem + STAGES * NIN * SA;                  // [SA] finalised node values
  double* slast = so + SA;                                // [ELEMS + 2]
  double* bsm = slast + ELEMS + 2;                        // [NMAT][NT][KC][32] if B_IN_SMEM
  uint64_t* bars = reinterpret_cast<uint64_t*>(bsm + (MT_::B_IN_SMEM ? NMAT * NT * KC * 32 : 0));
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const bool periodic = G.periodic != 0;
  const double mnu = -C.nu;

  // ---- B fragments (constant per CTA)
  double breg[MT_::B_IN_SMEM ? 1 : NMAT * NT * KC];
  if (MT_::B_IN_SMEM) {
    for (int q = tid; q < NMAT * NT * KC * 32; q += THREADS) {
      const int l = q & 31, r = q >> 5;
      const int kc = r % KC, nt = (r / KC) % NT, mat = r / (KC * NT);
      bsm[q] = bfrag_value<N>(C, mat == 2 ? 2 : mat, nt, kc, l);
    }
  } else {
#pragma unroll
    for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
          breg[(mat * NT + nt) * KC + kc] = bfrag_value<N>(C, mat, nt, kc, lane);
  }
  auto bget = [&](int mat, int nt, int kc) -> double {
    if (MT_::B_IN_SMEM) return bsm[((mat * NT + nt) * KC + kc) * 32 + lane];
    return breg[(mat * NT + nt) * KC + kc];
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto tile_of = [&](int T, int64_t& bofs, int64_t& e0, int& nel, bool& boundary) {
    const int b = T / tiles_per_ring;
    const int tl = T - b * tiles_per_ring;
    bofs = (int64_t)b * G.ndof;
    e0 = (int64_t)tl * ELEMS;
    nel = (int)min((int64_t)ELEMS, G.E - e0);
    boundary = (tl == 0) || (tl == tiles_per_ring - 1);
  };
  auto issue = [&](int T, int s) {
    int64_t bofs, e0;
    int nel;
    bool boundary;
    tile_of(T, bofs, e0, nel, boundary);
    if (boundary) return;
    const int64_t gg0 = bofs + (e0 - 1) * N;
    const int64_t a0 = gg0 & ~(int64_t)1;
    const int shift = (int)(gg0 - a0);
    const int cnt = (nel + 1) * N + 1;
    const uint32_t bytes = (uint32_t)(((cnt + shift) * 8 + 15) & ~15);
    mbar_expect_tx(&bars[s], NIN * bytes);
    bulk_g2s(stage_buf + (s * NIN + 0) * SA, A.u + a0, bytes, &bars[s]);
    if (NIN == 2) bulk_g2s(stage_buf + (s * NIN + 1) * SA, A.w + a0, bytes, &bars[s]);
  };
  if (tid == 0) {
    for (int p = 0; p < STAGES - 1; ++p) {
      const int T = blockIdx.x + p * gridDim.x;
      if (T < total_tiles) issue(T, p);
    }
  }

  bool bad_u = false, bad_w = false, bad_y = false;
  uint32_t phases = 0;
  int iter = 0;
  for (int T = blockIdx.x; T < total_tiles; T += gridDim.x, ++iter) {
    const int s = iter % STAGES;
    if (tid == 0) {
      const int Tn = T + (STAGES - 1) * gridDim.x;
      if (Tn < total_tiles) issue(Tn, (iter + STAGES - 1) % STAGES);
    }
    int64_t bofs, e0;
    int nel;
    bool boundary;
    tile_of(T, bofs, e0, nel, boundary);
    const double* su = stage_buf + (s * NIN + 0) * SA;
    const double* sw = stage_buf + (s * NIN + 1) * SA;
    int shift;
    const int64_t g0 = (e0 - 1) * N;
    if (boundary) {
      shift = 0;
      double* wu = stage_buf + (s * NIN + 0) * SA;
      double* ww = stage_buf + (s * NIN + 1) * SA;
      const int cnt = (nel + 1) * N + 1;
      for (int k = tid; k < cnt; k += THREADS) {
        int64_t g = g0 + k;
        bool valid = true;
        if (g < 0) {
          if (periodic) g += G.ndof; else valid = false;
        } else if (g >= G.ndof) {
          g -= G.ndof;
        }
        wu[k] = valid ? __ldg(A.u + bofs + g) : 0.0;
        if (NIN == 2) ww[k] = valid ? __ldg(A.w + bofs + g) : 0.0;
      }
      // partial tile: zero the slab beyond the last element so padded m-tiles stay finite
      for (int k = cnt + tid; k < (ELEMS + 1) * N + 1; k += THREADS) {
        wu[k] = 0.0;
        if (NIN == 2) ww[k] = 0.0;
      }
      __syncthreads();
    } else {
      shift = (int)((bofs + g0) & 1);
      while (!mbar_try_wait(&bars[s], (phases >> s) & 1u)) {
      }
      phases ^= (1u << s);
    }

    // ---- tensor-core contraction: warp w owns m-tiles w, w+8, ...
    for (int mt = warp; mt < MT_::MT; mt += THREADS / 32) {
      const int el = 8 * mt + (lane >> 2);          // local element of this lane's A/C row
      const bool live = el < nel;
      const int64_t eg = e0 + el;
      const int base = shift + (el + 1) * N;        // slab offset of element el's node 0
      double au[KC], aw[(OP != OP_RHS) ? KC : 1], at[(OP == OP_JACT) ? KC : 1];
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int j = 4 * kc + (lane & 3);
        au[kc] = su[base + j];
        if (live) bad_u |= nonfinite(au[kc]);
        if (OP != OP_RHS) {
          aw[kc] = sw[base + j];
          if (live) bad_w |= nonfinite(aw[kc]);
          if (OP == OP_JACT) {
            aw[kc] = jt_scale<N>(C, aw[kc], j, eg, G);
            at[kc] = __dmul_rn(au[kc], aw[kc]);
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        double k0 = 0.0, k1 = 0.0, p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const double ak = (OP == OP_RHS) ? au[kc] : aw[kc];
          dmma884(k0, k1, ak, bget(0, nt, kc));            // K x            (x = u, v or zm)
          dmma884(p0, p1, au[kc], bget(1, nt, kc));        // Dw u
          if (OP == OP_JAC) dmma884(q0, q1, aw[kc], bget(1, nt, kc));   // Dw v
          if (OP == OP_JACT) dmma884(q0, q1, at[kc], bget(2, nt, kc));  // Dw^T (u o zm)
        }
        if (live) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = 8 * nt + 2 * (lane & 3) + h;
            const double kx = h ? k1 : k0, du = h ? p1 : p0, qq = h ? q1 : q0;
            const double ui = su[base + i];
            double r;
            if (OP == OP_RHS) {
              r = __dsub_rn(__dmul_rn(kx, mnu), __dmul_rn(ui, du));
            } else if (OP == OP_JAC) {
              const double vi = sw[base + i];
              r = __dsub_rn(__dsub_rn(__dmul_rn(kx, mnu), __dmul_rn(vi, du)), __dmul_rn(ui, qq));
            } else {
              const double zi = jt_scale<N>(C, sw[base + i], i, eg, G);
              r = __dsub_rn(__dsub_rn(__dmul_rn(kx, mnu), __dmul_rn(zi, du)), qq);
            }
            if (i == N) {
              slast[el + 1] = r;
            } else if (i == 0) {
              so[el * N] = r;
            } else {
              so[el * N + i] = (OP == OP_JACT) ? r : __dmul_rn(r, C.minv[i]);
            }
          }
        }
      }
    }
    if (tid == 0) {  // row N of the halo element (left neighbour tile), scalar
      double hl = 0.0;
      if (periodic || e0 > 0) {
        double x[n], y[(OP != OP_RHS) ? n : 1], t[(OP == OP_JACT) ? n : 1];
        const int64_t eh = (e0 == 0) ? G.E - 1 : e0 - 1;
#pragma unroll
        for (int j = 0; j < n; ++j) {
          x[j] = su[shift + j];
          if (OP != OP_RHS) {
            y[j] = sw[shift + j];
            if (OP == OP_JACT) y[j] = jt_scale<N>(C, y[j], j, eh, G);
          }
        }
        if (OP == OP_JACT) {
#pragma unroll
          for (int j = 0; j < n; ++j) t[j] = __dmul_rn(x[j], y[j]);
        }
        hl = elem_row<N, OP>(C, x, y, t, N);
      }
      slast[0] = hl;
    }
    __syncthreads();

    // ---- interface nodes: element e-1's row N + element e's row 0 (grid.py:157-161)
    const bool last_tile = (e0 + nel == G.E);
    for (int el = tid; el <= nel; el += THREADS) {
      const int64_t g = e0 * N + (int64_t)el * N;
      if (el < nel) {
        double v = __dadd_rn(slast[el], so[el * N]);
        if (OP != OP_JACT) v = __dmul_rn(v, (!periodic && g == 0) ? C.minv[N] : C.minv[0]);
        if (!periodic && g == 0) v = __dmul_rn(v, 0.0);
        so[el * N] = v;
      } else if (!periodic && last_tile) {  // Dirichlet end node E*N
        double v = slast[el];
        if (OP != OP_JACT) v = __dmul_rn(v, C.minv[N + 1]);
        so[el * N] = __dmul_rn(v, 0.0);
      }
    }
    const int nout = nel * N + ((!periodic && last_tile) ? 1 : 0);
    const int64_t gout = bofs + e0 * N;
    const bool bulk = (EPI == EPI_STORE) && !boundary && ((gout & 1) == 0);
    if (bulk) fence_proxy_async_smem();
    __syncthreads();
    if (bulk) {
      if (tid == 0) {
        bulk_s2g(A.out + gout, so, (uint32_t)(nout * 8));
        bulk_commit();
        bulk_wait_read<0>();
      }
    } else {
      for (int k = tid; k < nout; k += THREADS) {
        const double v = so[k];
        const int64_t ga = gout + k;
        if (EPI == EPI_STORE) {
          A.out[ga] = v;
        } else {  // EPI_RK: base + dt * combination (timeloop.py:114-127)
          if (A.out) A.out[ga] = v;
          double yv;
          if (A.epi.n == 1) {
            const double kk = A.epi.ptr[0] ? __ldg(A.epi.ptr[0] + ga) : v;
            yv = __dadd_rn(__ldg(A.base + ga), __dmul_rn(__dmul_rn(A.dt, A.epi.coef[0]), kk));
          } else {
            double sacc = 0.0;
            for (int j = 0; j < A.epi.n; ++j) {
              const double kk = A.epi.ptr[j] ? __ldg(A.epi.ptr[j] + ga) : v;
              const double term = __dmul_rn(A.epi.coef[j], kk);
              sacc = (j == 0) ? term : __dadd_rn(sacc, term);
            }
            yv = __dadd_rn(__ldg(A.base + ga), __dmul_rn(A.dt, sacc));
          }
          if (A.check) bad_y |= nonfinite(yv);
          A.Y[ga] = yv;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) bulk_wait_all();
  if (bad_u || bad_w || bad_y)
    atomicOr(A.flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) |
                         (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0) |
                         (bad_y ? SEM1D_FLAG_STEP_NONFINITE : 0));
}

// ============================================================================
// Warp-specialised tensor-core kernel.  Warp CW (the last) is the TMA
// producer: it waits until a stage is released, loads the unaligned or wrapped
// pieces of the slab with its lanes and the 16-byte-aligned body with one bulk
// copy per input, then arms the stage's "full" mbarrier.  Warps 0..CW-1 are
// DMMA consumers, each owning WE consecutive elements of the tile: they
// contract with mma.m8n8k4.f64, form the shared interface node in registers
// (shuffle from the neighbouring lane; the row N of the element left of the
// warp is recomputed warp-cooperatively), stage their finished node range in
// shared memory and write it back with their own bulk store.  There is no
// CTA-wide barrier inside the tile loop.
// ============================================================================

#ifndef WS_FIN_INT
#define WS_FIN_INT 1
#endif
#if WS_FIN_INT
typedef unsigned ws_fin_t;
#define WS_FIN_ACC(acc, x) (acc) |= nonfinite_bit(x)
#define WS_FIN_BAD(acc) ((acc) != 0u)
#else
typedef double ws_fin_t;
#define WS_FIN_ACC(acc, x) (acc) = fma((x), 0.0, (acc))
#define WS_FIN_BAD(acc) ((acc) != (acc))
#endif

// round 2: F on 512-element tiles at 2 CTAs/SM (77.5 -> 76.9 us); J / J^T keep 256
#ifndef WS_ELEMS8
#define WS_ELEMS8 512
#endif
// n = 32: consumer warps per operator (A/B, config 3): 8 warps x 2 interleaved m-tiles with
// each shared-memory B fragment feeding both (mtile_compute_multi): F / J 55.4 / 73.8 us
// (63.0 / 82.3 at 16 x 1), J^T 90.1 us (97.4 at 16 x 1, which spilled at the 96-register cap).
// J and J^T (round 2): 4 warps x 2 m-tiles on 64-element tiles at 2 CTAs/SM, so the two
// CTAs of an SM run their DMMA and epilogue phases independently: J 67.2 -> 66.4 us,
// J^T 69.7 -> 67.0 us; F measured 47.5 either way (and 48.5 at 3 CTAs/SM).
#ifndef WS_CW32
#define WS_CW32 8
#endif
#ifndef WS_CW32_J
#define WS_CW32_J 4
#endif
#ifndef WS_CW32_JT
#define WS_CW32_JT 4
#endif
#ifndef WS_ELEMS32
#define WS_ELEMS32 128
#endif
// (J / J^T tiles at n = 32: 2 m-tiles per consumer warp, 16 * CW elements)

// Occupancy per operator at n = 8, A/B-measured on config 2 (round 1:
// profiles/r1_ab_occupancy.json; re-measured in round 2, profiles/r2_ws_ab_cfg2.jsonl):
// F on 512-element tiles at 2 CTAs/SM, J at 2 (deeper pipeline: 106.4 -> 103.9 us), J^T at 3
// (109.2 us at 2)
#ifndef WS_MINB_F8
#define WS_MINB_F8 2
#endif
#ifndef WS_MINB_J8
#define WS_MINB_J8 2
#endif
#ifndef WS_MINB_JT8
#define WS_MINB_JT8 3
#endif
// output staging buffers: 2 lets a warp compute tile t+1 while the bulk store of
// tile t still reads its staging (F has the shared memory to spare)
#ifndef WS_OUTB_F
#define WS_OUTB_F 2
#endif
#ifndef WS_OUTB_J
#define WS_OUTB_J 1
#endif
template <int OP>
constexpr int ws_outb() { return OP == OP_RHS ? WS_OUTB_F : WS_OUTB_J; }

#ifndef WS_MINB32
#define WS_MINB32 2
#endif
#ifndef WS_MINB32_F
#define WS_MINB32_F 1
#endif
// WS_EO (see the comment at bfrag_eo_value): the plain applies at n % 16 == 0 on the reflection
// split.  F at n = 32 then has half the DMMAs per tile and fewer live registers, and runs 64-element
// tiles on 4 consumer warps at 3 CTAs/SM (128 registers; config 3: 35.5 us at 1 CTA/SM x 8 warps,
// 34.5 at 2 x 4, 32.3 at 3 x 4)
#ifndef WS_EO
#define WS_EO 1
#endif
#ifndef WS_EO_ADJ
#define WS_EO_ADJ 1
#endif
template <int N, int EPI, int NZ>
constexpr bool ws_eo() {
  // plain applies, and (WS_EO_ADJ) the adjoint stage, whose J^T contraction is the plain one and
  // whose recurrence epilogue keeps its association; the RK stage keeps the full matrices
  return WS_EO && (N + 1) % 16 == 0 && ((EPI == EPI_STORE && NZ < 0) || (WS_EO_ADJ && EPI == EPI_ADJ && NZ >= 0));
}
#ifndef WS_MINB32_F_EO
#define WS_MINB32_F_EO 3
#endif
#ifndef WS_CW32_EO
#define WS_CW32_EO 4
#endif
#ifndef WS_ELEMS32_EO
#define WS_ELEMS32_EO 64
#endif
// NZ >= 0: the adjoint-stage variant (J^T with the z = b lam + sum_j a_j l_j prologue and
// the l / lam_out epilogue, adjoint.py:54-61) reading NZ l_j slabs besides U and lam
template <int N, int OP, int NZ = -1, bool EO = false>
constexpr int ws_minb() {
  if constexpr (NZ >= 0) return ((N + 1) == 32 && NZ > 0) ? 1 : 2;
  if constexpr (EO && (N + 1) == 32 && OP == OP_RHS) return WS_MINB32_F_EO;
  return ((N + 1) > 16) ? (OP == OP_RHS ? WS_MINB32_F : WS_MINB32)
                        : ((N + 1) == 16 ? 2 : (OP == OP_RHS ? WS_MINB_F8 : (OP == OP_JAC ? WS_MINB_J8 : WS_MINB_JT8)));
}

// ws-kernel B fragments with permuted output columns: DMMA output column
// c = 8nt + 2kq + h holds element row sigma(c) = 4(2nt + h) + kq, i.e. exactly the
// node this lane already holds as its A-fragment column for kc = 2nt + h.  The
// pointwise terms (u_i, v_i, zm_i, M^-1_i) then come from registers, not smem.
template <int N>
__device__ __forceinline__ double bfrag_perm(const Consts<N>& C, int mat, int nt, int kc, int lane) {
  constexpr int n = N + 1;
  const int c = 8 * nt + (lane >> 2);            // B column = DMMA output column
  const int i = 4 * (2 * (c >> 3) + (c & 1)) + ((c >> 1) & 3);
  const int j = 4 * kc + (lane & 3);
  if (mat == 0) return C.K[i * n + j];
  if (mat == 1) return C.Dw[i * n + j];
  return C.Dw[j * n + i];
}

// WS_EO: the plain applies at n % 16 == 0 (N = 15, 31: config 3) on the reflection (even/odd)
// split of K, Dw and Dw^T.  GLL nodes and weights are symmetric about the element midpoint, so
// K is centrosymmetric (K[N-i][N-j] = K[i][j]) and Dw, Dw^T anti-centrosymmetric.  With
// s_j = x_j + x_{N-j}, d_j = x_j - x_{N-j} (j < n/2) every n x n product becomes two
// (n/2) x (n/2) products on the half-length vectors,
//   (M x)_i = (Me s)_i + (Mo d)_i,  (M x)_{N-i} = +-((Me s)_i - (Mo d)_i)   (+ K, - Dw / Dw^T),
// i.e. n^2/32 DMMA m8n8k4 per product instead of n^2/16 -- these kernels are bound by the
// FP64 datapath the DMMAs occupy, not by HBM -- for n/4 + n/4 extra FP64 adds per lane.  The
// half blocks are at least one 8-column n-tile wide for n >= 16, so no DMMA column is wasted
// (n = 8 has 4-wide blocks: only F, whose two matrices share their input, gains there, see
// sem1d_tilerf.cuh).  Lane (rr, kq) holds node pairs (j, N - j), j = 4kc + kq, kc < n/8, and
// receives output rows i and N - i for the same set: rows 0 and N both sit in lane kq = 0.
// Sections of the fragment table: [Ke, Ko, De, Do, Te, To] and, for F on periodic rings,
// [Ke', Ko', De', Do'] with -nu M^-1_i / M^-1_i folded into row i (T = Dw^T).  The blocks are
// formed from both halves of each matrix (the host matrices are centrosymmetric to about one
// ulp only).  RK-stage and adjoint-stage launches keep the full-matrix fragments: their
// epilogues promise the reference's association (the adaptive Kutta-3 error estimate is a
// cancellation at the tolerance level).

// Double-double helpers for forming the half blocks.  A block entry is a signed sum of four
// scaled matrix entries that may cancel; rounding each product and partial sum would perturb
// the effective matrix by an ulp of its LARGEST mirrored entry, which on smooth inputs (where
// K u cancels to a small result) costs as much accuracy as the contraction itself.  So the
// four terms are formed as exact products (two_prod), summed in double-double, and rounded
// once.  Only IEEE operations and FMA: the host table and the in-kernel construction agree
// bit for bit.
struct DD {
  double hi, lo;
};
__host__ __device__ inline double dd_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
__host__ __device__ inline double dd_add1(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double t = a + b;
  return t;
#endif
}
__host__ __device__ inline DD dd_two_sum(double a, double b) {
  const double s = dd_add1(a, b), bb = dd_add1(s, -a);
  return {s, dd_add1(dd_add1(a, -dd_add1(s, -bb)), dd_add1(b, -bb))};
}
__host__ __device__ inline DD dd_two_prod(double a, double b) {
  const double p = dd_fma(a, b, 0.0);
  return {p, dd_fma(a, b, -p)};
}
__host__ __device__ inline DD dd_add(DD x, DD y) {
  DD s = dd_two_sum(x.hi, y.hi);
  return dd_two_sum(s.hi, dd_add1(s.lo, dd_add1(x.lo, y.lo)));
}
__host__ __device__ inline DD dd_mul(DD x, double y) {
  DD p = dd_two_prod(x.hi, y);
  return dd_two_sum(p.hi, dd_add1(p.lo, dd_fma(x.lo, y, 0.0)));
}
__host__ __device__ inline DD dd_neg(DD x) { return {-x.hi, -x.lo}; }
// even (par 0) / odd (par 1) half-block entry (i, j), i, j < n/2, of the matrix whose entries
// term(r, s) returns (as double-doubles): centrosymmetric (centro) or anti-centrosymmetric;
// formed from both halves, 1/4 ((M[i][j] +- M[N-i][N-j]) +- (M[i][N-j] +- M[N-i][j]))
template <class Term>
__host__ __device__ inline double eo_block_entry(Term term, bool centro, int par, int i, int j, int N) {
  DD b = term(N - i, N - j), d = term(N - i, j);
  if (!centro) {
    b = dd_neg(b);
    d = dd_neg(d);
  }
  const DD ab = dd_add(term(i, j), b), cd = dd_add(term(i, N - j), d);
  const DD t = dd_add(ab, par == 0 ? cd : dd_neg(cd));
  return 0.25 * dd_add1(t.hi, t.lo);
}

// sec: 0..5 = Ke, Ko, De, Do, Te, To; 6..9 = the prescaled Ke', Ko', De', Do' (F and J on periodic
// rings); 10..15 = J^T on periodic rings with M^-1 and -nu folded in, so z enters unscaled:
// K''e, K''o of K diag(-nu M^-1), De', Do' again, T''e, T''o of -Dw^T diag(M^-1) (negated: its
// products accumulate into the K'' chains)
template <int N>
__host__ __device__ inline double bfrag_eo_value(const double* K, const double* Dw, const double* minv, double nu,
                                                 int sec, int nt, int kc, int lane) {
  constexpr int n = N + 1;
  const bool jt = sec >= 10 && sec != 12 && sec != 13;   // column-scaled K'' / T''
  if (sec == 12 || sec == 13) sec -= 4;                  // De', Do'
  const bool pre = !jt && sec >= 6;
  const int mat = jt ? sec - 10 : (pre ? sec - 6 : sec);
  const int m = mat >> 1, par = mat & 1;
  const int c = 8 * nt + (lane >> 2);
  const int i = 4 * (2 * (c >> 3) + (c & 1)) + ((c >> 1) & 3);   // output row, < n/2
  const int j = 4 * kc + (lane & 3);                             // input node, < n/2
  auto mv = [&](int r) -> double { return minv[(r == 0 || r == N) ? 0 : r]; };
  auto term = [&](int r, int s) -> DD {
    const double b = m == 0 ? K[r * n + s] : (m == 1 ? Dw[r * n + s] : Dw[s * n + r]);
    if (jt) return m == 0 ? dd_mul(dd_two_prod(-nu, mv(s)), b) : dd_neg(dd_two_prod(b, mv(s)));
    if (pre) return m == 0 ? dd_mul(dd_two_prod(-nu, mv(r)), b) : dd_two_prod(b, mv(r));
    return DD{b, 0.0};
  };
  return eo_block_entry(term, m == 0, par, i, j, N);
}

#ifndef WS_ELEMS8_J
#define WS_ELEMS8_J 256
#endif
template <int N, int OP = OP_RHS, int NZ = -1, bool EO = false>
struct WsTile {
  static constexpr int n = N + 1;
  static constexpr bool ADJ = NZ >= 0;
  // inputs staged per tile: u; v / z / lam; the adjoint stage's NZ l_j fields
  static constexpr int NIN = (OP == OP_RHS) ? 1 : 2 + (ADJ ? NZ : 0);
  // consumer warps: n = 32 per operator (see WS_CW32 above), else 8
  static constexpr int CW =
      (n == 32) ? (ADJ ? 4 : (OP == OP_JACT ? WS_CW32_JT : (OP == OP_JAC ? WS_CW32_J : (EO ? WS_CW32_EO : WS_CW32)))) : 8;
  static constexpr int THREADS = 32 * (CW + 1);
  // the adjoint stage stages up to 4 inputs: half-size tiles keep 2 CTAs/SM at n = 8 and 16
  static constexpr int ELEMS =
      ADJ ? (n == 8 ? 128 : 64)
          : (n == 8) ? (OP == OP_RHS ? WS_ELEMS8 : WS_ELEMS8_J)
                     : (n == 32 ? (OP == OP_RHS ? (EO ? WS_ELEMS32_EO : WS_ELEMS32) : 16 * CW) : MmaTile<N>::ELEMS);
  static constexpr int WE = ELEMS / CW;                          // elements per consumer warp
  static constexpr int WMT = WE / 8;                             // m-tiles per warp
  static constexpr int NT = n / 8, KC = n / 4;
  static constexpr int SLAB = (ELEMS + 1) * N + 1;
  static constexpr int SLAB_ALLOC = ((SLAB + 1) + 1) & ~1;
  static constexpr int OUT = ((ELEMS * N + 2) + 1) & ~1;         // per-CTA output staging
  static constexpr bool B_IN_SMEM = (n > 16);
};

// Programmatic dependent launch (the apply kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel may start its prologue while
// the previous kernel in the stream drains; griddep_wait() blocks until that kernel has
// completed and its memory is visible, so it precedes every global access of the data path.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// PRE (F on periodic rings): the K / Dw fragments carry -nu M^-1_i / M^-1_i of the output row,
// so kx and du are already scaled and the row is M^-1-scaled F
template <int N, int OP, bool PRE = false>
__device__ __forceinline__ double combine_rows(double kx, double du, double qq, double ui,
                                               double wi, double mnu) {
  if (OP == OP_RHS) return PRE ? __dsub_rn(kx, __dmul_rn(ui, du)) : __dsub_rn(__dmul_rn(kx, mnu), __dmul_rn(ui, du));
  if (OP == OP_JAC)
    return __dsub_rn(__dsub_rn(__dmul_rn(kx, mnu), __dmul_rn(wi, du)), __dmul_rn(ui, qq));
  return __dsub_rn(__dsub_rn(__dmul_rn(kx, mnu), __dmul_rn(wi, du)), qq);
}

// Second input of the ws kernel as the consumers read it: the staged v / z slab (a plain
// pointer), or for the adjoint stage (NZ >= 0) z of adjoint.py:58-60 formed at fragment-load
// time from the staged lam and l_j slabs, in the reference's order:
// z = ((b lam + a_0 l_0) + a_1 l_1) + ...
template <int NZ>
struct WSrc {
  const double* w;
  const double* l[NZ > 0 ? NZ : 1];
  double b;
  double a[NZ > 0 ? NZ : 1];
  __device__ __forceinline__ double operator[](int i) const {
    double z = __dmul_rn(b, w[i]);
#pragma unroll
    for (int j = 0; j < NZ; ++j) z = __dadd_rn(z, __dmul_rn(a[j], l[j][i]));
    return z;
  }
};

// One DMMA m-tile: 8 elements (A rows) x n rows, pointwise-combined.  Lane
// (rr, kq) ends with rows i = 8nt + 2kq + h of element rr in r[nt][h].
// EDGE = tile touches a Dirichlet end (masking / special M^-1 entries).
template <int N, int OP, bool EDGE>
struct MTileOut {
  double r[N / 8 + 1][2];
};

// LAST: only the last output n-tile (rows 4(2NT-2+h)+kq, which hold row N): the producer's
// halo rows of the ws kernel need nothing else (n = 32: 16 of F's 64 DMMAs per halo m-tile)
template <int N, int OP, bool EDGE, class BGet, bool PRE = false, bool LAST = false, class WS = const double*>
__device__ __forceinline__ void mtile_compute(const Consts<N>& C, const Geo& G, const double* su,
                                              const WS& sw, int base, int64_t eg,
                                              const double* minv_a, const double (*minv_p)[2],
                                              double mnu, int kq, BGet bget, ws_fin_t& fin_u,
                                              ws_fin_t& fin_w, double (&r)[(N + 1) / 8][2]) {
  constexpr int n = N + 1, NT = n / 8, KC = n / 4;
  const bool eslow = EDGE && (eg == 0 || eg == G.E - 1);
  double au[KC], aw[(OP != OP_RHS) ? KC : 1], at[(OP == OP_JACT) ? KC : 1];
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int j = 4 * kc + kq;
    au[kc] = su[base + j];
    WS_FIN_ACC(fin_u, au[kc]);
    if (OP != OP_RHS) {
      aw[kc] = sw[base + j];
      WS_FIN_ACC(fin_w, aw[kc]);
      if (OP == OP_JACT) {
        aw[kc] = eslow ? jt_scale<N>(C, aw[kc], j, eg, G) : __dmul_rn(aw[kc], minv_a[kc]);
        at[kc] = __dmul_rn(au[kc], aw[kc]);
      }
    }
  }
#pragma unroll
  for (int nt = LAST ? NT - 1 : 0; nt < NT; ++nt) {
    double k0 = 0.0, k1 = 0.0, p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      dmma884(k0, k1, (OP == OP_RHS) ? au[kc] : aw[kc], bget(0, nt, kc));   // K x
      dmma884(p0, p1, au[kc], bget(1, nt, kc));                            // Dw u
      if (OP == OP_JAC) dmma884(q0, q1, aw[kc], bget(1, nt, kc));          // Dw v
      if (OP == OP_JACT) dmma884(q0, q1, at[kc], bget(2, nt, kc));         // Dw^T (u o zm)
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      // permuted output column (2kq+h of n-tile nt) = node 4(2nt+h)+kq = A column kc'
      const int kcp = 2 * nt + h;
      const double ui = au[kcp];
      double wi = 0.0;
      if (OP == OP_JAC) wi = aw[kcp];
      if (OP == OP_JACT) wi = aw[kcp];   // already zm = mask(z M^-1)
      r[nt][h] = combine_rows<N, OP, PRE>(h ? k1 : k0, h ? p1 : p0, h ? q1 : q0, ui, wi, mnu);
    }
  }
}

#ifndef WS_ILV
#define WS_ILV 1
#endif
// J^T at n = 8 on interleaved rows too (round 2: 107.1 -> 106.6 us; round 1 had measured it
// slower, 126.9 vs 112.2, before the fragment table and the other kernel changes)
#ifndef WS_ILV_JT7
#define WS_ILV_JT7 1
#endif
// n = 32: output n-tiles per accumulation group in mtile_compute_multi (A/B on config 3:
// 1 / 2 / 4 -> J^T 90.0 / 88.3 / 88.0 us, F and J flat within 0.3%; 4 slowed J to 75.8 us)
// F on periodic rings: -nu M^-1 / M^-1 folded into the K / Dw fragments (2 FP64 multiplies per
// node fewer on the pipe the DMMAs share)
#ifndef WS_PRE_F
#define WS_PRE_F 1
#endif
// round 2 (config 3, 64-element J / J^T tiles): 4 n-tiles per group for F and J^T
// (47.27 -> 47.0 us, 67.0 -> 66.1 us), 2 for J (66.4 against 67.15 at 4)
#ifndef WS_NTG_FT
#define WS_NTG_FT 4
#endif
#ifndef WS_NTG
#define WS_NTG 2
#endif
// Warp-local element held by row rr of m-tile q (apply_ws_kernel).  ILV (WMT = 2 or 4):
// interleaved rows, so the 64-bit slab loads/stores of a half-warp (rows 4h..4h+3, nodes
// N*e + kq) hit 16 distinct banks for odd N -- the half-warp's elements are congruent mod 4
// and distinct mod 16 (the contiguous mapping puts rows N apart: 4-way conflicts at N = 31).
// Same mapping as ring_elem of the sweep kernels.
template <int WMT, bool ILV>
__device__ __forceinline__ int ws_le(int q, int rr) {
  if constexpr (ILV && WMT == 2) return 4 * (rr & 3) + 2 * (rr >> 2) + q;
  else if constexpr (ILV && WMT == 4) return 4 * rr + q;
  else return 8 * q + rr;
}
// ILV: row of m-tile WMT-1 holding the left neighbour of (rr > 0, m-tile 0)
template <int WMT>
__device__ __forceinline__ int ws_left_row(int rr) {
  if constexpr (WMT == 2) return rr >= 4 ? rr - 4 : rr + 3;
  else return rr > 0 ? rr - 1 : 0;
}

// Q m-tiles of one warp at once (elements wbase/weg + ws_le(q, rr)): the loops over the output
// n-tiles and k-chunks are outermost, so each B fragment -- read from shared memory when
// the n x n matrices do not fit the register file (n = 32) -- feeds Q DMMAs instead of one.
template <int N, int OP, bool EDGE, int Q, bool ILV, class BGet, bool PRE = false, class WS = const double*>
__device__ __forceinline__ void mtile_compute_multi(const Consts<N>& C, const Geo& G, const double* su,
                                                    const WS& sw, int wbase, int64_t weg, int rr,
                                                    const double* minv_a, double mnu, int kq, BGet bget,
                                                    ws_fin_t& fin_u, ws_fin_t& fin_w,
                                                    double (&r)[Q][(N + 1) / 8][2]) {
  constexpr int n = N + 1, NT = n / 8, KC = n / 4;
  double au[Q][KC], aw[Q][(OP != OP_RHS) ? KC : 1], at[Q][(OP == OP_JACT) ? KC : 1];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int le = ws_le<Q, ILV>(q, rr);
    const int64_t eg = weg + le;
    const int base = wbase + le * N;
    const bool eslow = EDGE && (eg == 0 || eg == G.E - 1);
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      const int j = 4 * kc + kq;
      au[q][kc] = su[base + j];
      WS_FIN_ACC(fin_u, au[q][kc]);
      if (OP != OP_RHS) {
        aw[q][kc] = sw[base + j];
        WS_FIN_ACC(fin_w, aw[q][kc]);
        if (OP == OP_JACT) {
          aw[q][kc] = eslow ? jt_scale<N>(C, aw[q][kc], j, eg, G) : __dmul_rn(aw[q][kc], minv_a[kc]);
          at[q][kc] = __dmul_rn(au[q][kc], aw[q][kc]);
        }
      }
    }
  }
  // NTG output n-tiles at a time: NTG x Q x (2 or 3) independent accumulator chains per warp
  // hide the DMMA -> DMMA latency of the k-chunk chains
  constexpr int NTGW = (OP == OP_JAC) ? WS_NTG : WS_NTG_FT;
  constexpr int NTG = (NT % NTGW == 0) ? NTGW : 1;
#pragma unroll
  for (int nt0 = 0; nt0 < NT; nt0 += NTG) {
    double k[NTG][Q][2], p[NTG][Q][2], qq[NTG][Q][2];
#pragma unroll
    for (int g = 0; g < NTG; ++g)
#pragma unroll
      for (int q = 0; q < Q; ++q) k[g][q][0] = k[g][q][1] = p[g][q][0] = p[g][q][1] = qq[g][q][0] = qq[g][q][1] = 0.0;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
#pragma unroll
      for (int g = 0; g < NTG; ++g) {
        const int nt = nt0 + g;
        const double b0 = bget(0, nt, kc), b1 = bget(1, nt, kc);
        const double b2 = (OP == OP_JACT) ? bget(2, nt, kc) : 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          dmma884(k[g][q][0], k[g][q][1], (OP == OP_RHS) ? au[q][kc] : aw[q][kc], b0);
          dmma884(p[g][q][0], p[g][q][1], au[q][kc], b1);
          if (OP == OP_JAC) dmma884(qq[g][q][0], qq[g][q][1], aw[q][kc], b1);
          if (OP == OP_JACT) dmma884(qq[g][q][0], qq[g][q][1], at[q][kc], b2);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < NTG; ++g)
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kcp = 2 * (nt0 + g) + h;
          const double wi = (OP == OP_RHS) ? 0.0 : aw[q][kcp];
          r[q][nt0 + g][h] = combine_rows<N, OP, PRE>(k[g][q][h], p[g][q][h], qq[g][q][h], au[q][kcp], wi, mnu);
        }
  }
}

// WS_EO form of mtile_compute / mtile_compute_multi (n % 16 == 0): Q m-tiles at once on the
// half-length sum / difference vectors.  base[q] = slab index of node 0 of the lane's element
// in m-tile q, eg[q] its global element.  Output: r[q][nt][h] is row 4(2nt + h) + kq for
// nt < NT/2 and row N - (4(2(nt - NT/2) + h) + kq) above (ws_row_eo).  minv_lo / minv_hi:
// M^-1 at nodes 4kc + kq and N - (4kc + kq).  LAST: only the n-tile that holds row N.
#ifndef WS_EO_NTG
#define WS_EO_NTG 1
#endif
// J and J^T on periodic rings with the pointwise scalings on the fragments, as F has them
// (WS_PRE_F): J = K'v - v o (Dw'u) - u o (Dw'v) is two DFMAs per row instead of three multiplies,
// two subtractions and the M^-1 product; J^T takes z unscaled, K'' = K diag(-nu M^-1) and
// T'' = -Dw^T diag(M^-1) accumulate into one pair of chains, and a row is one DFMA
#ifndef WS_EO_PRE
#define WS_EO_PRE 1
#endif
// A/B only (off): the producer warp's halo rows (row N of the element left of each consumer
// warp) as dot products on the FP64 vector pipe instead of a halo m-tile of 16-24 DMMAs.  The
// idea was that the producer warps of all resident CTAs share one SM sub-partition with two
// consumer warps and lengthen its DMMA queue by 25%.  Measured on config 3 it loses, and the
// times become unstable from launch to launch: F 35.8-36.2 us against 31.8, J 44-51.5 against
// 47.9, J^T 53.7-55.6 against 47.0 -- vector FP64 work interleaved into the consumers' DMMA
// phases on that sub-partition costs more than the DMMAs it replaces.
#ifndef WS_EO_HALO
#define WS_EO_HALO 0
#endif
#ifndef WS_PROD_SLEEP
#define WS_PROD_SLEEP 0
#endif
// bit OP set: that operator takes its m-tiles one at a time even with the fragments in shared
// memory (register pressure: 6 half-length vectors and 6 accumulator pairs per m-tile for J^T)
#ifndef WS_EO_Q1
#define WS_EO_Q1 7
#endif
// A/B only: J^T in two DMMA passes per n-tile group (K zm + Dw^T (u o zm) first, then Dw u on
// sums and differences formed after the first pass, four half-length vectors live instead of
// six).  Config 3: 58.6 us against 48.8 in one pass -- two short phases per m-tile leave the
// FP64 datapath idle more often than the one-pass form's spills cost.
#ifndef WS_EO_JT2P
#define WS_EO_JT2P 0
#endif
template <int N, int OP, bool EDGE, int Q, class BGet, bool PRE, bool LAST, class WS>
__device__ __forceinline__ void mtile_compute_eo(const Consts<N>& C, const Geo& G, const double* su, const WS& sw,
                                                 const int (&base)[Q], const int64_t (&eg)[Q],
                                                 const double* minv_lo, const double* minv_hi, double mnu,
                                                 int kq, BGet bget, ws_fin_t& fin_u, ws_fin_t& fin_w,
                                                 double (&r)[Q][(N + 1) / 8][2]) {
  constexpr int n = N + 1, NT2 = n / 16, H = n / 8;
  constexpr int HX = (OP != OP_RHS) ? H : 1, HT = (OP == OP_JACT) ? H : 1;
  constexpr bool TWOPASS = WS_EO_JT2P && OP == OP_JACT;
  double us[Q][H], ud[Q][H], xs[Q][HX], xd[Q][HX], ts[Q][HT], td[Q][HT];
  // the second input at node j of m-tile q as the contraction sees it (J^T: masked z M^-1)
  auto second = [&](int q, int kc, bool hi, bool acc) -> double {
    const int j = hi ? N - (4 * kc + kq) : 4 * kc + kq;
    double w = sw[base[q] + j];
    if (acc) WS_FIN_ACC(fin_w, w);
    if (OP == OP_JACT && !PRE) {                 // (PRE: M^-1 rides on the fragments)
      const bool eslow = EDGE && (eg[q] == 0 || eg[q] == G.E - 1);
      w = eslow ? jt_scale<N>(C, w, j, eg[q], G) : __dmul_rn(w, hi ? minv_hi[kc] : minv_lo[kc]);
    }
    return w;
  };
#pragma unroll
  for (int q = 0; q < Q; ++q) {
#pragma unroll
    for (int kc = 0; kc < H; ++kc) {
      const int j = 4 * kc + kq;
      const double a0 = su[base[q] + j], a1 = su[base[q] + N - j];
      WS_FIN_ACC(fin_u, a0);
      WS_FIN_ACC(fin_u, a1);
      if (!TWOPASS) {
        us[q][kc] = __dadd_rn(a0, a1);
        ud[q][kc] = __dsub_rn(a0, a1);
      }
      if (OP != OP_RHS) {
        const double w0 = second(q, kc, false, true), w1 = second(q, kc, true, true);
        xs[q][kc] = __dadd_rn(w0, w1);
        xd[q][kc] = __dsub_rn(w0, w1);
        if (OP == OP_JACT) {
          const double t1 = __dmul_rn(a1, w1);   // u o zm sums / differences: one product, two DFMAs
          ts[q][kc] = __fma_rn(a0, w0, t1);
          td[q][kc] = __fma_rn(a0, w0, -t1);
        }
      }
    }
  }
  constexpr int NTG = (!LAST && NT2 % WS_EO_NTG == 0) ? WS_EO_NTG : 1;
#pragma unroll
  for (int nt0 = 0; nt0 < (LAST ? 1 : NT2); nt0 += NTG) {
    // even (s) and odd (d) parts of K x, Dw u and Dw v / Dw^T (u o zm): 4 or 6 independent
    // accumulator chains per m-tile and n-tile
    double ke[NTG][Q][2], ko[NTG][Q][2], pe[NTG][Q][2], po[NTG][Q][2], qe[NTG][Q][2], qo[NTG][Q][2];
#pragma unroll
    for (int g = 0; g < NTG; ++g)
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) ke[g][q][h] = ko[g][q][h] = pe[g][q][h] = po[g][q][h] = qe[g][q][h] = qo[g][q][h] = 0.0;
#pragma unroll
    for (int kc = 0; kc < H; ++kc) {
#pragma unroll
      for (int g = 0; g < NTG; ++g) {
        const int nt = nt0 + g;
        const double bke = bget(0, nt, kc), bko = bget(1, nt, kc), bde = bget(2, nt, kc), bdo = bget(3, nt, kc);
        const double bte = (OP == OP_JACT) ? bget(4, nt, kc) : 0.0, bto = (OP == OP_JACT) ? bget(5, nt, kc) : 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          dmma884(ke[g][q][0], ke[g][q][1], (OP == OP_RHS) ? us[q][kc] : xs[q][kc], bke);
          dmma884(ko[g][q][0], ko[g][q][1], (OP == OP_RHS) ? ud[q][kc] : xd[q][kc], bko);
          if (!TWOPASS) {
            dmma884(pe[g][q][0], pe[g][q][1], us[q][kc], bde);
            dmma884(po[g][q][0], po[g][q][1], ud[q][kc], bdo);
          }
          if (OP == OP_JAC) {
            dmma884(qe[g][q][0], qe[g][q][1], xs[q][kc], bde);
            dmma884(qo[g][q][0], qo[g][q][1], xd[q][kc], bdo);
          }
          if (OP == OP_JACT && PRE) {
            // T'' is negated and its hi rows are O - E: with A = K''e zs + T''o td and
            // B = K''o zd + T''e ts, rows i and N - i of K''z + T''t are A + B and A - B
            dmma884(ko[g][q][0], ko[g][q][1], ts[q][kc], bte);
            dmma884(ke[g][q][0], ke[g][q][1], td[q][kc], bto);
          } else if (OP == OP_JACT) {
            dmma884(qe[g][q][0], qe[g][q][1], ts[q][kc], bte);
            dmma884(qo[g][q][0], qo[g][q][1], td[q][kc], bto);
          }
        }
      }
    }
    if (TWOPASS) {
      if (nt0 == 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
          for (int kc = 0; kc < H; ++kc) {
            const int j = 4 * kc + kq;
            const double a0 = su[base[q] + j], a1 = su[base[q] + N - j];
            us[q][kc] = __dadd_rn(a0, a1);
            ud[q][kc] = __dsub_rn(a0, a1);
          }
      }
#pragma unroll
      for (int kc = 0; kc < H; ++kc)
#pragma unroll
        for (int g = 0; g < NTG; ++g) {
          const double bde = bget(2, nt0 + g, kc), bdo = bget(3, nt0 + g, kc);
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            dmma884(pe[g][q][0], pe[g][q][1], us[q][kc], bde);
            dmma884(po[g][q][0], po[g][q][1], ud[q][kc], bdo);
          }
        }
    }
#pragma unroll
    for (int g = 0; g < NTG; ++g)
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kcp = 2 * (nt0 + g) + h;       // output rows 4kcp + kq and N - (4kcp + kq)
          // pointwise factors come back from the staged slabs (cheaper than 4 n registers per m-tile)
          const double u0 = su[base[q] + 4 * kcp + kq], u1 = su[base[q] + N - (4 * kcp + kq)];
          const double w0 = (OP == OP_RHS) ? 0.0 : second(q, kcp, false, false);
          const double w1 = (OP == OP_RHS) ? 0.0 : second(q, kcp, true, false);
          const double k0 = __dadd_rn(ke[g][q][h], ko[g][q][h]), k1 = __dsub_rn(ke[g][q][h], ko[g][q][h]);
          const double p0 = __dadd_rn(pe[g][q][h], po[g][q][h]), p1 = __dsub_rn(po[g][q][h], pe[g][q][h]);
          if (PRE && OP == OP_RHS) {             // K'u - u o (Dw'u): one DFMA per row
            r[q][nt0 + g][h] = __fma_rn(-u0, p0, k0);
            r[q][NT2 + nt0 + g][h] = __fma_rn(-u1, p1, k1);
          } else if (PRE && OP == OP_JACT) {     // K''z + T''t - z o (Dw'u): one DFMA per row
            r[q][nt0 + g][h] = __fma_rn(-w0, p0, k0);
            r[q][NT2 + nt0 + g][h] = __fma_rn(-w1, p1, k1);
          } else {
            const double q0 = __dadd_rn(qe[g][q][h], qo[g][q][h]), q1 = __dsub_rn(qo[g][q][h], qe[g][q][h]);
            if (PRE && OP == OP_JAC) {           // K'v - v o (Dw'u) - u o (Dw'v): two DFMAs per row
              r[q][nt0 + g][h] = __fma_rn(-u0, q0, __fma_rn(-w0, p0, k0));
              r[q][NT2 + nt0 + g][h] = __fma_rn(-u1, q1, __fma_rn(-w1, p1, k1));
            } else {
              r[q][nt0 + g][h] = combine_rows<N, OP, PRE>(k0, p0, q0, u0, w0, mnu);
              r[q][NT2 + nt0 + g][h] = combine_rows<N, OP, PRE>(k1, p1, q1, u1, w1, mnu);
            }
          }
        }
  }
}
// row held in r[.][nt][h] by lane kq in the WS_EO layout
template <int N>
__device__ __forceinline__ int ws_row_eo(int nt, int h, int kq) {
  constexpr int NT2 = (N + 1) / 16;
  return nt < NT2 ? 4 * (2 * nt + h) + kq : N - (4 * (2 * (nt - NT2) + h) + kq);
}

// NZ >= 0 (OP_JACT, EPI_ADJ): one adjoint stage, adjoint.py:54-61 (see WSrc and the EPI_ADJ
// epilogue below); the same arithmetic and association as apply_kernel<N, OP_JACT, PRO_ADJ, EPI_ADJ>
template <int N, int OP, int EPI, int STAGES, int NZ = -1>
__global__ void __launch_bounds__(WsTile<N, OP, NZ, ws_eo<N, EPI, NZ>()>::THREADS, ws_minb<N, OP, NZ, ws_eo<N, EPI, NZ>()>())
    apply_ws_kernel(const __grid_constant__ Consts<N> C, const Geo G, const Args A,
                    const int tiles_per_ring, const int total_tiles, const double* __restrict__ frag) {
  using W = WsTile<N, OP, NZ, ws_eo<N, EPI, NZ>()>;
  static_assert(!W::ADJ || (OP == OP_JACT && EPI == EPI_ADJ), "adjoint stage = J^T with the EPI_ADJ epilogue");
  constexpr int ELEMS = W::ELEMS, WE = W::WE, WMT = W::WMT, NT = W::NT, KC = W::KC;
  constexpr int NIN = W::NIN;
  constexpr int NMAT = (OP == OP_JACT) ? 3 : 2;
  // WS_EO: half-size blocks, [Ke, Ko, De, Do (, Te, To)][NT/2][KC/2][32]; rows 0 and N in lane kq = 0
  constexpr bool EO = ws_eo<N, EPI, NZ>();
  constexpr int NMAT_EO = (OP == OP_JACT) ? 6 : 4, NT2 = NT / 2, KC2 = KC / 2;
  constexpr int BTOT = EO ? NMAT_EO * NT2 * KC2 * 32 : NMAT * NT * KC * 32;   // B fragments of this kernel
  constexpr int RN_NT = EO ? NT2 : NT - 1, RN_H = EO ? 0 : 1, RN_KQ = EO ? 0 : 3;   // where row N lands
  constexpr int SA = W::SLAB_ALLOC;
  extern __shared__ __align__(16) double smem[];
  double* stage_buf = smem;                                   // [STAGES][NIN][SA]
  constexpr int OUTB = ws_outb<OP>();
  double* ostage = smem + STAGES * NIN * SA;                  // [OUTB][OUT]
  double* hrow = ostage + OUTB * W::OUT;                      // [STAGES][CW] warp halo rows
  double* bsm = hrow + STAGES * W::CW;                        // B fragments (n = 32)
  double* hal = bsm + (W::B_IN_SMEM ? BTOT : 0);              // WS_EO_HALO: 3 scaled matrix rows / columns N
  uint64_t* full = reinterpret_cast<uint64_t*>(hal + (EO ? 3 * (N + 1) : 0));
  uint64_t* empty = full + STAGES;
  uint64_t* halo = empty + STAGES;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const bool periodic = G.periodic != 0;
  // the next kernel may be scheduled as soon as SM resources free up (its data path waits)
  griddep_launch_dependents();

  // tile cursor for the loads (runs STAGES-1 tiles ahead of the halo cursor)
  auto tile_coords = [&](int T, int& tl, int64_t& bofs) {
    const int b = T / tiles_per_ring;
    tl = T - b * tiles_per_ring;
    bofs = (int64_t)b * G.ndof;
  };
  auto load_tile = [&](int T, int s) {
    int tl;
    int64_t bofs;
    tile_coords(T, tl, bofs);
    const int64_t e0 = (int64_t)tl * ELEMS;
    const int nel = (int)min((int64_t)ELEMS, G.E - e0);
    const int cnt = (nel + 1) * N + 1;
    const int64_t g0 = (e0 - 1) * N;
    const int sh = (int)((bofs + g0) & 1);
    const int64_t lo = g0 < 0 ? 0 : g0;
    const int64_t hi = min(g0 + cnt, G.ndof);
    int64_t alo, ahi;
    if (g0 >= 0 && g0 + cnt + 1 <= G.ndof) {
      // interior tile: widen the body outward to 16-byte boundaries (the extra
      // doubles lie inside this ring), so no lane has to load anything itself
      alo = ((bofs + g0) & ~(int64_t)1) - bofs;
      ahi = ((bofs + g0 + cnt + 1) & ~(int64_t)1) - bofs;
    } else {
      alo = ((bofs + lo + 1) & ~(int64_t)1) - bofs;
      ahi = ((bofs + hi) & ~(int64_t)1) - bofs;
      if (ahi < alo) ahi = alo;
    }
    const int k0 = (int)(alo - g0), k1 = (int)(ahi - g0);
    // inputs: u; v / z / lam; the adjoint stage's l_j
    double* dst[NIN];
    const double* src[NIN];
#pragma unroll
    for (int i = 0; i < NIN; ++i) {
      dst[i] = stage_buf + (s * NIN + i) * SA + sh;
      src[i] = (i == 0 ? A.u : (i == 1 ? A.w : A.zin.ptr[i - 2])) + bofs;
    }
    auto scalar_piece = [&](int kb, int ke) {
      for (int k = kb + lane; k < ke; k += 32) {
        int64_t g = g0 + k;
        bool valid = true;
        if (g < 0) {
          if (periodic) g += G.ndof; else valid = false;
        } else if (g >= G.ndof) {
          g -= G.ndof;
        }
#pragma unroll
        for (int i = 0; i < NIN; ++i) dst[i][k] = valid ? __ldg(src[i] + g) : 0.0;
      }
    };
    if (k0 > 0) scalar_piece(0, k0);
    if (k1 < cnt) scalar_piece(k1, cnt);
    for (int k = cnt + lane; k < (ELEMS + 1) * N + 1; k += 32) {  // ragged tile: finite pad
#pragma unroll
      for (int i = 0; i < NIN; ++i) dst[i][k] = 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)((ahi - alo) * 8);
      mbar_expect_tx(&full[s], NIN * bytes);
      if (bytes > 0) {
#pragma unroll
        for (int i = 0; i < NIN; ++i) bulk_g2s(dst[i] + k0, src[i] + alo, bytes, &full[s]);
      }
    }
  };
  // the consumers' second input for stage s (slab pointer, or the adjoint stage's z)
  auto wsrc = [&](int s, int sh) {
    const double* w = stage_buf + (s * NIN + 1) * SA + sh;
    if constexpr (W::ADJ) {
      WSrc<NZ> r;
      r.w = w;
      r.b = A.b;
#pragma unroll
      for (int j = 0; j < (NZ > 0 ? NZ : 1); ++j) {
        r.l[j] = stage_buf + (s * NIN + 2 + (j < NZ ? j : 0)) * SA + sh;
        r.a[j] = A.zin.coef[j];
      }
      return r;
    } else {
      return w;
    }
  };
  int issued = 0;  // tiles issued so far (iteration index of the next load)
  auto issue_next = [&](int T) {
    const int s = issued % STAGES;
    while (!mbar_try_wait(&empty[s], ((issued / STAGES) & 1) ^ 1)) {
      if (WS_PROD_SLEEP) __nanosleep(WS_PROD_SLEEP);   // the producer shares its sub-partition with consumers
    }
    load_tile(T, s);
    ++issued;
  };
  // the producer initialises the barriers; with the fragment table in shared memory (n = 32,
  // a 16-24 KB copy) it also puts the first STAGES-1 tile loads in flight before the CTA-wide
  // prologue, hiding their HBM latency behind it (config 3: F/J/J^T -5%; at n = 8, whose
  // prologue is short, the early issue measured 2% slower for F)
  constexpr bool EARLY = W::B_IN_SMEM;
  auto issue_first = [&]() {
    griddep_wait();              // inputs may come from the previous kernel in the stream
    for (int p = 0; p < STAGES - 1; ++p) {
      const int T = blockIdx.x + p * gridDim.x;
      if (T < total_tiles) issue_next(T);
    }
  };
  if (EARLY ? (warp == W::CW && lane == 0) : tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W::CW);
      mbar_init(&halo[s], 1);
    }
    fence_mbar_init();
  }
  if constexpr (EARLY) {
    if (warp == W::CW) {
      __syncwarp();
      issue_first();
    }
  }
  // B fragments: a coalesced copy of the plan's device table (bfrag_perm order; J^T's Dw^T
  // table follows Dw's), else built from kernel-parameter space (lane-divergent reads: 13% of
  // the stall samples of the config-3 F kernel)
  // F on a periodic ring reads the prescaled fragments (second part of the plan's table)
  // (plain applies only: the RK-stage epilogue keeps the reference's association, which the
  // adaptive Kutta-3 error estimate -- a cancellation at the tolerance level -- is sensitive to)
  // WS_EO: J and J^T too (sections 6..9 and 10..15 of the reflection-split table)
  const bool pre = WS_PRE_F && (OP == OP_RHS || (EO && WS_EO_PRE)) && EPI == EPI_STORE && periodic && frag != nullptr;
  constexpr int PRE_SEC = (OP == OP_JACT) ? 10 : 6;          // first prescaled section of this operator
  if (EO) {
    if (frag) frag += 5 * NT * KC * 32 + (pre ? PRE_SEC * NT2 * KC2 * 32 : 0);
  } else if (pre) {
    frag += 3 * NT * KC * 32;
  }
  if (W::B_IN_SMEM) {
    constexpr int TOT = BTOT, PER = (TOT + W::THREADS - 1) / W::THREADS;
    if (frag) {                    // every load in flight before the first store
      double t[PER];
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int q = tid + r * W::THREADS;
        t[r] = q < TOT ? __ldg(frag + q) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int q = tid + r * W::THREADS;
        if (q < TOT) bsm[q] = t[r];
      }
    }
    for (int q = tid; q < TOT && !frag; q += W::THREADS) {
      {
        const int l = q & 31, r = q >> 5;
        if constexpr (EO) {
          const int kc = r % KC2, nt = (r / KC2) % NT2, mat = r / (KC2 * NT2);
          bsm[q] = bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, mat + (pre ? PRE_SEC : 0), nt, kc, l);
        } else {
        const int kc = r % KC, nt = (r / KC) % NT, mat = r / (KC * NT);
        bsm[q] = bfrag_perm<N>(C, mat, nt, kc, l);
        }
      }
    }
  }
  if constexpr (EO) {
    // WS_EO_HALO: row N of the prescaled matrices (the producer's halo rows are three dot
    // products per element on the FP64 vector pipe instead of 16-24 DMMAs)
    if (WS_EO_HALO && pre) {
      constexpr int n = N + 1;
      const double m0 = C.minv[0];
      for (int j = tid; j < n; j += W::THREADS) {
        const double mj = C.minv[(j == 0 || j == N) ? 0 : j];
        hal[j] = (OP == OP_JACT) ? __dmul_rn(C.K[N * n + j], __dmul_rn(-C.nu, mj))
                                 : __dmul_rn(C.K[N * n + j], __dmul_rn(-C.nu, m0));
        hal[n + j] = __dmul_rn(C.Dw[N * n + j], m0);
        hal[2 * n + j] = -__dmul_rn(C.Dw[j * n + N], mj);
      }
    }
  }
  __syncthreads();

  // per-lane constants (all warps): B fragments, M^-1 at fragment positions
  double breg[W::B_IN_SMEM ? 1 : (EO ? NMAT_EO * NT2 * KC2 : NMAT * NT * KC)];
  if (!W::B_IN_SMEM && EO) {
#pragma unroll
    for (int mat = 0; mat < NMAT_EO; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
        for (int kc = 0; kc < KC2; ++kc)
          breg[(mat * NT2 + nt) * KC2 + kc] =
              frag ? __ldg(frag + ((mat * NT2 + nt) * KC2 + kc) * 32 + lane)
                   : bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, mat + (pre ? PRE_SEC : 0), nt, kc, lane);
  }
  if (!W::B_IN_SMEM && !EO) {
#pragma unroll
    for (int mat = 0; mat < NMAT; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
          breg[(mat * NT + nt) * KC + kc] =
              frag ? __ldg(frag + ((mat * NT + nt) * KC + kc) * 32 + lane) : bfrag_perm<N>(C, mat, nt, kc, lane);
  }
  auto bget = [&](int mat, int nt, int kc) -> double {
    if (EO) {
      if (W::B_IN_SMEM) return bsm[((mat * NT2 + nt) * KC2 + kc) * 32 + lane];
      return breg[(mat * NT2 + nt) * KC2 + kc];
    }
    if (W::B_IN_SMEM) return bsm[((mat * NT + nt) * KC + kc) * 32 + lane];
    return breg[(mat * NT + nt) * KC + kc];
  };
  const int kq = lane & 3, rr = lane >> 2;
  const double mnu = -C.nu;
  double minv_a[KC];                                // M^-1 at A columns j = 4kc + kq
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int j = 4 * kc + kq;
    minv_a[kc] = C.minv[(j == 0 || j == N) ? 0 : j];
  }
  double minv_p[NT][2];                             // M^-1 at output rows i = 8nt + 2kq + h
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = 8 * nt + 2 * kq + h;
      minv_p[nt][h] = C.minv[(i == 0 || i == N) ? 0 : i];
    }
  double minv_hi[KC2 > 0 ? KC2 : 1];                // WS_EO: M^-1 at the mirrored nodes N - (4kc + kq)
#pragma unroll
  for (int kc = 0; kc < KC2; ++kc) {
    const int j = N - (4 * kc + kq);
    minv_hi[kc] = C.minv[(j == 0 || j == N) ? 0 : j];
  }
  // row held in r[nt][h] by this lane, and M^-1 there
  auto row_of = [&](int nt, int h) -> int {
    if constexpr (EO) return ws_row_eo<N>(nt, h, kq);
    else return 4 * (2 * nt + h) + kq;
  };
  auto minv_row = [&](int nt, int h) -> double {
    if constexpr (EO) return nt < NT2 ? minv_a[2 * nt + h] : minv_hi[2 * (nt - NT2) + h];
    else return minv_a[2 * nt + h];
  };
  const double minv_if = C.minv[0];
  ws_fin_t fin_u = 0, fin_w = 0;
  bool bad_y = false;

  // ------------------------------------------------------------------ producer
  if (warp == W::CW) {
    if constexpr (!EARLY) issue_first();
    int it = 0;
    for (int T = blockIdx.x; T < total_tiles; T += gridDim.x, ++it) {
      // row N of the element left of each consumer warp: one DMMA m-tile whose
      // row rr is tile-local element rr*WE - 1 (slab base rr*WE*N).  Done before
      // the next issue so the consumers' halo wait never sits behind a refill.
      const int s = it % STAGES;
      int tl;
      int64_t bofs;
      tile_coords(T, tl, bofs);
      const int64_t e0 = (int64_t)tl * ELEMS;
      const int sh = (int)((bofs + (e0 - 1) * N) & 1);
      const double* su = stage_buf + (s * NIN + 0) * SA + sh;
      const auto sw = wsrc(s, sh);
      while (!mbar_try_wait(&full[s], (it / STAGES) & 1)) {
      }
#pragma unroll 1
      for (int hm = 0; hm < (W::CW + 7) / 8; ++hm) {  // one halo m-tile per 8 consumer warps
        // consumer warp whose left neighbour this is (rows past the last warp repeat it)
        const int wq = min(hm * 8 + rr, W::CW - 1);
        const int64_t eh = e0 + wq * WE - 1;
        const int64_t ehw = (eh < 0) ? G.E - 1 : eh;
        double r[NT][2];
        ws_fin_t du_ = 0, dw_ = 0;
        using BG = decltype(bget);
        if (EO && WS_EO_HALO && pre) {
          // row N of element eh on the vector pipe: lane (rr, kq) sums the products of nodes
          // j = kq, kq + 4, ..., the four partial sums meet by two butterfly shuffles
          constexpr int n = N + 1;
          const int hbase = wq * WE * N;
          double kx = 0.0, du = 0.0, qq = 0.0;
#pragma unroll
          for (int m = 0; m < n / 4; ++m) {
            const int j = 4 * m + kq;
            const double uj = su[hbase + j];
            du = __fma_rn(hal[n + j], uj, du);
            if (OP == OP_RHS) {
              kx = __fma_rn(hal[j], uj, kx);
            } else {
              const double wj = sw[hbase + j];
              kx = __fma_rn(hal[j], wj, kx);
              if (OP == OP_JAC) qq = __fma_rn(hal[n + j], wj, qq);
              else kx = __fma_rn(hal[2 * n + j], __dmul_rn(uj, wj), kx);
            }
          }
#pragma unroll
          for (int x = 1; x <= 2; x <<= 1) {
            kx = __dadd_rn(kx, __shfl_xor_sync(0xffffffffu, kx, x));
            du = __dadd_rn(du, __shfl_xor_sync(0xffffffffu, du, x));
            if (OP == OP_JAC) qq = __dadd_rn(qq, __shfl_xor_sync(0xffffffffu, qq, x));
          }
          const double uN = su[hbase + N];
          double row;
          if (OP == OP_RHS) row = __fma_rn(-uN, du, kx);
          else if (OP == OP_JAC) row = __fma_rn(-uN, qq, __fma_rn(-sw[hbase + N], du, kx));
          else row = __fma_rn(-sw[hbase + N], du, kx);
          r[RN_NT][RN_H] = row;                      // (pre: periodic ring, every halo row exists)
        } else if constexpr (EO) {
          const int hb[1] = {wq * WE * N};
          const int64_t he[1] = {ehw};
          using WSrcT = decltype(sw);
          if (!periodic && (tl == 0 || tl == tiles_per_ring - 1))
            mtile_compute_eo<N, OP, true, 1, BG, false, true, WSrcT>(C, G, su, sw, hb, he, minv_a, minv_hi, mnu, kq, bget,
                                                                    du_, dw_, reinterpret_cast<double (&)[1][NT][2]>(r));
          else if (pre)
            mtile_compute_eo<N, OP, false, 1, BG, true, true, WSrcT>(C, G, su, sw, hb, he, minv_a, minv_hi, mnu, kq, bget,
                                                                    du_, dw_, reinterpret_cast<double (&)[1][NT][2]>(r));
          else
            mtile_compute_eo<N, OP, false, 1, BG, false, true, WSrcT>(C, G, su, sw, hb, he, minv_a, minv_hi, mnu, kq, bget,
                                                                     du_, dw_, reinterpret_cast<double (&)[1][NT][2]>(r));
        } else
        if (!periodic && (tl == 0 || tl == tiles_per_ring - 1))
          mtile_compute<N, OP, true, BG, false, true>(C, G, su, sw, wq * WE * N, ehw, minv_a, minv_p, mnu, kq, bget,
                                                      du_, dw_, r);
        else if (pre)
          mtile_compute<N, OP, false, BG, true, true>(C, G, su, sw, wq * WE * N, ehw, minv_a, minv_p, mnu, kq, bget,
                                                      du_, dw_, r);
        else
          mtile_compute<N, OP, false, BG, false, true>(C, G, su, sw, wq * WE * N, ehw, minv_a, minv_p, mnu, kq, bget,
                                                       du_, dw_, r);
        if (kq == RN_KQ && hm * 8 + rr < W::CW) hrow[s * W::CW + wq] = (!periodic && eh < 0) ? 0.0 : r[RN_NT][RN_H];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&halo[s]);
      const int Tn = T + (STAGES - 1) * gridDim.x;
      if (Tn < total_tiles) issue_next(Tn);
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  int it = 0;
  int tl = blockIdx.x % tiles_per_ring;
  int bidx = blockIdx.x / tiles_per_ring;
  for (int T = blockIdx.x; T < total_tiles; T += gridDim.x, ++it) {
    const int s = it % STAGES;
    const int64_t bofs = (int64_t)bidx * G.ndof;
    const int64_t e0 = (int64_t)tl * ELEMS;
    const int nel = (int)min((int64_t)ELEMS, G.E - e0);
    const int sh = (int)((bofs + (e0 - 1) * N) & 1);
    const bool edge = !periodic && (tl == 0 || tl == tiles_per_ring - 1);
    const double* su = stage_buf + (s * NIN + 0) * SA + sh;
    const auto sw = wsrc(s, sh);
    const int wel0 = warp * WE;
    const int wnel = min(WE, nel - wel0);
    double* wout = ostage + (it % OUTB) * W::OUT + warp * WE * N;   // this warp's node staging
    while (!mbar_try_wait(&full[s], (it / STAGES) & 1)) {
    }
    if (wnel > 0) {
      if (lane == 0) bulk_wait_read<OUTB - 1>();   // the store out of this buffer has drained
      __syncwarp();
      double carry = 0.0;
      auto body = [&](auto edge_tag, auto pre_tag) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        constexpr bool PRE = decltype(pre_tag)::value;
        constexpr bool MULTI = W::B_IN_SMEM && (WMT > 1);
        // interleaved rows: A/B (config 2 / 3) F 86.5 -> 85.3 us, J 111.9 -> 111.0 (n = 8);
        // F 59.9 -> 55.4, J 77.9 -> 73.8 (n = 32); J^T at n = 8 measured slower (126.9 vs 112.2)
        constexpr bool ILVW = WS_ILV && (WMT == 2 || WMT == 4) && !(OP == OP_JACT && N == 7 && !WS_ILV_JT7);
        double rq[WMT][NT][2];
        if constexpr (EO) {
          // Q m-tiles per call: all of the warp's with the fragments in shared memory (each
          // fragment read feeds Q DMMAs), else one at a time
          constexpr int QE = (MULTI && !(WS_EO_Q1 & (1 << OP))) ? WMT : 1;
#pragma unroll
          for (int q0 = 0; q0 < WMT; q0 += QE) {
            int eb[QE];
            int64_t ee[QE];
#pragma unroll
            for (int q = 0; q < QE; ++q) {
              const int le = ws_le<WMT, ILVW>(q0 + q, rr);
              eb[q] = (wel0 + le + 1) * N;
              ee[q] = e0 + wel0 + le;
            }
            mtile_compute_eo<N, OP, EDGE, QE, decltype(bget), PRE, false, decltype(sw)>(
                C, G, su, sw, eb, ee, minv_a, minv_hi, mnu, kq, bget, fin_u, fin_w,
                reinterpret_cast<double (&)[QE][NT][2]>(rq[q0]));
          }
        } else if constexpr (MULTI) {
          mtile_compute_multi<N, OP, EDGE, WMT, ILVW, decltype(bget), PRE>(C, G, su, sw, (wel0 + 1) * N, e0 + wel0, rr,
                                                                          minv_a, mnu, kq, bget, fin_u, fin_w, rq);
        } else {
#pragma unroll
          for (int q = 0; q < WMT; ++q) {
            const int le = ws_le<WMT, ILVW>(q, rr);
            mtile_compute<N, OP, EDGE, decltype(bget), PRE, false>(C, G, su, sw, (wel0 + le + 1) * N, e0 + wel0 + le, minv_a,
                                                            minv_p, mnu, kq, bget, fin_u, fin_w, rq[q]);
          }
        }
        // interface value of element le's node 0 (v = left row N + own row 0, or row 0 alone
        // for the warp's first element until the halo arrives): M^-1 / Dirichlet mask, staged
        auto put_row0 = [&](int le, bool first, double left, double row0) {
          const int64_t eg = e0 + wel0 + le;
          double v = first ? row0 : __dadd_rn(left, row0);
          if (!first) {
            if (EDGE && eg == 0) {
              if (OP != OP_JACT) v = __dmul_rn(v, C.minv[N]);
              v = __dmul_rn(v, 0.0);
            } else if (OP != OP_JACT && !PRE) {
              v = __dmul_rn(v, minv_if);
            }
          }
          wout[le * N] = v;
        };
#pragma unroll
        for (int q = 0; q < WMT; ++q) {
          const int le = ws_le<WMT, ILVW>(q, rr);    // warp-local element of this lane
          const bool live = le < wnel;
          const int64_t eg = e0 + wel0 + le;
          const double (&r)[NT][2] = rq[q];
          // interior rows -> staging; rows 0 and N stay in registers
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int i = row_of(nt, h);             // permuted row (= A column)
              if (live && i != 0 && i != N)
                wout[le * N + i] = (OP == OP_JACT || PRE) ? r[nt][h] : __dmul_rn(r[nt][h], minv_row(nt, h));
            }
          if constexpr (!ILVW) {
            const double row0 = r[0][0];              // valid in lanes kq == 0
            const double rowN = r[RN_NT][RN_H];       // valid in lanes kq == 3 (WS_EO: kq == 0)
            double left = __shfl_up_sync(0xffffffffu, rowN, RN_KQ == 3 ? 1 : 4);
            if (rr == 0) left = carry;                // q == 0: patched after the halo arrives
            carry = __shfl_sync(0xffffffffu, rowN, 28 + RN_KQ);
            if (kq == 0 && live) put_row0(le, q == 0 && rr == 0, left, row0);
          }
          if (EDGE && kq == RN_KQ && live && eg == G.E - 1) {  // Dirichlet end node E*N
            double v = r[RN_NT][RN_H];
            if (OP != OP_JACT) v = __dmul_rn(v, C.minv[N + 1]);
            wout[(le + 1) * N] = __dmul_rn(v, 0.0);
          }
        }
        if constexpr (ILVW) {
          // left neighbour of (q, rr): (q-1, rr) in lane 4rr+3; of (0, rr > 0): m-tile WMT-1
          // of row ws_left_row(rr); (0, 0) is the warp's first element (halo)
#pragma unroll
          for (int q = 0; q < WMT; ++q) {
            const double left = q > 0 ? __shfl_down_sync(0xffffffffu, rq[q - 1][RN_NT][RN_H], RN_KQ)
                                      : __shfl_sync(0xffffffffu, rq[WMT - 1][RN_NT][RN_H], 4 * ws_left_row<WMT>(rr) + RN_KQ);
            const int le = ws_le<WMT, ILVW>(q, rr);
            if (kq == 0 && le < wnel) put_row0(le, q == 0 && rr == 0, left, rq[q][0][0]);
          }
        }
      };
      if (edge) body(std::integral_constant<bool, true>{}, std::integral_constant<bool, false>{});
      else if (pre) body(std::integral_constant<bool, false>{}, std::integral_constant<bool, OP == OP_RHS || EO>{});
      else body(std::integral_constant<bool, false>{}, std::integral_constant<bool, false>{});
      // first interface node of the warp: needs the halo row from the producer
      while (!mbar_try_wait(&halo[s], (it / STAGES) & 1)) {
      }
      if (lane == 0) {
        const int64_t eg = e0 + wel0;
        double v = __dadd_rn(hrow[s * W::CW + warp], wout[0]);
        if (!periodic && eg == 0) {
          if (OP != OP_JACT) v = __dmul_rn(v, C.minv[N]);
          v = __dmul_rn(v, 0.0);
        } else if (OP != OP_JACT && !pre) {
          v = __dmul_rn(v, minv_if);
        }
        wout[0] = v;
      }
    } else {
      while (!mbar_try_wait(&halo[s], (it / STAGES) & 1)) {
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done reading stage s
    if (wnel > 0) {
      const bool owns_end = !periodic && (e0 + wel0 + wnel == G.E);
      const int cnt_w = wnel * N + (owns_end ? 1 : 0);
      const int64_t gw = bofs + (e0 + wel0) * N;    // absolute index of the warp's first node
      const bool bulk = (EPI == EPI_STORE) && ((gw & 1) == 0) && ((cnt_w & 1) == 0);
      if (bulk) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          bulk_s2g(A.out + gw, wout, (uint32_t)(cnt_w * 8));
          bulk_commit();
        }
      } else {
        // four nodes per lane at a time: every global read of a chunk (base, terms) is in
        // flight before its arithmetic, instead of one dependent round trip per node (the
        // stores of a chunk may alias the next chunk's inputs, so chunks stay ordered)
        constexpr int U4 = 4;
        if constexpr (EPI == EPI_STORE) {            // unaligned warp range of a plain apply
          for (int k = lane; k < cnt_w; k += 32) A.out[gw + k] = wout[k];
        } else
        for (int kb = lane; kb < cnt_w; kb += 32 * U4) {
          double v[U4], x[U4];
          bool live[U4];
#pragma unroll
          for (int r = 0; r < U4; ++r) {
            live[r] = kb + 32 * r < cnt_w;
            v[r] = live[r] ? wout[kb + 32 * r] : 0.0;
          }
          if (EPI == EPI_STORE) {
#pragma unroll
            for (int r = 0; r < U4; ++r)
              if (live[r]) A.out[gw + kb + 32 * r] = v[r];
          } else if (EPI == EPI_ADJ) {
            double l[U4];
#pragma unroll
            for (int r = 0; r < U4; ++r) l[r] = __dmul_rn(A.dt, v[r]);  // l = dt * J^T(U) z (adjoint.py:58-60)
            if (A.Y) {
              // lam + l_0 + l_1 + ...                          (adjoint.py:61)
#pragma unroll
              for (int r = 0; r < U4; ++r) x[r] = live[r] ? __ldg(A.base + gw + kb + 32 * r) : 0.0;
              for (int j = 0; j < A.epi.n; ++j) {
                const double* pj = A.epi.ptr[j];
                double t[U4];
#pragma unroll
                for (int r = 0; r < U4; ++r) t[r] = (pj && live[r]) ? __ldg(pj + gw + kb + 32 * r) : l[r];
#pragma unroll
                for (int r = 0; r < U4; ++r) x[r] = __dadd_rn(x[r], t[r]);
              }
            }
#pragma unroll
            for (int r = 0; r < U4; ++r) {
              if (!live[r]) continue;
              if (A.out) A.out[gw + kb + 32 * r] = l[r];
              if (A.Y) A.Y[gw + kb + 32 * r] = x[r];
            }
          } else {  // EPI_RK: base + dt * combination (timeloop.py:114-127)
            double bv[U4];
#pragma unroll
            for (int r = 0; r < U4; ++r) bv[r] = live[r] ? __ldg(A.base + gw + kb + 32 * r) : 0.0;
            if (A.epi.n == 1) {
              const double* p0 = A.epi.ptr[0];
#pragma unroll
              for (int r = 0; r < U4; ++r) x[r] = (p0 && live[r]) ? __ldg(p0 + gw + kb + 32 * r) : v[r];
              const double c = __dmul_rn(A.dt, A.epi.coef[0]);
#pragma unroll
              for (int r = 0; r < U4; ++r) x[r] = __dadd_rn(bv[r], __dmul_rn(c, x[r]));
            } else {
#pragma unroll
              for (int r = 0; r < U4; ++r) x[r] = 0.0;
              for (int j = 0; j < A.epi.n; ++j) {
                const double* pj = A.epi.ptr[j];
                double t[U4];
#pragma unroll
                for (int r = 0; r < U4; ++r) t[r] = (pj && live[r]) ? __ldg(pj + gw + kb + 32 * r) : v[r];
#pragma unroll
                for (int r = 0; r < U4; ++r) {
                  const double term = __dmul_rn(A.epi.coef[j], t[r]);
                  x[r] = (j == 0) ? term : __dadd_rn(x[r], term);
                }
              }
#pragma unroll
              for (int r = 0; r < U4; ++r) x[r] = __dadd_rn(bv[r], __dmul_rn(A.dt, x[r]));
            }
#pragma unroll
            for (int r = 0; r < U4; ++r) {
              if (!live[r]) continue;
              if (A.out) A.out[gw + kb + 32 * r] = v[r];
              if (A.check) bad_y |= nonfinite(x[r]);
              A.Y[gw + kb + 32 * r] = x[r];
            }
          }
        }
        __syncwarp();
        // an empty group keeps one commit per tile, so wait_group.read<OUTB-1> above
        // always refers to the store out of the buffer about to be reused
        if (OUTB > 1 && lane == 0) bulk_commit();
      }
    }
    tl += gridDim.x;
    while (tl >= tiles_per_ring) {
      tl -= tiles_per_ring;
      ++bidx;
    }
  }
  if (lane == 0) bulk_wait_all();
  const bool bad_u = WS_FIN_BAD(fin_u), bad_w = WS_FIN_BAD(fin_w);
  if (bad_u || bad_w || bad_y)
    atomicOr(A.flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) |
                         (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0) |
                         (bad_y ? SEM1D_FLAG_STEP_NONFINITE : 0));
}

// Pipeline depth: enough stages that ~100 KB of slab loads can be in flight per
// CTA (two CTAs per SM for n <= 16), since HBM at ~1.5 us loaded latency needs
// >= 64 KB outstanding per SM (Little's law).
// doubles of the kernel's shared-memory B-fragment table (EO: the reflection-split blocks)
template <int N, int OP, int NZ, bool EO>
constexpr int ws_bsm_doubles() {
  using W = WsTile<N, OP, NZ, EO>;
  if (!W::B_IN_SMEM) return 0;
  return EO ? ((OP == OP_JACT) ? 6 : 4) * (W::NT / 2) * (W::KC / 2) * 32 : ((OP == OP_JACT) ? 3 : 2) * W::NT * W::KC * 32;
}

template <int N, int OP, int NZ = -1, bool EO = false>
constexpr int ws_stages() {
  using W = WsTile<N, OP, NZ, EO>;
  constexpr int NIN = W::NIN;
  // shared-memory budget that keeps ws_minb CTAs resident (227 KB per SM)
  constexpr int mb = ws_minb<N, OP, NZ, EO>();
  constexpr int budget = (mb == 1 ? 180 : (mb == 2 ? 104 : (mb == 3 ? 72 : (mb == 4 ? 54 : 44)))) * 1024;
  constexpr int per = NIN * W::SLAB_ALLOC * 8;
  constexpr int st = (budget - ws_outb<OP>() * W::OUT * 8 - ws_bsm_doubles<N, OP, NZ, EO>() * 8) / per;
  return st < 2 ? 2 : (st > 8 ? 8 : st);
}

template <int N, int OP, int STAGES, int NZ = -1, bool EO = false>
constexpr size_t ws_smem_bytes() {
  using W = WsTile<N, OP, NZ, EO>;
  constexpr int NIN = W::NIN;
  return sizeof(double) * ((size_t)STAGES * NIN * W::SLAB_ALLOC + ws_outb<OP>() * W::OUT + STAGES * W::CW +
                           ws_bsm_doubles<N, OP, NZ, EO>() + (EO ? 3 * (N + 1) : 0)) +
         sizeof(uint64_t) * 3 * STAGES;
}

template <int N, int OP, int STAGES>
constexpr size_t mma_smem_bytes() {
  using MT_ = MmaTile<N>;
  constexpr int NIN = (OP == OP_RHS) ? 1 : 2;
  constexpr int NMAT = (OP == OP_JACT) ? 3 : 2;
  return sizeof(double) * ((size_t)(STAGES * NIN + 1) * MT_::SLAB_ALLOC + MT_::ELEMS + 2 +
                           (MT_::B_IN_SMEM ? NMAT * MT_::NT * MT_::KC * 32 : 0)) +
         sizeof(uint64_t) * STAGES;
}

template <int N, int OP, int STAGES>
constexpr size_t tma_smem_bytes() {
  constexpr int NIN = (OP == OP_RHS) ? 1 : 2;
  return sizeof(double) * ((size_t)(STAGES * NIN + 1) * TmaTile<N>::SLAB_ALLOC + TmaTile<N>::TPB + 2) +
         sizeof(uint64_t) * STAGES;
}

template <int N, int OP>
constexpr size_t apply_smem_bytes() {
  return sizeof(double) *
         ((OP == OP_RHS ? 2 : 3) * (size_t)Tile<N>::SLAB_ALLOC + Tile<N>::TPB + 1);
}

}  // namespace sem1d
