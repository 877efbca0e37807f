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

#include <cuda_runtime.h>
#include <stdint.h>

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

__device__ __forceinline__ bool nonfinite(double v) { return !isfinite(v); }

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
