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

template <int N, int OP>
constexpr size_t apply_smem_bytes() {
  return sizeof(double) *
         ((OP == OP_RHS ? 2 : 3) * (size_t)Tile<N>::SLAB_ALLOC + Tile<N>::TPB + 1);
}

}  // namespace sem1d
