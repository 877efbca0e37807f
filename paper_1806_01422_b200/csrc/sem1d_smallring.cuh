// sem1d_smallring.cuh -- whole sweeps of SMALL rings in one launch (BASELINE
// config 1: E = 16, N = 9, where per-stage launches and host syncs would cost
// more than the arithmetic).  One CTA per ring, one thread per (element, row):
// thread (e, i) contracts row i of element e with K / Dw held in shared memory
// (DFMA; n = N+1 need not be a multiple of 8), rows are assembled into nodes
// after one barrier (node e*N = row N of e-1 + row 0 of e, the same two-term sum
// as grid.py:157-161), and each thread then owns at most one node, so the RK
// and stage-adjoint arithmetic of timeloop.py:111-130 / adjoint.py:54-61 runs
// in registers.  Periodic and homogeneous-Dirichlet rings; E*(N+1) <= 1024.
#pragma once

#include "sem1d_ensemble.cuh"

namespace sem1d {

struct SmallGeo {
  int E, N, ndof, periodic;
};

// row i of element e for OP = RHS (x = state) or JACT (x = state, z = zm)
template <int N, int OP>
__device__ __forceinline__ double small_row(const double* sK, const double* sDw, const double* x,
                                            const double* z, int e, int i, double mnu) {
  constexpr int n = N + 1;
  const double* xe = x + e * N;
  if (OP == OP_RHS) {
    double ku = 0.0, du = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      ku = fma(sK[i * n + j], xe[j], ku);
      du = fma(sDw[i * n + j], xe[j], du);
    }
    return __dsub_rn(__dmul_rn(ku, mnu), __dmul_rn(xe[i], du));
  } else {
    const double* ze = z + e * N;
    double kz = 0.0, du = 0.0, dt = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      kz = fma(sK[i * n + j], ze[j], kz);
      du = fma(sDw[i * n + j], xe[j], du);
      dt = fma(sDw[j * n + i], __dmul_rn(xe[j], ze[j]), dt);
    }
    return __dsub_rn(__dsub_rn(__dmul_rn(kz, mnu), __dmul_rn(ze[i], du)), dt);
  }
}

// Assemble the owned node of thread (e, i) from the rows (needs a barrier before).
// Owned: node e*N + i for i < N, plus node E*N (Dirichlet) by thread (E-1, N).
__device__ __forceinline__ bool small_owned(const SmallGeo& G, int e, int i, int& g) {
  const int N = G.N;
  if (e >= G.E) return false;
  if (i < N) { g = e * N + i; return true; }
  if (!G.periodic && e == G.E - 1) { g = G.E * N; return true; }
  return false;
}

template <int N>
__device__ __forceinline__ double small_assemble(const SmallGeo& G, const double* srow, int e, int i) {
  constexpr int n = N + 1;
  if (i == 0) {
    if (e == 0) {
      if (!G.periodic) return srow[0];
      return __dadd_rn(srow[(G.E - 1) * n + N], srow[0]);
    }
    return __dadd_rn(srow[(e - 1) * n + N], srow[e * n]);
  }
  return srow[e * n + i];   // interior row, or row N of the last Dirichlet element
}

// per-node M^-1 / mask (sem1d.h pattern positions)
template <int N>
__device__ __forceinline__ void small_pattern(const Consts<N>& C, const SmallGeo& G, int g,
                                              double& minv, bool& masked) {
  masked = false;
  if (!G.periodic && (g == 0 || g == G.E * N)) {
    masked = true;
    minv = (g == 0) ? C.minv[N] : C.minv[N + 1];
  } else {
    minv = C.minv[g % N];
  }
}

// SCH: compile-time tableau (TabC: 0 Euler, 1 Kutta-3, 2 RK4) -- the stage loops unroll and
// the coefficients become immediates; same values and association as the runtime tableau
template <int N, int SCH>
__global__ void __launch_bounds__(1024, 1)
    small_forward_kernel(const __grid_constant__ Consts<N> C, const SmallGeo G, const EnsArgs A) {
  constexpr int n = N + 1;
  using TB = TabC<SCH>;
  extern __shared__ __align__(16) double smem[];
  const int ndof = G.ndof;
  double* sK = smem;
  double* sDw = sK + n * n;
  double* su = sDw + n * n;                 // ndof + 1 (periodic mirror)
  double* sU = su + ndof + 2;
  double* srow = sU + ndof + 2;             // E * n rows
  const int tid = threadIdx.x;
  const int e = tid / n, i = tid - (tid / n) * n;
  const int64_t b = blockIdx.x, nb = gridDim.x;
  const double mnu = -C.nu;
  for (int k = tid; k < n * n; k += blockDim.x) { sK[k] = C.K[k]; sDw[k] = C.Dw[k]; }
  const double* u0 = A.u0 + b * ndof;
  for (int k = tid; k < ndof; k += blockDim.x) su[k] = u0[k];
  __syncthreads();
  if (tid == 0 && G.periodic) su[ndof] = su[0];
  int g = 0;
  const bool owns = small_owned(G, e, i, g);
  double minv = 1.0;
  bool masked = false;
  if (owns) small_pattern<N>(C, G, g, minv, masked);
  if (A.traj && owns) A.traj[b * ndof + g] = su[g];
  double fin = 0.0, kkeep = 0.0, acc = 0.0;
  bool bad = false;
  __syncthreads();
  for (int step = 0; step < A.nsteps; ++step) {
    const double dt = A.dts[step];
#pragma unroll
    for (int st = 0; st < TB::s; ++st) {
      const double* src = (st == 0) ? su : sU;
      if (e < G.E) {
        if (owns) fin = fma(src[g], 0.0, fin);
        srow[tid] = small_row<N, OP_RHS>(sK, sDw, src, nullptr, e, i, mnu);
      }
      __syncthreads();
      if (owns) {
        double kk = __dmul_rn(small_assemble<N>(G, srow, e, i), minv);
        if (masked) kk = __dmul_rn(kk, 0.0);
        const double term = __dmul_rn(TB::b(st), kk);
        acc = (st == 0) ? term : __dadd_rn(acc, term);
        if (st + 1 < TB::s) {
          double y;
          if (TB::nterm(st + 1) == 1) {
            y = __dadd_rn(su[g], __dmul_rn(__dmul_rn(dt, TB::a(st + 1, st)), kk));
          } else {
            double sacc = __dmul_rn(TB::a(st + 1, 0), (st == 0) ? kk : kkeep);
#pragma unroll
            for (int jj = 1; jj <= st; ++jj)
              sacc = __dadd_rn(sacc, __dmul_rn(TB::a(st + 1, jj), (jj == st) ? kk : kkeep));
            y = __dadd_rn(su[g], __dmul_rn(dt, sacc));
          }
          sU[g] = y;
          if (g == 0 && G.periodic) sU[ndof] = y;
          if (st == 0) kkeep = kk;
        } else {
          const double un = __dadd_rn(su[g], __dmul_rn(dt, acc));
          bad |= !isfinite(un);
          su[g] = un;
          if (g == 0 && G.periodic) su[ndof] = un;
        }
      }
      __syncthreads();
    }
    if (A.traj && owns) A.traj[((int64_t)(step + 1) * nb + b) * ndof + g] = su[g];
  }
  if (owns) A.u_final[b * ndof + g] = su[g];
  if (fin != fin || bad)
    atomicOr(&A.flags[b], (fin != fin ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad ? SEM1D_FLAG_STEP_NONFINITE : 0));
}

template <int N, int SCH>
__global__ void __launch_bounds__(1024, 1)
    small_adjoint_kernel(const __grid_constant__ Consts<N> C, const SmallGeo G, const EnsAdjArgs A) {
  constexpr int n = N + 1;
  using TB = TabC<SCH>;
  extern __shared__ __align__(16) double smem[];
  const int ndof = G.ndof, pad = ndof + 2;
  double* sK = smem;
  double* sDw = sK + n * n;
  double* sUs = sDw + n * n;                // U_0 .. U_{s-1}: 4 arrays
  double* sz = sUs + 4 * pad;               // zm
  double* srow = sz + pad;                  // E * n rows
  const int tid = threadIdx.x;
  const int e = tid / n, i = tid - (tid / n) * n;
  const int64_t b = blockIdx.x, nb = gridDim.x;
  const double mnu = -C.nu;
  constexpr int S = TB::s;
  for (int k = tid; k < n * n; k += blockDim.x) { sK[k] = C.K[k]; sDw[k] = C.Dw[k]; }
  int g = 0;
  const bool owns = small_owned(G, e, i, g);
  double minv = 1.0;
  bool masked = false;
  if (owns) small_pattern<N>(C, G, g, minv, masked);
  double lam = owns ? A.lam_in[b * ndof + g] : 0.0;
  double fin = 0.0;
  // this thread's trajectory value of the next step, loaded one step ahead
  auto traj_at = [&](int step) { return A.traj[((int64_t)step * nb + b) * ndof + g]; };
  double unext = (owns && A.nsteps > 0) ? traj_at(A.nsteps - 1) : 0.0;
  __syncthreads();
  for (int step = A.nsteps - 1; step >= 0; --step) {
    const double dt = A.dts[step];
    if (owns) {
      sUs[g] = unext;
      if (g == 0 && G.periodic) sUs[ndof] = unext;
      if (step > 0) unext = traj_at(step - 1);
    }
    __syncthreads();
    // stage states U_1..U_{S-1} (timeloop.rk3_stages)
    double kkeep = 0.0;
#pragma unroll
    for (int st = 0; st + 1 < S; ++st) {
      const double* src = sUs + st * pad;
      if (e < G.E) srow[tid] = small_row<N, OP_RHS>(sK, sDw, src, nullptr, e, i, mnu);
      __syncthreads();
      if (owns) {
        double kk = __dmul_rn(small_assemble<N>(G, srow, e, i), minv);
        if (masked) kk = __dmul_rn(kk, 0.0);
        double y;
        if (TB::nterm(st + 1) == 1) {
          y = __dadd_rn(sUs[g], __dmul_rn(__dmul_rn(dt, TB::a(st + 1, st)), kk));
        } else {
          double sacc = __dmul_rn(TB::a(st + 1, 0), (st == 0) ? kk : kkeep);
#pragma unroll
          for (int jj = 1; jj <= st; ++jj)
            sacc = __dadd_rn(sacc, __dmul_rn(TB::a(st + 1, jj), (jj == st) ? kk : kkeep));
          y = __dadd_rn(sUs[g], __dmul_rn(dt, sacc));
        }
        double* dst = sUs + (st + 1) * pad;
        dst[g] = y;
        if (g == 0 && G.periodic) dst[ndof] = y;
        if (st == 0) kkeep = kk;
      }
      __syncthreads();
    }
    // stage-adjoint chain i = S-1..0 (adjoint.py:58-61), lam' = ((lam + l_0) + l_1) + ...
    double l[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int st = S - 1; st >= 0; --st) {
      if (owns) {
        double z = __dmul_rn(TB::b(st), lam);
#pragma unroll
        for (int jj = st + 1; jj < S; ++jj)
          if (TB::a(jj, st) != 0.0) z = __dadd_rn(z, __dmul_rn(TB::a(jj, st), l[jj]));
        fin = fma(z, 0.0, fin);
        double zm = __dmul_rn(z, minv);
        if (masked) zm = __dmul_rn(zm, 0.0);
        sz[g] = zm;
        if (g == 0 && G.periodic) sz[ndof] = zm;
      }
      __syncthreads();
      if (e < G.E) srow[tid] = small_row<N, OP_JACT>(sK, sDw, sUs + st * pad, sz, e, i, mnu);
      __syncthreads();
      if (owns) {
        double jt = small_assemble<N>(G, srow, e, i);
        if (masked) jt = __dmul_rn(jt, 0.0);
        l[st] = __dmul_rn(dt, jt);
      }
      __syncthreads();
    }
    if (owns) {
      double acc = lam;
#pragma unroll
      for (int st = 0; st < S; ++st) acc = __dadd_rn(acc, l[st]);
      lam = acc;
    }
  }
  if (owns) A.lam_out[b * ndof + g] = lam;
  if (fin != fin) atomicOr(&A.flags[b], SEM1D_FLAG_INPUT2_NONFINITE);
}

inline size_t small_fwd_smem(int N, int ndof, int E) {
  const int n = N + 1;
  return sizeof(double) * (2 * n * n + 2 * (ndof + 2) + E * n);
}
inline size_t small_adj_smem(int N, int ndof, int E) {
  const int n = N + 1;
  return sizeof(double) * (2 * n * n + 5 * (ndof + 2) + E * n);
}

}  // namespace sem1d
