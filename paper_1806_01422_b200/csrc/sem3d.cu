// sem3d.cu -- 3D periodic boxes: sum-factorised Burgers F(u), J(u)v, J(u)^T z
// (reference ops.py:63-81,109-115,127-257 and grid.py:112-146).
//
// Field layout (the reference's): 3 components, each a scalar lattice of
// P1*P2*P3 nodes, P_a = E_a*N, node (g1,g2,g3) at (g1*P2 + g2)*P3 + g3.
// Element (e1,e2,e3) is e = (e1*E2 + e2)*E3 + e3; its local node (i,j,k) is global
// ((e1 N + i) mod P1, ...).
//
// Two kernels per apply:
//  * elem3d_kernel<N, OP>: one CTA per element, one thread per (a,b) pencil of the
//    n x n x n block.  The element's u (and v or M^-1 z) are staged in shared memory;
//    each of the three phases contracts one axis (K_a, Dw, Dw^T: n^2 FMAs per pencil
//    output row), multiplies by the transverse mass weights and accumulates; phase 3
//    forms the element result in the reference's evaluation order
//        F:   ((K0 u_i + K1 u_i) + K2 u_i) * (-nu) - u_0 D0 u_i - u_1 D1 u_i - u_2 D2 u_i
//        J:   (sum K w_i)(-nu) - sum_j (w_j D_j u_i + u_j D_j w_i)
//        J^T: (sum K z_i)(-nu) - sum_j (z_j D_i u_j + D_j^T (u_j z_i))
//    and writes the (3, nelem, n, n, n) element blocks to a scratch buffer.
//  * gather3d_kernel<N>: one thread per global node and component sums its (up to 8)
//    element contributions (Q^T) and applies M^-1 (F, J) -- the reference's gather +
//    _finish.  Deterministic: a fixed summation order, no atomics.
// FP64 on the CUDA cores (the DMMA m8n8k4 shape fits only n = 8 and 16; a tensor-core
// variant is the next step).  Degrees 1..12 (the element block of J^T must fit smem).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "sem1d.h"
#include "sem1d_devguard.cuh"

namespace sem1d {
int set_error(int code, const std::string& msg);   // sem1d_capi.cu
int sem1d_path_override();                          // sem1d_capi.cu: 0 auto, 1 no tensor cores
}

struct sem3d_plan {
  int N, n;
  int64_t E[3], P[3], nscalar, nelem;
  double nu;
  double* cbuf;   // device: K[3][n*n], Dw[n*n], T[3][n*n], minv[(N+1)^3], mass[(N+1)^3]
  int device;     // the device current at sem3d_plan_create; every call runs there
};

namespace sem1d {
int plan3_device(const sem3d_plan* p) { return p ? p->device : -1; }
}  // namespace sem1d

namespace {

constexpr int S3_MAX_N = 12;
// output rows contracted together per pencil: independent FMA chains
#ifndef S3_UNROLL
#define S3_UNROLL 4
#endif
constexpr int kUnrollF = S3_UNROLL;
enum { OP3_RHS = 0, OP3_JAC = 1, OP3_JACT = 2 };

int fail(int code, const std::string& m) { return sem1d::set_error(code, m); }
int cuda_fail(cudaError_t e, const char* where) {
  return fail(SEM1D_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

struct Geo3 {
  int64_t E1, E2, E3, P1, P2, P3, nscalar, nelem;
  double mnu;
};

__device__ __forceinline__ bool nonfin3(double x) {
  return ((unsigned)__double2hiint(x) & 0x7ff00000u) == 0x7ff00000u;
}

// Padded shared-memory block strides per n (node (i,j,k) at i*SI + j*SJ + k): chosen by an
// exhaustive search so that the pencil loads of all three phases (lanes = (a,b) pencils)
// hit at most 3 lanes per double bank (unpadded n = 8 put 16 lanes on one bank).
constexpr int pad_j(int n) {
  return (n == 3 || n == 4 || n == 8 || n == 10) ? 1 : 0;
}
constexpr int pad_i(int n) {
  return n == 3 ? 1 : (n == 6 ? 1 : (n == 7 ? 3 : (n == 9 ? 2 : (n == 12 || n == 13 ? 1 : 0))));
}

template <int N>
struct L3 {
  static constexpr int n = N + 1, n2 = n * n, n3 = n * n * n;
  static constexpr int SJ = n + pad_j(n), SI = n * SJ + pad_i(n), BLK = n * SI;   // padded block
  static constexpr int THREADS = ((n2 + 31) / 32) * 32;
  // shared arrays (doubles): consts 7 n^2, fields, scratch
  static constexpr int CONSTS = 7 * n2;
  static constexpr int arrays(int op) { return op == OP3_RHS ? 4 : 7; }
  static constexpr size_t smem(int op) { return sizeof(double) * ((size_t)CONSTS + (size_t)arrays(op) * BLK); }
};

// element e -> global scalar index of local node (i, j, k)
__device__ __forceinline__ int64_t node_index(const Geo3& G, int64_t e1, int64_t e2, int64_t e3, int N, int i,
                                              int j, int k) {
  int64_t g1 = e1 * N + i, g2 = e2 * N + j, g3 = e3 * N + k;
  if (g1 >= G.P1) g1 -= G.P1;
  if (g2 >= G.P2) g2 -= G.P2;
  if (g3 >= G.P3) g3 -= G.P3;
  return (g1 * G.P2 + g2) * G.P3 + g3;
}

// One axis contraction of a pencil: y[i] = sum_l A[i][l] x[l] (A row-major n x n in smem)
// The axis contractions are dense matrix products (the reference runs them through BLAS
// dgemm, ops.py:63-81), so they use FMA; only the pointwise terms keep the reference's
// separately rounded multiply / add.
template <int n>
__device__ __forceinline__ double contract_row(const double* A, const double (&x)[n], int i) {
  double acc = A[i * n] * x[0];
#pragma unroll
  for (int l = 1; l < n; ++l) acc = fma(A[i * n + l], x[l], acc);
  return acc;
}
template <int n>
__device__ __forceinline__ double contract_row_t(const double* A, const double (&x)[n], int i) {
  double acc = A[i] * x[0];
#pragma unroll
  for (int l = 1; l < n; ++l) acc = fma(A[l * n + i], x[l], acc);
  return acc;
}

// padded block offset of node (i, j, k), and of position p along axis `ax` of pencil (a,b)
template <int N>
__device__ __forceinline__ int bidx(int i, int j, int k) {
  return i * L3<N>::SI + j * L3<N>::SJ + k;
}
template <int N>
__device__ __forceinline__ int off(int ax, int a, int b, int p) {
  return ax == 0 ? bidx<N>(p, a, b) : (ax == 1 ? bidx<N>(a, p, b) : bidx<N>(a, b, p));
}

template <int N, int OP>
__global__ void __launch_bounds__(L3<N>::THREADS) elem3d_kernel(const Geo3 G, const double* __restrict__ cbuf,
                                                               const double* __restrict__ u,
                                                               const double* __restrict__ w, double* loc,
                                                               int* flag) {
  using L = L3<N>;
  constexpr int n = L::n, n2 = L::n2, n3 = L::n3;
  extern __shared__ __align__(16) double sm[];
  double* sK = sm;                  // [3][n2]
  double* sD = sK + 3 * n2;         // Dw [n2]
  double* sT = sD + n2;             // transverse weights [3][n2]
  constexpr int B = L::BLK;         // padded block size
  double* sU = sT + 3 * n2;         // [3][B] state
  double* sW = sU + 3 * B;          // [3][B] v (J) / M^-1 z (J^T); unused for F
  double* ACC = (OP == OP3_RHS) ? sW : sW + 3 * B;    // [B] per-node accumulator
  const int tid = threadIdx.x;
  for (int k = tid; k < 7 * n2; k += blockDim.x) sK[k] = cbuf[k];
  const int64_t e = blockIdx.x;
  const int64_t e3 = e % G.E3, e12 = e / G.E3, e2 = e12 % G.E2, e1 = e12 / G.E2;
  const double* minv_pat = cbuf + 7 * n2;     // [(N+1)^3] by position class
  unsigned bad_u = 0, bad_w = 0;
  for (int q = tid; q < n3; q += blockDim.x) {
    const int i = q / n2, j = (q / n) % n, k = q % n;
    const int64_t g = node_index(G, e1, e2, e3, N, i, j, k);
    const int qb = bidx<N>(i, j, k);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = u[c * G.nscalar + g];
      bad_u |= nonfin3(x);
      sU[c * B + qb] = x;
      if (OP != OP3_RHS) {
        double y = w[c * G.nscalar + g];
        bad_w |= nonfin3(y);
        if (OP == OP3_JACT) {
          // position class per axis: 0 = wrap interface, 1..N-1 interior, N = interface
          const int64_t gg[3] = {(e1 * N + i) % G.P1, (e2 * N + j) % G.P2, (e3 * N + k) % G.P3};
          int cl[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int r = (int)(gg[a] % N);
            cl[a] = (r != 0) ? r : (gg[a] == 0 ? 0 : N);
          }
          y = __dmul_rn(y, minv_pat[(cl[0] * (N + 1) + cl[1]) * (N + 1) + cl[2]]);
        }
        sW[c * B + qb] = y;
      }
    }
  }
  if (bad_u || bad_w)
    atomicOr(flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0));
  __syncthreads();
  const bool act = tid < n2;
  const int a = tid / n, b = tid % n;
  for (int ci = 0; ci < 3; ++ci) {
    const double* Ui = sU + ci * B;
    const double* Wi = sW + ci * B;
    for (int ax = 0; ax < 3; ++ax) {
      if (act) {
        // each phase adds its axis' whole contribution at the nodes of the pencil (a, b):
        //   F:   -nu K_ax u_i - u_ax D_ax u_i          J: -nu K_ax w_i - w_ax D_ax u_i - u_ax D_ax w_i
        //   J^T: -nu K_ax z_i - D_ax^T (u_ax z_i) [- sum_j z_j D_ax u_j on the axis ax == ci]
        const double t = sT[ax * n2 + a * n + b];
        const double* Ka = sK + ax * n2;
        double xu[n], xw[n], xt[n], x0[n], x1[n], x2[n];
#pragma unroll
        for (int l = 0; l < n; ++l) {
          const int o = off<N>(ax, a, b, l);
          xu[l] = Ui[o];
          if (OP != OP3_RHS) xw[l] = Wi[o];
          if (OP == OP3_JACT) xt[l] = __dmul_rn(sU[ax * B + o], xw[l]);
        }
        const bool own = (OP == OP3_JACT) && (ax == ci);
        if (own) {
#pragma unroll
          for (int l = 0; l < n; ++l) {
            const int o = off<N>(ax, a, b, l);
            x0[l] = sU[o];
            x1[l] = sU[B + o];
            x2[l] = sU[2 * B + o];
          }
        }
#pragma unroll(kUnrollF)
        for (int p = 0; p < n; ++p) {
          const int o = off<N>(ax, a, b, p);
          double c;
          if (OP == OP3_RHS) {
            c = __dsub_rn(__dmul_rn(__dmul_rn(contract_row<n>(Ka, xu, p), t), G.mnu),
                          __dmul_rn(sU[ax * B + o], __dmul_rn(contract_row<n>(sD, xu, p), t)));
          } else if (OP == OP3_JAC) {
            c = __dmul_rn(__dmul_rn(contract_row<n>(Ka, xw, p), t), G.mnu);
            c = __dsub_rn(c, __dmul_rn(sW[ax * B + o], __dmul_rn(contract_row<n>(sD, xu, p), t)));
            c = __dsub_rn(c, __dmul_rn(sU[ax * B + o], __dmul_rn(contract_row<n>(sD, xw, p), t)));
          } else {
            c = __dsub_rn(__dmul_rn(__dmul_rn(contract_row<n>(Ka, xw, p), t), G.mnu),
                          __dmul_rn(contract_row_t<n>(sD, xt, p), t));
            if (own) {
              c = __dsub_rn(c, __dmul_rn(sW[o], __dmul_rn(contract_row<n>(sD, x0, p), t)));
              c = __dsub_rn(c, __dmul_rn(sW[B + o], __dmul_rn(contract_row<n>(sD, x1, p), t)));
              c = __dsub_rn(c, __dmul_rn(sW[2 * B + o], __dmul_rn(contract_row<n>(sD, x2, p), t)));
            }
          }
          ACC[o] = (ax == 0) ? c : __dadd_rn(ACC[o], c);
        }
      }
      __syncthreads();
    }
    // element block of component ci -> scratch (coalesced: contiguous n^3 run)
    double* dst = loc + ((int64_t)ci * G.nelem + e) * n3;
    for (int q = tid; q < n3; q += blockDim.x) dst[q] = ACC[bidx<N>(q / n2, (q / n) % n, q % n)];
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------
// n = 8 (N = 7): the axis contractions on the FP64 tensor cores.  One element per CTA,
// four warps, each warp two tiles of 8 pencils.  A contraction along the phase axis is
// D[pencil][i] = sum_l X[pencil][l] M[i][l]: DMMA m8n8k4 with the element data as the A
// operand (lane: pencil lane>>2, l = 4kc + lane&3, loaded from the padded block) and the
// constant matrix as the B operand (lane: M[i = lane>>2][l = 4kc + lane&3], held in
// registers for the whole kernel); the lane receives outputs i = 2(lane&3) + {0,1} of
// pencil lane>>2.  Phases, scratch arrays and the final evaluation order are those of
// elem3d_kernel.
// ----------------------------------------------------------------------------

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int OP>
__global__ void __launch_bounds__(128) elem3d_mma_kernel(const Geo3 G, const double* __restrict__ cbuf,
                                                        const double* __restrict__ u,
                                                        const double* __restrict__ w, double* loc, int* flag) {
  constexpr int N = 7;
  using L = L3<N>;
  constexpr int n = 8, n2 = 64, n3 = 512;
  constexpr int B = L::BLK;
  extern __shared__ __align__(16) double sm[];
  double* sU = sm;                                   // [3][B]
  double* sW = sU + 3 * B;                           // [3][B] (J, J^T)
  double* ACC = (OP == OP3_RHS) ? sW : sW + 3 * B;   // [B] per-node accumulator
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, kq = lane & 3;
  // B fragments: K_ax (3), Dw, Dw^T -- M[i = r][l = 4kc + kq]; transverse weights of the
  // lane's two pencils per axis
  double bK[3][2], bD[2], bDt[2], tw[3][2];
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    const int l = 4 * kc + kq;
#pragma unroll
    for (int a = 0; a < 3; ++a) bK[a][kc] = cbuf[a * n2 + r * n + l];
    bD[kc] = cbuf[3 * n2 + r * n + l];
    bDt[kc] = cbuf[3 * n2 + l * n + r];
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int tt = 0; tt < 2; ++tt) tw[a][tt] = cbuf[4 * n2 + a * n2 + (2 * warp + tt) * n + r];
  const int64_t e = blockIdx.x;
  const int64_t e3 = e % G.E3, e12 = e / G.E3, e2 = e12 % G.E2, e1 = e12 / G.E2;
  const double* minv_pat = cbuf + 7 * n2;
  unsigned bad_u = 0, bad_w = 0;
  for (int q = tid; q < n3; q += blockDim.x) {
    const int i = q >> 6, j = (q >> 3) & 7, k = q & 7;
    const int64_t g = node_index(G, e1, e2, e3, N, i, j, k);
    const int qb = bidx<N>(i, j, k);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = u[c * G.nscalar + g];
      bad_u |= nonfin3(x);
      sU[c * B + qb] = x;
      if (OP != OP3_RHS) {
        double y = w[c * G.nscalar + g];
        bad_w |= nonfin3(y);
        if (OP == OP3_JACT) {
          const int64_t gg[3] = {(e1 * N + i) % G.P1, (e2 * N + j) % G.P2, (e3 * N + k) % G.P3};
          int cl[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int rr = (int)(gg[a] % N);
            cl[a] = (rr != 0) ? rr : (gg[a] == 0 ? 0 : N);
          }
          y = __dmul_rn(y, minv_pat[(cl[0] * (N + 1) + cl[1]) * (N + 1) + cl[2]]);
        }
        sW[c * B + qb] = y;
      }
    }
  }
  if (bad_u || bad_w)
    atomicOr(flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0));
  __syncthreads();
  // Phases unrolled (compile-time axis: every shared-memory offset is a per-thread base plus
  // an immediate).  The pencil's transverse weight t scales the A fragment and -nu rides on
  // the K fragment, so an output is one DFMA (F) instead of four multiplies and a subtract:
  //   F:   K'(t u_i) - u_ax D(t u_i)                 (K' = -nu K)
  //   J:   K'(t w_i) - w_ax D(t u_i) - u_ax D(t w_i)
  //   J^T: K'(t z_i) - D^T(t u_ax z_i) [- sum_j z_j D(t u_j) on the axis ax == ci]
  // (the same terms and order as elem3d_kernel, rounded differently: 1e-13 apart)
  double bKn[3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) bKn[a][kc] = __dmul_rn(G.mnu, bK[a][kc]);
#pragma unroll
  for (int ci = 0; ci < 3; ++ci) {
    const double* Ui = sU + ci * B;
    const double* Wi = sW + ci * B;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const int pt = 2 * warp + tt;                 // pencil tile: pencils (a = pt, b = 0..7)
        // offset of position p along the axis of the lane's pencil (pt, r)
        const int ob = ax == 0 ? pt * L::SJ + r : (ax == 1 ? pt * L::SI + r : pt * L::SI + r * L::SJ);
        const int st = ax == 0 ? L::SI : (ax == 1 ? L::SJ : 1);
        const double t = tw[ax][tt];
        double xu[2], xw[2];
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          const int o = ob + (4 * kc + kq) * st;
          xu[kc] = __dmul_rn(t, Ui[o]);
          if (OP != OP3_RHS) xw[kc] = __dmul_rn(t, Wi[o]);
        }
        double c[2];
        if (OP == OP3_RHS) {
          double k0 = 0.0, k1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int kc = 0; kc < 2; ++kc) {
            dmma8(k0, k1, xu[kc], bKn[ax][kc]);
            dmma8(d0, d1, xu[kc], bD[kc]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int o = ob + (2 * kq + h) * st;
            c[h] = __fma_rn(-sU[ax * B + o], h ? d1 : d0, h ? k1 : k0);
          }
        } else if (OP == OP3_JAC) {
          double k0 = 0.0, k1 = 0.0, p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
          for (int kc = 0; kc < 2; ++kc) {
            dmma8(k0, k1, xw[kc], bKn[ax][kc]);
            dmma8(p0, p1, xu[kc], bD[kc]);
            dmma8(q0, q1, xw[kc], bD[kc]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int o = ob + (2 * kq + h) * st;
            const double v = __fma_rn(-sW[ax * B + o], h ? p1 : p0, h ? k1 : k0);
            c[h] = __fma_rn(-sU[ax * B + o], h ? q1 : q0, v);
          }
        } else {
          const double* Ua = sU + ax * B;
          double xt[2];
#pragma unroll
          for (int kc = 0; kc < 2; ++kc) xt[kc] = __dmul_rn(Ua[ob + (4 * kc + kq) * st], xw[kc]);
          double k0 = 0.0, k1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
          for (int kc = 0; kc < 2; ++kc) {
            dmma8(k0, k1, xw[kc], bKn[ax][kc]);
            dmma8(t0, t1, xt[kc], bDt[kc]);
          }
          double ej[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          const bool own = (ax == ci);
          if (own) {
#pragma unroll
            for (int kc = 0; kc < 2; ++kc) {
              const int o = ob + (4 * kc + kq) * st;
#pragma unroll
              for (int jj = 0; jj < 3; ++jj) dmma8(ej[jj][0], ej[jj][1], __dmul_rn(t, sU[jj * B + o]), bD[kc]);
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int o = ob + (2 * kq + h) * st;
            double v = __dsub_rn(h ? k1 : k0, h ? t1 : t0);
            if (own) {
#pragma unroll
              for (int jj = 0; jj < 3; ++jj) v = __fma_rn(-sW[jj * B + o], ej[jj][h], v);
            }
            c[h] = v;
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int o = ob + (2 * kq + h) * st;
          ACC[o] = (ax == 0) ? c[h] : __dadd_rn(ACC[o], c[h]);
        }
      }
      __syncthreads();
    }
    double* dst = loc + ((int64_t)ci * G.nelem + e) * n3;
    for (int q = tid; q < n3; q += blockDim.x) dst[q] = ACC[bidx<N>(q >> 6, (q >> 3) & 7, q & 7)];
    __syncthreads();
  }
}

// Q^T + M^-1: one CTA per (component, g1, g2) row, threads along g3.  The contributions
// of the element blocks sharing a node are summed per axis with (element k-1, local N)
// before (element k, local 0); the row's axis-1/2 candidates are computed once per CTA
// and the per-thread index math is division by the compile-time N.
template <int N>
__global__ void __launch_bounds__(128) gather3d_kernel(const Geo3 G, const double* __restrict__ cbuf,
                                                      const double* __restrict__ loc, double* out, int scale) {
  constexpr int n = N + 1, n3 = n * n * n;
  const double* minv_pat = cbuf + 7 * n * n;
  const int P1 = (int)G.P1, P2 = (int)G.P2, P3 = (int)G.P3;
  const int row = blockIdx.x;                          // (c * P1 + g1) * P2 + g2
  const int g2 = row % P2, t1 = row / P2, g1 = t1 % P1, c = t1 / P1;
  int e1c[2], l1c[2], e2c[2], l2c[2], n1, n2c, cl1, cl2;
  {
    const int k = g1 / N, r = g1 - k * N;
    if (r) { n1 = 1; e1c[0] = k; l1c[0] = r; cl1 = r; }
    else { n1 = 2; e1c[0] = k ? k - 1 : (int)G.E1 - 1; l1c[0] = N; e1c[1] = k; l1c[1] = 0; cl1 = g1 ? N : 0; }
  }
  {
    const int k = g2 / N, r = g2 - k * N;
    if (r) { n2c = 1; e2c[0] = k; l2c[0] = r; cl2 = r; }
    else { n2c = 2; e2c[0] = k ? k - 1 : (int)G.E2 - 1; l2c[0] = N; e2c[1] = k; l2c[1] = 0; cl2 = g2 ? N : 0; }
  }
  const double* lc = loc + (int64_t)c * G.nelem * n3;
  double* orow = out + ((int64_t)(c * P1 + g1) * P2 + g2) * P3;
  const int E2 = (int)G.E2, E3 = (int)G.E3;
  for (int g3 = threadIdx.x; g3 < P3; g3 += blockDim.x) {
    const int k = g3 / N, r = g3 - k * N;
    int e3c[2], l3c[2], n3c, cl3;
    if (r) { n3c = 1; e3c[0] = k; l3c[0] = r; cl3 = r; }
    else { n3c = 2; e3c[0] = k ? k - 1 : E3 - 1; l3c[0] = N; e3c[1] = k; l3c[1] = 0; cl3 = g3 ? N : 0; }
    double acc = 0.0;
    for (int x = 0; x < n1; ++x)
      for (int y = 0; y < n2c; ++y)
        for (int z = 0; z < n3c; ++z) {
          const int64_t e = ((int64_t)e1c[x] * E2 + e2c[y]) * E3 + e3c[z];
          acc = __dadd_rn(acc, __ldg(lc + e * n3 + (l1c[x] * n + l2c[y]) * n + l3c[z]));
        }
    if (scale) acc = __dmul_rn(acc, minv_pat[(cl1 * (N + 1) + cl2) * (N + 1) + cl3]);
    orow[g3] = acc;
  }
}

// terminal condition (adjoint.py:33-47): J = d^T M d, lam = 2 M d (periodic: no mask)
__global__ void __launch_bounds__(256) terminal3d_kernel(const Geo3 G, int N, const double* __restrict__ mass_pat,
                                                        const double* uN, const double* ud, double* lam,
                                                        double* partial) {
  __shared__ double red[256];
  double acc = 0.0;
  const int64_t total = 3 * G.nscalar;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t % G.nscalar;
    const int64_t g3 = g % G.P3, g12 = g / G.P3, g2 = g12 % G.P2, g1 = g12 / G.P2;
    const int64_t gg[3] = {g1, g2, g3};
    int cl[3];
    for (int a = 0; a < 3; ++a) {
      const int r = (int)(gg[a] % N);
      cl[a] = (r != 0) ? r : (gg[a] == 0 ? 0 : N);
    }
    const double m = mass_pat[(cl[0] * (N + 1) + cl[1]) * (N + 1) + cl[2]];
    const double d = __dsub_rn(uN[t], ud[t]);
    const double md = __dmul_rn(m, d);
    lam[t] = __dmul_rn(2.0, md);
    acc = __dadd_rn(acc, __dmul_rn(d, md));
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void sum_partials3d(const double* partial, int np, double* out) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += 256) acc = __dadd_rn(acc, partial[i]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

Geo3 geo(const sem3d_plan* p) {
  Geo3 G;
  G.E1 = p->E[0]; G.E2 = p->E[1]; G.E3 = p->E[2];
  G.P1 = p->P[0]; G.P2 = p->P[1]; G.P3 = p->P[2];
  G.nscalar = p->nscalar;
  G.nelem = p->nelem;
  G.mnu = -p->nu;
  return G;
}

template <int OP>
cudaError_t launch_elem_mma(const sem3d_plan* p, const double* u, const double* w, double* loc, int* flag,
                            cudaStream_t s) {
  auto kern = elem3d_mma_kernel<OP>;
  constexpr size_t smem = sizeof(double) * (size_t)L3<7>::BLK * (OP == OP3_RHS ? 4 : 7);
  static sem1d::DevCache attr;     // the attribute is per (kernel, device)
  int& done = attr.here();
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    done = 1;
  }
  kern<<<(unsigned)p->nelem, 128, smem, s>>>(geo(p), p->cbuf, u, w, loc, flag);
  return cudaGetLastError();
}

template <int N, int OP>
cudaError_t launch_elem(const sem3d_plan* p, const double* u, const double* w, double* loc, int* flag,
                        cudaStream_t s) {
  if constexpr (N == 7) {
    if (sem1d::sem1d_path_override() == 0) return launch_elem_mma<OP>(p, u, w, loc, flag, s);
  }
  auto kern = elem3d_kernel<N, OP>;
  constexpr size_t smem = L3<N>::smem(OP);
  static sem1d::DevCache attr;     // the attribute is per (kernel, device)
  int& done = attr.here();
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    done = 1;
  }
  kern<<<(unsigned)p->nelem, L3<N>::THREADS, smem, s>>>(geo(p), p->cbuf, u, w, loc, flag);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_gather(const sem3d_plan* p, const double* loc, double* out, int scale, cudaStream_t s) {
  const int64_t rows = 3 * p->P[0] * p->P[1];
  if (rows > 0x7fffffffLL) return cudaErrorInvalidValue;
  gather3d_kernel<N><<<(unsigned)rows, 128, 0, s>>>(geo(p), p->cbuf, loc, out, scale);
  return cudaGetLastError();
}

template <int N>
cudaError_t apply_n(const sem3d_plan* p, int op, const double* u, const double* w, double* out, double* loc,
                    int* flag, cudaStream_t s) {
  cudaError_t e;
  if (op == OP3_RHS) e = launch_elem<N, OP3_RHS>(p, u, nullptr, loc, flag, s);
  else if (op == OP3_JAC) e = launch_elem<N, OP3_JAC>(p, u, w, loc, flag, s);
  else e = launch_elem<N, OP3_JACT>(p, u, w, loc, flag, s);
  if (e != cudaSuccess) return e;
  return launch_gather<N>(p, loc, out, op != OP3_JACT, s);
}

cudaError_t dispatch3(const sem3d_plan* p, int op, const double* u, const double* w, double* out, double* loc,
                      int* flag, cudaStream_t s) {
  switch (p->N) {
#define S3_CASE(NN) \
  case NN: return apply_n<NN>(p, op, u, w, out, loc, flag, s);
    S3_CASE(1) S3_CASE(2) S3_CASE(3) S3_CASE(4) S3_CASE(5) S3_CASE(6)
    S3_CASE(7) S3_CASE(8) S3_CASE(9) S3_CASE(10) S3_CASE(11) S3_CASE(12)
#undef S3_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

extern "C" {

int sem3d_max_degree(void) { return S3_MAX_N; }

int sem3d_plan_create(const int64_t* elements, int degree, double nu, const double* K3, const double* Dw,
                      const double* T3, const double* minv_pattern, const double* mass_pattern,
                      sem3d_plan** out) {
  if (!out || !elements || !K3 || !Dw || !T3 || !minv_pattern || !mass_pattern)
    return fail(SEM1D_EINVAL, "sem3d_plan_create: NULL argument");
  if (degree < 1 || degree > S3_MAX_N)
    return fail(SEM1D_EINVAL, "sem3d_plan_create: degree must be in 1..12");
  const int n = degree + 1;
  sem3d_plan* p = new (std::nothrow) sem3d_plan();
  if (!p) return fail(SEM1D_EINVAL, "sem3d_plan_create: out of host memory");
  p->N = degree;
  p->n = n;
  p->nu = nu;
  if (cudaGetDevice(&p->device) != cudaSuccess) p->device = 0;
  p->nscalar = 1;
  p->nelem = 1;
  for (int a = 0; a < 3; ++a) {
    if (elements[a] < 1) {
      delete p;
      return fail(SEM1D_EINVAL, "sem3d_plan_create: elements must be >= 1");
    }
    p->E[a] = elements[a];
    p->P[a] = elements[a] * degree;
    p->nscalar *= p->P[a];
    p->nelem *= p->E[a];
  }
  const int pat = (degree + 1) * (degree + 1) * (degree + 1);
  std::vector<double> host(7 * n * n + 2 * pat);
  std::memcpy(host.data(), K3, sizeof(double) * 3 * n * n);
  std::memcpy(host.data() + 3 * n * n, Dw, sizeof(double) * n * n);
  std::memcpy(host.data() + 4 * n * n, T3, sizeof(double) * 3 * n * n);
  std::memcpy(host.data() + 7 * n * n, minv_pattern, sizeof(double) * pat);
  std::memcpy(host.data() + 7 * n * n + pat, mass_pattern, sizeof(double) * pat);
  cudaError_t e = cudaMalloc(&p->cbuf, sizeof(double) * host.size());
  if (e == cudaSuccess) e = cudaMemcpy(p->cbuf, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (p->cbuf) cudaFree(p->cbuf);
    delete p;
    return cuda_fail(e, "sem3d_plan_create");
  }
  *out = p;
  return SEM1D_OK;
}

int sem3d_plan_destroy(sem3d_plan* p) {
  sem1d::DeviceGuard guard_(p ? p->device : -1);
  if (!p) return SEM1D_OK;
  if (p->cbuf) cudaFree(p->cbuf);
  delete p;
  return SEM1D_OK;
}

int64_t sem3d_plan_ndof(const sem3d_plan* p) { return p ? 3 * p->nscalar : -1; }

int64_t sem3d_work_size(const sem3d_plan* p) {
  sem1d::DeviceGuard guard_(p ? p->device : -1);
  if (!p) return -1;
  return 3 * p->nelem * (int64_t)p->n * p->n * p->n + 4096;
}

static int run3(const sem3d_plan* p, int op, const double* u, const double* w, double* out, double* work,
                int* flag, void* stream, const char* name) {
  sem1d::DeviceGuard guard_(p ? p->device : -1);
  if (!p || !u || !out || !work || !flag || (op != OP3_RHS && !w))
    return fail(SEM1D_EINVAL, std::string(name) + ": bad argument");
  if (out == u || out == w) return fail(SEM1D_EINVAL, std::string(name) + ": output must not alias an input");
  cudaError_t e = dispatch3(p, op, u, w, out, work, flag, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, name);
}

int sem3d_rhs(const sem3d_plan* p, const double* u, double* f, double* work, int* flag, void* stream) {
  sem1d::DeviceGuard guard_(p ? p->device : -1);
  return run3(p, OP3_RHS, u, nullptr, f, work, flag, stream, "sem3d_rhs");
}
int sem3d_jac(const sem3d_plan* p, const double* u, const double* v, double* out, double* work, int* flag,
              void* stream) {
  sem1d::DeviceGuard guard_(p ? p->device : -1);
  return run3(p, OP3_JAC, u, v, out, work, flag, stream, "sem3d_jac");
}
int sem3d_jact(const sem3d_plan* p, const double* u, const double* z, double* out, double* work, int* flag,
               void* stream) {
  sem1d::DeviceGuard guard_(p ? p->device : -1);
  return run3(p, OP3_JACT, u, z, out, work, flag, stream, "sem3d_jact");
}

int sem3d_terminal(const sem3d_plan* p, const double* uN, const double* ud, double* lam, double* J,
                   double* work, void* stream) {
  sem1d::DeviceGuard guard_(p ? p->device : -1);
  if (!p || !uN || !ud || !lam || !J || !work) return fail(SEM1D_EINVAL, "sem3d_terminal: bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int pat = (p->N + 1) * (p->N + 1) * (p->N + 1);
  const int blocks = 148 * 4;
  terminal3d_kernel<<<blocks, 256, 0, s>>>(geo(p), p->N, p->cbuf + 7 * p->n * p->n + pat, uN, ud, lam, work);
  sum_partials3d<<<1, 256, 0, s>>>(work, blocks, J);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem3d_terminal");
}

}  // extern "C"
