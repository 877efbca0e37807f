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

namespace sem1d {
int set_error(int code, const std::string& msg);   // sem1d_capi.cu
}

struct sem3d_plan {
  int N, n;
  int64_t E[3], P[3], nscalar, nelem;
  double nu;
  double* cbuf;   // device: K[3][n*n], Dw[n*n], T[3][n*n], minv[(N+1)^3], mass[(N+1)^3]
};

namespace {

constexpr int S3_MAX_N = 12;
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

template <int N>
struct L3 {
  static constexpr int n = N + 1, n2 = n * n, n3 = n * n * n;
  static constexpr int THREADS = ((n2 + 31) / 32) * 32;
  // shared arrays (doubles): consts 7 n^2, fields, scratch
  static constexpr int CONSTS = 7 * n2;
  static constexpr int arrays(int op) { return op == OP3_RHS ? 6 : (op == OP3_JAC ? 11 : 12); }
  static constexpr size_t smem(int op) { return sizeof(double) * ((size_t)CONSTS + (size_t)arrays(op) * n3); }
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
template <int n>
__device__ __forceinline__ double contract_row(const double* A, const double (&x)[n], int i) {
  double acc = __dmul_rn(A[i * n], x[0]);
#pragma unroll
  for (int l = 1; l < n; ++l) acc = __dadd_rn(acc, __dmul_rn(A[i * n + l], x[l]));
  return acc;
}
template <int n>
__device__ __forceinline__ double contract_row_t(const double* A, const double (&x)[n], int i) {
  double acc = __dmul_rn(A[i], x[0]);
#pragma unroll
  for (int l = 1; l < n; ++l) acc = __dadd_rn(acc, __dmul_rn(A[l * n + i], x[l]));
  return acc;
}

// node offset inside an n^3 block for phase `ax` (0,1,2), pencil (a,b), position p along ax
template <int n>
__device__ __forceinline__ int off(int ax, int a, int b, int p) {
  return ax == 0 ? (p * n + a) * n + b : (ax == 1 ? (a * n + p) * n + b : (a * n + b) * n + p);
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
  double* sU = sT + 3 * n2;         // [3][n3] state
  double* sW = sU + 3 * n3;         // [3][n3] v (J) / M^-1 z (J^T); unused for F
  double* scr = (OP == OP3_RHS) ? sW : sW + 3 * n3;   // scratch arrays
  const int tid = threadIdx.x;
  for (int k = tid; k < 7 * n2; k += blockDim.x) sK[k] = cbuf[k];
  const int64_t e = blockIdx.x;
  const int64_t e3 = e % G.E3, e12 = e / G.E3, e2 = e12 % G.E2, e1 = e12 / G.E2;
  const double* minv_pat = cbuf + 7 * n2;     // [(N+1)^3] by position class
  unsigned bad_u = 0, bad_w = 0;
  for (int q = tid; q < n3; q += blockDim.x) {
    const int i = q / n2, j = (q / n) % n, k = q % n;
    const int64_t g = node_index(G, e1, e2, e3, N, i, j, k);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = u[c * G.nscalar + g];
      bad_u |= nonfin3(x);
      sU[c * n3 + q] = x;
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
        sW[c * n3 + q] = y;
      }
    }
  }
  if (bad_u || bad_w)
    atomicOr(flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0));
  __syncthreads();
  const bool act = tid < n2;
  const int a = tid / n, b = tid % n;
  double* KS = scr;                 // sum_j K_j x_i (accumulated over the phases)
  double* const* dummy = nullptr;
  (void)dummy;
  for (int ci = 0; ci < 3; ++ci) {
    const double* Ui = sU + ci * n3;
    const double* Wi = sW + ci * n3;
    for (int ax = 0; ax < 3; ++ax) {
      if (act) {
        const double t = sT[ax * n2 + a * n + b];
        const double* Ka = sK + ax * n2;
        double xu[n], xw[n];
#pragma unroll
        for (int l = 0; l < n; ++l) {
          const int o = off<n>(ax, a, b, l);
          xu[l] = Ui[o];
          if (OP != OP3_RHS) xw[l] = Wi[o];
        }
        if (OP == OP3_RHS) {
          double* D0 = scr + n3;
          double* D1 = scr + 2 * n3;
#pragma unroll 1
          for (int p = 0; p < n; ++p) {
            const int o = off<n>(ax, a, b, p);
            const double kt = __dmul_rn(contract_row<n>(Ka, xu, p), t);
            const double dt = __dmul_rn(contract_row<n>(sD, xu, p), t);
            if (ax == 0) {
              KS[o] = kt;
              D0[o] = dt;
            } else if (ax == 1) {
              KS[o] = __dadd_rn(KS[o], kt);
              D1[o] = dt;
            } else {
              double acc = __dmul_rn(__dadd_rn(KS[o], kt), G.mnu);
              acc = __dsub_rn(acc, __dmul_rn(sU[o], D0[o]));
              acc = __dsub_rn(acc, __dmul_rn(sU[n3 + o], D1[o]));
              acc = __dsub_rn(acc, __dmul_rn(sU[2 * n3 + o], dt));
              KS[o] = acc;                       // element result (in place)
            }
          }
        } else if (OP == OP3_JAC) {
          // D_ax u_i and D_ax w_i per node, kept for the final combination
          double* Du = scr + n3 + 2 * ax * n3;   // [3][2] arrays: (Du, Dw) per axis 0,1
          double* Dv = Du + n3;
#pragma unroll 1
          for (int p = 0; p < n; ++p) {
            const int o = off<n>(ax, a, b, p);
            const double kt = __dmul_rn(contract_row<n>(Ka, xw, p), t);
            const double du = __dmul_rn(contract_row<n>(sD, xu, p), t);
            const double dw = __dmul_rn(contract_row<n>(sD, xw, p), t);
            if (ax == 0) {
              KS[o] = kt;
              Du[o] = du;
              Dv[o] = dw;
            } else if (ax == 1) {
              KS[o] = __dadd_rn(KS[o], kt);
              Du[o] = du;
              Dv[o] = dw;
            } else {
              const double* Du0 = scr + n3;
              const double* Dv0 = Du0 + n3;
              const double* Du1 = Du0 + 2 * n3;
              const double* Dv1 = Du1 + n3;
              double acc = __dmul_rn(__dadd_rn(KS[o], kt), G.mnu);
              acc = __dsub_rn(acc, __dmul_rn(sW[o], Du0[o]));
              acc = __dsub_rn(acc, __dmul_rn(sU[o], Dv0[o]));
              acc = __dsub_rn(acc, __dmul_rn(sW[n3 + o], Du1[o]));
              acc = __dsub_rn(acc, __dmul_rn(sU[n3 + o], Dv1[o]));
              acc = __dsub_rn(acc, __dmul_rn(sW[2 * n3 + o], du));
              acc = __dsub_rn(acc, __dmul_rn(sU[2 * n3 + o], dw));
              KS[o] = acc;
            }
          }
        } else {
          // J^T: K_ax z_i, T_ax = D_ax^T (u_ax o z_i), and on the phase ax == ci the
          // three E_j = z_j (D_ci u_j)
          double* Ej = scr + n3;                 // [3] arrays
          double* Tj = scr + 4 * n3;             // [2] arrays (T_0, T_1)
          double xt[n];
          const double* Ua = sU + ax * n3;
#pragma unroll
          for (int l = 0; l < n; ++l) {
            const int o = off<n>(ax, a, b, l);
            xt[l] = __dmul_rn(Ua[o], xw[l]);
          }
          double xu1[n], xu2[n], xu0[n];
          const bool own = (ax == ci);
          if (own) {
#pragma unroll
            for (int l = 0; l < n; ++l) {
              const int o = off<n>(ax, a, b, l);
              xu0[l] = sU[o];
              xu1[l] = sU[n3 + o];
              xu2[l] = sU[2 * n3 + o];
            }
          }
#pragma unroll 1
          for (int p = 0; p < n; ++p) {
            const int o = off<n>(ax, a, b, p);
            const double kt = __dmul_rn(contract_row<n>(Ka, xw, p), t);
            const double tt = __dmul_rn(contract_row_t<n>(sD, xt, p), t);
            double e0 = 0.0, e1v = 0.0, e2v = 0.0;
            if (own) {
              e0 = __dmul_rn(sW[o], __dmul_rn(contract_row<n>(sD, xu0, p), t));
              e1v = __dmul_rn(sW[n3 + o], __dmul_rn(contract_row<n>(sD, xu1, p), t));
              e2v = __dmul_rn(sW[2 * n3 + o], __dmul_rn(contract_row<n>(sD, xu2, p), t));
            }
            if (ax < 2) {
              KS[o] = (ax == 0) ? kt : __dadd_rn(KS[o], kt);
              Tj[ax * n3 + o] = tt;
              if (own) {
                Ej[o] = e0;
                Ej[n3 + o] = e1v;
                Ej[2 * n3 + o] = e2v;
              }
            } else {
              const double E0 = own ? e0 : Ej[o];
              const double E1 = own ? e1v : Ej[n3 + o];
              const double E2 = own ? e2v : Ej[2 * n3 + o];
              double acc = __dmul_rn(__dadd_rn(KS[o], kt), G.mnu);
              acc = __dsub_rn(acc, E0);
              acc = __dsub_rn(acc, Tj[o]);
              acc = __dsub_rn(acc, E1);
              acc = __dsub_rn(acc, Tj[n3 + o]);
              acc = __dsub_rn(acc, E2);
              acc = __dsub_rn(acc, tt);
              KS[o] = acc;
            }
          }
        }
      }
      __syncthreads();
    }
    // element block of component ci -> scratch (coalesced: contiguous n^3 run)
    double* dst = loc + ((int64_t)ci * G.nelem + e) * n3;
    for (int q = tid; q < n3; q += blockDim.x) dst[q] = KS[q];
    __syncthreads();
  }
}

// Q^T + M^-1: one thread per (component, global node); contributions of the element
// blocks that share the node, per axis (element k-1, local N) before (element k, local 0).
template <int N>
__global__ void __launch_bounds__(256) gather3d_kernel(const Geo3 G, const double* __restrict__ cbuf,
                                                      const double* __restrict__ loc, double* out, int scale) {
  constexpr int n = N + 1, n3 = n * n * n;
  const int64_t total = 3 * G.nscalar;
  const double* minv_pat = cbuf + 7 * n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / G.nscalar);
    const int64_t g = t - c * G.nscalar;
    const int64_t g3 = g % G.P3, g12 = g / G.P3, g2 = g12 % G.P2, g1 = g12 / G.P2;
    const int64_t gg[3] = {g1, g2, g3};
    const int64_t EE[3] = {G.E1, G.E2, G.E3};
    int64_t ea[3][2];
    int la[3][2], na[3], cl[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int64_t k = gg[a] / N;
      const int r = (int)(gg[a] - k * N);
      if (r != 0) {
        na[a] = 1;
        ea[a][0] = k;
        la[a][0] = r;
        cl[a] = r;
      } else {
        na[a] = 2;
        const int64_t km = (k == 0) ? EE[a] - 1 : k - 1;
        ea[a][0] = km;       // element k-1 (local N) first
        la[a][0] = N;
        ea[a][1] = k;
        la[a][1] = 0;
        cl[a] = (gg[a] == 0) ? 0 : N;
      }
    }
    double acc = 0.0;
    for (int x = 0; x < na[0]; ++x)
      for (int y = 0; y < na[1]; ++y)
        for (int z = 0; z < na[2]; ++z) {
          const int64_t e = (ea[0][x] * G.E2 + ea[1][y]) * G.E3 + ea[2][z];
          const int q = (la[0][x] * n + la[1][y]) * n + la[2][z];
          acc = __dadd_rn(acc, __ldg(loc + ((int64_t)c * G.nelem + e) * n3 + q));
        }
    if (scale) acc = __dmul_rn(acc, minv_pat[(cl[0] * (N + 1) + cl[1]) * (N + 1) + cl[2]]);
    out[t] = acc;
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

template <int N, int OP>
cudaError_t launch_elem(const sem3d_plan* p, const double* u, const double* w, double* loc, int* flag,
                        cudaStream_t s) {
  auto kern = elem3d_kernel<N, OP>;
  constexpr size_t smem = L3<N>::smem(OP);
  static bool done = false;
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    done = true;
  }
  kern<<<(unsigned)p->nelem, L3<N>::THREADS, smem, s>>>(geo(p), p->cbuf, u, w, loc, flag);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_gather(const sem3d_plan* p, const double* loc, double* out, int scale, cudaStream_t s) {
  const int64_t total = 3 * p->nscalar;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  gather3d_kernel<N><<<grid, 256, 0, s>>>(geo(p), p->cbuf, loc, out, scale);
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
  if (!p) return SEM1D_OK;
  if (p->cbuf) cudaFree(p->cbuf);
  delete p;
  return SEM1D_OK;
}

int64_t sem3d_plan_ndof(const sem3d_plan* p) { return p ? 3 * p->nscalar : -1; }

int64_t sem3d_work_size(const sem3d_plan* p) {
  if (!p) return -1;
  return 3 * p->nelem * (int64_t)p->n * p->n * p->n + 4096;
}

static int run3(const sem3d_plan* p, int op, const double* u, const double* w, double* out, double* work,
                int* flag, void* stream, const char* name) {
  if (!p || !u || !out || !work || !flag || (op != OP3_RHS && !w))
    return fail(SEM1D_EINVAL, std::string(name) + ": bad argument");
  if (out == u || out == w) return fail(SEM1D_EINVAL, std::string(name) + ": output must not alias an input");
  cudaError_t e = dispatch3(p, op, u, w, out, work, flag, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, name);
}

int sem3d_rhs(const sem3d_plan* p, const double* u, double* f, double* work, int* flag, void* stream) {
  return run3(p, OP3_RHS, u, nullptr, f, work, flag, stream, "sem3d_rhs");
}
int sem3d_jac(const sem3d_plan* p, const double* u, const double* v, double* out, double* work, int* flag,
              void* stream) {
  return run3(p, OP3_JAC, u, v, out, work, flag, stream, "sem3d_jac");
}
int sem3d_jact(const sem3d_plan* p, const double* u, const double* z, double* out, double* work, int* flag,
               void* stream) {
  return run3(p, OP3_JACT, u, z, out, work, flag, stream, "sem3d_jact");
}

int sem3d_terminal(const sem3d_plan* p, const double* uN, const double* ud, double* lam, double* J,
                   double* work, void* stream) {
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
