// sem1d_krylov.cu -- the implicit (Crank-Nicolson) path and the adaptive Kutta-3
// controller on the device.
//
//  * sem1d_gmres: restarted GMRES with modified Gram-Schmidt and Givens rotations,
//    the algorithm scipy.sparse.linalg.gmres (scipy 1.18.1, the reference's own
//    unpinned dependency, pyproject.toml:10-13) runs for the reference's
//    _gmres_solve (timeloop.py:133-151): x0 = 0, rtol = gmres_tol, atol = 0,
//    restart = min(restart, n), maxiter = ceil(gmres_max / restart), the inner
//    stop on the Givens residual estimate with the gh-8400 tolerance control, the
//    true-residual check after every cycle, and one counted matvec per Arnoldi
//    column plus one per cycle (the reference's gmres_iters).  The operator is
//    the shifted Jacobian x + alpha * J(p) x or x + alpha * J(p)^T x.
//  * sem1d_cn_step: full Newton on v - u - dt/2 (f(u) + f(v)) = 0 with GMRES on
//    (I - dt/2 J(v)) (timeloop.py:154-186).
//  * sem1d_cn_adjoint_step: (I - dt/2 J(u_{n+1}))^T mu = lam, lam_n = mu + dt/2 J^T(u_n) mu
//    (adjoint.py:64-69).
//  * sem1d_rk_error_norm: the embedded-pair weighted error of timeloop.py:198-218.
//
// The Krylov vectors never leave HBM: the matvec is the library's own J / J^T kernel
// followed by ONE fused pass that applies the shift and accumulates |w|^2 and the first
// projection; each modified Gram-Schmidt step is one pass that subtracts the previous
// projection and accumulates the next one.  The small Hessenberg problem (at most
// restart+1 values per column) is solved on the host, which reads one column per
// Arnoldi step -- the same decision points as the reference's loop.
//
// Reductions are deterministic: a fixed grid of KB CTAs writes one partial per CTA,
// and the last CTA to finish (threadfence + ticket) combines the KB partials in a
// fixed tree order.  Element arithmetic follows the reference's numpy evaluation
// order with no FMA contraction.
#include <cuda_runtime.h>

#include "sem1d_devguard.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "sem1d.h"

namespace sem1d {
int set_error(int code, const std::string& msg);   // sem1d_capi.cu
int64_t plan_batch(const sem1d_plan* p);           // sem1d_capi.cu
int plan_device(const sem1d_plan* p);              // sem1d_capi.cu
int plan3_device(const sem3d_plan* p);             // sem3d.cu
}  // namespace sem1d

namespace {

constexpr int KT = 256;                 // threads per CTA
constexpr int KB = 4 * 148;             // CTAs per reduction launch: one resident wave (4 per SM), fixed
constexpr int KU = 4;                   // grid-strided elements per thread with loads issued together
constexpr int RED_DOUBLES = 2 * KB + 2; // partials (2 slots) + ticket
constexpr int MAX_RESTART = 64;

int fail(int code, const std::string& m) { return sem1d::set_error(code, m); }
int cuda_fail(cudaError_t e, const char* where) {
  return fail(SEM1D_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ reductions

template <bool MAX>
__device__ __forceinline__ double red_op(double a, double b) {
  return MAX ? fmax(a, b) : __dadd_rn(a, b);
}

template <int R, bool MAX>
__device__ __forceinline__ void block_reduce(double (&v)[R], double (*sred)[KT / 32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[r] = red_op<MAX>(v[r], __shfl_xor_sync(0xffffffffu, v[r], o));
    if (lane == 0) sred[r][warp] = v[r];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = sred[r][0];
      for (int w = 1; w < KT / 32; ++w) acc = red_op<MAX>(acc, sred[r][w]);
      v[r] = acc;
    }
  }
}

// Grid-wide deterministic reduction of R values per thread; thread 0 of the last CTA
// writes out[0..R-1].  Must be called by every thread of every CTA (gridDim.x == KB).
template <int R, bool MAX>
__device__ __forceinline__ void grid_reduce(double (&v)[R], double* work, double* out) {
  __shared__ double sred[R][KT / 32];
  __shared__ bool last;
  unsigned* ticket = reinterpret_cast<unsigned*>(work + 2 * KB);
  block_reduce<R, MAX>(v, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) work[r * KB + blockIdx.x] = v[r];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double w[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {          // fixed order: thread t combines partials t, t+KT, ...
    w[r] = __ldcg(work + r * KB + threadIdx.x);
    for (int k = threadIdx.x + KT; k < KB; k += KT) w[r] = red_op<MAX>(w[r], __ldcg(work + r * KB + k));
  }
  __syncthreads();                       // sred reuse
  block_reduce<R, MAX>(w, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) out[r] = w[r];
    *ticket = 0u;                        // ready for the next launch on this stream
  }
}

__device__ __forceinline__ bool nonfin(double x) {
  return ((unsigned)__double2hiint(x) & 0x7ff00000u) == 0x7ff00000u;
}

// ------------------------------------------------------------------ kernels

// Grid-strided element loop with KU loads in flight per thread: LOAD(u, i) fills the
// registers of slot u, STEP(u, i) consumes them (all loads of a batch precede its stores,
// so aliasing between outputs and inputs cannot serialise them).
#define KR_LOOP(n, LOAD, STEP)                                                          \
  {                                                                                     \
    const int64_t S_ = (int64_t)gridDim.x * KT;                                         \
    int64_t i0_ = blockIdx.x * (int64_t)KT + threadIdx.x;                               \
    for (; i0_ + (KU - 1) * S_ < (n); i0_ += KU * S_) {                                 \
      _Pragma("unroll") for (int u = 0; u < KU; ++u) { const int64_t i = i0_ + u * S_; (void)i; LOAD } \
      _Pragma("unroll") for (int u = 0; u < KU; ++u) { const int64_t i = i0_ + u * S_; (void)i; STEP } \
    }                                                                                   \
    for (; i0_ < (n); i0_ += S_) {                                                      \
      const int u = 0;                                                                  \
      const int64_t i = i0_;                                                            \
      (void)i;                                                                          \
      LOAD STEP                                                                         \
    }                                                                                   \
  }

__global__ void __launch_bounds__(KT, 4) k_dot(int64_t n, const double* x, const double* y, double* work,
                                            double* out) {
  double v[1] = {0.0};
  double a[KU], b[KU];
  KR_LOOP(n, { a[u] = __ldg(x + i); b[u] = __ldg(y + i); },
          { v[0] = __dadd_rn(v[0], __dmul_rn(a[u], b[u])); })
  grid_reduce<1, false>(v, work, out);
}

// w = x + alpha t;  out[0] = w.w, out[1] = z.w (z may be NULL)
__global__ void __launch_bounds__(KT, 4) k_shift_dot2(int64_t n, const double* x, const double* t, double alpha,
                                                   double* w, const double* z, double* work, double* out) {
  double v[2] = {0.0, 0.0};
  double a[KU], b[KU], c[KU];
  KR_LOOP(n, { a[u] = x[i]; b[u] = t[i]; c[u] = z ? z[i] : 0.0; },
          {
            const double wi = __dadd_rn(a[u], __dmul_rn(alpha, b[u]));
            w[i] = wi;
            v[0] = __dadd_rn(v[0], __dmul_rn(wi, wi));
            v[1] = __dadd_rn(v[1], __dmul_rn(c[u], wi));
          })
  grid_reduce<2, false>(v, work, out);
}

// y -= a[0] * x (modified Gram-Schmidt update);  out[0] = z.y_new (z == y: |y_new|^2)
__global__ void __launch_bounds__(KT, 4) k_axpy_dot(int64_t n, const double* a, const double* x, double* y,
                                                 const double* z, double* work, double* out) {
  const double av = __ldcg(a);
  const bool self = (z == y);
  double v[1] = {0.0};
  double xa[KU], ya[KU], za[KU];
  KR_LOOP(n, { xa[u] = __ldg(x + i); ya[u] = y[i]; za[u] = self ? 0.0 : __ldg(z + i); },
          {
            const double yi = __dsub_rn(ya[u], __dmul_rn(av, xa[u]));
            y[i] = yi;
            v[0] = __dadd_rn(v[0], __dmul_rn(self ? yi : za[u], yi));
          })
  grid_reduce<1, false>(v, work, out);
}

__global__ void __launch_bounds__(KT, 4) k_scale(int64_t n, const double* x, double s, double* y) {
  double a[KU];
  KR_LOOP(n, { a[u] = x[i]; }, { y[i] = __dmul_rn(a[u], s); })
}

struct Coefs {
  double c[MAX_RESTART + 1];
};

// x += sum_k c_k V_k   (scipy: x += y @ v[:col+1, :])
__global__ void __launch_bounds__(KT, 4) k_lincomb(int64_t n, int m, const Coefs c, const double* V,
                                                int64_t ld, double* x) {
  for (int64_t i = blockIdx.x * (int64_t)KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    double acc = __dmul_rn(c.c[0], V[i]);
    for (int k = 1; k < m; ++k) acc = __dadd_rn(acc, __dmul_rn(c.c[k], V[k * ld + i]));
    x[i] = __dadd_rn(x[i], acc);
  }
}

// r = b - (x + alpha t);  out[0] = r.r   (scipy: r = b - matvec(x))
__global__ void __launch_bounds__(KT, 4) k_residual(int64_t n, const double* b, const double* x, const double* t,
                                                 double alpha, double* r, double* work, double* out) {
  double v[1] = {0.0};
  double ba[KU], xa[KU], ta[KU];
  KR_LOOP(n, { ba[u] = __ldg(b + i); xa[u] = __ldg(x + i); ta[u] = __ldg(t + i); },
          {
            const double ri = __dsub_rn(ba[u], __dadd_rn(xa[u], __dmul_rn(alpha, ta[u])));
            r[i] = ri;
            v[0] = __dadd_rn(v[0], __dmul_rn(ri, ri));
          })
  grid_reduce<1, false>(v, work, out);
}

// nr = -((v - u) - h (fu + fv))  (timeloop.py:168 with the sign of the GMRES rhs -r);
// out[0] = |r|^2; a non-finite r sets flag bit 1
__global__ void __launch_bounds__(KT, 4) k_cn_residual(int64_t n, const double* v, const double* u_,
                                                    const double* fu, const double* fv, double h, double* nr,
                                                    double* work, double* out, int* flag) {
  double acc[1] = {0.0};
  bool bad = false;
  double va[KU], ua[KU], fa[KU], ga[KU];
  KR_LOOP(n, { va[u] = __ldg(v + i); ua[u] = __ldg(u_ + i); fa[u] = __ldg(fu + i); ga[u] = __ldg(fv + i); },
          {
            const double ri = __dsub_rn(__dsub_rn(va[u], ua[u]), __dmul_rn(h, __dadd_rn(fa[u], ga[u])));
            bad |= nonfin(ri);
            nr[i] = -ri;
            acc[0] = __dadd_rn(acc[0], __dmul_rn(ri, ri));
          })
  if (bad) atomicOr(flag, 1);
  grid_reduce<1, false>(acc, work, out);
}

__global__ void __launch_bounds__(KT, 4) k_add(int64_t n, const double* x, const double* y, double* out) {
  double a[KU], b[KU];
  KR_LOOP(n, { a[u] = x[i]; b[u] = y[i]; }, { out[i] = __dadd_rn(a[u], b[u]); })
}

// Embedded-pair error (timeloop.py:205-210): u_hat = u + dt k2, err = u_new - u_hat,
// tol = tol_a + max(|u_new|, |u_hat|) tol_r, ratio = |err| / tol;
// out[0] = sum sqrt(ratio) (form 0, "rms": the reference's mean of square roots) or max ratio
template <bool MAX>
__global__ void __launch_bounds__(KT, 4) k_rk_error(int64_t n, const double* un, const double* u_, const double* k2,
                                                 double dt, double ta, double tr, double* work, double* out) {
  double v[1] = {0.0};
  double na[KU], ua[KU], ka[KU];
  KR_LOOP(n, { na[u] = __ldg(un + i); ua[u] = __ldg(u_ + i); ka[u] = __ldg(k2 + i); },
          {
            const double uh = __dadd_rn(ua[u], __dmul_rn(dt, ka[u]));
            const double e = __dsub_rn(na[u], uh);
            const double tol = __dadd_rn(ta, __dmul_rn(fmax(fabs(na[u]), fabs(uh)), tr));
            const double ratio = __ddiv_rn(fabs(e), tol);
            v[0] = MAX ? fmax(v[0], ratio) : __dadd_rn(v[0], __dsqrt_rn(ratio));
          })
  grid_reduce<1, MAX>(v, work, out);
}

// ---- stage compositions for operators without fused stage kernels (3D) ----------

struct Terms {
  const double* p[SEM1D_MAX_TERMS];
  double c[SEM1D_MAX_TERMS];
  int n;
};

// Y = base + (dt c0) K0 (one term) or base + dt ((c0 K0 + c1 K1) + ...)  -- the association
// of timeloop.py:114-127 / sem1d_rk_stage; a non-finite Y sets SEM1D_FLAG_STEP_NONFINITE
__global__ void __launch_bounds__(KT, 4) k_rk_combine(int64_t n, const double* base, double dt, const Terms T,
                                                      double* Y, int check, int* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    double y;
    if (T.n == 1) {
      y = __dadd_rn(base[i], __dmul_rn(__dmul_rn(dt, T.c[0]), T.p[0][i]));
    } else {
      double acc = __dmul_rn(T.c[0], T.p[0][i]);
      for (int j = 1; j < T.n; ++j) acc = __dadd_rn(acc, __dmul_rn(T.c[j], T.p[j][i]));
      y = __dadd_rn(base[i], __dmul_rn(dt, acc));
    }
    if (check) bad |= nonfin(y);
    Y[i] = y;
  }
  if (bad) atomicOr(flag, SEM1D_FLAG_STEP_NONFINITE);
}

// z = b lam + sum_j a_j l_j (left to right, adjoint.py:58-60 / sem1d_adj_stage)
__global__ void __launch_bounds__(KT, 4) k_adj_combine(int64_t n, const double* lam, double b, const Terms T,
                                                       double* z) {
  for (int64_t i = blockIdx.x * (int64_t)KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    double acc = __dmul_rn(b, lam[i]);
    for (int j = 0; j < T.n; ++j) acc = __dadd_rn(acc, __dmul_rn(T.c[j], T.p[j][i]));
    z[i] = acc;
  }
}

// out = ((x + t0) + t1) + ...   (lam + l_1 + l_2 + ..., adjoint.py:61)
__global__ void __launch_bounds__(KT, 4) k_accumulate(int64_t n, const double* x, const Terms T, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    double acc = x[i];
    for (int j = 0; j < T.n; ++j) acc = __dadd_rn(acc, T.p[j][i]);
    out[i] = acc;
  }
}

bool make_terms(int nt, const double* const* ptrs, const double* coefs, Terms& T) {
  if (nt < 0 || nt > SEM1D_MAX_TERMS) return false;
  std::memset(&T, 0, sizeof(T));
  T.n = nt;
  for (int j = 0; j < nt; ++j) {
    if (!ptrs[j]) return false;
    T.p[j] = ptrs[j];
    T.c[j] = coefs ? coefs[j] : 1.0;
  }
  return true;
}

int ew_grid(int64_t n) {
  const int64_t b = (n + KT - 1) / KT;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, KB));
}

// ------------------------------------------------------------------ host drivers

struct Vec {
  cudaStream_t s;
  int64_t n;
  double* red;    // RED_DOUBLES reduction work (ticket zero-initialised by the caller)
  double* scal;   // device scalars
};

// LAPACK dlartg (3.10 algorithm, as scipy's lartg calls it): c, s, r with r = sign(f) sqrt(f^2+g^2)
void lartg(double f, double g, double& c, double& s, double& r) {
  const double safmin = 2.2250738585072014e-308, safmax = 1.0 / safmin;
  const double rtmin = std::sqrt(safmin), rtmax = std::sqrt(safmax / 2);
  const double f1 = std::fabs(f), g1 = std::fabs(g);
  if (g == 0.0) {
    c = 1.0; s = 0.0; r = f;
  } else if (f == 0.0) {
    c = 0.0; s = std::copysign(1.0, g); r = g1;
  } else if (f1 > rtmin && f1 < rtmax && g1 > rtmin && g1 < rtmax) {
    const double d = std::sqrt(f * f + g * g);
    c = f1 / d;
    r = std::copysign(d, f);
    s = g / r;
  } else {
    const double u = std::min(safmax, std::max(safmin, std::max(f1, g1)));
    const double fs = f / u, gs = g / u;
    const double d = std::sqrt(fs * fs + gs * gs);
    c = std::fabs(fs) / d;
    r = std::copysign(d, f);
    s = gs / r;
    r *= u;
  }
}

// The operator the Krylov drivers run on: a 1D plan (sem1d_*) or a 3D plan (sem3d_*,
// which also needs its element-block scratch).
struct OpIf {
  const void* plan;
  int is3d;
  double* work3d;
  int64_t n;
  int rhs(const double* u, double* f, int* flag, void* s) const {
    return is3d ? sem3d_rhs(static_cast<const sem3d_plan*>(plan), u, f, work3d, flag, s)
                : sem1d_rhs(static_cast<const sem1d_plan*>(plan), u, f, flag, s);
  }
  int jac(const double* u, const double* v, double* out, int* flag, void* s) const {
    return is3d ? sem3d_jac(static_cast<const sem3d_plan*>(plan), u, v, out, work3d, flag, s)
                : sem1d_jac(static_cast<const sem1d_plan*>(plan), u, v, out, flag, s);
  }
  int jact(const double* u, const double* z, double* out, int* flag, void* s) const {
    return is3d ? sem3d_jact(static_cast<const sem3d_plan*>(plan), u, z, out, work3d, flag, s)
                : sem1d_jact(static_cast<const sem1d_plan*>(plan), u, z, out, flag, s);
  }
};

struct Gmres {
  const OpIf* plan;
  int op;                 // 0: J(p), 1: J(p)^T
  const double* p;        // linearisation point
  double alpha;           // operator x + alpha * J x
  Vec v;
  double* V;              // (restart+1) x n basis
  double* t;              // J output
  int* flag;
  int64_t matvecs = 0;

  int jop(const double* x, double* out) {
    return op == 0 ? plan->jac(p, x, out, flag, v.s) : plan->jact(p, x, out, flag, v.s);
  }
};

int rd(const Vec& v, int k, double* host) {   // read k device scalars (syncs the stream)
  cudaError_t e = cudaMemcpyAsync(host, v.scal, sizeof(double) * k, cudaMemcpyDeviceToHost, v.s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(v.s);
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "krylov readback");
}

int dev_norm(const Vec& v, const double* x, double* res) {
  k_dot<<<KB, KT, 0, v.s>>>(v.n, x, x, v.red, v.scal);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "krylov dot");
  double h;
  int rc = rd(v, 1, &h);
  *res = std::sqrt(h);
  return rc;
}

int read_flag(const Vec& v, int* dflag, int* host) {
  cudaError_t e = cudaMemcpyAsync(host, dflag, sizeof(int), cudaMemcpyDeviceToHost, v.s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(v.s);
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "krylov flag readback");
}

// scipy 1.18.1 gmres(A, b, x0=None, rtol, atol=0, restart, maxiter), iterative.py:593-817,
// restated.  x (n doubles) receives the solution.  Returns 0 and *info (0 = converged,
// else maxiter) or an error code.
int gmres_run(Gmres& G, const double* b, double* x, double rtol, int restart, int maxiter, int* info,
              int* nonfinite) {
  const Vec& v = G.v;
  const int64_t n = v.n;
  cudaError_t e;
  double bnrm2;
  int rc = dev_norm(v, b, &bnrm2);
  if (rc) return rc;
  *info = 0;
  *nonfinite = 0;
  const double atol = rtol * bnrm2;           // _get_atol_rtol: max(atol=0, rtol * |b|)
  if (bnrm2 == 0.0) {                         // return b, 0
    e = cudaMemcpyAsync(x, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, v.s);
    return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "gmres copy");
  }
  const double eps = 2.220446049250313e-16;
  restart = (int)std::min<int64_t>(restart, n);
  double ptol_max_factor = 1.0;
  double ptol = bnrm2 * std::min(ptol_max_factor, atol / bnrm2);   // Mb_nrm2 = |b| (no preconditioner)
  double presid = 0.0, rnorm = 0.0;
  std::vector<double> h((size_t)restart * (restart + 1)), givens((size_t)restart * 2), S(restart + 1),
      col_h(restart + 3);
  auto H = [&](int c, int k) -> double& { return h[(size_t)c * (restart + 1) + k]; };
  e = cudaMemsetAsync(x, 0, sizeof(double) * n, v.s);
  if (e != cudaSuccess) return cuda_fail(e, "gmres init");
  double* V0 = G.V;
  // iteration 0: x = 0, so r = b.copy() (no matvec); |r| = |b| >= atol unless rtol >= 1
  e = cudaMemcpyAsync(V0, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, v.s);
  if (e != cudaSuccess) return cuda_fail(e, "gmres copy");
  double rn0 = bnrm2;
  if (rn0 < atol) return SEM1D_OK;
  for (int iteration = 0; iteration < maxiter; ++iteration) {
    // v[0] = r / |r| (r sits in V[0]); iteration 0 knows |r| = |b|, later cycles computed it
    const double tmp0 = (iteration == 0) ? rn0 : rnorm;
    k_scale<<<ew_grid(n), KT, 0, v.s>>>(n, V0, 1.0 / tmp0, V0);
    std::fill(S.begin(), S.end(), 0.0);
    std::fill(h.begin(), h.end(), 0.0);
    S[0] = tmp0;
    bool breakdown = false;
    int col = 0;
    for (col = 0; col < restart; ++col) {
      double* vc = G.V + (int64_t)col * n;
      double* w = G.V + (int64_t)(col + 1) * n;      // w is built in place of v[col+1]
      rc = G.jop(vc, G.t);
      if (rc) return rc;
      ++G.matvecs;
      // w = v_col + alpha J v_col; scal[col+1] = |w|^2 (h0), scal[0] = v_0 . w
      k_shift_dot2<<<KB, KT, 0, v.s>>>(n, vc, G.t, G.alpha, w, G.V, v.red, v.scal + col + 1);
      // shift_dot2 wrote scal[col+1] = w.w and scal[col+2] = v0.w; move v0.w to scal[0]
      // by running the MGS chain on scal[col+2] first: k = 0 uses it
      for (int k = 0; k <= col; ++k) {
        const double* a = (k == 0) ? v.scal + col + 2 : v.scal + 3 + col + k;   // h[col,k] on device
        double* outk = (k < col) ? v.scal + 3 + col + k + 1 : v.scal + 3 + 2 * col + 1 + 1;
        const double* z = (k < col) ? G.V + (int64_t)(k + 1) * n : w;          // next projection / |w|^2
        k_axpy_dot<<<KB, KT, 0, v.s>>>(n, a, G.V + (int64_t)k * n, w, z, v.red, outk);
      }
      e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(e, "gmres arnoldi");
      // read h0^2, h[col,0..col], h1^2
      const int nread = 3 + 2 * col + 3;
      std::vector<double> sc(nread);
      rc = rd(v, nread, sc.data());
      if (rc) return rc;
      const double h0 = std::sqrt(sc[col + 1]);
      H(col, 0) = sc[col + 2];
      for (int k = 1; k <= col; ++k) H(col, k) = sc[3 + col + k];
      const double h1 = std::sqrt(sc[3 + 2 * col + 2]);
      H(col, col + 1) = h1;
      if (!(std::isfinite(h0) && std::isfinite(h1))) {
        *nonfinite = 1;
        return SEM1D_OK;
      }
      if (h1 <= eps * h0) {                        // exact solution indicator
        H(col, col + 1) = 0.0;
        breakdown = true;
      } else {
        k_scale<<<ew_grid(n), KT, 0, v.s>>>(n, w, 1.0 / h1, w);
      }
      for (int k = 0; k < col; ++k) {               // past rotations
        const double c = givens[2 * k], s = givens[2 * k + 1];
        const double n0 = H(col, k), n1 = H(col, k + 1);
        H(col, k) = c * n0 + s * n1;
        H(col, k + 1) = -s * n0 + c * n1;
      }
      double c, s, mag;
      lartg(H(col, col), H(col, col + 1), c, s, mag);
      givens[2 * col] = c;
      givens[2 * col + 1] = s;
      H(col, col) = mag;
      H(col, col + 1) = 0.0;
      const double tmp = -s * S[col];
      S[col] = c * S[col];
      S[col + 1] = tmp;
      presid = std::fabs(tmp);
      if (presid <= ptol || breakdown) break;
    }
    if (col == restart) col = restart - 1;          // the for loop ran to completion
    if (H(col, col) == 0.0) S[col] = 0.0;
    std::vector<double> y(S.begin(), S.begin() + col + 1);
    for (int k = col; k > 0; --k) {
      if (y[k] != 0.0) {
        y[k] /= H(k, k);
        const double tk = y[k];
        for (int j = 0; j < k; ++j) y[j] -= tk * H(k, j);
      }
    }
    if (y[0] != 0.0) y[0] /= H(0, 0);
    Coefs cf;
    std::memset(&cf, 0, sizeof(cf));
    for (int k = 0; k <= col; ++k) cf.c[k] = y[k];
    k_lincomb<<<ew_grid(n), KT, 0, v.s>>>(n, col + 1, cf, G.V, n, x);
    // r = b - matvec(x) into V[0]
    rc = G.jop(x, G.t);
    if (rc) return rc;
    ++G.matvecs;
    k_residual<<<KB, KT, 0, v.s>>>(n, b, x, G.t, G.alpha, V0, v.red, v.scal);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "gmres residual");
    double r2;
    rc = rd(v, 1, &r2);
    if (rc) return rc;
    rnorm = std::sqrt(r2);
    if (!std::isfinite(rnorm)) {
      *nonfinite = 1;
      return SEM1D_OK;
    }
    if (rnorm <= atol) break;
    if (breakdown) break;
    if (presid <= ptol)
      ptol_max_factor = std::max(eps, 0.25 * ptol_max_factor);
    else
      ptol_max_factor = std::min(1.0, 1.5 * ptol_max_factor);
    ptol = presid * std::min(ptol_max_factor, atol / rnorm);
  }
  *info = (rnorm <= atol) ? 0 : maxiter;
  return SEM1D_OK;
}

bool check_params(const sem1d_cn_params* P, int64_t n) {
  return P && P->gmres_restart >= 1 && P->gmres_restart <= MAX_RESTART && P->gmres_max >= 1 &&
         P->newton_max >= 0 && n > 0;
}

struct Layout {          // device workspace (doubles)
  double *V, *t, *fu, *nr, *delta, *red, *scal;
};

Layout layout(double* work, int64_t n, int restart) {
  Layout L;
  L.V = work;
  L.t = L.V + (int64_t)(restart + 1) * n;
  L.fu = L.t + n;
  L.nr = L.fu + n;
  L.delta = L.nr + n;
  L.red = L.delta + n;
  L.scal = L.red + RED_DOUBLES;
  return L;
}

int gmres_impl(const OpIf& op, int transpose, const double* p, double alpha, const double* b, double* x,
               const sem1d_cn_params* P, double* work, int* flag, sem1d_cn_stats* st, void* stream) {
  if (!p || !b || !x || !work || !flag || !st)
    return fail(SEM1D_EINVAL, "gmres: bad argument (device pointers)");
  const int64_t n = op.n;
  const OpIf* plan = &op;
  if (!check_params(P, n)) return fail(SEM1D_EINVAL, "sem1d_gmres: bad parameters (1 <= restart <= 64)");
  const int restart = (int)std::min<int64_t>(P->gmres_restart, n);
  const Layout L = layout(work, n, P->gmres_restart);
  Gmres G{plan, transpose ? 1 : 0, p, alpha, Vec{static_cast<cudaStream_t>(stream), n, L.red, L.scal},
          L.V, L.t, flag};
  const int maxiter = std::max(1, (P->gmres_max + restart - 1) / restart);
  int info = 0, nonfinite = 0;
  const int rc = gmres_run(G, b, x, P->gmres_tol, restart, maxiter, &info, &nonfinite);
  st->gmres_iters += G.matvecs;
  if (transpose) st->jact_applies += G.matvecs; else st->jac_applies += G.matvecs;
  st->gmres_info = nonfinite ? -1 : info;
  st->status = nonfinite ? SEM1D_CN_INPUT_NONFINITE : (info ? SEM1D_CN_GMRES_FAILED : SEM1D_CN_OK);
  return rc;
}

int cn_step_impl(const OpIf& op, const double* u, double* v, double dt, const sem1d_cn_params* P,
                 double* work, int* flag, sem1d_cn_stats* st, void* stream) {
  if (!u || !v || u == v || !work || !flag || !st)
    return fail(SEM1D_EINVAL, "cn_step: bad argument (v must not alias u)");
  const int64_t n = op.n;
  const OpIf* plan = &op;
  if (!check_params(P, n)) return fail(SEM1D_EINVAL, "sem1d_cn_step: bad parameters (1 <= restart <= 64)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Layout L = layout(work, n, P->gmres_restart);
  Vec vv{s, n, L.red, L.scal};
  st->status = SEM1D_CN_OK;
  int rc, hflag = 0;
  cudaError_t e;
  // fu = f(u) (timeloop.py:166); the input check of apply_rhs raises NumericFailure
  if ((rc = plan->rhs(u, L.fu, flag, stream))) return rc;
  st->rhs_applies += 1;
  if ((rc = read_flag(vv, flag, &hflag))) return rc;
  if (hflag) { st->status = SEM1D_CN_INPUT_NONFINITE; return SEM1D_OK; }
  e = cudaMemcpyAsync(v, u, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "cn copy");
  double unorm;
  if ((rc = dev_norm(vv, u, &unorm))) return rc;
  const double tol = P->newton_tol * (1.0 + unorm);
  const double h = 0.5 * dt;
  int iters = 0;
  while (true) {
    if ((rc = plan->rhs(v, L.t, flag, stream))) return rc;          // f(v)
    st->rhs_applies += 1;
    int* rflag = reinterpret_cast<int*>(L.scal + 3 * MAX_RESTART + 8);
    e = cudaMemsetAsync(rflag, 0, sizeof(int), s);
    if (e != cudaSuccess) return cuda_fail(e, "cn memset");
    k_cn_residual<<<KB, KT, 0, s>>>(n, v, u, L.fu, L.t, h, L.nr, L.red, L.scal, rflag);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "cn residual");
    double r2;
    if ((rc = rd(vv, 1, &r2))) return rc;
    int rbad = 0;
    if ((rc = read_flag(vv, flag, &hflag))) return rc;
    if ((rc = read_flag(vv, rflag, &rbad))) return rc;
    if (hflag) { st->status = SEM1D_CN_INPUT_NONFINITE; break; }
    if (rbad) { st->status = SEM1D_CN_RESIDUAL_NONFINITE; break; }
    const double rn = std::sqrt(r2);
    st->last_residual = rn;
    if (rn <= tol) break;
    if (iters >= P->newton_max) { st->status = SEM1D_CN_NEWTON_STALLED; break; }
    // (I - dt/2 J(v)) delta = -r   (timeloop.py:178-181)
    const int restart = (int)std::min<int64_t>(P->gmres_restart, n);
    Gmres G{plan, 0, v, -h, vv, L.V, L.t, flag};
    int info = 0, nonfinite = 0;
    rc = gmres_run(G, L.nr, L.delta, P->gmres_tol, restart,
                   std::max(1, (P->gmres_max + restart - 1) / restart), &info, &nonfinite);
    st->gmres_iters += G.matvecs;
    st->jac_applies += G.matvecs;
    if (rc) return rc;
    if ((rc = read_flag(vv, flag, &hflag))) return rc;
    if (hflag || nonfinite) { st->status = SEM1D_CN_INPUT_NONFINITE; st->gmres_info = -1; break; }
    if (info != 0) { st->status = SEM1D_CN_GMRES_FAILED; st->gmres_info = info; break; }
    k_add<<<ew_grid(n), KT, 0, s>>>(n, v, L.delta, v);                   // v = v + delta
    ++iters;
  }
  st->newton_iters += iters;
  e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_cn_step");
}

int cn_adjoint_impl(const OpIf& op, const double* u_n, const double* u_np1, const double* lam, double* lam_out,
                    double dt, const sem1d_cn_params* P, double* work, int* flag, sem1d_cn_stats* st,
                    void* stream) {
  if (!u_n || !u_np1 || !lam || !lam_out || lam_out == lam || !work || !flag || !st)
    return fail(SEM1D_EINVAL, "cn_adjoint_step: bad argument (lam_out must not alias lam)");
  const int64_t n = op.n;
  const OpIf* plan = &op;
  if (!check_params(P, n)) return fail(SEM1D_EINVAL, "sem1d_cn_adjoint_step: bad parameters");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Layout L = layout(work, n, P->gmres_restart);
  Vec vv{s, n, L.red, L.scal};
  st->status = SEM1D_CN_OK;
  const double h = 0.5 * dt;
  const int restart = (int)std::min<int64_t>(P->gmres_restart, n);
  // (I - dt/2 J(u_{n+1}))^T mu = lam  (adjoint.py:65-68); mu in delta
  Gmres G{plan, 1, u_np1, -h, vv, L.V, L.t, flag};
  int info = 0, nonfinite = 0, rc;
  rc = gmres_run(G, lam, L.delta, P->gmres_tol, restart, std::max(1, (P->gmres_max + restart - 1) / restart),
                 &info, &nonfinite);
  st->gmres_iters += G.matvecs;
  st->jact_applies += G.matvecs;
  if (rc) return rc;
  int hflag = 0;
  if ((rc = read_flag(vv, flag, &hflag))) return rc;
  if (hflag || nonfinite) { st->status = SEM1D_CN_INPUT_NONFINITE; st->gmres_info = -1; return SEM1D_OK; }
  if (info != 0) { st->status = SEM1D_CN_GMRES_FAILED; st->gmres_info = info; return SEM1D_OK; }
  // lam_n = mu + dt/2 J^T(u_n) mu  (adjoint.py:69)
  if ((rc = plan->jact(u_n, L.delta, L.t, flag, stream))) return rc;
  st->jact_applies += 1;
  k_shift_dot2<<<KB, KT, 0, s>>>(n, L.delta, L.t, h, lam_out, nullptr, L.red, L.scal);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_cn_adjoint_step");
}

}  // namespace

extern "C" {

int64_t sem1d_cn_work_size(const sem1d_plan* plan, int restart) {
  sem1d::DeviceGuard guard_(sem1d::plan_device(plan));
  if (!plan || restart < 1 || restart > MAX_RESTART) return -1;
  const int64_t n = sem1d_plan_ndof(plan);
  return (int64_t)(restart + 1) * n + 4 * n + RED_DOUBLES + 3 * MAX_RESTART + 16 + 2;
}

int sem1d_gmres(const sem1d_plan* plan, int transpose, const double* p, double alpha, const double* b,
                double* x, const sem1d_cn_params* P, double* work, int* flag, sem1d_cn_stats* st,
                void* stream) {
  sem1d::DeviceGuard guard_(sem1d::plan_device(plan));
  if (!plan || sem1d::plan_batch(plan) != 1) return fail(SEM1D_EINVAL, "sem1d_gmres: needs a batch-1 plan");
  return gmres_impl(OpIf{plan, 0, nullptr, sem1d_plan_ndof(plan)}, transpose, p, alpha, b, x, P, work, flag,
                    st, stream);
}

int sem1d_cn_step(const sem1d_plan* plan, const double* u, double* v, double dt, const sem1d_cn_params* P,
                  double* work, int* flag, sem1d_cn_stats* st, void* stream) {
  sem1d::DeviceGuard guard_(sem1d::plan_device(plan));
  if (!plan || sem1d::plan_batch(plan) != 1) return fail(SEM1D_EINVAL, "sem1d_cn_step: needs a batch-1 plan");
  return cn_step_impl(OpIf{plan, 0, nullptr, sem1d_plan_ndof(plan)}, u, v, dt, P, work, flag, st, stream);
}

int sem1d_cn_adjoint_step(const sem1d_plan* plan, const double* u_n, const double* u_np1, const double* lam,
                          double* lam_out, double dt, const sem1d_cn_params* P, double* work, int* flag,
                          sem1d_cn_stats* st, void* stream) {
  sem1d::DeviceGuard guard_(sem1d::plan_device(plan));
  if (!plan || sem1d::plan_batch(plan) != 1)
    return fail(SEM1D_EINVAL, "sem1d_cn_adjoint_step: needs a batch-1 plan");
  return cn_adjoint_impl(OpIf{plan, 0, nullptr, sem1d_plan_ndof(plan)}, u_n, u_np1, lam, lam_out, dt, P, work,
                         flag, st, stream);
}

// 3D: `work` = the Krylov workspace for n = ndof, then the element-block scratch
static int64_t krylov_doubles(int64_t n, int restart) {
  return (int64_t)(restart + 1) * n + 4 * n + RED_DOUBLES + 3 * MAX_RESTART + 16 + 2;
}

int64_t sem3d_cn_work_size(const sem3d_plan* plan, int restart) {
  sem1d::DeviceGuard guard_(sem1d::plan3_device(plan));
  if (!plan || restart < 1 || restart > MAX_RESTART) return -1;
  return krylov_doubles(sem3d_plan_ndof(plan), restart) + sem3d_work_size(plan);
}

static OpIf op3(const sem3d_plan* plan, double* work, int restart) {
  const int64_t n = sem3d_plan_ndof(plan);
  return OpIf{plan, 1, work + krylov_doubles(n, restart), n};
}

int sem3d_gmres(const sem3d_plan* plan, int transpose, const double* p, double alpha, const double* b, double* x,
                const sem1d_cn_params* P, double* work, int* flag, sem1d_cn_stats* st, void* stream) {
  sem1d::DeviceGuard guard_(sem1d::plan3_device(plan));
  if (!plan || !P || !work) return fail(SEM1D_EINVAL, "sem3d_gmres: bad argument");
  return gmres_impl(op3(plan, work, P->gmres_restart), transpose, p, alpha, b, x, P, work, flag, st, stream);
}

int sem3d_cn_step(const sem3d_plan* plan, const double* u, double* v, double dt, const sem1d_cn_params* P,
                  double* work, int* flag, sem1d_cn_stats* st, void* stream) {
  sem1d::DeviceGuard guard_(sem1d::plan3_device(plan));
  if (!plan || !P || !work) return fail(SEM1D_EINVAL, "sem3d_cn_step: bad argument");
  return cn_step_impl(op3(plan, work, P->gmres_restart), u, v, dt, P, work, flag, st, stream);
}

int sem3d_cn_adjoint_step(const sem3d_plan* plan, const double* u_n, const double* u_np1, const double* lam,
                          double* lam_out, double dt, const sem1d_cn_params* P, double* work, int* flag,
                          sem1d_cn_stats* st, void* stream) {
  sem1d::DeviceGuard guard_(sem1d::plan3_device(plan));
  if (!plan || !P || !work) return fail(SEM1D_EINVAL, "sem3d_cn_adjoint_step: bad argument");
  return cn_adjoint_impl(op3(plan, work, P->gmres_restart), u_n, u_np1, lam, lam_out, dt, P, work, flag, st,
                         stream);
}

int sem1d_vec_dot(int64_t n, const double* x, const double* y, double* work, double* out, void* stream) {
  if (n < 1 || !x || !y || !work || !out) return fail(SEM1D_EINVAL, "sem1d_vec_dot: bad argument");
  k_dot<<<KB, KT, 0, static_cast<cudaStream_t>(stream)>>>(n, x, y, work, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_vec_dot");
}

int sem1d_rk_error_norm(int64_t n, const double* u_new, const double* u, const double* k2, double dt,
                        double tol_a, double tol_r, int max_form, double* work, double* out, void* stream) {
  if (n < 1 || !u_new || !u || !k2 || !work || !out) return fail(SEM1D_EINVAL, "sem1d_rk_error_norm: bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (max_form)
    k_rk_error<true><<<KB, KT, 0, s>>>(n, u_new, u, k2, dt, tol_a, tol_r, work, out);
  else
    k_rk_error<false><<<KB, KT, 0, s>>>(n, u_new, u, k2, dt, tol_a, tol_r, work, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_rk_error_norm");
}

int64_t sem1d_reduce_work_size(void) { return RED_DOUBLES; }

int sem1d_vec_rk_combine(int64_t n, const double* base, double dt, int nterms, const double* const* terms,
                         const double* coef, double* Y, int check, int* flag, void* stream) {
  Terms T;
  if (n < 1 || !base || !Y || nterms < 1 || !terms || !coef || !make_terms(nterms, terms, coef, T) ||
      (check && !flag))
    return fail(SEM1D_EINVAL, "sem1d_vec_rk_combine: bad argument");
  k_rk_combine<<<ew_grid(n), KT, 0, static_cast<cudaStream_t>(stream)>>>(n, base, dt, T, Y, check, flag);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_vec_rk_combine");
}

int sem1d_vec_adj_combine(int64_t n, const double* lam, double b, int nl, const double* const* l_terms,
                          const double* a, double* z, void* stream) {
  Terms T;
  if (n < 1 || !lam || !z || (nl > 0 && (!l_terms || !a)) || !make_terms(nl, l_terms, a, T))
    return fail(SEM1D_EINVAL, "sem1d_vec_adj_combine: bad argument");
  k_adj_combine<<<ew_grid(n), KT, 0, static_cast<cudaStream_t>(stream)>>>(n, lam, b, T, z);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_vec_adj_combine");
}

int sem1d_vec_accumulate(int64_t n, const double* x, int nt, const double* const* terms, double* out,
                         void* stream) {
  Terms T;
  if (n < 1 || !x || !out || (nt > 0 && !terms) || !make_terms(nt, terms, nullptr, T))
    return fail(SEM1D_EINVAL, "sem1d_vec_accumulate: bad argument");
  k_accumulate<<<ew_grid(n), KT, 0, static_cast<cudaStream_t>(stream)>>>(n, x, T, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_vec_accumulate");
}

int sem1d_vec_scale(int64_t n, const double* x, double s, double* y, void* stream) {
  if (n < 1 || !x || !y) return fail(SEM1D_EINVAL, "sem1d_vec_scale: bad argument");
  k_scale<<<ew_grid(n), KT, 0, static_cast<cudaStream_t>(stream)>>>(n, x, s, y);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_vec_scale");
}

}  // extern "C"
