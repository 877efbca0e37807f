// sem1d_capi.cu -- the extern "C" boundary (include/sem1d.h): plans, argument
// validation, dispatch by degree, and the small non-templated kernels
// (terminal condition, scatter, gather).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "sem1d_launch.cuh"

using namespace sem1d;

namespace sem1d {
#define SEM_DECL(NN) \
  extern template cudaError_t launch_apply<NN>(const PlanView&, int, const Args&, cudaStream_t); \
  extern template cudaError_t launch_ens_forward<NN>(const PlanView&, const EnsArgs&, cudaStream_t); \
  extern template cudaError_t launch_ens_adjoint<NN>(const PlanView&, const EnsAdjArgs&, cudaStream_t); \
  extern template cudaError_t launch_tile_step<NN>(const PlanView&, int, TileStepArgs, cudaStream_t);
SEM_DECL(1) SEM_DECL(2) SEM_DECL(3) SEM_DECL(4) SEM_DECL(5) SEM_DECL(6) SEM_DECL(7) SEM_DECL(8)
SEM_DECL(9) SEM_DECL(10) SEM_DECL(11) SEM_DECL(12) SEM_DECL(13) SEM_DECL(14) SEM_DECL(15)
SEM_DECL(16) SEM_DECL(17) SEM_DECL(18) SEM_DECL(19) SEM_DECL(20) SEM_DECL(21) SEM_DECL(22)
SEM_DECL(23) SEM_DECL(24) SEM_DECL(25) SEM_DECL(26) SEM_DECL(27) SEM_DECL(28) SEM_DECL(29)
SEM_DECL(30) SEM_DECL(31) SEM_DECL(32)
#undef SEM_DECL
}  // namespace sem1d

namespace sem1d {
static int g_path_override = 0;
int sem1d_path_override() { return g_path_override; }
static int g_tile_variant = 0;
int sem1d_tile_variant() { return g_tile_variant; }
}  // namespace sem1d

struct sem1d_plan {
  int N;
  int64_t E, ndof, batch;
  int periodic;
  double nu;
  std::vector<double> packed;  // Consts<N> image
  std::vector<double> mass, minv;
  int adv = 0;                 // 0 Burgers, 1 linear (constant speed), 2 none (ops.py:147-212)
  double speed = 0.0;
  double* dconst = nullptr;    // advection kinds: device K[n*n], Dw[n*n], minv[N+2]
  // tensor-core apply kernels (N+1 % 8 == 0): the permuted B-fragment table
  // [K, Dw, Dw^T][n/8][n/4][32 lanes] in device memory, built on first use, so a kernel
  // prologue is a coalesced copy instead of lane-divergent kernel-parameter reads
  mutable double* dfrag = nullptr;
  mutable std::once_flag frag_once;
  mutable cudaError_t frag_err = cudaSuccess;
  int device = 0;              // the device current at sem1d_plan_create; every call runs there
};

namespace {
thread_local std::string g_err;
}  // namespace

namespace sem1d {
// shared with the other translation units of the library (sem1d_krylov.cu)
int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
}  // namespace sem1d

namespace {

int fail(int code, const std::string& msg) { return sem1d::set_error(code, msg); }
}  // namespace

namespace sem1d {
int64_t plan_batch(const sem1d_plan* p) { return p ? p->batch : 0; }
int plan_device(const sem1d_plan* p) { return p ? p->device : -1; }
}  // namespace sem1d

namespace {

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SEM1D_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// bfrag_eo_value<N> for the two degrees that use it (N + 1 a multiple of 16, N <= 32)
double eo_value(int N, const double* K, const double* Dw, const double* minv, double nu, int sec, int nt,
                int kc, int l) {
  return N == 15 ? sem1d::bfrag_eo_value<15>(K, Dw, minv, nu, sec, nt, kc, l)
                 : sem1d::bfrag_eo_value<31>(K, Dw, minv, nu, sec, nt, kc, l);
}

// Host image of bfrag_perm (sem1d_device.cuh) for every (mat, nt, kc, lane): a permutation of
// K / Dw entries, so the device table is bit-identical to the in-kernel construction.
cudaError_t ensure_frag(const sem1d_plan* p) {
  const int n = p->N + 1;
  if (n % 8 != 0) return cudaSuccess;
  std::call_once(p->frag_once, [p, n]() {
    const int NT = n / 8, KC = n / 4;
    const double* K = p->packed.data();
    const double* Dw = K + n * n;
    // [K, Dw, Dw^T] as bfrag_perm, then [K, Dw] with the output row's -nu M^-1_i / M^-1_i folded
    // in (bfrag_pre; periodic rings, interface rows take pattern entry 0)
    const double* minv = p->minv.data();
    std::vector<double> h((size_t)5 * NT * KC * 32);
    for (int mat = 0; mat < 5; ++mat)
      for (int nt = 0; nt < NT; ++nt)
        for (int kc = 0; kc < KC; ++kc)
          for (int l = 0; l < 32; ++l) {
            const int c = 8 * nt + (l >> 2);
            const int i = 4 * (2 * (c >> 3) + (c & 1)) + ((c >> 1) & 3);
            const int j = 4 * kc + (l & 3);
            const int m = mat < 3 ? mat : mat - 3;
            double b = m == 0 ? K[i * n + j] : (m == 1 ? Dw[i * n + j] : Dw[j * n + i]);
            if (mat >= 3) {
              const double mi = minv[(i == 0 || i == p->N) ? 0 : i];
              volatile double sc = (mat == 3) ? (-p->nu) * mi : mi;   // one rounding, as on the device
              b = b * sc;
            }
            h[(((size_t)mat * NT + nt) * KC + kc) * 32 + l] = b;
          }
    // n % 16 == 0: the reflection-split (WS_EO) sections follow, [Ke, Ko, De, Do, Te, To], the
    // prescaled [Ke', Ko', De', Do'] and J^T's [K''e, K''o, De', Do', T''e, T''o], each
    // [n/16][n/8][32] (bfrag_eo_value, sem1d_device.cuh)
    if (n % 16 == 0) {
      const int NT2 = NT / 2, KC2 = KC / 2;
      const size_t base = h.size();
      h.resize(base + (size_t)16 * NT2 * KC2 * 32);
      for (int sec = 0; sec < 16; ++sec)
        for (int nt = 0; nt < NT2; ++nt)
          for (int kc = 0; kc < KC2; ++kc)
            for (int l = 0; l < 32; ++l)
              h[base + (((size_t)sec * NT2 + nt) * KC2 + kc) * 32 + l] =
                  eo_value(p->N, K, Dw, minv, p->nu, sec, nt, kc, l);
    }
    double* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(double) * h.size());
    if (e == cudaSuccess) e = cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess && d) {
      cudaFree(d);
      d = nullptr;
    }
    p->frag_err = e;
    p->dfrag = d;
  });
  return p->frag_err;
}

PlanView view(const sem1d_plan* p) {
  PlanView v;
  v.consts = p->packed.data();
  v.frag = p->dfrag;
  v.geo.E = p->E;
  v.geo.ndof = p->ndof;
  v.geo.periodic = p->periodic;
  v.batch = p->batch;
  return v;
}

cudaError_t dispatch(const sem1d_plan* p, int kind, const Args& a, cudaStream_t s) {
  cudaError_t fe = ensure_frag(p);
  if (fe != cudaSuccess) return fe;
  const PlanView v = view(p);
  switch (p->N) {
#define SEM_CASE(NN) \
  case NN: return launch_apply<NN>(v, kind, a, s);
    SEM_CASE(1) SEM_CASE(2) SEM_CASE(3) SEM_CASE(4) SEM_CASE(5) SEM_CASE(6) SEM_CASE(7)
    SEM_CASE(8) SEM_CASE(9) SEM_CASE(10) SEM_CASE(11) SEM_CASE(12) SEM_CASE(13) SEM_CASE(14)
    SEM_CASE(15) SEM_CASE(16) SEM_CASE(17) SEM_CASE(18) SEM_CASE(19) SEM_CASE(20) SEM_CASE(21)
    SEM_CASE(22) SEM_CASE(23) SEM_CASE(24) SEM_CASE(25) SEM_CASE(26) SEM_CASE(27) SEM_CASE(28)
    SEM_CASE(29) SEM_CASE(30) SEM_CASE(31) SEM_CASE(32)
#undef SEM_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t dispatch_ens_forward(const sem1d_plan* p, const EnsArgs& a, cudaStream_t s) {
  const PlanView v = view(p);
  switch (p->N) {
#define SEM_CASE(NN) \
  case NN: return launch_ens_forward<NN>(v, a, s);
    SEM_CASE(1) SEM_CASE(2) SEM_CASE(3) SEM_CASE(4) SEM_CASE(5) SEM_CASE(6) SEM_CASE(7)
    SEM_CASE(8) SEM_CASE(9) SEM_CASE(10) SEM_CASE(11) SEM_CASE(12) SEM_CASE(13) SEM_CASE(14)
    SEM_CASE(15) SEM_CASE(16) SEM_CASE(17) SEM_CASE(18) SEM_CASE(19) SEM_CASE(20) SEM_CASE(21)
    SEM_CASE(22) SEM_CASE(23) SEM_CASE(24) SEM_CASE(25) SEM_CASE(26) SEM_CASE(27) SEM_CASE(28)
    SEM_CASE(29) SEM_CASE(30) SEM_CASE(31) SEM_CASE(32)
#undef SEM_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t dispatch_ens_adjoint(const sem1d_plan* p, const EnsAdjArgs& a, cudaStream_t s) {
  const PlanView v = view(p);
  switch (p->N) {
#define SEM_CASE(NN) \
  case NN: return launch_ens_adjoint<NN>(v, a, s);
    SEM_CASE(1) SEM_CASE(2) SEM_CASE(3) SEM_CASE(4) SEM_CASE(5) SEM_CASE(6) SEM_CASE(7)
    SEM_CASE(8) SEM_CASE(9) SEM_CASE(10) SEM_CASE(11) SEM_CASE(12) SEM_CASE(13) SEM_CASE(14)
    SEM_CASE(15) SEM_CASE(16) SEM_CASE(17) SEM_CASE(18) SEM_CASE(19) SEM_CASE(20) SEM_CASE(21)
    SEM_CASE(22) SEM_CASE(23) SEM_CASE(24) SEM_CASE(25) SEM_CASE(26) SEM_CASE(27) SEM_CASE(28)
    SEM_CASE(29) SEM_CASE(30) SEM_CASE(31) SEM_CASE(32)
#undef SEM_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t dispatch_tile(const sem1d_plan* p, int kind, const TileStepArgs& a, cudaStream_t s) {
  const PlanView v = view(p);
  switch (p->N) {
#define SEM_CASE(NN) \
  case NN: return launch_tile_step<NN>(v, kind, a, s);
    SEM_CASE(1) SEM_CASE(2) SEM_CASE(3) SEM_CASE(4) SEM_CASE(5) SEM_CASE(6) SEM_CASE(7)
    SEM_CASE(8) SEM_CASE(9) SEM_CASE(10) SEM_CASE(11) SEM_CASE(12) SEM_CASE(13) SEM_CASE(14)
    SEM_CASE(15) SEM_CASE(16) SEM_CASE(17) SEM_CASE(18) SEM_CASE(19) SEM_CASE(20) SEM_CASE(21)
    SEM_CASE(22) SEM_CASE(23) SEM_CASE(24) SEM_CASE(25) SEM_CASE(26) SEM_CASE(27) SEM_CASE(28)
    SEM_CASE(29) SEM_CASE(30) SEM_CASE(31) SEM_CASE(32)
#undef SEM_CASE
    default: return cudaErrorInvalidValue;
  }
}

// Butcher tableaux of the schemes on the path (timeloop.py:24-27; RK4 classic)
bool make_tableau(int scheme, Tableau& t) {
  std::memset(&t, 0, sizeof(t));
  if (scheme == 0) {            // euler
    t.s = 1; t.b[0] = 1.0;
  } else if (scheme == 1) {     // rk3 (Kutta-3)
    t.s = 3;
    t.a[1][0] = 0.5;
    t.a[2][0] = -1.0; t.a[2][1] = 2.0;
    t.b[0] = 1.0 / 6.0; t.b[1] = 2.0 / 3.0; t.b[2] = 1.0 / 6.0;
    t.keep[0] = 1;
  } else if (scheme == 2) {     // rk4
    t.s = 4;
    t.a[1][0] = 0.5; t.a[2][1] = 0.5; t.a[3][2] = 1.0;
    t.b[0] = 1.0 / 6.0; t.b[1] = 1.0 / 3.0; t.b[2] = 1.0 / 3.0; t.b[3] = 1.0 / 6.0;
  } else {
    return false;
  }
  for (int i = 1; i < t.s; ++i)
    for (int j = 0; j < i; ++j) t.nterm[i] += (t.a[i][j] != 0.0);
  return true;
}

bool valid_plan(const sem1d_plan* p) { return p != nullptr && p->N >= 1 && p->N <= SEM1D_MAX_DEGREE; }
// fused stage / step / ensemble kernels implement Burgers advection only; plans with another
// advection kind compose their stages from F / J^T applies and the vector kernels
bool valid_burgers(const sem1d_plan* p) { return valid_plan(p) && p->adv == 0; }

Args blank_args() {
  Args a;
  std::memset(&a, 0, sizeof(a));
  return a;
}

int fill_combo(Combo& c, int n, const double* const* ptrs, const double* coef, bool need_coef,
               const char* what) {
  if (n < 0 || n > SEM1D_MAX_TERMS) return fail(SEM1D_EINVAL, std::string(what) + ": bad term count");
  if (n > 0 && ptrs == nullptr) return fail(SEM1D_EINVAL, std::string(what) + ": null term list");
  if (n > 0 && need_coef && coef == nullptr) return fail(SEM1D_EINVAL, std::string(what) + ": null coefficients");
  c.n = n;
  for (int j = 0; j < n; ++j) {
    c.ptr[j] = ptrs[j];
    c.coef[j] = need_coef ? coef[j] : 1.0;
  }
  return SEM1D_OK;
}

// ---------------------------------------------------------------- small kernels

struct Pattern {
  double mass[SEM1D_MAX_DEGREE + 2];
  int N;
};

__device__ __forceinline__ double pat_at(const Pattern& P, int64_t g, const Geo& G) {
  if (!G.periodic) {
    if (g == 0) return P.mass[P.N];
    if (g == G.E * P.N) return P.mass[P.N + 1];
  }
  return P.mass[g % P.N];
}

constexpr int RED_TPB = 256;
constexpr int RED_ITEMS = 16;

__device__ double block_sum_fixed(double v, double* sh) {
  // fixed-shape tree: deterministic for a given blockDim
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = RED_TPB / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

// d = uN - ud; md = M d; lam = mask(2 md); partial sums of d*md   (adjoint.py:39-47)
__global__ void __launch_bounds__(RED_TPB)
    terminal_kernel(const Pattern P, const Geo G, const double* __restrict__ uN,
                    const double* __restrict__ ud, double* __restrict__ lam,
                    double* __restrict__ work, int nblk) {
  __shared__ double sh[RED_TPB];
  const int64_t bofs = (int64_t)blockIdx.y * G.ndof;
  const int64_t start = (int64_t)blockIdx.x * RED_TPB * RED_ITEMS;
  double acc = 0.0;
  for (int it = 0; it < RED_ITEMS; ++it) {
    const int64_t g = start + (int64_t)it * RED_TPB + threadIdx.x;
    if (g < G.ndof) {
      const double d = __dsub_rn(uN[bofs + g], ud[bofs + g]);
      const double md = __dmul_rn(pat_at(P, g, G), d);
      double l = __dmul_rn(2.0, md);
      if (!G.periodic && (g == 0 || g == G.E * P.N)) l = __dmul_rn(l, 0.0);
      lam[bofs + g] = l;
      acc = __dadd_rn(acc, __dmul_rn(d, md));
    }
  }
  const double s = block_sum_fixed(acc, sh);
  if (threadIdx.x == 0) work[(int64_t)blockIdx.y * nblk + blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_TPB)
    terminal_finish(const double* __restrict__ work, int nblk, double* __restrict__ J_out) {
  __shared__ double sh[RED_TPB];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nblk; i += RED_TPB) acc = __dadd_rn(acc, work[(int64_t)blockIdx.x * nblk + i]);
  const double s = block_sum_fixed(acc, sh);
  if (threadIdx.x == 0) J_out[blockIdx.x] = s;
}

// local[b, e, i] = u[b, (e*N + i) mod ndof]                      (grid.py:165-169)
__global__ void scatter_kernel(const Geo G, int N, const double* __restrict__ u,
                               double* __restrict__ local) {
  const int n = N + 1;
  const int64_t total = G.E * n;
  const int64_t bofs_u = (int64_t)blockIdx.y * G.ndof, bofs_l = (int64_t)blockIdx.y * total;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = k / n;
    const int i = (int)(k - e * n);
    int64_t g = e * N + i;
    if (g >= G.ndof) g -= G.ndof;
    local[bofs_l + k] = u[bofs_u + g];
  }
}

// out[g] = (0 + first contribution) + second contribution         (grid.py:157-161)
__global__ void gather_kernel(const Geo G, int N, const double* __restrict__ local,
                              double* __restrict__ out) {
  const int n = N + 1;
  const int64_t bofs_o = (int64_t)blockIdx.y * G.ndof, bofs_l = (int64_t)blockIdx.y * G.E * n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G.ndof;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = g / N;
    const int i = (int)(g - e * N);
    double v;
    if (i != 0) {
      v = __dadd_rn(0.0, local[bofs_l + e * n + i]);
    } else if (G.periodic) {
      // bincount visits table positions in ravel order
      const int64_t eprev = (e == 0) ? G.E - 1 : e - 1;
      const double a = local[bofs_l + e * n];
      const double b = local[bofs_l + eprev * n + N];
      v = (e == 0) ? __dadd_rn(__dadd_rn(0.0, a), b) : __dadd_rn(__dadd_rn(0.0, b), a);
    } else {
      if (e == 0) {
        v = __dadd_rn(0.0, local[bofs_l]);
      } else if (e == G.E) {
        v = __dadd_rn(0.0, local[bofs_l + (e - 1) * n + N]);
      } else {
        v = __dadd_rn(__dadd_rn(0.0, local[bofs_l + (e - 1) * n + N]), local[bofs_l + e * n]);
      }
    }
    out[bofs_o + g] = v;
  }
}

unsigned grid_for(int64_t work, int tpb) {
  int64_t b = (work + tpb - 1) / tpb;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

extern "C" {

int sem1d_version(void) { return 1; }

int sem1d_set_kernel_path(int path) {
  if (path < 0 || path > 3) return fail(SEM1D_EINVAL, "sem1d_set_kernel_path: path must be 0..3");
  sem1d::g_path_override = path;
  return SEM1D_OK;
}
const char* sem1d_last_error(void) { return g_err.c_str(); }

int sem1d_set_tile_variant(int variant) {
  if (variant < 0 || variant > 3)
    return fail(SEM1D_EINVAL, "sem1d_set_tile_variant: 0 (auto), 1 (shared-memory tiles), 2 (N = 7 forward at "
                              "128-element tiles), 3 (N = 7 forward at 192-element tiles)");
  g_tile_variant = variant;
  return SEM1D_OK;
}
int sem1d_max_degree(void) { return SEM1D_MAX_DEGREE; }

// ---- LINEAR / NONE advection (ops.py:147-212 branches) --------------------------------
// One thread per (problem, global node): the node's (at most two) element rows
//   row_i(x) = (K x)_i * (-nu) - a (Dw x)_i          (F, J: x = u resp. v)
//   row_i(x) = (K x)_i * (-nu) - a (Dw^T x)_i        (J^T:  x = mask(M^-1 z))
// summed in the reference gather order ((element k-1, local N) + (element k, local 0)),
// then M^-1 and the Dirichlet mask (F, J) or the mask (J^T).  For these operators J(u)v
// does not depend on u, which is still checked for NaN/Inf like ops.py:216-223 does.
namespace {
__device__ __forceinline__ bool nonfin_adv(double x) {
  return ((unsigned)__double2hiint(x) & 0x7ff00000u) == 0x7ff00000u;
}

__device__ __forceinline__ double adv_minv(const double* mi, int N, int64_t g, int64_t ndof, int periodic) {
  if (!periodic && g == 0) return mi[N];
  if (!periodic && g == ndof - 1) return mi[N + 1];
  return mi[g % N];
}

__global__ void adv_apply_kernel(int N, int64_t E, int64_t ndof, int periodic, double mnu, double a, int mode,
                                 int op, const double* __restrict__ cst, const double* __restrict__ u,
                                 const double* __restrict__ w, double* __restrict__ out, int* flag) {
  extern __shared__ double sc[];
  const int n = N + 1;
  for (int k = threadIdx.x; k < 2 * n * n + N + 2; k += blockDim.x) sc[k] = cst[k];
  __syncthreads();
  const double* K = sc;
  const double* Dw = sc + n * n;
  const double* mi = sc + 2 * n * n;
  const int64_t b = blockIdx.y;
  const double* ub = u + b * ndof;
  const double* xb = (op == 0 ? u : w) + b * ndof;
  unsigned bad_u = 0, bad_w = 0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ndof; g += (int64_t)gridDim.x * blockDim.x) {
    bad_u |= nonfin_adv(ub[g]);
    if (op != 0) bad_w |= nonfin_adv(w[b * ndof + g]);
    const int64_t k = g / N;
    const int r = (int)(g - k * N);
    // contributing (element, local row) pairs in gather order
    int64_t ee[2];
    int rr[2], cnt = 0;
    if (r != 0) {
      ee[0] = k; rr[0] = r; cnt = 1;
    } else if (periodic) {
      if (k == 0) { ee[0] = 0; rr[0] = 0; ee[1] = E - 1; rr[1] = N; }
      else { ee[0] = k - 1; rr[0] = N; ee[1] = k; rr[1] = 0; }
      cnt = 2;
    } else {
      if (k == 0) { ee[0] = 0; rr[0] = 0; cnt = 1; }
      else if (k == E) { ee[0] = E - 1; rr[0] = N; cnt = 1; }
      else { ee[0] = k - 1; rr[0] = N; ee[1] = k; rr[1] = 0; cnt = 2; }
    }
    double acc = 0.0;
    for (int c = 0; c < cnt; ++c) {
      const int64_t base = ee[c] * N;
      const int i = rr[c];
      double kx = 0.0, dx = 0.0;
      for (int j = 0; j < n; ++j) {
        int64_t gj = base + j;
        if (periodic && gj >= ndof) gj -= ndof;
        double x = xb[gj];
        if (op == 2) {                           // J^T input: mask(z M^-1)
          x = __dmul_rn(x, adv_minv(mi, N, gj, ndof, periodic));
          if (!periodic && (gj == 0 || gj == ndof - 1)) x = __dmul_rn(x, 0.0);
        }
        kx = fma(K[i * n + j], x, kx);
        if (mode == 1) dx = fma(op == 2 ? Dw[j * n + i] : Dw[i * n + j], x, dx);
      }
      double row = __dmul_rn(kx, mnu);
      if (mode == 1) row = __dsub_rn(row, __dmul_rn(a, dx));
      acc = (c == 0) ? row : __dadd_rn(acc, row);
    }
    if (op != 2) acc = __dmul_rn(acc, adv_minv(mi, N, g, ndof, periodic));
    if (!periodic && (g == 0 || g == ndof - 1)) acc = __dmul_rn(acc, 0.0);
    out[b * ndof + g] = acc;
  }
  if (bad_u || bad_w)
    atomicOr(flag, (bad_u ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad_w ? SEM1D_FLAG_INPUT2_NONFINITE : 0));
}

int run_adv(const sem1d_plan* p, int op, const double* u, const double* w, double* out, int* flag, void* stream,
            const char* name) {
  const int n = p->N + 1;
  const size_t smem = sizeof(double) * (2 * n * n + p->N + 2);
  const int64_t blocks = std::min<int64_t>((p->ndof + 255) / 256, 148 * 8);
  dim3 grid((unsigned)std::max<int64_t>(1, blocks), (unsigned)p->batch);
  adv_apply_kernel<<<grid, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      p->N, p->E, p->ndof, p->periodic, -p->nu, p->speed, p->adv, op, p->dconst, u, w, out, flag);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, name);
}
}  // namespace

int sem1d_plan_set_advection(sem1d_plan* plan, int mode, double speed) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!plan || mode < 0 || mode > 2 || !std::isfinite(speed))
    return fail(SEM1D_EINVAL, "sem1d_plan_set_advection: bad argument (mode 0 burgers, 1 linear, 2 none)");
  plan->adv = mode;
  plan->speed = (mode == 1) ? speed : 0.0;
  if (mode != 0 && !plan->dconst) {
    const int n = plan->N + 1;
    std::vector<double> h(2 * n * n + plan->N + 2);
    std::memcpy(h.data(), plan->packed.data(), sizeof(double) * 2 * n * n);     // K, Dw
    std::memcpy(h.data() + 2 * n * n, plan->minv.data(), sizeof(double) * (plan->N + 2));
    cudaError_t e = cudaMalloc(&plan->dconst, sizeof(double) * h.size());
    if (e == cudaSuccess) e = cudaMemcpy(plan->dconst, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "sem1d_plan_set_advection");
  }
  return SEM1D_OK;
}

int sem1d_plan_create(int64_t n_elements, int degree, int periodic, double nu, const double* K,
                      const double* Dw, const double* mass_pattern, const double* minv_pattern,
                      int64_t batch, sem1d_plan** out) {
  if (out == nullptr) return fail(SEM1D_EINVAL, "plan_create: null output");
  *out = nullptr;
  if (degree < 1 || degree > SEM1D_MAX_DEGREE)
    return fail(SEM1D_EINVAL, "plan_create: degree must be in [1, " +
                                  std::to_string(SEM1D_MAX_DEGREE) + "]");
  if (n_elements < 1) return fail(SEM1D_EINVAL, "plan_create: need at least one element");
  if (periodic && n_elements * degree < 2)
    return fail(SEM1D_EINVAL, "plan_create: periodic axis needs E*N >= 2");
  if (batch < 1 || batch > 65535) return fail(SEM1D_EINVAL, "plan_create: batch must be in [1, 65535]");
  if (!K || !Dw || !mass_pattern || !minv_pattern) return fail(SEM1D_EINVAL, "plan_create: null constant");
  if (!std::isfinite(nu) || nu < 0.0) return fail(SEM1D_EINVAL, "plan_create: viscosity must be >= 0");
  const int n = degree + 1;
  const int64_t nb = (n_elements + 127) / 128;
  if (nb > 2147483647LL) return fail(SEM1D_EINVAL, "plan_create: too many elements");
  sem1d_plan* p = new (std::nothrow) sem1d_plan();
  if (!p) return fail(SEM1D_EINVAL, "plan_create: out of host memory");
  p->N = degree;
  p->E = n_elements;
  p->periodic = periodic ? 1 : 0;
  p->ndof = n_elements * degree + (periodic ? 0 : 1);
  p->batch = batch;
  p->nu = nu;
  if (cudaGetDevice(&p->device) != cudaSuccess) p->device = 0;
  p->mass.assign(mass_pattern, mass_pattern + degree + 2);
  p->minv.assign(minv_pattern, minv_pattern + degree + 2);
  // Consts<N> image: K[n*n], Dw[n*n], minv[N+2], mass[N+2], nu
  p->packed.reserve(2 * n * n + 2 * (degree + 2) + 1);
  p->packed.insert(p->packed.end(), K, K + n * n);
  p->packed.insert(p->packed.end(), Dw, Dw + n * n);
  p->packed.insert(p->packed.end(), minv_pattern, minv_pattern + degree + 2);
  p->packed.insert(p->packed.end(), mass_pattern, mass_pattern + degree + 2);
  p->packed.push_back(nu);
  *out = p;
  return SEM1D_OK;
}

int sem1d_plan_destroy(sem1d_plan* plan) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (plan && plan->dconst) cudaFree(plan->dconst);
  if (plan && plan->dfrag) cudaFree(plan->dfrag);
  delete plan;
  return SEM1D_OK;
}

int64_t sem1d_plan_ndof(const sem1d_plan* plan) { return plan ? plan->ndof : -1; }

static int run_apply(const sem1d_plan* p, int kind, const Args& a, void* stream, const char* name) {
  cudaError_t e = dispatch(p, kind, a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, name);
  return SEM1D_OK;
}

int sem1d_rhs(const sem1d_plan* plan, const double* u, double* f, int* flag, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_plan(plan) || !u || !f || !flag) return fail(SEM1D_EINVAL, "sem1d_rhs: bad argument");
  if (plan->adv) return run_adv(plan, 0, u, nullptr, f, flag, stream, "sem1d_rhs");
  Args a = blank_args();
  a.u = u; a.out = f; a.flag = flag;
  return run_apply(plan, 0, a, stream, "sem1d_rhs");
}

int sem1d_jac(const sem1d_plan* plan, const double* u, const double* v, double* out, int* flag,
              void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_plan(plan) || !u || !v || !out || !flag) return fail(SEM1D_EINVAL, "sem1d_jac: bad argument");
  if (plan->adv) return run_adv(plan, 1, u, v, out, flag, stream, "sem1d_jac");
  Args a = blank_args();
  a.u = u; a.w = v; a.out = out; a.flag = flag;
  return run_apply(plan, 1, a, stream, "sem1d_jac");
}

int sem1d_jact(const sem1d_plan* plan, const double* u, const double* z, double* out, int* flag,
               void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_plan(plan) || !u || !z || !out || !flag) return fail(SEM1D_EINVAL, "sem1d_jact: bad argument");
  if (plan->adv) return run_adv(plan, 2, u, z, out, flag, stream, "sem1d_jact");
  Args a = blank_args();
  a.u = u; a.w = z; a.out = out; a.flag = flag;
  return run_apply(plan, 2, a, stream, "sem1d_jact");
}

int sem1d_rk_stage(const sem1d_plan* plan, const double* U_in, double* k_out, const double* base,
                   int nterms, const double* const* terms, const double* coef, double dt, double* Y,
                   int check_step, int* flag, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !U_in || !base || !Y || !flag || nterms < 1)
    return fail(SEM1D_EINVAL, "sem1d_rk_stage: bad argument");
  Args a = blank_args();
  a.u = U_in; a.out = k_out; a.flag = flag; a.base = base; a.dt = dt; a.Y = Y;
  a.check = check_step ? 1 : 0;
  int rc = fill_combo(a.epi, nterms, terms, coef, true, "sem1d_rk_stage");
  if (rc) return rc;
  return run_apply(plan, 3, a, stream, "sem1d_rk_stage");
}

int sem1d_adj_stage(const sem1d_plan* plan, const double* U, const double* lam, double b, int nl,
                    const double* const* l_terms, const double* acoef, double dt, double* l_out,
                    int nacc, const double* const* acc_terms, double* lam_out, int* flag,
                    void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !U || !lam || !flag) return fail(SEM1D_EINVAL, "sem1d_adj_stage: bad argument");
  Args a = blank_args();
  a.u = U; a.w = lam; a.b = b; a.out = l_out; a.flag = flag; a.base = lam; a.dt = dt; a.Y = lam_out;
  int rc = fill_combo(a.zin, nl, l_terms, acoef, true, "sem1d_adj_stage(z)");
  if (rc) return rc;
  if (lam_out) {
    rc = fill_combo(a.epi, nacc, acc_terms, nullptr, false, "sem1d_adj_stage(acc)");
    if (rc) return rc;
  }
  return run_apply(plan, 4, a, stream, "sem1d_adj_stage");
}

int sem1d_ens_forward(const sem1d_plan* plan, const double* u0, double* traj, double* u_final,
                      const double* dts, int nsteps, int scheme, int* flags, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !u0 || !u_final || !dts || !flags || nsteps < 0)
    return fail(SEM1D_EINVAL, "sem1d_ens_forward: bad argument");
  EnsArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_ens_forward: unknown scheme");
  a.u0 = u0; a.traj = traj; a.u_final = u_final; a.dts = dts; a.nsteps = nsteps; a.flags = flags;
  cudaError_t e = dispatch_ens_forward(plan, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_ens_forward: ring too large for one CTA (needs E*(N+1) <= 1024, "
                              "or periodic, N+1 in {8,16,24,32}, E a multiple of 8, E <= 256)");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_ens_forward");
  return SEM1D_OK;
}

int sem1d_ens_adjoint(const sem1d_plan* plan, const double* traj, const double* lam_in,
                      double* lam_out, const double* dts, int nsteps, int scheme, int* flags,
                      void* stream) {
  return sem1d_ens_adjoint_ex(plan, traj, lam_in, lam_out, dts, nsteps, scheme, 1, flags, stream);
}

int sem1d_ens_adjoint_ex(const sem1d_plan* plan, const double* traj, const double* lam_in,
                         double* lam_out, const double* dts, int nsteps, int scheme, int check,
                         int* flags, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !traj || !lam_in || !lam_out || !dts || !flags || nsteps < 0)
    return fail(SEM1D_EINVAL, "sem1d_ens_adjoint: bad argument");
  EnsAdjArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_ens_adjoint: unknown scheme");
  a.traj = traj; a.lam_in = lam_in; a.lam_out = lam_out; a.dts = dts; a.nsteps = nsteps; a.flags = flags;
  a.check = check ? 1 : 0;
  cudaError_t e = dispatch_ens_adjoint(plan, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_ens_adjoint: ring too large for one CTA (needs E*(N+1) <= 1024, "
                              "or periodic, N+1 in {8,16,24,32}, E a multiple of 8, E <= 256)");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_ens_adjoint");
  return SEM1D_OK;
}

int sem1d_step_supported(const sem1d_plan* plan) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan)) return 0;
  const int te = ((plan->N + 1) == 8) ? 8 * TILE_WF8 * TILE_WMT8 : ((plan->N + 1) == 32 ? 64 : 128);
  return (plan->periodic && plan->batch == 1 && (plan->N + 1) % 8 == 0 && plan->E >= 2 * te) ? 1 : 0;
}

int sem1d_rk_step(const sem1d_plan* plan, const double* u, double* u_new, double dt, int scheme,
                  int* flag, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !u || !u_new || !flag || u == u_new)
    return fail(SEM1D_EINVAL, "sem1d_rk_step: bad argument (u_new must not alias u)");
  TileStepArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_rk_step: unknown scheme");
  a.u = u; a.out = u_new; a.flag = flag; a.dt = dt; a.check = 1;
  cudaError_t e = dispatch_tile(plan, 0, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_rk_step: needs a periodic batch-1 ring, N+1 in {8,16,24,32}, E >= 2 tiles");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_rk_step");
  return SEM1D_OK;
}

int sem1d_adj_step(const sem1d_plan* plan, const double* u, const double* lam, double* lam_out,
                   double dt, int scheme, int* flag, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !u || !lam || !lam_out || !flag || lam == lam_out)
    return fail(SEM1D_EINVAL, "sem1d_adj_step: bad argument (lam_out must not alias lam)");
  TileStepArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_adj_step: unknown scheme");
  a.u = u; a.lam = lam; a.out = lam_out; a.flag = flag; a.dt = dt; a.check = 1;
  cudaError_t e = dispatch_tile(plan, 1, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_adj_step: needs a periodic batch-1 ring, N+1 in {8,16,24,32}, E >= 2 tiles");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_adj_step");
  return SEM1D_OK;
}

int sem1d_rk_step_ex(const sem1d_plan* plan, const double* u, double* u_new, double* const* stages,
                     double dt, int scheme, int check, int tile_lo, int tile_cnt, int* flag, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !u || !u_new || !flag || u == u_new)
    return fail(SEM1D_EINVAL, "sem1d_rk_step_ex: bad argument (u_new must not alias u)");
  TileStepArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_rk_step_ex: unknown scheme");
  if (stages) {
    if (a.tab.s < 2) return fail(SEM1D_EINVAL, "sem1d_rk_step_ex: a one-stage scheme has no stage states");
    for (int i = 0; i + 1 < a.tab.s; ++i) {
      if (!stages[i]) return fail(SEM1D_EINVAL, "sem1d_rk_step_ex: NULL stage buffer");
      a.stages[i] = stages[i];
    }
  }
  a.u = u; a.out = u_new; a.flag = flag; a.dt = dt; a.check = check ? 1 : 0;
  a.tile_lo = tile_lo; a.tile_cnt = tile_cnt;
  cudaError_t e = dispatch_tile(plan, 0, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_rk_step_ex: needs a periodic batch-1 ring, N+1 in {8,16,24,32}, E >= 2 tiles");
  if (e == cudaErrorInvalidValue)
    return fail(SEM1D_EINVAL, "sem1d_rk_step_ex: bad tile range (ranges need N = 7)");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_rk_step_ex");
  return SEM1D_OK;
}

int sem1d_adj_step_ex(const sem1d_plan* plan, const double* u, const double* const* stages, const double* lam,
                      double* lam_out, double dt, int scheme, int check, int tile_lo, int tile_cnt, int* flag,
                      void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !u || !lam || !lam_out || !flag || lam == lam_out)
    return fail(SEM1D_EINVAL, "sem1d_adj_step_ex: bad argument (lam_out must not alias lam)");
  TileStepArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_adj_step_ex: unknown scheme");
  if (stages) {
    if (a.tab.s < 2) return fail(SEM1D_EINVAL, "sem1d_adj_step_ex: a one-stage scheme has no stage states");
    for (int i = 0; i + 1 < a.tab.s; ++i) {
      if (!stages[i]) return fail(SEM1D_EINVAL, "sem1d_adj_step_ex: NULL stage buffer");
      a.stin[i] = stages[i];
    }
  }
  a.u = u; a.lam = lam; a.out = lam_out; a.flag = flag; a.dt = dt; a.check = check ? 1 : 0;
  a.tile_lo = tile_lo; a.tile_cnt = tile_cnt;
  cudaError_t e = dispatch_tile(plan, 1, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_adj_step_ex: needs a periodic batch-1 ring, N+1 in {8,16,24,32}, E >= 2 tiles");
  if (e == cudaErrorInvalidValue)
    return fail(SEM1D_EINVAL, "sem1d_adj_step_ex: bad tile range (ranges need N = 7)");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_adj_step_ex");
  return SEM1D_OK;
}

int sem1d_step_tiling(const sem1d_plan* plan, int kind, int stored, int scheme, int* ntiles, int* owned,
                      int* ghost) {
  DeviceGuard guard_(plan ? plan->device : -1);
  Tableau tab;
  if (!valid_burgers(plan) || !ntiles || !owned || !ghost || (kind != 0 && kind != 1) || !make_tableau(scheme, tab))
    return fail(SEM1D_EINVAL, "sem1d_step_tiling: bad argument");
  if (!sem1d_step_supported(plan)) return fail(SEM1D_EINVAL, "sem1d_step_tiling: no whole-step kernels for this plan");
  const PlanView v = view(plan);
  cudaError_t e = cudaErrorNotSupported;
  switch (plan->N) {
    case 7: e = tile_layout<7>(v, kind, stored != 0, tab.s, ntiles, owned, ghost); break;
    case 15: e = tile_layout<15>(v, kind, stored != 0, tab.s, ntiles, owned, ghost); break;
    case 23: e = tile_layout<23>(v, kind, stored != 0, tab.s, ntiles, owned, ghost); break;
    case 31: e = tile_layout<31>(v, kind, stored != 0, tab.s, ntiles, owned, ghost); break;
    default: break;
  }
  return e == cudaSuccess ? SEM1D_OK : fail(SEM1D_EINVAL, "sem1d_step_tiling: no whole-step kernels for this plan");
}

int sem1d_step_stages_supported(const sem1d_plan* plan) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!sem1d_step_supported(plan)) return 0;
  switch (plan->N) {
    case 7: return stages_fit<7>() ? 1 : 0;
    case 15: return stages_fit<15>() ? 1 : 0;
    case 23: return stages_fit<23>() ? 1 : 0;
    case 31: return stages_fit<31>() ? 1 : 0;
    default: return 0;
  }
}

int sem1d_rk_step_stages(const sem1d_plan* plan, const double* u, double* u_new, double* const* stages,
                         double dt, int scheme, int* flag, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !u || !u_new || !flag || !stages || u == u_new)
    return fail(SEM1D_EINVAL, "sem1d_rk_step_stages: bad argument");
  TileStepArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_rk_step_stages: unknown scheme");
  if (a.tab.s < 2) return fail(SEM1D_EINVAL, "sem1d_rk_step_stages: a one-stage scheme has no stage states");
  for (int i = 0; i + 1 < a.tab.s; ++i) {
    if (!stages[i]) return fail(SEM1D_EINVAL, "sem1d_rk_step_stages: NULL stage buffer");
    a.stages[i] = stages[i];
  }
  a.u = u; a.out = u_new; a.flag = flag; a.dt = dt; a.check = 1;
  cudaError_t e = dispatch_tile(plan, 0, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_rk_step_stages: needs a periodic batch-1 ring, N+1 in {8,16,24,32}");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_rk_step_stages");
  return SEM1D_OK;
}

int sem1d_adj_step_stages(const sem1d_plan* plan, const double* u, const double* const* stages,
                          const double* lam, double* lam_out, double dt, int scheme, int* flag, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_burgers(plan) || !u || !lam || !lam_out || !flag || !stages || lam == lam_out)
    return fail(SEM1D_EINVAL, "sem1d_adj_step_stages: bad argument (lam_out must not alias lam)");
  TileStepArgs a;
  std::memset(&a, 0, sizeof(a));
  if (!make_tableau(scheme, a.tab)) return fail(SEM1D_EINVAL, "sem1d_adj_step_stages: unknown scheme");
  if (a.tab.s < 2) return fail(SEM1D_EINVAL, "sem1d_adj_step_stages: a one-stage scheme has no stage states");
  for (int i = 0; i + 1 < a.tab.s; ++i) {
    if (!stages[i]) return fail(SEM1D_EINVAL, "sem1d_adj_step_stages: NULL stage buffer");
    a.stin[i] = stages[i];
  }
  a.u = u; a.lam = lam; a.out = lam_out; a.flag = flag; a.dt = dt; a.check = 1;
  cudaError_t e = dispatch_tile(plan, 1, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(SEM1D_EINVAL, "sem1d_adj_step_stages: needs a periodic batch-1 ring, N+1 in {8,16,24,32}");
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_adj_step_stages");
  return SEM1D_OK;
}

int64_t sem1d_terminal_work_size(const sem1d_plan* plan) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_plan(plan)) return -1;
  const int64_t per = RED_TPB * RED_ITEMS;
  return plan->batch * ((plan->ndof + per - 1) / per);
}

int sem1d_terminal(const sem1d_plan* plan, const double* uN, const double* ud, double* lam,
                   double* J_out, double* work, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_plan(plan) || !uN || !ud || !lam || !J_out || !work)
    return fail(SEM1D_EINVAL, "sem1d_terminal: bad argument");
  Pattern P;
  std::memset(&P, 0, sizeof(P));
  P.N = plan->N;
  for (int i = 0; i < plan->N + 2; ++i) P.mass[i] = plan->mass[i];
  const Geo G = view(plan).geo;
  const int64_t per = RED_TPB * RED_ITEMS;
  const int nblk = (int)((plan->ndof + per - 1) / per);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  terminal_kernel<<<dim3(nblk, (unsigned)plan->batch), RED_TPB, 0, s>>>(P, G, uN, ud, lam, work, nblk);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_terminal");
  terminal_finish<<<(unsigned)plan->batch, RED_TPB, 0, s>>>(work, nblk, J_out);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sem1d_terminal(finish)");
  return SEM1D_OK;
}

int sem1d_scatter(const sem1d_plan* plan, const double* u, double* local, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_plan(plan) || !u || !local) return fail(SEM1D_EINVAL, "sem1d_scatter: bad argument");
  const Geo G = view(plan).geo;
  scatter_kernel<<<dim3(grid_for(plan->E * (plan->N + 1), 256), (unsigned)plan->batch), 256, 0,
                   static_cast<cudaStream_t>(stream)>>>(G, plan->N, u, local);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_scatter");
}

int sem1d_gather(const sem1d_plan* plan, const double* local, double* out, void* stream) {
  DeviceGuard guard_(plan ? plan->device : -1);
  if (!valid_plan(plan) || !local || !out) return fail(SEM1D_EINVAL, "sem1d_gather: bad argument");
  const Geo G = view(plan).geo;
  gather_kernel<<<dim3(grid_for(plan->ndof, 256), (unsigned)plan->batch), 256, 0,
                  static_cast<cudaStream_t>(stream)>>>(G, plan->N, local, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SEM1D_OK : cuda_fail(e, "sem1d_gather");
}

}  // extern "C"
