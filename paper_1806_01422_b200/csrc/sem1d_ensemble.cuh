// sem1d_ensemble.cuh -- ring-resident sweeps (BASELINE config 4: many small
// independent problems).  One CTA owns one periodic/Dirichlet ring whose
// fields fit in shared memory and runs every RK step of the forward sweep
// there; only the trajectory leaves the SM (one bulk store per step), so a
// 1000-step forward sweep costs 8 bytes per DOF per step of HBM traffic and
// is FP64-tensor-core bound.  The backward sweep (sem1d_ens_adjoint) streams
// the trajectory back in the same way.
//
// Mapping: 8 consumer warps; a warp owns ring elements in m-tiles of 8
// (DMMA m8n8k4.f64, permuted output columns as in apply_ws_kernel), lane
// (rr, kq) owns nodes 4kc + kq of element rr for kc = 0..KC-1 except node N,
// which is the right neighbour's node 0.  Interface node 0 = row N of the
// left element (shfl within the warp, shared-memory exchange across warps,
// ring wrap from the last warp) + row 0 of the element.
#pragma once

#include "sem1d_device.cuh"

namespace sem1d {

// periodic ring kernels (tile steps, ensembles): -nu M^-1 / M^-1 folded into the K / Dw
// B fragments of the F apply (ring_rhs<PRE>); A/B 0.456 vs 0.480 ms per RK4 step
#ifndef TILE_PRE
#define TILE_PRE 1
#endif
// the shared-memory ring / tile kernels (ens_forward_kernel, tile_step_kernel, tile_adj_kernel) at
// n % 16 == 0 (N = 15, 31) on the reflection split (ring_rhs / ring_jact EO)
#ifndef TILE_EO
#define TILE_EO 1
#endif
// the ensemble adjoint at N = 15 on the reflection split (ring_rhs / ring_jact EO): 8 + 12 DMMAs
// per m-tile for F + J^T instead of 16 + 24
#ifndef ENS_ADJ_EO
#define ENS_ADJ_EO 1
#endif
#ifndef ENS_ADJ_NOCHK
#define ENS_ADJ_NOCHK 0   // timing experiment only: no cotangent checks in the ensemble adjoint
#endif
#ifndef SEM1D_FIN_INT
#define SEM1D_FIN_INT 1
#endif

struct Tableau {
  double a[4][4];    // a[i][j], j < i
  double b[4];
  int s;             // stages (1..4)
  int keep[4];       // keep[j] != 0: k_j must be stored for a later combination row
  int nterm[4];      // nonzero terms of row i (i >= 1)
};

struct EnsArgs {
  const double* u0;      // (batch, ndof)
  double* traj;          // (nsteps+1, batch, ndof), step-major, or nullptr
  double* u_final;       // (batch, ndof)
  const double* dts;     // (nsteps) device
  int nsteps;
  int* flags;            // (batch) per-problem flag bits
  Tableau tab;
};

// warps per ring: forward 8 warps x 4 m-tiles at 2 rings per SM (see ENS_FWD_WARPS),
// the backward sweep 8 warps x 4 m-tiles (A/B on config 4, profiles/)
template <int N, int WARPS = 8>
struct EnsCfg {
  static constexpr int n = N + 1;
  static constexpr int W = WARPS;
  static constexpr int THREADS = 32 * W;
  static constexpr int NT = n / 8, KC = n / 4;
};
// forward sweep: 8 warps x 4 interleaved m-tiles with 2 rings (CTAs) per SM, so one ring's
// stage barriers overlap the other's DMMAs (config 4 forward 213.4 -> 205.9 ms against
// 16 warps x 2 with one ring per SM)
#ifndef ENS_FWD_WARPS
#define ENS_FWD_WARPS 8
#endif
#ifndef ENS_FWD_MINB
#define ENS_FWD_MINB 2
#endif
constexpr int kEnsFwdWarps = ENS_FWD_WARPS;
constexpr int kEnsAdjWarps = 8;
#ifndef TILE_WF16
#define TILE_WF16 8     // tile forward warps at n = 16 (x 16/W m-tiles; 8 x 2 with ring_elem ILV: 0.178 vs 0.203 ms at 16 x 1)
#endif
#ifndef TILE_WF24
#define TILE_WF24 8     // n = 24 tile forward: 8 x 2 interleaved (0.146 vs 0.164 ms at 16 x 1)
#endif
#ifndef ILV_SIMPLE2
#define ILV_SIMPLE2 0
#endif
#ifndef TILE_ILV
#define TILE_ILV 1      // tile kernels: interleaved m-tile rows (ring_elem)
#endif
#ifndef ENS_ILV
#define ENS_ILV 1       // ensemble kernels: interleaved rows when E is a multiple of 8*WMT
#endif
#ifndef ENS_ADJ_W16
#define ENS_ADJ_W16 1
#endif
// backward-sweep warps at n = 16: 16 x 2 interleaved m-tiles with the B fragments in a
// shared-memory table (ens_adj_bsm).  Round 1 measured it slower (804 vs 764 ms, the
// 128-register cap spilled); after round 2's kernel changes it is faster: config-4 adjoint
// 443.3 -> 431.0 ms (8 warps x 4 with register B fragments: 253 registers, 2 warps per
// sub-partition)
template <int N>
constexpr int ens_adj_warps() { return (ENS_ADJ_W16 && (N + 1) == 16) ? 16 : kEnsAdjWarps; }
template <int N>
constexpr bool ens_adj_bsm() { return ens_adj_warps<N>() == 16; }
// n = 32: 8 warps (255 registers per thread; at 16 warps the 128-register cap spilled)
template <int N>
constexpr int ens_fwd_warps() { return (N + 1) == 32 ? 8 : kEnsFwdWarps; }

// Element held by row rr of a warp's m-tile q.  ILV (interleaved; E a multiple of
// 8*WMT_MAX, WMT_MAX = 2 or 4): a 64-bit LDS/STS is served per half-warp, whose 16 lanes
// read rows rr = 4h..4h+3 at nodes 4kc + kq, i.e. doubles N*e + kq.  For odd N they hit 16
// distinct banks iff the half-warp's 4 elements are congruent mod 4 and distinct mod 16;
// the contiguous mapping (rows N apart) is a 4-way conflict at N = 15.  WMT_MAX = 4:
// e = 4 rr + q (16 h + 4 a + q); WMT_MAX = 2: e = 4 a + 2 h + q (a = rr & 3, h = rr >> 2).
// Each element's arithmetic is unchanged, so results are bit-identical.
template <int WMT_MAX, bool ILV>
__device__ __forceinline__ int ring_elem(int warp, int q, int rr) {
  if constexpr (ILV && WMT_MAX == 2 && !ILV_SIMPLE2) return 16 * warp + 4 * (rr & 3) + 2 * (rr >> 2) + q;
  else if constexpr (ILV && WMT_MAX > 1) return 8 * WMT_MAX * warp + WMT_MAX * rr + q;
  else return 8 * (warp * WMT_MAX + q) + rr;
}
// Row whose m-tile WMT_MAX-1 holds the left neighbour of (rr, m-tile 0), rr > 0 (ILV)
template <int WMT_MAX>
__device__ __forceinline__ int ring_left_row(int rr) {
  if constexpr (WMT_MAX == 2 && !ILV_SIMPLE2) return rr >= 4 ? rr - 4 : rr + 3;
  else return rr > 0 ? rr - 1 : 0;
}

// Reflection (even/odd) split in the ring kernels (EO template flag of ring_rhs / ring_jact,
// n % 16 == 0; see bfrag_eo_value in sem1d_device.cuh): lane (rr, kq) holds the node pairs
// (j, N - j), j = 4kc + kq, kc < n/8.  Slot kc of a per-lane array is node ring_node(kc, kq);
// rows 0 and N (the replica of the right neighbour's node 0) both sit in lane kq = 0.
template <int N, bool EO>
__device__ __forceinline__ int ring_node(int kc, int kq) {
  constexpr int H = (N + 1) / 8;
  if constexpr (EO) return kc < H ? 4 * kc + kq : N - (4 * (kc - H) + kq);
  else return 4 * kc + kq;
}

// One operator application over the whole ring held in shared memory.
// src: node values (ndof + 1 entries; entry ndof mirrors node 0 if periodic).
// EO (PRE only): bget(0..3, nt, kc) = Ke', Ko', De', Do' blocks, nt < NT/2, kc < KC/2.
// Output: kv[q][kc] = (M^-1-scaled) F at the nodes owned by this lane, for
// m-tile q of this warp (node 4kc+kq of element 8*(warp + q*W) + rr ... see body).
template <int N, int WMT_MAX, class BGet, bool WRAP = true, bool PRE = false, bool ILV = false, bool EO = false>
__device__ __forceinline__ void ring_rhs(const Consts<N>& C, const Geo& G, const double* src,
                                         double* xfer, BGet bget, const double* minv_a,
                                         double mnu, int warp, int lane,
                                         double (&kv)[WMT_MAX][(N + 1) / 4], unsigned& fin) {
  // PRE: the B fragments carry -nu M^-1_i (K) and M^-1_i (Dw) on output row i (periodic
  // rings: one M^-1 per local row, the interface rows share M^-1_0), so the row value is
  // already the M^-1-scaled F: two FP64 ops per node fewer on the pipe the DMMAs use
  constexpr int KC = (N + 1) / 4, NT = (N + 1) / 8, W = EnsCfg<N>::W;
  static_assert(!EO || (PRE && (N + 1) % 16 == 0), "reflection split: prescaled fragments, n % 16 == 0");
  constexpr int RKQ = EO ? 0 : 3;             // lane (kq) that holds row N
  const int kq = lane & 3, rr = lane >> 2;
  const int E = (int)G.E;
  const int mt_total = E / 8;
  double carry = 0.0;
  double row0_first = 0.0;
  double row0s[WMT_MAX], rowNs[WMT_MAX];
#pragma unroll
  for (int q = 0; q < WMT_MAX; ++q) {
    const int mt = warp * WMT_MAX + q;        // this warp's m-tiles
    if (mt >= mt_total) break;
    const int e = ring_elem<WMT_MAX, ILV>(warp, q, rr);
    const int base = e * N;
    if constexpr (EO) {
      constexpr int H = KC / 2, NT2 = NT / 2;
      double lo[H], hi[H], sv[H], dv[H];
#pragma unroll
      for (int kc = 0; kc < H; ++kc) {
        lo[kc] = src[base + 4 * kc + kq];
        hi[kc] = src[base + N - (4 * kc + kq)];
        fin |= nonfinite_bit(lo[kc]) | nonfinite_bit(hi[kc]);
        sv[kc] = __dadd_rn(lo[kc], hi[kc]);
        dv[kc] = __dsub_rn(lo[kc], hi[kc]);
      }
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt) {
        double ke[2] = {0.0, 0.0}, ko[2] = {0.0, 0.0}, pe[2] = {0.0, 0.0}, po[2] = {0.0, 0.0};
#pragma unroll
        for (int kc = 0; kc < H; ++kc) {
          dmma884(ke[0], ke[1], sv[kc], bget(0, nt, kc));
          dmma884(ko[0], ko[1], dv[kc], bget(1, nt, kc));
          dmma884(pe[0], pe[1], sv[kc], bget(2, nt, kc));
          dmma884(po[0], po[1], dv[kc], bget(3, nt, kc));
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {           // rows 4(2nt + h) + kq and their mirrors
          kv[q][2 * nt + h] = __fma_rn(-lo[2 * nt + h], __dadd_rn(pe[h], po[h]), __dadd_rn(ke[h], ko[h]));
          kv[q][H + 2 * nt + h] = __fma_rn(-hi[2 * nt + h], __dsub_rn(po[h], pe[h]), __dsub_rn(ke[h], ko[h]));
        }
      }
      const double row0 = kv[q][0], rowN = kv[q][H];   // both in lane kq = 0
      if (ILV && WMT_MAX > 1) {
        row0s[q] = row0;
        rowNs[q] = rowN;
      } else {
        double left = __shfl_up_sync(0xffffffffu, rowN, 4);
        if (rr == 0) left = carry;
        carry = __shfl_sync(0xffffffffu, rowN, 28);
        if (q == 0) row0_first = row0;
        if (kq == 0) kv[q][0] = __dadd_rn(left, row0);
      }
    } else {
    double au[KC];
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      au[kc] = src[base + 4 * kc + kq];
#if SEM1D_FIN_INT
      fin |= nonfinite_bit(au[kc]);
#else
      fin |= (au[kc] - au[kc] != 0.0) ? 1u : 0u;
#endif
    }
    double r[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double k0 = 0.0, k1 = 0.0, p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        dmma884(k0, k1, au[kc], bget(0, nt, kc));
        dmma884(p0, p1, au[kc], bget(1, nt, kc));
      }
      if (PRE) {                        // one DFMA: the FP64 pipe is shared with the DMMAs
        r[nt][0] = __fma_rn(-au[2 * nt], p0, k0);
        r[nt][1] = __fma_rn(-au[2 * nt + 1], p1, k1);
      } else {
        r[nt][0] = __dsub_rn(__dmul_rn(k0, mnu), __dmul_rn(au[2 * nt], p0));
        r[nt][1] = __dsub_rn(__dmul_rn(k1, mnu), __dmul_rn(au[2 * nt + 1], p1));
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) kv[q][2 * nt + h] = PRE ? r[nt][h] : __dmul_rn(r[nt][h], minv_a[2 * nt + h]);
    const double row0 = r[0][0];
    const double rowN = r[NT - 1][1];
    if (ILV && WMT_MAX > 1) {
      row0s[q] = row0;
      rowNs[q] = rowN;
    } else {
      double left = __shfl_up_sync(0xffffffffu, rowN, 1);
      if (rr == 0) left = carry;
      carry = __shfl_sync(0xffffffffu, rowN, 31);
      if (q == 0) row0_first = row0;           // lane 0 patches it after the exchange
      if (kq == 0) kv[q][0] = PRE ? __dadd_rn(left, row0) : __dmul_rn(__dadd_rn(left, row0), minv_a[0]);
    }
    }
  }
  if (ILV && WMT_MAX > 1 && warp * WMT_MAX < mt_total) {
    // left neighbour of (q, rr): (q-1, rr) in lane 4rr+3; of (0, rr): (WMT_MAX-1, ring_left_row)
#pragma unroll
    for (int q = 0; q < WMT_MAX; ++q) {
      const double left = q > 0 ? __shfl_down_sync(0xffffffffu, rowNs[q - 1], RKQ)
                                : __shfl_sync(0xffffffffu, rowNs[WMT_MAX - 1], 4 * ring_left_row<WMT_MAX>(rr) + RKQ);
      if (kq == 0 && (q > 0 || rr > 0))
        kv[q][0] = PRE ? __dadd_rn(left, row0s[q]) : __dmul_rn(__dadd_rn(left, row0s[q]), minv_a[0]);
    }
    carry = rowNs[WMT_MAX - 1];
    row0_first = row0s[0];
  }
  if (lane == 28 + RKQ && warp * WMT_MAX < mt_total) xfer[warp] = carry;   // row N of the warp's last element
  __syncthreads();
  if (lane == 0 && warp * WMT_MAX < mt_total) {
    // left neighbour of the warp's first element: previous warp (ring wrap from the last;
    // an open chain's first node stays incomplete -- it lies in the ghost margin)
    const int wl = (warp == 0) ? (WRAP ? (mt_total - 1) / WMT_MAX : -1) : warp - 1;
    const double v = wl >= 0 ? __dadd_rn(xfer[wl], row0_first) : row0_first;
    kv[0][0] = PRE ? v : __dmul_rn(v, minv_a[0]);
  }
  (void)W;
}

// B fragment of ring_rhs<PRE = true>: output row i of K scaled by -nu M^-1_i, of Dw by M^-1_i
// (periodic rings: row i < N has M^-1 pattern entry i, rows 0 and N the interface entry 0)
template <int N>
__device__ __forceinline__ double bfrag_pre(const Consts<N>& C, int mat, int nt, int kc, int lane) {
  const int c = 8 * nt + (lane >> 2);
  const int i = 4 * (2 * (c >> 3) + (c & 1)) + ((c >> 1) & 3);      // permuted output row
  const double mi = C.minv[(i == 0 || i == N) ? 0 : i];
  const double b = bfrag_perm<N>(C, mat, nt, kc, lane);
  return mat == 0 ? __dmul_rn(b, __dmul_rn(-C.nu, mi)) : __dmul_rn(b, mi);
}

// B fragments of ring_jact<PREJ = true> (tile adjoint steps; the ensemble adjoint passes dt = 1
// since its dt varies per step): dt and M^-1 folded in, so the
// stage input z enters unscaled and the row value is already the stage's l contribution:
// K column j by -nu dt M^-1_j, Dw row i (the z o (Dw u) term) by dt M^-1_i, Dw^T column j
// by dt M^-1_j (periodic rings: the interface rows/columns take the pattern entry 0)
template <int N>
__device__ __forceinline__ double bfrag_adj(const Consts<N>& C, int mat, int nt, int kc, int lane, double dt) {
  const int c = 8 * nt + (lane >> 2);
  const int i = 4 * (2 * (c >> 3) + (c & 1)) + ((c >> 1) & 3);      // permuted output row
  const int j = 4 * kc + (lane & 3);                                  // input node
  const double mi = C.minv[(i == 0 || i == N) ? 0 : i];
  const double mj = C.minv[(j == 0 || j == N) ? 0 : j];
  const double b = bfrag_perm<N>(C, mat, nt, kc, lane);
  if (mat == 0) return __dmul_rn(b, __dmul_rn(__dmul_rn(-C.nu, dt), mj));
  if (mat == 1) return __dmul_rn(b, __dmul_rn(dt, mi));
  return -__dmul_rn(b, __dmul_rn(dt, mj));     // negated: accumulates into the K chain
}

// Reflection-split blocks of the ring_jact<PREJ, EO> fragments (bfrag_adj's matrices; the ensemble
// adjoint passes dt = 1): mat 0 / 1 = even / odd block of K'' = K diag(-nu dt M^-1) (centrosymmetric),
// mat 2 / 3 of Dw'' = diag(dt M^-1) Dw and mat 4 / 5 of T'' = -Dw^T diag(dt M^-1) (both
// anti-centrosymmetric).  Formed from both halves of each matrix, as bfrag_eo_value does.
template <int N>
__device__ __forceinline__ double bfrag_eo_adj(const Consts<N>& C, int mat, int nt, int kc, int lane, double dt = 1.0) {
  constexpr int n = N + 1;
  const int m = mat >> 1, par = mat & 1;
  const int c = 8 * nt + (lane >> 2);
  const int i = 4 * (2 * (c >> 3) + (c & 1)) + ((c >> 1) & 3);
  const int j = 4 * kc + (lane & 3);
  auto mv = [&](int r) -> double { return C.minv[(r == 0 || r == N) ? 0 : r]; };
  // exact products summed in double-double and rounded once (eo_block_entry)
  auto term = [&](int r, int s) -> DD {
    if (m == 0) return dd_mul(dd_mul(dd_two_prod(-C.nu, dt), mv(s)), C.K[r * n + s]);
    if (m == 1) return dd_mul(dd_two_prod(dt, mv(r)), C.Dw[r * n + s]);
    return dd_neg(dd_mul(dd_two_prod(dt, mv(s)), C.Dw[s * n + r]));
  };
  return eo_block_entry(term, m == 0, par, i, j, N);
}

// Compile-time Butcher tableaux of the sweep kernels (same values as make_tableau:
// 0 euler, 1 Kutta-3 of timeloop.py:24-27, 2 classic RK4): with the stage count and
// coefficients constant the stage loops unroll and every tableau branch folds away
// (a runtime tableau made integer/branch instructions half of the adjoint step's issue)
template <int SCH>
struct TabC {
  static constexpr int s = SCH == 0 ? 1 : (SCH == 1 ? 3 : 4);
  __host__ __device__ static constexpr double a(int i, int j) {
    return SCH == 1 ? ((i == 1 && j == 0) ? 0.5 : (i == 2 && j == 0) ? -1.0 : (i == 2 && j == 1) ? 2.0 : 0.0)
         : SCH == 2 ? (((i == 1 && j == 0) || (i == 2 && j == 1)) ? 0.5 : (i == 3 && j == 2) ? 1.0 : 0.0)
                    : 0.0;
  }
  __host__ __device__ static constexpr double b(int i) {
    return SCH == 0 ? 1.0
         : SCH == 1 ? (i == 1 ? 2.0 / 3.0 : 1.0 / 6.0)
                    : ((i == 0 || i == 3) ? 1.0 / 6.0 : 1.0 / 3.0);
  }
  __host__ __device__ static constexpr int nterm(int i) {
    int n = 0;
    for (int j = 0; j < i; ++j) n += a(i, j) != 0.0;
    return n;
  }
  __host__ __device__ static constexpr int keep(int j) { return (SCH == 1 && j == 0) ? 1 : 0; }
};

// Forward sweep of one ring per CTA: periodic rings, E a multiple of 8 with
// E/8 <= 8 * WMT_MAX.  Trajectory state n+1 is written after step n.
template <int N, int WMT_MAX, bool ILV, int SCH>
__global__ void __launch_bounds__(EnsCfg<N, ens_fwd_warps<N>()>::THREADS, ((N + 1) == 32 ? 1 : ENS_FWD_MINB))
    ens_forward_kernel(const __grid_constant__ Consts<N> C, const Geo G, const EnsArgs A) {
  constexpr int n = N + 1, KC = EnsCfg<N>::KC, NT = EnsCfg<N>::NT;
  constexpr int THREADS = EnsCfg<N, ens_fwd_warps<N>()>::THREADS;
  extern __shared__ __align__(16) double smem[];
  const int ndof = (int)G.ndof;
  const int pad = (ndof + 2 + 1) & ~1;        // ndof + mirror node, 16-byte multiple
  double* su = smem;                          // base state u_n
  double* sU = su + pad;                      // current stage input
  double* sk = sU + pad;                      // stored slope k_0 (RK3 only)
  double* xfer = sk + pad;                    // [W] warp exchange
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  const int64_t b = blockIdx.x;
  const double* u0 = A.u0 + b * G.ndof;
  const double mnu = -C.nu;
  using TB = TabC<SCH>;                       // compile-time tableau: stage loop unrolls

  // reflection split (ring_node layout, ring_rhs EO) for n % 16 == 0: Ke', Ko', De', Do' blocks
  constexpr bool EO = TILE_EO && (N + 1) % 16 == 0 && TILE_PRE;
  constexpr int NT2 = NT / 2, KH = KC / 2;
  double breg[EO ? 4 * NT2 * KH : 2 * NT * KC];
  if constexpr (EO) {
#pragma unroll
    for (int mat = 0; mat < 4; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
        for (int kc = 0; kc < KH; ++kc)
          breg[(mat * NT2 + nt) * KH + kc] = bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, 6 + mat, nt, kc, lane);
  } else {
#pragma unroll
    for (int mat = 0; mat < 2; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) breg[(mat * NT + nt) * KC + kc] = (TILE_PRE ? bfrag_pre<N>(C, mat, nt, kc, lane) : bfrag_perm<N>(C, mat, nt, kc, lane));
  }
  auto bget = [&](int mat, int nt, int kc) -> double {
    if constexpr (EO) return breg[(mat * NT2 + nt) * KH + kc];
    else return breg[(mat * NT + nt) * KC + kc];
  };
  double minv_a[KC];
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int j = 4 * kc + kq;
    minv_a[kc] = C.minv[(j == 0 || j == N) ? 0 : j];
  }

  for (int k = tid; k < ndof; k += THREADS) su[k] = u0[k];
  if (tid == 0) su[ndof] = u0[0];
  __syncthreads();
  const int64_t nb = gridDim.x;
  if (A.traj) {
    double* t0 = A.traj + b * G.ndof;
    for (int k = tid; k < ndof; k += THREADS) t0[k] = su[k];
  }

  const int mt_total = (int)G.E / 8;
  unsigned fin = 0u;
  bool bad_step = false;
  double acc[WMT_MAX][KC];
  double kv[WMT_MAX][KC];
  for (int step = 0; step < A.nsteps; ++step) {
    const double dt = A.dts[step];
#pragma unroll
    for (int i = 0; i < TB::s; ++i) {
      const double* src = (i == 0) ? su : sU;
      ring_rhs<N, WMT_MAX, decltype(bget), true, TILE_PRE != 0, ILV, EO>(C, G, src, xfer, bget, minv_a, mnu, warp, lane, kv,
                                                               fin);
      // (ring_rhs ended with a barrier: every warp is done reading src)
#pragma unroll
      for (int q = 0; q < WMT_MAX; ++q) {
        const int mt = warp * WMT_MAX + q;
        if (mt >= mt_total) break;
        const int e = ring_elem<WMT_MAX, ILV>(warp, q, rr);
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const int j = ring_node<N, EO>(kc, kq);
          if (j == N) continue;               // node N belongs to the next element
          const int g = e * N + j;
          const double kk = kv[q][kc];
          // acc = b0 k0 + b1 k1 + ... left to right (timeloop.py:127), fused multiply-adds
          // (the FP64 pipe is shared with the DMMAs: 3 instead of 7 operations per node)
          acc[q][kc] = (i == 0) ? __dmul_rn(TB::b(i), kk) : __fma_rn(TB::b(i), kk, acc[q][kc]);
          if (i + 1 < TB::s) {
            double y;
            if (TB::nterm(i + 1) == 1) {
              // single term: u + (dt * a) * k  (timeloop.py:114)
              y = __fma_rn(__dmul_rn(dt, TB::a(i + 1, i)), kk, su[g]);
            } else {
              // u + dt * (a0 k0 + a1 k1)  (timeloop.py:116)
              double sacc = __dmul_rn(TB::a(i + 1, 0), (i == 0) ? kk : sk[g]);
#pragma unroll
              for (int jj = 1; jj <= i; ++jj)
                sacc = __fma_rn(TB::a(i + 1, jj), (jj == i) ? kk : sk[g], sacc);
              y = __fma_rn(dt, sacc, su[g]);
            }
            sU[g] = y;
            if (g == 0) sU[ndof] = y;
            if (i == 0 && TB::keep(0)) sk[g] = kk;
          } else {
            const double un = __fma_rn(dt, acc[q][kc], su[g]);
            bad_step |= nonfinite_bit(un) != 0u;
            su[g] = un;
            if (g == 0) su[ndof] = un;
          }
        }
      }
      __syncthreads();
    }
    if (A.traj) {
      double* tn = A.traj + ((int64_t)(step + 1) * nb + b) * G.ndof;
      for (int k = tid; k < ndof; k += THREADS) tn[k] = su[k];
    }
  }
  double* uf = A.u_final + b * G.ndof;
  for (int k = tid; k < ndof; k += THREADS) uf[k] = su[k];
  const bool bad_in = fin != 0u;
  if (bad_in || bad_step)
    atomicOr(&A.flags[b], (bad_in ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad_step ? SEM1D_FLAG_STEP_NONFINITE : 0));
  (void)n;
}

// J^T over the ring held in shared memory: usrc = linearisation point, zsrc =
// zm = mask(z M^-1) already scaled (ops.py:252-254).  Output (no M^-1, ops.py:256):
// jv[q][kc] at the nodes owned by this lane, interface nodes summed.
// PREJ: fragments from bfrag_adj, zsrc holds the unscaled stage input z, and the output is
// dt * J^T(M^-1 z) (the M^-1 and dt products ride on the DMMAs)
// ZS: the stage input is zs * zsrc (the first transposed stage reads b_{s-1} lam straight
// from the lam slab)
// EO (PREJ only): bget(0..5, nt, kc) = K''e, K''o, De', Do', T''e, T''o blocks (bfrag_eo_adj);
// the even K'' chain also takes T''o td and the odd one T''e ts, so that with A = K''e zs + T''o td
// and B = K''o zd + T''e ts rows i and N - i of K''z + T''t are A + B and A - B
template <int N, int WMT_MAX, class BGet, bool WRAP = true, bool ILV = false, bool PREJ = false, bool ZS = false,
          bool EO = false>
__device__ __forceinline__ void ring_jact(const Consts<N>& C, const Geo& G, const double* usrc,
                                          const double* zsrc, double* xfer, BGet bget,
                                          double mnu, int warp, int lane,
                                          double (&jv)[WMT_MAX][(N + 1) / 4], double zs = 1.0) {
  constexpr int KC = (N + 1) / 4, NT = (N + 1) / 8;
  static_assert(!EO || (PREJ && (N + 1) % 16 == 0), "reflection split: prescaled fragments, n % 16 == 0");
  constexpr int RKQ = EO ? 0 : 3;             // lane (kq) that holds row N
  const int kq = lane & 3, rr = lane >> 2;
  const int mt_total = (int)G.E / 8;
  double carry = 0.0, row0_first = 0.0;
  double row0s[WMT_MAX], rowNs[WMT_MAX];
#pragma unroll
  for (int q = 0; q < WMT_MAX; ++q) {
    const int mt = warp * WMT_MAX + q;
    if (mt >= mt_total) break;
    const int base = ring_elem<WMT_MAX, ILV>(warp, q, rr) * N;
    if constexpr (EO) {
      constexpr int H = KC / 2, NT2 = NT / 2;
      double zl[H], zh[H], us[H], ud[H], zs_[H], zd_[H], ts[H], td[H];
#pragma unroll
      for (int kc = 0; kc < H; ++kc) {
        const int j0 = base + 4 * kc + kq, j1 = base + N - (4 * kc + kq);
        const double u0 = usrc[j0], u1 = usrc[j1];
        zl[kc] = ZS ? __dmul_rn(zs, zsrc[j0]) : zsrc[j0];
        zh[kc] = ZS ? __dmul_rn(zs, zsrc[j1]) : zsrc[j1];
        const double t1 = __dmul_rn(u1, zh[kc]);
        us[kc] = __dadd_rn(u0, u1);
        ud[kc] = __dsub_rn(u0, u1);
        zs_[kc] = __dadd_rn(zl[kc], zh[kc]);
        zd_[kc] = __dsub_rn(zl[kc], zh[kc]);
        ts[kc] = __fma_rn(u0, zl[kc], t1);        // u0 z0 + u1 z1 and u0 z0 - u1 z1: one product
        td[kc] = __fma_rn(u0, zl[kc], -t1);       // and two DFMAs instead of two and two adds
      }
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt) {
        double ca[2] = {0.0, 0.0}, cb[2] = {0.0, 0.0}, pe[2] = {0.0, 0.0}, po[2] = {0.0, 0.0};
#pragma unroll
        for (int kc = 0; kc < H; ++kc) {
          dmma884(ca[0], ca[1], zs_[kc], bget(0, nt, kc));   // K''e zs
          dmma884(cb[0], cb[1], zd_[kc], bget(1, nt, kc));   // K''o zd
          dmma884(pe[0], pe[1], us[kc], bget(2, nt, kc));    // De' us
          dmma884(po[0], po[1], ud[kc], bget(3, nt, kc));    // Do' ud
          dmma884(cb[0], cb[1], ts[kc], bget(4, nt, kc));    // + T''e ts
          dmma884(ca[0], ca[1], td[kc], bget(5, nt, kc));    // + T''o td
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          jv[q][2 * nt + h] = __fma_rn(-zl[2 * nt + h], __dadd_rn(pe[h], po[h]), __dadd_rn(ca[h], cb[h]));
          jv[q][H + 2 * nt + h] = __fma_rn(-zh[2 * nt + h], __dsub_rn(po[h], pe[h]), __dsub_rn(ca[h], cb[h]));
        }
      }
      const double row0 = jv[q][0], rowN = jv[q][H];   // both in lane kq = 0
      if (ILV && WMT_MAX > 1) {
        row0s[q] = row0;
        rowNs[q] = rowN;
      } else {
        double left = __shfl_up_sync(0xffffffffu, rowN, 4);
        if (rr == 0) left = carry;
        carry = __shfl_sync(0xffffffffu, rowN, 28);
        if (q == 0) row0_first = row0;
        if (kq == 0) jv[q][0] = __dadd_rn(left, row0);
      }
    } else {
    double au[KC], az[KC], at[KC];
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      au[kc] = usrc[base + 4 * kc + kq];
      az[kc] = ZS ? __dmul_rn(zs, zsrc[base + 4 * kc + kq]) : zsrc[base + 4 * kc + kq];
      at[kc] = __dmul_rn(au[kc], az[kc]);
    }
    double r[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double k0 = 0.0, k1 = 0.0, p0 = 0.0, p1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        dmma884(k0, k1, az[kc], bget(0, nt, kc));   // K zm
        dmma884(p0, p1, au[kc], bget(1, nt, kc));   // Dw u
        if (PREJ) dmma884(k0, k1, at[kc], bget(2, nt, kc));   // - Dw^T (u o zm) into the K chain
        else dmma884(t0, t1, at[kc], bget(2, nt, kc));        // Dw^T (u o zm)
      }
      if (PREJ) {                    // one DFMA per value (FP64 pipe shared with the DMMAs)
        r[nt][0] = __fma_rn(-az[2 * nt], p0, k0);
        r[nt][1] = __fma_rn(-az[2 * nt + 1], p1, k1);
      } else {
        r[nt][0] = __dsub_rn(__dsub_rn(__dmul_rn(k0, mnu), __dmul_rn(az[2 * nt], p0)), t0);
        r[nt][1] = __dsub_rn(__dsub_rn(__dmul_rn(k1, mnu), __dmul_rn(az[2 * nt + 1], p1)), t1);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) jv[q][2 * nt + h] = r[nt][h];
    const double row0 = r[0][0], rowN = r[NT - 1][1];
    if (ILV && WMT_MAX > 1) {
      row0s[q] = row0;
      rowNs[q] = rowN;
    } else {
      double left = __shfl_up_sync(0xffffffffu, rowN, 1);
      if (rr == 0) left = carry;
      carry = __shfl_sync(0xffffffffu, rowN, 31);
      if (q == 0) row0_first = row0;
      if (kq == 0) jv[q][0] = __dadd_rn(left, row0);
    }
    }
  }
  if (ILV && WMT_MAX > 1 && warp * WMT_MAX < mt_total) {
#pragma unroll
    for (int q = 0; q < WMT_MAX; ++q) {
      const double left = q > 0 ? __shfl_down_sync(0xffffffffu, rowNs[q - 1], RKQ)
                                : __shfl_sync(0xffffffffu, rowNs[WMT_MAX - 1], 4 * ring_left_row<WMT_MAX>(rr) + RKQ);
      if (kq == 0 && (q > 0 || rr > 0)) jv[q][0] = __dadd_rn(left, row0s[q]);
    }
    carry = rowNs[WMT_MAX - 1];
    row0_first = row0s[0];
  }
  if (lane == 28 + RKQ && warp * WMT_MAX < mt_total) xfer[warp] = carry;
  __syncthreads();
  if (lane == 0 && warp * WMT_MAX < mt_total) {
    const int wl = (warp == 0) ? (WRAP ? (mt_total - 1) / WMT_MAX : -1) : warp - 1;
    jv[0][0] = wl >= 0 ? __dadd_rn(xfer[wl], row0_first) : row0_first;
  }
}

struct EnsAdjArgs {
  const double* traj;     // (nsteps+1, batch, ndof) step-major forward trajectory
  const double* lam_in;   // (batch, ndof) terminal seed
  double* lam_out;        // (batch, ndof) dJ/du0
  const double* dts;
  int nsteps;
  int* flags;
  Tableau tab;
  int check;              // 1: classify every stage's cotangent (INPUT2 bit); 0: test only lam_out
                          // (STEP bit; the caller re-runs a flagged sweep with check = 1)
};

// Backward sweep of one ring per CTA (adjoint.py:54-61 generalised, every step in
// shared memory): stage states recomputed from the stored u_n (s-1 F applies), then
// l_i = dt J^T(U_i)(b_i lam + sum_{j>i} a_ji l_j) for i = s-1..0 and
// lam <- lam + (l_{s-1} + ... + l_0).
template <int N, int WMT_MAX, bool ILV, int SCH, bool CHK = true>
__global__ void __launch_bounds__(EnsCfg<N, ens_adj_warps<N>()>::THREADS, 1)
    ens_adjoint_kernel(const __grid_constant__ Consts<N> C, const Geo G, const EnsAdjArgs A) {
  constexpr int KC = EnsCfg<N>::KC, NT = EnsCfg<N>::NT;
  constexpr int THREADS = EnsCfg<N, ens_adj_warps<N>()>::THREADS;
  extern __shared__ __align__(16) double smem[];
  const int ndof = (int)G.ndof;
  const int pad = (ndof + 2 + 1) & ~1;
  using TB = TabC<SCH>;                       // compile-time tableau: stage loops unroll
  constexpr int S = TB::s;
  // z of stage i-1 goes into the dead stage-state slab U_i and the first transposed stage reads
  // b_{s-1} lam from the lam slab, so the slab a z buffer took holds the NEXT step's trajectory
  // state, prefetched by one bulk copy while this step runs
  double* su = smem;                          // u_n (= U_0)
  double* spre = su + pad;                    // u_{n-1} in flight
  double* sUs = spre + pad;                   // U_1 .. U_{S-1}: S-1 arrays
  double* sk = sUs + 3 * pad;                 // k_0 (RK3 recompute) / an older l (RK3 chain)
  double* slam = sk + pad;                    // lam (owner-only, + wrap mirror)
  double* xfer = slam + pad;
  uint64_t* pbar = reinterpret_cast<uint64_t*>(xfer + 32);
  double* sB = xfer + 34;                     // B-fragment table (ens_adj_bsm), per lane
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  const int64_t b = blockIdx.x, nb = gridDim.x;
  const double mnu = -C.nu;
  auto Uarr = [&](int i) -> double* { return i == 0 ? su : sUs + (i - 1) * pad; };

  // B fragments: registers at 8 warps; at 16 warps (128-register cap) shared memory,
  // laid out per lane (in registers the compiler re-reads them from parameter space
  // with lane-divergent indices)
  constexpr bool BSM = ens_adj_bsm<N>();
  // reflection split (ring_node layout): N = 15 with the fragment table in shared memory
  constexpr bool EO = ENS_ADJ_EO && N == 15 && BSM && TILE_PRE;
  constexpr int NT2 = NT / 2, KH = KC / 2;
  double breg[BSM ? 1 : 3 * NT * KC];
  double bpre[(BSM || !TILE_PRE) ? 1 : 2 * NT * KC];
  if constexpr (EO) {
    // [K''e, K''o, De', Do', T''e, T''o, Ke', Ko'][NT/2][KC/2][32]
    for (int q = tid; q < 8 * NT2 * KH * 32; q += THREADS) {
      const int l = q & 31, f = q >> 5, kc = f % KH, nt = (f / KH) % NT2, mat = f / (KH * NT2);
      sB[q] = mat < 6 ? bfrag_eo_adj<N>(C, mat, nt, kc, l) : bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, mat, nt, kc, l);
    }
  } else if constexpr (BSM) {
    for (int q = tid; q < 5 * NT * KC * 32; q += THREADS) {
      const int l = q & 31, f = q >> 5, kc = f % KC, nt = (f / KC) % NT, mat = f / (KC * NT);
      sB[q] = mat < 3 ? bfrag_adj<N>(C, mat, nt, kc, l, 1.0)
                      : (TILE_PRE ? bfrag_pre<N>(C, mat - 3, nt, kc, l) : bfrag_perm<N>(C, mat - 3, nt, kc, l));
    }
  } else {
#pragma unroll
    for (int mat = 0; mat < 3; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) breg[(mat * NT + nt) * KC + kc] = bfrag_adj<N>(C, mat, nt, kc, lane, 1.0);
    if (TILE_PRE) {
#pragma unroll
      for (int mat = 0; mat < 2; ++mat)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int kc = 0; kc < KC; ++kc) bpre[(mat * NT + nt) * KC + kc] = bfrag_pre<N>(C, mat, nt, kc, lane);
    }
  }
  auto bget = [&](int mat, int nt, int kc) -> double {
    if constexpr (EO) return sB[((mat * NT2 + nt) * KH + kc) * 32 + lane];
    else if constexpr (BSM) return sB[((mat * NT + nt) * KC + kc) * 32 + lane];
    else return breg[(mat * NT + nt) * KC + kc];
  };
  auto bpget = [&](int mat, int nt, int kc) -> double {
    if constexpr (EO) return sB[(((mat < 2 ? 6 + mat : mat) * NT2 + nt) * KH + kc) * 32 + lane];
    else if constexpr (BSM) return sB[(((mat + 3) * NT + nt) * KC + kc) * 32 + lane];
    else return TILE_PRE ? bpre[(mat * NT + nt) * KC + kc] : breg[(mat * NT + nt) * KC + kc];
  };
  double minv_a[KC];
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int j = 4 * kc + kq;
    minv_a[kc] = C.minv[(j == 0 || j == N) ? 0 : j];
  }
  const int mt_total = (int)G.E / 8;
  const double* lin = A.lam_in + b * G.ndof;
  for (int k = tid; k < ndof; k += THREADS) slam[k] = lin[k];
  if (tid == 0) slam[ndof] = lin[0];
  unsigned fin = 0u;
  double kv[WMT_MAX][KC], lnext[WMT_MAX][KC], lacc[WMT_MAX][KC];
  // trajectory states arrive by bulk copy when a state is a 16-byte multiple (every row of the
  // step-major trajectory is then 16-byte aligned)
  const bool bulk = ((ndof * 8) & 15) == 0;
  const uint32_t sbytes = (uint32_t)(ndof * 8);
  auto traj_row = [&](int step) { return A.traj + ((int64_t)step * nb + b) * G.ndof; };
  if (tid == 0) {
    mbar_init(pbar, 1);
    fence_mbar_init();
    if (bulk && A.nsteps > 0) {
      mbar_expect_tx(pbar, sbytes);
      bulk_g2s(su, traj_row(A.nsteps - 1), sbytes, pbar);
    }
  }
  uint32_t pphase = 0;

  for (int step = A.nsteps - 1; step >= 0; --step) {
    const double dt = A.dts[step];
    const double* un = traj_row(step);
    __syncthreads();   // previous step's readers of su / sUs are done
    if (bulk) {
      while (!mbar_try_wait(pbar, pphase)) {
      }
      pphase ^= 1u;
    } else {
      for (int k = tid; k < ndof; k += THREADS) su[k] = un[k];
    }
    if (tid == 0) su[ndof] = bulk ? su[0] : un[0];
    __syncthreads();
    if (bulk && step > 0 && tid == 0) {   // u_{n-1} into the buffer u_{n+1} left
      mbar_expect_tx(pbar, sbytes);
      bulk_g2s(spre, traj_row(step - 1), sbytes, pbar);
    }
    // ---- stage states U_1..U_{S-1} (timeloop.rk3_stages, adjoint.py:56)
#pragma unroll
    for (int i = 0; i + 1 < S; ++i) {
      ring_rhs<N, WMT_MAX, decltype(bpget), true, TILE_PRE != 0, ILV, EO>(C, G, Uarr(i), xfer, bpget, minv_a, mnu, warp,
                                                                lane, kv, fin);
      double* dst = Uarr(i + 1);
#pragma unroll
      for (int q = 0; q < WMT_MAX; ++q) {
        const int mt = warp * WMT_MAX + q;
        if (mt >= mt_total) break;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const int j = ring_node<N, EO>(kc, kq);
          if (j == N) continue;
          const int g = ring_elem<WMT_MAX, ILV>(warp, q, rr) * N + j;
          const double kk = kv[q][kc];
          double y;
          if (TB::nterm(i + 1) == 1) {
            y = __fma_rn(__dmul_rn(dt, TB::a(i + 1, i)), kk, su[g]);
          } else {
            double sacc = __dmul_rn(TB::a(i + 1, 0), (i == 0) ? kk : sk[g]);
#pragma unroll
            for (int jj = 1; jj <= i; ++jj)
              sacc = __fma_rn(TB::a(i + 1, jj), (jj == i) ? kk : sk[g], sacc);
            y = __fma_rn(dt, sacc, su[g]);
          }
          dst[g] = y;
          if (g == 0) dst[ndof] = y;
          if (i == 0 && TB::keep(0)) sk[g] = kk;
        }
      }
      __syncthreads();
    }
    // ---- stage-adjoint chain, i = S-1 .. 0 (M^-1 and -nu ride on the J^T fragments, so z
    // enters unscaled); z_i = b_i lam + a_{i+1,i} l_{i+1} + a_{i+2,i} l_{i+2} (adjoint.py:58-60)
    // lnext / sk hold l / dt (the ring J^T output): dt rides on the coefficients
    auto zval = [&](int i, int g, int q, int kc) -> double {
      double z = __dmul_rn(TB::b(i), slam[g]);
      if (i + 1 < S && TB::a(i + 1, i) != 0.0) z = __fma_rn(__dmul_rn(TB::a(i + 1, i), dt), lnext[q][kc], z);
      if (i + 2 < S && TB::a(i + 2, i) != 0.0) z = __fma_rn(__dmul_rn(TB::a(i + 2, i), dt), sk[g], z);
      return z;
    };
    if constexpr (!ENS_ADJ_NOCHK && CHK) {
#pragma unroll
      for (int q = 0; q < WMT_MAX; ++q) {
        const int mt = warp * WMT_MAX + q;
        if (mt >= mt_total) break;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const int j = ring_node<N, EO>(kc, kq);
          if (j == N) continue;
          const int g = ring_elem<WMT_MAX, ILV>(warp, q, rr) * N + j;
          const double z = zval(S - 1, g, q, kc);
          fin |= nonfinite_bit(z);
        }
      }
    }
    // per stage: J^T apply (its internal barrier ends every read of its z and U_i), then
    // accumulate l_i and form z_{i-1} (into the dead U_i) in one pass -- two barriers per stage
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      if (i == S - 1)
        ring_jact<N, WMT_MAX, decltype(bget), true, ILV, true, true, EO>(C, G, Uarr(i), slam, xfer, bget, mnu, warp, lane,
                                                                   kv, TB::b(S - 1));
      else
        ring_jact<N, WMT_MAX, decltype(bget), true, ILV, true, false, EO>(C, G, Uarr(i), Uarr(i + 1), xfer, bget, mnu, warp, lane,
                                                             kv);
      double* zdst = Uarr(i);
#pragma unroll
      for (int q = 0; q < WMT_MAX; ++q) {
        const int mt = warp * WMT_MAX + q;
        if (mt >= mt_total) break;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const int j = ring_node<N, EO>(kc, kq);
          if (j == N) continue;
          const int g = ring_elem<WMT_MAX, ILV>(warp, q, rr) * N + j;
          const double l = kv[q][kc];                       // l_i / dt
          lacc[q][kc] = (i == S - 1) ? l : __dadd_rn(lacc[q][kc], l);
          if (i + 1 < S && S == 3) sk[g] = lnext[q][kc];   // RK3: keep l_{i+1} for z_{i-1}
          lnext[q][kc] = l;
          if (i == 0) {
            const double lv = __fma_rn(dt, lacc[q][kc], slam[g]);
            slam[g] = lv;
            if (g == 0) slam[ndof] = lv;
          } else {
            const double z = zval(i - 1, g, q, kc);
            if (!ENS_ADJ_NOCHK && CHK) fin |= nonfinite_bit(z);
            zdst[g] = z;
            if (g == 0) zdst[ndof] = z;
          }
        }
      }
      __syncthreads();
    }
    if (bulk) {                                // swap the trajectory buffers
      double* t = su;
      su = spre;
      spre = t;
    }
  }
  double* lo = A.lam_out + b * G.ndof;
  unsigned bad_out = 0u;
  for (int k = tid; k < ndof; k += THREADS) {
    lo[k] = slam[k];
    if (!CHK) bad_out |= nonfinite_bit(slam[k]);
  }
  if (fin || bad_out)
    atomicOr(&A.flags[b], (fin ? SEM1D_FLAG_INPUT2_NONFINITE : 0) | (bad_out ? SEM1D_FLAG_STEP_NONFINITE : 0));
}

template <int N>
constexpr size_t ens_adj_smem_bytes(int ndof) {
  constexpr size_t frag = ens_adj_bsm<N>() ? 5 * EnsCfg<N>::NT * EnsCfg<N>::KC * 32 : 0;
  return sizeof(double) * (7 * (size_t)((ndof + 2 + 1) & ~1) + 34 + frag);
}

// ============================================================================
// Temporally blocked steps for LARGE periodic rings.  A CTA takes a tile of TE
// = 8*W*WMT consecutive elements, of which the outer H on each side are ghost
// elements recomputed from the neighbouring tiles' data: H = s for a forward
// step (the valid range shrinks by one element per stage), H = 2s-1 for an
// adjoint step (s-1 stage recomputes + s transposed applies).  Everything
// between the tile load and the store of the central TE-2H elements stays in
// shared memory, so one RK step moves 16 B/DOF and one adjoint step 24 B/DOF
// (plus the ghost margin) instead of one HBM round trip per stage.
// ============================================================================

#ifndef TILE_MINB8
#define TILE_MINB8 2
#endif
#ifndef TILE_WMT8
#define TILE_WMT8 4
#endif
#ifndef TILE_WA8
#define TILE_WA8 8      // recompute adjoint at n = 8: 8 warps x 4 m-tiles, 7 slabs, 2 CTAs/SM (0.624 ms; 0.649 at 8 x 2 x 3)
#endif
#ifndef TILE_WF8
#define TILE_WF8 8
#endif
#ifndef TILE_WMTA8
#define TILE_WMTA8 4
#endif
#ifndef TILE_WA16
#define TILE_WA16 8
#endif
#ifndef TILE_WL8
#define TILE_WL8 8      // stored-stage adjoint at n = 8: 8 warps x 2 m-tiles, 3 CTAs/SM (0.445 vs 0.472 ms at 4 x 2 x 6)
#endif
#ifndef TILE_WMTL8
#define TILE_WMTL8 2
#endif
#ifndef TILE_ADJ_MINB8
#define TILE_ADJ_MINB8 2
#endif

struct TileStepArgs {
  const double* u;        // state u_n (forward input / adjoint linearisation point)
  const double* lam;      // adjoint: lam_{n+1}
  double* out;            // forward: u_{n+1}; adjoint: lam_n
  int* flag;
  double dt;
  int H;                  // ghost elements per side
  int ntiles;             // ceil(E / (TE - 2H))
  Tableau tab;
  double* stages[3];      // forward: also write the stage states U_1..U_{s-1} (NULL: don't)
  const double* stin[3];  // adjoint: read U_1..U_{s-1} instead of recomputing them (NULL: recompute)
  int check;              // 1: classify non-finite stage inputs (STATE bit); 0: outputs only
                          // (register-resident N = 7 kernels; the others always classify)
  int tile_lo, tile_cnt;  // N = 7 kernels: run ring tiles (tile_lo + k) mod ntiles, k < tile_cnt
                          // (tile_cnt 0: every tile); the other kernels need tile_cnt 0
};

// Tile loader shared by the step kernels: interior tiles arrive by one bulk
// copy (issued one tile ahead, completion on an mbarrier); tiles whose node
// range wraps around the ring end are loaded synchronously by the whole CTA.
struct TileLoad {
  int64_t g0;      // first node (mod ndof)
  int sh;          // 16-byte alignment shift of the smem copy
  bool bulk;       // loaded by cp.async.bulk
};

__device__ __forceinline__ TileLoad tile_load_plan(int t, int T, int H, int N, int LEN, int64_t ndof) {
  TileLoad L;
  // t * T - H lies in [-H, E + T): at most one wrap either way (no 64-bit modulo: ncu put
  // 7% of the register-resident step kernel's stall samples on it)
  int64_t g0 = ((int64_t)t * T - H) * N;
  if (g0 < 0) g0 += ndof;
  if (g0 >= ndof) g0 -= ndof;
  L.g0 = g0;
  L.sh = (int)(g0 & 1);
  const int64_t a0 = g0 - L.sh;
  const int64_t bytes = ((int64_t)(LEN + L.sh) * 8 + 15) & ~15LL;
  L.bulk = (a0 * 8 + bytes <= ndof * 8);
  if (!L.bulk) L.sh = 0;
  return L;
}

__device__ __forceinline__ void tile_issue(const TileLoad& L, int LEN, const double* src, double* dst,
                                           uint64_t* bar, int nsrc, const double* src2, double* dst2) {
  const int64_t a0 = L.g0 - L.sh;
  const uint32_t bytes = (uint32_t)((((int64_t)(LEN + L.sh)) * 8 + 15) & ~15LL);
  mbar_expect_tx(bar, nsrc * bytes);
  bulk_g2s(dst, src + a0, bytes, bar);
  if (nsrc == 2) bulk_g2s(dst2, src2 + a0, bytes, bar);
}

// first 16-byte aligned double after the two mbarriers (the n = 32 B-fragment table)
template <int N>
__device__ __forceinline__ double* bar_smem_end(double* p) {
  return reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}

// n slabs of the same tile range under ONE arrive.expect_tx (a second arm could let the
// phase complete before all copies are registered)
__device__ __forceinline__ void tile_issue_n(const TileLoad& L, int LEN, const double* const (&src)[5],
                                             double* const (&dst)[5], uint64_t* bar, int nsrc) {
  const int64_t a0 = L.g0 - L.sh;
  const uint32_t bytes = (uint32_t)((((int64_t)(LEN + L.sh)) * 8 + 15) & ~15LL);
  mbar_expect_tx(bar, nsrc * bytes);
#pragma unroll
  for (int i = 0; i < 5; ++i)            // compile-time bound: the pointer arrays stay in registers
    if (i < nsrc) bulk_g2s(dst[i], src[i] + a0, bytes, bar);
}

// resident CTAs per SM (A/B: a 64-register cap for two CTAs made the n = 8 step 2x slower)
template <int N>
constexpr int tile_minb() { return (N + 1) == 8 ? TILE_MINB8 : 1; }
#ifndef TILE_ADJ_LD_MINB8
#define TILE_ADJ_LD_MINB8 3
#endif
template <int N, int MODE = 0>
constexpr int tile_adj_minb() { return (N + 1) == 8 ? (MODE == 1 ? TILE_ADJ_LD_MINB8 : TILE_ADJ_MINB8) : 1; }

// MODE 0: plain step; 1: also store the stage states U_1..U_{s-1} (north_star item 4)
template <int N, int W, int WMT, int SCH, int MODE>
__global__ void __launch_bounds__(32 * W, tile_minb<N>())
    tile_step_kernel(const __grid_constant__ Consts<N> C, const Geo G, const TileStepArgs A) {
  constexpr int KC = (N + 1) / 4, NT = (N + 1) / 8;
  constexpr int TE = 8 * W * WMT;
  constexpr int LEN = TE * N + 1;
  constexpr int PAD = ((LEN + 2) + 1) & ~1;
  extern __shared__ __align__(16) double smem[];
  double* sbuf = smem;                        // [2][PAD] double-buffered tile loads (base u)
  double* sU = sbuf + 2 * PAD;                // stage input / new state
  double* sk = sU + PAD;                      // k_0 (RK3)
  double* xfer = sk + PAD;                    // [W]
  uint64_t* bar = reinterpret_cast<uint64_t*>(xfer + 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  using TB = TabC<SCH>;                       // compile-time tableau: stage loops unroll
  constexpr int H = TB::s;                    // ghost elements per side (= the launcher's A.H)
  constexpr int T = TE - 2 * H;
  constexpr bool STG = MODE == 1;
  const int64_t ndof = G.ndof;
  const double mnu = -C.nu;
  Geo Gt = G;
  Gt.E = TE;
  // reflection split (ring_node layout, ring_rhs EO) for n % 16 == 0: Ke', Ko', De', Do' blocks
  constexpr bool EO = TILE_EO && (N + 1) % 16 == 0 && TILE_PRE;
  constexpr int NT2 = NT / 2, KH = KC / 2;
  double breg[EO ? 4 * NT2 * KH : 2 * NT * KC];
  if constexpr (EO) {
#pragma unroll
    for (int mat = 0; mat < 4; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
        for (int kc = 0; kc < KH; ++kc)
          breg[(mat * NT2 + nt) * KH + kc] = bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, 6 + mat, nt, kc, lane);
  } else {
#pragma unroll
    for (int mat = 0; mat < 2; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) breg[(mat * NT + nt) * KC + kc] = (TILE_PRE ? bfrag_pre<N>(C, mat, nt, kc, lane) : bfrag_perm<N>(C, mat, nt, kc, lane));
  }
  auto bget = [&](int mat, int nt, int kc) -> double {
    if constexpr (EO) return breg[(mat * NT2 + nt) * KH + kc];
    else return breg[(mat * NT + nt) * KC + kc];
  };
  double minv_a[KC];
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int j = 4 * kc + kq;
    minv_a[kc] = C.minv[(j == 0 || j == N) ? 0 : j];
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_launch_dependents();               // PDL: the next step's prologue may start
  griddep_wait();                             // ... and this step's data path waits for ours
  if (tid == 0 && blockIdx.x < A.ntiles) {
    const TileLoad L = tile_load_plan(blockIdx.x, T, H, N, LEN, ndof);
    if (L.bulk) tile_issue(L, LEN, A.u, sbuf, &bar[0], 1, nullptr, nullptr);
  }
  unsigned fin = 0u;
  bool bad = false;
  uint32_t phase = 0;
  double kv[WMT][KC], acc[WMT][KC];
  int it = 0;
  for (int t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++it) {
    const int b = it & 1;
    double* sb = sbuf + b * PAD;
    const TileLoad L = tile_load_plan(t, T, H, N, LEN, ndof);
    if (L.bulk) {
      while (!mbar_try_wait(&bar[b], (phase >> b) & 1u)) {
      }
      phase ^= (1u << b);
    } else {
      for (int k = tid; k < LEN; k += 32 * W) {
        int64_t g = L.g0 + k;
        while (g >= ndof) g -= ndof;
        sb[k] = __ldg(A.u + g);
      }
      __syncthreads();
    }
    // prefetch the next tile into the other buffer (free: its tile ended with a barrier)
    if (tid == 0 && t + (int)gridDim.x < A.ntiles) {
      const TileLoad Ln = tile_load_plan(t + gridDim.x, T, H, N, LEN, ndof);
      if (Ln.bulk) tile_issue(Ln, LEN, A.u, sbuf + (b ^ 1) * PAD, &bar[b ^ 1], 1, nullptr, nullptr);
    }
    const double* su = sb + L.sh;
    if (tid == 0) sU[LEN - 1] = su[LEN - 1];   // the chain's last node is never owned
#pragma unroll
    for (int st = 0; st < TB::s; ++st) {
      if (STG && tid == 0) bulk_wait_read<0>();   // the previous stage's store has read sU
      const double* src = (st == 0) ? su : sU;
      ring_rhs<N, WMT, decltype(bget), false, TILE_PRE != 0, TILE_ILV != 0, EO>(C, Gt, src, xfer, bget, minv_a, mnu, warp, lane, kv,
                                                            fin);
      const double tb = TB::b(st);
      const bool last = (st + 1 == TB::s);
      const bool one = !last && TB::nterm(st + 1) == 1;
      const double c1 = last ? 0.0 : __dmul_rn(A.dt, TB::a(st + 1, st));
#pragma unroll
      for (int q = 0; q < WMT; ++q) {
        const int e = ring_elem<WMT, TILE_ILV != 0>(warp, q, rr);
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const int j = ring_node<N, EO>(kc, kq);
          if (j == N) continue;
          const int g = e * N + j;
          const double kk = kv[q][kc];
          acc[q][kc] = (st == 0) ? __dmul_rn(tb, kk) : __fma_rn(tb, kk, acc[q][kc]);
          if (!last) {
            double y;
            if (one) {
              y = __fma_rn(c1, kk, su[g]);
            } else {
              double sacc = __dmul_rn(TB::a(st + 1, 0), (st == 0) ? kk : sk[g]);
#pragma unroll
              for (int jj = 1; jj <= st; ++jj)
                sacc = __fma_rn(TB::a(st + 1, jj), (jj == st) ? kk : sk[g], sacc);
              y = __fma_rn(A.dt, sacc, su[g]);
            }
            sU[g] = y;
            if (st == 0 && TB::keep(0)) sk[g] = kk;
          } else {
            const double un = __fma_rn(A.dt, acc[q][kc], su[g]);
            if (e >= H && e < H + T) bad |= !isfinite(un);
            sU[g] = un;                         // every warp is past its last read of sU
          }
        }
      }
      if (STG) fence_proxy_async_smem();   // sU is read by the bulk store below
      __syncthreads();
      if (STG && st + 1 < TB::s) {  // stage state U_{st+1} of the owned elements
        const int64_t e_o = (int64_t)t * T;
        const int no = (int)min((int64_t)T, G.E - e_o) * N;
        double* dst = A.stages[st] + e_o * N;
        const double* src = sU + H * N;
        if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0 && (no & 1) == 0) {
          if (tid == 0) {                     // one async bulk store; read-drained before sU is rewritten
            bulk_s2g(dst, src, (uint32_t)(no * 8));
            bulk_commit();
          }
        } else {
          for (int k = tid; k < no; k += 32 * W) dst[k] = src[k];
        }
      }
    }
    const int64_t e_out0 = (int64_t)t * T;
    const int nout_el = (int)min((int64_t)T, G.E - e_out0);
    for (int k = tid; k < nout_el * N; k += 32 * W) A.out[e_out0 * N + k] = sU[H * N + k];
    __syncthreads();
  }
  if (STG && tid == 0) bulk_wait_all();
  if (fin || bad)
    atomicOr(A.flag, (fin ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad ? SEM1D_FLAG_STEP_NONFINITE : 0));
}

// MODE 0: stage states recomputed (H = 2s-1); 1: read from the forward run's stored
// states (H = s)
template <int N, int W, int WMT, int SCH, int MODE>
__global__ void __launch_bounds__(32 * W, tile_adj_minb<N, MODE>())
    tile_adj_kernel(const __grid_constant__ Consts<N> C, const Geo G, const TileStepArgs A) {
  constexpr int KC = (N + 1) / 4, NT = (N + 1) / 8;
  constexpr int TE = 8 * W * WMT;
  constexpr int LEN = TE * N + 1;
  constexpr int PAD = ((LEN + 2) + 1) & ~1;
  extern __shared__ __align__(16) double smem[];
  double* sbu = smem;                         // [2][PAD] u_n loads (= U_0)
  double* sbl = sbu + 2 * PAD;                // [2][PAD] lam loads (accumulated in place)
  // stage states: recomputed into [3][PAD], or (stored by the forward step) prefetched with
  // the tile into [2][3][PAD]
  constexpr bool LD = MODE == 1;
  using TB = TabC<SCH>;                       // compile-time tableau: stage loops unroll
  constexpr int S = TB::s;
  // z of stage i-1 goes into the (dead) stage-state slab U_i and the first stage reads
  // b_{s-1} lam from the lam slab, so there is no z slab; k (Kutta-3's older l) only for s = 3
  // -- RK4: 10 slabs with stored stages, 7 with recompute
  double* sUs = sbl + 2 * PAD;
  double* sk = sUs + (LD ? 6 : 3) * PAD;
  double* xfer = sk + (S == 3 ? PAD : 0);
  uint64_t* bar = reinterpret_cast<uint64_t*>(xfer + 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  constexpr int H = LD ? S : 2 * S - 1;       // ghost elements per side (= the launcher's A.H)
  constexpr int T = TE - 2 * H;
  auto issue = [&](const TileLoad& Lx, int buf) {
    const double* srcs[5] = {A.u, A.lam, A.stin[0], A.stin[1], A.stin[2]};
    double* dsts[5] = {sbu + buf * PAD, sbl + buf * PAD, sUs + (buf * 3 + 0) * PAD, sUs + (buf * 3 + 1) * PAD,
                       sUs + (buf * 3 + 2) * PAD};
    tile_issue_n(Lx, LEN, srcs, dsts, &bar[buf], LD ? S + 1 : 2);
  };
  const int64_t ndof = G.ndof;
  const double mnu = -C.nu;
  Geo Gt = G;
  Gt.E = TE;
  double* su = sbu;
  double* slam = sbl;
  double* sUb = sUs;                          // this tile's stage-state slabs
  auto Uarr = [&](int i) -> double* { return i == 0 ? su : sUb + (i - 1) * PAD; };
  // B fragments (K, Dw, Dw^T and, for the stage recompute, K / Dw with -nu M^-1 / M^-1 folded
  // in): registers up to n = 24; at n = 32 (160 values per lane) shared memory, laid out
  // per lane -- in registers the compiler re-reads them from kernel-parameter space with
  // lane-divergent indices (19x slower)
  constexpr bool BSM = (N + 1) == 32;
  // reflection split (ring_node layout, ring_rhs / ring_jact EO) for n % 16 == 0:
  // [K''e, K''o, Dw''e, Dw''o, T''e, T''o] with dt folded in, and the recompute's [Ke', Ko', De', Do']
  constexpr bool EO = TILE_EO && (N + 1) % 16 == 0 && TILE_PRE;
  constexpr int NT2 = NT / 2, KH = KC / 2;
  double breg[BSM ? 1 : (EO ? 6 * NT2 * KH : 3 * NT * KC)];
  double bpre[(BSM || !TILE_PRE) ? 1 : (EO ? 4 * NT2 * KH : 2 * NT * KC)];
  double* sB = bar_smem_end<N>(reinterpret_cast<double*>(bar + 2));
  if constexpr (EO && BSM) {
    for (int q = tid; q < 10 * NT2 * KH * 32; q += blockDim.x) {
      const int l = q & 31, f = q >> 5, kc = f % KH, nt = (f / KH) % NT2, mat = f / (KH * NT2);
      sB[q] = mat < 6 ? bfrag_eo_adj<N>(C, mat, nt, kc, l, A.dt) : bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, mat, nt, kc, l);
    }
  } else if constexpr (EO) {
#pragma unroll
    for (int mat = 0; mat < 6; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
        for (int kc = 0; kc < KH; ++kc) breg[(mat * NT2 + nt) * KH + kc] = bfrag_eo_adj<N>(C, mat, nt, kc, lane, A.dt);
#pragma unroll
    for (int mat = 0; mat < 4; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
        for (int kc = 0; kc < KH; ++kc)
          bpre[(mat * NT2 + nt) * KH + kc] = bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, 6 + mat, nt, kc, lane);
  } else if constexpr (BSM) {
    for (int q = tid; q < 5 * NT * KC * 32; q += blockDim.x) {
      const int l = q & 31, f = q >> 5, kc = f % KC, nt = (f / KC) % NT, mat = f / (KC * NT);
      sB[q] = mat < 3 ? bfrag_adj<N>(C, mat, nt, kc, l, A.dt)
                      : (TILE_PRE ? bfrag_pre<N>(C, mat - 3, nt, kc, l) : bfrag_perm<N>(C, mat - 3, nt, kc, l));
    }
  } else {
#pragma unroll
    for (int mat = 0; mat < 3; ++mat)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) breg[(mat * NT + nt) * KC + kc] = bfrag_adj<N>(C, mat, nt, kc, lane, A.dt);
    if (TILE_PRE) {
#pragma unroll
      for (int mat = 0; mat < 2; ++mat)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int kc = 0; kc < KC; ++kc) bpre[(mat * NT + nt) * KC + kc] = bfrag_pre<N>(C, mat, nt, kc, lane);
    }
  }
  auto bget = [&](int mat, int nt, int kc) -> double {
    if constexpr (EO && BSM) return sB[((mat * NT2 + nt) * KH + kc) * 32 + lane];
    else if constexpr (EO) return breg[(mat * NT2 + nt) * KH + kc];
    else if constexpr (BSM) return sB[((mat * NT + nt) * KC + kc) * 32 + lane];
    else return breg[(mat * NT + nt) * KC + kc];
  };
  auto bpget = [&](int mat, int nt, int kc) -> double {
    if constexpr (EO && BSM) return sB[(((6 + mat) * NT2 + nt) * KH + kc) * 32 + lane];
    else if constexpr (EO) return bpre[(mat * NT2 + nt) * KH + kc];
    else if constexpr (BSM) return sB[(((mat + 3) * NT + nt) * KC + kc) * 32 + lane];
    else return TILE_PRE ? bpre[(mat * NT + nt) * KC + kc] : breg[(mat * NT + nt) * KC + kc];
  };
  double minv_a[KC];
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int j = 4 * kc + kq;
    minv_a[kc] = C.minv[(j == 0 || j == N) ? 0 : j];
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_launch_dependents();               // PDL: the next step's prologue may start
  griddep_wait();                             // ... and this step's data path waits for ours
  if (tid == 0 && blockIdx.x < A.ntiles) {
    const TileLoad L = tile_load_plan(blockIdx.x, T, H, N, LEN, ndof);
    if (L.bulk) issue(L, 0);
  }
  unsigned fin = 0u;
  uint32_t phase = 0;
  double kv[WMT][KC], lnext[WMT][KC], lacc[WMT][KC];
  int it = 0;
  for (int t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++it) {
    const int bsel = it & 1;
    const TileLoad L = tile_load_plan(t, T, H, N, LEN, ndof);
    if (L.bulk) {
      while (!mbar_try_wait(&bar[bsel], (phase >> bsel) & 1u)) {
      }
      phase ^= (1u << bsel);
    } else {
      for (int k = tid; k < LEN; k += 32 * W) {
        int64_t g = L.g0 + k;
        while (g >= ndof) g -= ndof;
        sbu[bsel * PAD + k] = __ldg(A.u + g);
        sbl[bsel * PAD + k] = __ldg(A.lam + g);
        if (LD)
          for (int i = 1; i < S; ++i) sUs[(bsel * 3 + i - 1) * PAD + k] = __ldg(A.stin[i - 1] + g);
      }
      __syncthreads();
    }
    if (tid == 0 && t + (int)gridDim.x < A.ntiles) {
      const TileLoad Ln = tile_load_plan(t + gridDim.x, T, H, N, LEN, ndof);
      if (Ln.bulk) issue(Ln, bsel ^ 1);
    }
    su = sbu + bsel * PAD + L.sh;
    slam = sbl + bsel * PAD + L.sh;
    sUb = LD ? sUs + bsel * 3 * PAD + L.sh : sUs;
    if (tid == 0 && !LD)
      for (int i = 1; i < S; ++i) Uarr(i)[LEN - 1] = su[LEN - 1];   // never-owned last node
#pragma unroll
    for (int i = 0; i + 1 < S && !LD; ++i) {
      ring_rhs<N, WMT, decltype(bpget), false, TILE_PRE != 0, TILE_ILV != 0, EO>(C, Gt, Uarr(i), xfer, bpget, minv_a, mnu, warp, lane,
                                                              kv, fin);
      double* dst = Uarr(i + 1);
#pragma unroll
      for (int q = 0; q < WMT; ++q) {
        const int e = ring_elem<WMT, TILE_ILV != 0>(warp, q, rr);
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const int j = ring_node<N, EO>(kc, kq);
          if (j == N) continue;
          const int g = e * N + j;
          const double kk = kv[q][kc];
          double y;
          if (TB::nterm(i + 1) == 1) {
            y = __fma_rn(__dmul_rn(A.dt, TB::a(i + 1, i)), kk, su[g]);
          } else {
            double sacc = __dmul_rn(TB::a(i + 1, 0), (i == 0) ? kk : sk[g]);
#pragma unroll
            for (int jj = 1; jj <= i; ++jj)
              sacc = __fma_rn(TB::a(i + 1, jj), (jj == i) ? kk : sk[g], sacc);
            y = __fma_rn(A.dt, sacc, su[g]);
          }
          dst[g] = y;
          if (i == 0 && TB::keep(0)) sk[g] = kk;
        }
      }
      __syncthreads();
    }
    // z of stage i (unscaled; M^-1 rides on the J^T fragments): b_i lam + sum_{j>i} a_ji l_j
    // with l_{i+1} in lnext and (Kutta-3) l_{i+2} in sk
    auto zval = [&](int i, int g, int q, int kc) -> double {
      double z = __dmul_rn(TB::b(i), slam[g]);
      if (i + 1 < S && TB::a(i + 1, i) != 0.0) z = __fma_rn(TB::a(i + 1, i), lnext[q][kc], z);
      if (i + 2 < S && TB::a(i + 2, i) != 0.0) z = __fma_rn(TB::a(i + 2, i), sk[g], z);
      return z;
    };
#pragma unroll
    for (int q = 0; q < WMT; ++q) {
      const int e = ring_elem<WMT, TILE_ILV != 0>(warp, q, rr);
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int j = ring_node<N, EO>(kc, kq);
        if (j == N) continue;
        const int g = e * N + j;
        const double z = zval(S - 1, g, q, kc);
        if (e >= H && e < H + T) fin |= nonfinite_bit(z);
      }
    }
    // per stage: J^T apply (its internal barrier ends every read of sz), then accumulate l_i
    // and form z_{i-1} in the same pass -- two barriers per stage
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      if (i == S - 1)
        ring_jact<N, WMT, decltype(bget), false, TILE_ILV != 0, true, true, EO>(C, Gt, Uarr(i), slam, xfer, bget, mnu, warp,
                                                                         lane, kv, TB::b(S - 1));
      else
        ring_jact<N, WMT, decltype(bget), false, TILE_ILV != 0, true, false, EO>(C, Gt, Uarr(i), Uarr(i + 1), xfer, bget, mnu, warp,
                                                                   lane, kv);
      double* zdst = Uarr(i);                   // U_i is dead once its J^T has run
#pragma unroll
      for (int q = 0; q < WMT; ++q) {
        const int e = ring_elem<WMT, TILE_ILV != 0>(warp, q, rr);
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const int j = ring_node<N, EO>(kc, kq);
          if (j == N) continue;
          const int g = e * N + j;
          const double l = kv[q][kc];           // already dt * J^T(M^-1 z)
          lacc[q][kc] = (i == S - 1) ? l : __dadd_rn(lacc[q][kc], l);
          if (i + 1 < S && S == 3) sk[g] = lnext[q][kc];
          lnext[q][kc] = l;
          if (i == 0) {
            slam[g] = __dadd_rn(slam[g], lacc[q][kc]);
          } else {
            const double z = zval(i - 1, g, q, kc);
            if (e >= H && e < H + T) fin |= nonfinite_bit(z);
            zdst[g] = z;
          }
        }
      }
      if (i > 0 && tid == 0) zdst[TE * N] = 0.0;   // last node of the open chain
      __syncthreads();
    }
    const int64_t e_out0 = (int64_t)t * T;
    const int nout_el = (int)min((int64_t)T, G.E - e_out0);
    for (int k = tid; k < nout_el * N; k += 32 * W) A.out[e_out0 * N + k] = slam[H * N + k];
    __syncthreads();
  }
  if (fin) atomicOr(A.flag, SEM1D_FLAG_INPUT2_NONFINITE);
}

template <int N>
struct TileCfg {
  // forward: TE = 256 elements for N = 7 (8 warps x 4 m-tiles, 2 CTAs per SM: the second
  // CTA's DMMA fills the first one's barrier waits; A/B 0.48 vs 0.54 ms per RK4 step at
  // 16 x 4 x 1), 128 for N = 15/23 (N = 15: 8 warps x 2 interleaved m-tiles), 64 for N = 31;
  // adjoint: 256 for N = 7 (8 warps x 4 m-tiles, 2 CTAs per SM with the 7-slab layout:
  // 0.624 ms vs 0.649 at 8 x 2 x 3, 0.682 at 4 x 4 x 3), 128 / 64 otherwise (the slabs must
  // fit the shared memory of the resident CTAs)
  static constexpr int W = (N + 1) == 32 ? 8 : ((N + 1) == 8 ? TILE_WF8 : ((N + 1) == 16 ? TILE_WF16 : TILE_WF24));
  // adjoint warps: 8 x 2 m-tiles for N = 15/23 (at 16 warps the 128-register cap made the
  // compiler re-read the B fragments from kernel-parameter space with lane-divergent
  // indices inside the DMMA loops: 6.9x the forward step)
  static constexpr int W_A = (N + 1) == 8 ? TILE_WA8 : ((N + 1) == 32 ? 8 : TILE_WA16);
  static constexpr int WMT_F = (N + 1) == 8 ? TILE_WMT8 : ((N + 1) == 32 ? 1 : 16 / W);
  static constexpr int WMT_A = (N + 1) == 8 ? TILE_WMTA8 : ((N + 1) == 32 ? 1 : 128 / (8 * TILE_WA16));
  // adjoint step reading stored stage states (fewer DMMAs, 10-11 slabs): its own warp shape
  static constexpr int W_L = (N + 1) == 8 ? TILE_WL8 : W_A;
  static constexpr int WMT_L = (N + 1) == 8 ? TILE_WMTL8 : WMT_A;
  static constexpr int TE_L = 8 * W_L * WMT_L;
  static constexpr int PAD_L = ((TE_L * N + 1 + 2) + 1) & ~1;
  static constexpr int TE_F = 8 * W * WMT_F;
  static constexpr int TE_A = 8 * W_A * WMT_A;
  static constexpr int PAD_F = ((TE_F * N + 1 + 2) + 1) & ~1;
  static constexpr int PAD_A = ((TE_A * N + 1 + 2) + 1) & ~1;
  static constexpr size_t fwd_smem = sizeof(double) * (4 * (size_t)PAD_F + 32) + 2 * sizeof(uint64_t);
  static constexpr size_t BFRAG = ((N + 1) == 32) ? sizeof(double) * 5 * ((N + 1) / 8) * ((N + 1) / 4) * 32 + 16 : 0;
  // recompute mode: u, lam double-buffered + U_1..U_3 (+ k for Kutta-3); the bound covers every
  // scheme, adj_smem_s<SCH> is the launch size
  static constexpr size_t adj_smem = sizeof(double) * (8 * (size_t)PAD_A + 32) + 2 * sizeof(uint64_t) + BFRAG;
  template <int SCH>
  static constexpr size_t adj_smem_s() {
    return sizeof(double) * ((SCH == 1 ? 8 : 7) * (size_t)PAD_A + 32) + 2 * sizeof(uint64_t) + BFRAG;
  }
  // adjoint step reading the stored stage states at the W_L x WMT_L shape: u, lam, U_1..U_3
  // double-buffered (+ k for Kutta-3); z lives in the dead U slabs, so RK4 needs 10 slabs
  // (6 CTAs/SM) -- the bound below (11) covers every scheme
  static constexpr size_t adj_smem_ld = sizeof(double) * (11 * (size_t)PAD_L + 32) + 2 * sizeof(uint64_t) + BFRAG;
  template <int SCH>
  static constexpr size_t adj_smem_ld_s() {
    return sizeof(double) * ((SCH == 1 ? 11 : 10) * (size_t)PAD_L + 32) + 2 * sizeof(uint64_t) + BFRAG;
  }
  static constexpr int TE_MAX = TE_F > TE_A ? TE_F : TE_A;
};

template <int N>
constexpr size_t ens_smem_bytes(int ndof) {
  return sizeof(double) * (3 * (size_t)((ndof + 2 + 1) & ~1) + 32);
}

}  // namespace sem1d
