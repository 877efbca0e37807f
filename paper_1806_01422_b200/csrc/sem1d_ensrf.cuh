// sem1d_ensrf.cuh -- register-resident ensemble forward sweep for n = 16 (BASELINE config 4:
// 4096 periodic rings of 256 elements at N = 15, 1000 RK steps each).
//
// ens_forward_kernel keeps every stage state in shared memory: each stage reads its DMMA A
// fragments from there and writes the next stage state back, behind two CTA barriers.  Here
// the stage state never leaves the registers, as in tile_step_rf_kernel (sem1d_tilerf.cuh):
//  * With the permuted output columns of the ws kernels (bfrag_perm), lane (rr, kq) of an
//    m-tile receives rows 4kc + kq (kc = 0..3) of its element -- exactly the nodes it holds as
//    its A fragments.  So U[q][kc] = stage state at node 4kc + kq of element e(q, rr), updated
//    in place; node 15 of lane kq = 3 is a replica of the right neighbour's node 0.
//  * Interface node 0 of element e = row 15 of element e-1 (the same lane for q > 0 under the
//    interleaved mapping e = 32w + 4rr + q, a shuffle for q = 0, the left warp for rr = q = 0)
//    + row 0 of e, summed as (left + right) like every other gather here.
//  * The replica is refreshed after each stage update the same way in the other direction.
//  * The base state u_n stays in shared memory (read once per node and stage, written by the
//    last stage) and leaves for the trajectory with one bulk store per step.
// Same stage arithmetic, association and flag bits as ens_forward_kernel; with ENSRF_EO = 0
// the results are bit-identical to it.
//
// ENSRF_EO (default): F on the reflection (even/odd) split of K' = -nu M^-1 K and Dw' = M^-1 Dw
// (see bfrag_eo_value in sem1d_device.cuh): lane (rr, kq) holds the node pairs (j, 15 - j),
// j = 4kc + kq, kc < 2, forms s = u_j + u_{15-j} and d = u_j - u_{15-j}, and 8 DMMAs per
// m-tile and stage (Ke s, Ko d, De s, Do d; two k-chunks each) replace 16.  Rows 0 and 15 (the
// replica of the right neighbour's node 0) then both sit in lane kq = 0, so the interface sum
// of elements e-1 | e inside a lane needs no shuffle.  F differs from the full-matrix form in
// the last bits only (the same products, summed in a different order).
#pragma once

#include "sem1d_ensemble.cuh"

namespace sem1d {

// tested on config 4 against ens_forward_kernel; 0 restores the shared-memory kernel
#ifndef ENS_RF
#define ENS_RF 1
#endif
#ifndef ENSRF_NOBAR
#define ENSRF_NOBAR 0       // timing experiment only (wrong results): no stage barriers
#endif
#ifndef ENSRF_EO
#define ENSRF_EO 1
#endif
#ifndef ENSRF_MINB
#define ENSRF_MINB 2       // rings (CTAs) per SM; 3 (80 registers, 72-128 B of spills): 138.7 ms against 128.0 on config 4
#endif

struct EnsRf {
  static constexpr int N = 15, KC = 4, NT = 2, WMT = 4, W = 8, THREADS = 32 * W;
  static size_t smem(int ndof, bool rk3) {
    const size_t pad = (size_t)((ndof + 2 + 1) & ~1);
    return sizeof(double) * ((rk3 ? 3 : 2) * pad + 2 * W);
  }
};

template <int SCH>
__global__ void __launch_bounds__(EnsRf::THREADS, ENSRF_MINB)
    ens_forward_rf_kernel(const __grid_constant__ Consts<15> C, const Geo G, const EnsArgs A) {
  constexpr int N = EnsRf::N, KC = EnsRf::KC, NT = EnsRf::NT, WMT = EnsRf::WMT, W = EnsRf::W;
  using TB = TabC<SCH>;
  extern __shared__ __align__(16) double smem[];
  const int ndof = (int)G.ndof;
  const int pad = (ndof + 2 + 1) & ~1;
  double* su = smem;                                   // base state u_n (+ mirror of node 0)
  double* sacc = su + pad;                             // b_0 k_0 + b_1 k_1 + ... per node
  double* sk = sacc + pad;                             // k_0 (Kutta-3 only)
  double* xF = su + (SCH == 1 ? 3 : 2) * pad;          // [W] row 15 of each warp's last element
  double* xU = xF + W;                                 // [W] node 0 of each warp's first element

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  const int nw = (int)G.E / 32;                        // warps holding elements
  const bool act = warp < nw;
  const int64_t b = blockIdx.x, nb = gridDim.x;

  constexpr bool EO = ENSRF_EO != 0;
  // node held in U[q][kc]; where the node-15 replica sits (lane kq = RKQ, slot RKC)
  auto node = [&](int kc) -> int { return EO ? (kc < 2 ? 4 * kc + kq : N - (4 * (kc - 2) + kq)) : 4 * kc + kq; };
  constexpr int RKQ = EO ? 0 : 3, RKC = EO ? 2 : 3, RLANE = 28 + RKQ;
  // EO: bk[0] = Ke', bk[1] = Ko', bd[0] = De', bd[1] = Do' (two k-chunks each)
  double bk[NT][KC], bd[NT][KC];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      if (EO) {
        bk[nt][kc] = kc < 2 ? bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, 6 + nt, 0, kc, lane) : 0.0;
        bd[nt][kc] = kc < 2 ? bfrag_eo_value<N>(C.K, C.Dw, C.minv, C.nu, 8 + nt, 0, kc, lane) : 0.0;
      } else {
        bk[nt][kc] = bfrag_pre<N>(C, 0, nt, kc, lane);
        bd[nt][kc] = bfrag_pre<N>(C, 1, nt, kc, lane);
      }
    }

  const double* u0 = A.u0 + b * G.ndof;
  for (int k = tid; k < ndof; k += EnsRf::THREADS) su[k] = u0[k];
  if (tid == 0) su[ndof] = u0[0];
  fence_proxy_async_smem();                            // su writes -> visible to the bulk copy
  __syncthreads();
  // su -> HBM in one bulk copy (every writer of su has fenced and passed a barrier)
  auto store_state = [&](double* dst) {
    if (tid == 0) {
      bulk_s2g(dst, su, (uint32_t)(ndof * 8));
      bulk_commit();
    }
  };
  if (A.traj) store_state(A.traj + b * G.ndof);

  int ebase[WMT];
  // the stage state lives in registers; the slope accumulator (one read-modify-write per
  // node and stage) in shared memory, which keeps the kernel within 128 registers
  double U[WMT][KC];
#pragma unroll
  for (int q = 0; q < WMT; ++q) {
    ebase[q] = (32 * warp + 4 * rr + q) * N;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) U[q][kc] = act ? su[ebase[q] + node(kc)] : 0.0;
  }
  unsigned fin = 0u;
  bool bad_step = false;
  const int wl = (warp + nw - 1) % (nw > 0 ? nw : 1), wr = (warp + 1) % (nw > 0 ? nw : 1);

  for (int step = 0; step < A.nsteps; ++step) {
    const double dt = A.dts[step];
    if (A.traj) {                                      // last step's store has read su
      if (tid == 0) bulk_wait_read<0>();
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TB::s; ++i) {
      const bool last = i + 1 == TB::s;
      const double c1 = last ? 0.0 : __dmul_rn(dt, TB::a(i + 1, i));
      // stage arithmetic of one owned node (ens_forward_kernel's, statement for statement)
      auto upd = [&](int q, int kc, double kk) {
        const int g = ebase[q] + node(kc);
        const double acc = (i == 0) ? __dmul_rn(TB::b(i), kk) : __fma_rn(TB::b(i), kk, sacc[g]);
        if (!last) {
          sacc[g] = acc;
          double y;
          if (TB::nterm(i + 1) == 1) {
            y = __fma_rn(c1, kk, su[g]);
          } else {
            double sacc = __dmul_rn(TB::a(i + 1, 0), (i == 0) ? kk : sk[g]);
#pragma unroll
            for (int jj = 1; jj <= i; ++jj) sacc = __fma_rn(TB::a(i + 1, jj), (jj == i) ? kk : sk[g], sacc);
            y = __fma_rn(dt, sacc, su[g]);
          }
          U[q][kc] = y;
          if (i == 0 && TB::keep(0)) sk[g] = kk;
        } else {
          const double un = __fma_rn(dt, acc, su[g]);
          bad_step |= nonfinite_bit(un) != 0u;
          su[g] = un;
          U[q][kc] = un;
        }
      };
      // (1) F of every m-tile; all owned nodes but the interface node 0 updated at once
      double F0[WMT], RN[WMT];
      if (act) {
#pragma unroll
        for (int q = 0; q < WMT; ++q) {
#pragma unroll
          for (int kc = 0; kc < KC; ++kc) fin |= nonfinite_bit(U[q][kc]);
          double Fv[KC];
          if (EO) {
            double ke[2] = {0.0, 0.0}, ko[2] = {0.0, 0.0}, pe[2] = {0.0, 0.0}, po[2] = {0.0, 0.0};
#pragma unroll
            for (int kc = 0; kc < 2; ++kc) {
              const double sv = __dadd_rn(U[q][kc], U[q][2 + kc]), dv = __dsub_rn(U[q][kc], U[q][2 + kc]);
              dmma884(ke[0], ke[1], sv, bk[0][kc]);
              dmma884(ko[0], ko[1], dv, bk[1][kc]);
              dmma884(pe[0], pe[1], sv, bd[0][kc]);
              dmma884(po[0], po[1], dv, bd[1][kc]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {            // rows 4h + kq and 15 - (4h + kq)
              Fv[h] = __fma_rn(-U[q][h], __dadd_rn(pe[h], po[h]), __dadd_rn(ke[h], ko[h]));
              Fv[2 + h] = __fma_rn(-U[q][2 + h], __dsub_rn(po[h], pe[h]), __dsub_rn(ke[h], ko[h]));
            }
          } else
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            double k0 = 0.0, k1 = 0.0, p0 = 0.0, p1 = 0.0;
#pragma unroll
            for (int kc = 0; kc < KC; ++kc) {
              dmma884(k0, k1, U[q][kc], bk[nt][kc]);
              dmma884(p0, p1, U[q][kc], bd[nt][kc]);
            }
            Fv[2 * nt] = __fma_rn(-U[q][2 * nt], p0, k0);
            Fv[2 * nt + 1] = __fma_rn(-U[q][2 * nt + 1], p1, k1);
          }
          F0[q] = Fv[0];
          RN[q] = Fv[RKC];
#pragma unroll
          for (int kc = 1; kc < KC; ++kc)
            if (kc != RKC || kq != RKQ) upd(q, kc, Fv[kc]);
        }
        if (lane == RLANE) xF[warp] = RN[WMT - 1];
      }
      if (!ENSRF_NOBAR) __syncthreads();
      // (2) interface nodes: + row 15 of the left element
      if (act) {
#pragma unroll
        for (int q = 0; q < WMT; ++q) {
          double left = q > 0 ? (EO ? RN[q - 1] : __shfl_down_sync(0xffffffffu, RN[q - 1], 3))
                              : __shfl_sync(0xffffffffu, RN[WMT - 1], 4 * ((rr + 7) & 7) + RKQ);
          if (q == 0 && lane == 0) left = xF[wl];
          upd(q, 0, kq == 0 ? __dadd_rn(left, F0[q]) : F0[q]);
        }
        if (lane == 0) xU[warp] = U[0][0];
      }
      if (last && A.traj) fence_proxy_async_smem();    // this step's su writes -> bulk store
      if (!ENSRF_NOBAR || last) __syncthreads();
      // (3) refresh the node-15 replicas: node 0 of the right element
      if (act) {
#pragma unroll
        for (int q = 0; q < WMT; ++q) {
          double right = q + 1 < WMT ? (EO ? U[q + 1 < WMT ? q + 1 : 0][0]
                                           : __shfl_up_sync(0xffffffffu, U[q + 1 < WMT ? q + 1 : 0][0], 3))
                                     : __shfl_sync(0xffffffffu, U[0][0], 4 * ((rr + 1) & 7));
          if (q == WMT - 1 && lane == RLANE) right = xU[wr];
          if (kq == RKQ) U[q][RKC] = right;
        }
      }
    }
    if (A.traj) store_state(A.traj + ((int64_t)(step + 1) * nb + b) * G.ndof);
  }
  if (A.traj && tid == 0) bulk_wait_read<0>();
  __syncthreads();
  double* uf = A.u_final + b * G.ndof;
  for (int k = tid; k < ndof; k += EnsRf::THREADS) uf[k] = su[k];
  if (tid == 0) bulk_wait_all();
  const bool bad_in = fin != 0u;
  if (bad_in || bad_step)
    atomicOr(&A.flags[b], (bad_in ? SEM1D_FLAG_STATE_NONFINITE : 0) | (bad_step ? SEM1D_FLAG_STEP_NONFINITE : 0));
}

}  // namespace sem1d
