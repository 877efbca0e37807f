// sem1d_tilerf.cuh -- register-resident temporally blocked RK steps for N = 7
// (n = 8 GLL points), the config-2/config-5 degree.
//
// Why a second tile kernel.  On sm_100a the FP64 tensor-core op (DMMA m8n8k4) and
// DFMA/DMUL/DADD share ONE issue resource: 4 DMMA + 32 DFMA per warp cost 143
// sub-partition cycles against 65 + 66 alone (tools/fp64_pipes.cu,
// profiles/r2_fp64_pipes.jsonl).  The shared-memory tile kernel (tile_step_kernel)
// spent 151 pipe-cycles per m-tile and stage against a 90-cycle floor: every stage
// round-tripped its state through shared memory behind two CTA-wide barriers, so the
// eight warps ran their DMMA phases in lock step and left the pipe idle in between.
//
// Here a stage never leaves the registers:
//  * Lane (rr, kq) of warp w holds, for m-tile q = 0..3, element e = 32w + 4rr + q
//    (the interleaved ring_elem mapping) at nodes kq and 7-kq.  The DMMA A fragment of
//    k-chunk 0 is node kq, of chunk 1 node 7-kq; the B fragments are permuted to match,
//    and the output columns are permuted so that the lane receives rows kq and 7-kq of
//    K u and Dw u -- the nodes it holds.  Lane kq = 0 holds both interface nodes 0 and 7.
//  * Interface node of elements e-1 | e: row 7 of e-1 and row 0 of e sit in the SAME
//    lane for q > 0, one shuffle for q = 0, one exchange with the left warp for the
//    warp's first element.  The replica of node 7 (the right neighbour's node 0) is
//    refreshed the same way after the stage update.
//  * The two warp-boundary exchanges of a stage use pairwise named barriers (bar.arrive
//    / bar.sync over 64 threads) between neighbouring warps instead of __syncthreads, so
//    warps drift against each other and one warp's pointwise epilogue overlaps another
//    warp's DMMAs.
//  * -nu M^-1 / M^-1 ride on the B fragments (row scaling, the bfrag_pre values); the
//    stage arithmetic is fused: F = fma(-u, Dw'u, K'u), acc = fma(b_i, F, acc),
//    U_{i+1} = fma(dt a_{i+1,i}, F, u), u_new = fma(dt, acc, u).
//  * Non-finite checks: CHK = 0 checks only the owned outputs (a non-finite stage input
//    always makes an owned output non-finite: NaN/Inf propagate through every term of
//    the step, and every b_i != 0), setting SEM1D_FLAG_STEP_NONFINITE; the run-ahead
//    integrate re-runs a flagged step with CHK = 1, which also classifies non-finite
//    stage inputs (SEM1D_FLAG_STATE_NONFINITE) and gives bitwise the same state.
//  * Tiles of 256 elements (H = s ghost elements per side) arrive by one bulk copy,
//    double-buffered; lanes read their values once per tile and store the owned
//    results straight from registers (each 32-byte sector fully written).
#pragma once

#include "sem1d_ensemble.cuh"

namespace sem1d {

// RF_BAR_NA: the non-.aligned barrier forms (no convergence requirement, so no divergence
// checks around them); RF_NOBAR / RF_NOSTORE: timing experiments only (wrong results)
#ifndef RF_BAR_NA
#define RF_BAR_NA 1
#endif
#ifndef RF_NOBAR
#define RF_NOBAR 0
#endif
#ifndef RF_NOSTORE
#define RF_NOSTORE 0
#endif
// RF_BULKOUT: results leave through shared memory and one bulk store per warp (the owned
// node range of its 32 elements is contiguous in HBM) instead of 8 scattered 32-byte
// register stores per lane
#ifndef RF_BULKOUT
#define RF_BULKOUT 1
#endif
__device__ __forceinline__ void nbar_arrive(int id, int nthreads) {
  if (RF_NOBAR) return;
  if (RF_BAR_NA) asm volatile("barrier.cta.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
  else asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void nbar_sync(int id, int nthreads) {
  if (RF_NOBAR) return;
  if (RF_BAR_NA) asm volatile("barrier.cta.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int WMT_ = 4>
struct RfCfg {
  static constexpr int N = 7, W = 8, WMT = WMT_, TE = 8 * W * WMT;   // 256 elements per tile at WMT 4
  static constexpr int LEN = TE * N + 1;
  static constexpr int PAD = ((LEN + 2) + 1) & ~1;
  // named barriers: 1..7 carry F (row 7) from warp w to w+1, 8..14 carry U (node 0) back
  static constexpr int BAR_F = 1, BAR_U = 8;
  // tile loads [2][PAD], output staging [2][PAD], exchange slots, 4 mbarriers
  static constexpr size_t smem = sizeof(double) * (4 * (size_t)PAD + 32) + 4 * sizeof(uint64_t);
};

// B fragment of the reflected layout: output column c -> row (c even ? c/2 : 7 - c/2),
// k-chunk 0 input node k, chunk 1 node 7 - k; row i scaled by -nu M^-1_i (K) or M^-1_i (Dw),
// the same one-rounding values as bfrag_pre
__device__ __forceinline__ double bfrag_rf(const Consts<7>& C, int mat, int kc, int lane) {
  const int c = lane >> 2, k = lane & 3;
  const int i = (c & 1) ? 7 - (c >> 1) : (c >> 1);
  const int j = kc == 0 ? k : 7 - k;
  const double mi = C.minv[(i == 0 || i == 7) ? 0 : i];
  return mat == 0 ? __dmul_rn(C.K[i * 8 + j], __dmul_rn(-C.nu, mi)) : __dmul_rn(C.Dw[i * 8 + j], mi);
}

// SCH: compile-time tableau (TabC); STG: also store U_1..U_{s-1}; CHK: classify stage inputs;
// WMT: m-tiles (8 elements each) per warp; MINB: resident CTAs per SM
template <int SCH, bool STG, bool CHK, int WMT, int MINB>
__global__ void __launch_bounds__(32 * RfCfg<WMT>::W, MINB)
    tile_step_rf_kernel(const __grid_constant__ Consts<7> C, const Geo G, const TileStepArgs A) {
  using CF = RfCfg<WMT>;
  constexpr int N = 7, W = CF::W, TE = CF::TE, LEN = CF::LEN, PAD = CF::PAD;
  using TB = TabC<SCH>;
  constexpr int S = TB::s, H = S, T = TE - 2 * H;
  extern __shared__ __align__(16) double smem[];
  double* sbuf = smem;                        // [2][PAD] tile loads
  double* sout = sbuf + 2 * PAD;              // [2][PAD] output staging (bulk stores)
  double* xF = sout + 2 * PAD;                // [16] row 7 of each warp's last element
  double* xU = xF + 16;                       // [16] node 0 of each warp's first element
  uint64_t* full = reinterpret_cast<uint64_t*>(xU + 16);
  uint64_t* empty = full + 2;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  const int e_lane = 8 * WMT * w + WMT * rr;  // tile element of m-tile 0 in this lane
  const int64_t ndof = G.ndof;
  double bk[2], bd[2];
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    bk[kc] = bfrag_rf(C, 0, kc, lane);
    bd[kc] = bfrag_rf(C, 1, kc, lane);
  }
  const double dt = A.dt;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], W);
    mbar_init(&empty[1], W);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_launch_dependents();               // PDL: the next step's prologue may start
  griddep_wait();                             // ... and this step's data path waits for ours
  // full[x]: a bulk tile landed in buffer x (phase bit per buffer, toggled by every waiter);
  // empty[x]: all W warps have read it (tracked by the issuing thread: pend = a bulk tile
  // was issued into x and its readers' arrivals are still owed)
  uint32_t fphase = 0u, ephase = 0u, pend = 0u;
  if (tid == 0 && blockIdx.x < A.ntiles) {
    const TileLoad L = tile_load_plan(blockIdx.x, T, H, N, LEN, ndof);
    if (L.bulk) {
      tile_issue(L, LEN, A.u, sbuf, &full[0], 1, nullptr, nullptr);
      pend |= 1u;
    }
  }
  unsigned bad_state = 0u, bad_out = 0u;
  int it = 0;
  for (int t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++it) {
    const int b = it & 1;
    const TileLoad L = tile_load_plan(t, T, H, N, LEN, ndof);
    double u0[WMT][2], U[WMT][2], acc[WMT][2], F[WMT][2];
    double k0[(SCH == 1) ? WMT : 1][2];       // Kutta-3: k_0 enters the third stage's row
    if (L.bulk) {
      while (!mbar_try_wait(&full[b], (fphase >> b) & 1u)) {
      }
      fphase ^= 1u << b;
      const double* su = sbuf + b * PAD + L.sh;
#pragma unroll
      for (int q = 0; q < WMT; ++q) {
        u0[q][0] = su[(e_lane + q) * N + kq];
        u0[q][1] = su[(e_lane + q) * N + 7 - kq];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);   // this warp is done with buffer b
    } else {                                   // tile wraps around the ring end: direct loads
#pragma unroll
      for (int q = 0; q < WMT; ++q) {
        int64_t g0 = L.g0 + (e_lane + q) * N + kq, g1 = L.g0 + (e_lane + q) * N + 7 - kq;
        while (g0 >= ndof) g0 -= ndof;
        while (g1 >= ndof) g1 -= ndof;
        u0[q][0] = __ldg(A.u + g0);
        u0[q][1] = __ldg(A.u + g1);
      }
    }
    // prefetch the next tile into the other buffer once every warp has read its last tile
    if (tid == 0 && t + (int)gridDim.x < A.ntiles) {
      const TileLoad Ln = tile_load_plan(t + gridDim.x, T, H, N, LEN, ndof);
      if (Ln.bulk) {
        const int x = b ^ 1;
        if (pend & (1u << x)) {
          while (!mbar_try_wait(&empty[x], (ephase >> x) & 1u)) {
          }
          ephase ^= 1u << x;
        }
        tile_issue(Ln, LEN, A.u, sbuf + x * PAD, &full[x], 1, nullptr, nullptr);
        pend |= 1u << x;
      }
    }
    // owned elements of this lane: tile element e in [H, H+T) and inside the ring
    const int64_t e_base = (int64_t)t * T - H;
    bool own[WMT];
#pragma unroll
    for (int q = 0; q < WMT; ++q) {
      const int e = e_lane + q;
      own[q] = e >= H && e < H + T && e_base + e < G.E;
      U[q][0] = u0[q][0];
      U[q][1] = u0[q][1];
    }
    // owned node range of this warp's elements, and the staging offset that gives the
    // shared-memory copy the parity of its global node index (16-byte bulk alignment)
    const int e_lo = max(8 * WMT * w, H);
    const int e_hi = (int)min((int64_t)min(8 * WMT * (w + 1), H + T), (int64_t)G.E - e_base);
    const int64_t gbase = e_base * N - ((e_base * N) & 1);   // even; staging index = g - gbase
    int obuf = 0;
    // write the owned values of v (one stage state or the new state) to dst[0..ndof)
    auto put = [&](const double (&v)[WMT][2], double* dst) {
      if (!RF_BULKOUT) {
#pragma unroll
        for (int q = 0; q < WMT; ++q) {
          if (!own[q]) continue;
          const int64_t g = (e_base + e_lane + q) * N;
          if (RF_NOSTORE && v[q][0] != 1.2345e300) continue;
          dst[g + kq] = v[q][0];
          if (kq != 0) dst[g + 7 - kq] = v[q][1];
        }
        return;
      }
      if (e_hi <= e_lo) return;                  // warp owns nothing (tile edge / ring end)
      double* so = sout + obuf * PAD;
      obuf ^= 1;
      if (lane == 0) bulk_wait_read<1>();        // the store out of this buffer two uses ago
      __syncwarp();
#pragma unroll
      for (int q = 0; q < WMT; ++q) {
        if (!own[q]) continue;
        const int64_t i0 = (e_base + e_lane + q) * N - gbase;
        so[i0 + kq] = v[q][0];
        if (kq != 0) so[i0 + 7 - kq] = v[q][1];
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int64_t g0 = (e_base + e_lo) * N, g1 = (e_base + e_hi) * N;
        const int64_t ga = (g0 + 1) & ~(int64_t)1, gb = g1 & ~(int64_t)1;
        if (g0 != ga) dst[g0] = so[g0 - gbase];
        if (g1 != gb) dst[gb] = so[gb - gbase];
        if (gb > ga) {
          bulk_s2g(dst + ga, so + (ga - gbase), (uint32_t)((gb - ga) * 8));
          bulk_commit();
        }
      }
    };
    auto mtile_F = [&](int q) {
      double ka = 0.0, kb = 0.0, da = 0.0, db = 0.0;
      dmma884(ka, kb, U[q][0], bk[0]);
      dmma884(da, db, U[q][0], bd[0]);
      dmma884(ka, kb, U[q][1], bk[1]);
      dmma884(da, db, U[q][1], bd[1]);
      F[q][0] = __fma_rn(-U[q][0], da, ka);     // node kq   (M^-1-scaled F)
      F[q][1] = __fma_rn(-U[q][1], db, kb);     // node 7-kq
    };
#pragma unroll
    for (int st = 0; st < S; ++st) {
      if (CHK) {
#pragma unroll
        for (int q = 0; q < WMT; ++q)
          if (own[q]) bad_state |= nonfinite_bit(U[q][0]) | (kq != 0 ? nonfinite_bit(U[q][1]) : 0u);
      }
      const bool last = st + 1 == S;
      const double bi = TB::b(st);
      const double c1 = last ? 0.0 : __dmul_rn(dt, TB::a(st + 1, st));
      auto update = [&](int q) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double k = F[q][h];
          acc[q][h] = (st == 0) ? __dmul_rn(bi, k) : __fma_rn(bi, k, acc[q][h]);
          if (!last) {
            if (TB::nterm(st + 1) == 1) {
              U[q][h] = __fma_rn(c1, k, u0[q][h]);
            } else {                              // Kutta-3 row 2: u + dt (a20 k0 + a21 k1)
              const double s = __fma_rn(TB::a(st + 1, st), k, __dmul_rn(TB::a(st + 1, 0), k0[q][h]));
              U[q][h] = __fma_rn(dt, s, u0[q][h]);
            }
            if (SCH == 1 && st == 0) k0[q][h] = k;
          } else {
            U[q][h] = __fma_rn(dt, acc[q][h], u0[q][h]);
          }
        }
      };
      // (1) the warp's last m-tile first: its row 7 is what the right warp waits for
      mtile_F(WMT - 1);
      double left = __shfl_up_sync(0xffffffffu, F[WMT - 1][1], 4);
      if (w < W - 1) {
        if (lane == 28) xF[w] = F[WMT - 1][1];
        if (!RF_BAR_NA) __syncwarp();
        nbar_arrive(CF::BAR_F + w, 64);
      }
      // (2) the other m-tiles
#pragma unroll
      for (int q = 0; q + 1 < WMT; ++q) mtile_F(q);
      // (3) interface node 0 of element e: + row 7 of element e-1 (lane kq = 0 holds both)
      if (w > 0) {
        nbar_sync(CF::BAR_F + w - 1, 64);
        if (lane == 0) left = xF[w - 1];
      } else if (lane == 0) {
        left = 0.0;                             // tile edge: ghost element, left incomplete
      }
      if (kq == 0) {
#pragma unroll
        for (int q = WMT - 1; q > 0; --q) F[q][0] = __dadd_rn(F[q - 1][1], F[q][0]);
        F[0][0] = __dadd_rn(left, F[0][0]);
      }
      // (4) stage update, m-tile 0 first: its node 0 is what the left warp waits for.  The
      // pairwise barriers also run after the last stage: warp w may arrive on BAR_F + w of the
      // next stage only after warp w+1 has passed this stage's sync on it (otherwise two of
      // w's arrivals could complete one barrier generation)
      update(0);
      double right = __shfl_down_sync(0xffffffffu, U[0][0], 4);
      if (w > 0) {
        if (!last && lane == 0) xU[w] = U[0][0];
        if (!RF_BAR_NA) __syncwarp();
        nbar_arrive(CF::BAR_U + w - 1, 64);
      }
#pragma unroll
      for (int q = 1; q < WMT; ++q) update(q);
      // (5) refresh the node-7 replica of lane kq = 0: node 0 of the right neighbour
      if (w < W - 1) {
        nbar_sync(CF::BAR_U + w, 64);
        if (lane == 28) right = xU[w + 1];
      }
      if (!last) {
        if (kq == 0) {
#pragma unroll
          for (int q = 0; q + 1 < WMT; ++q) U[q][1] = U[q + 1][0];
          U[WMT - 1][1] = right;
        }
        if (STG) put(U, A.stages[st]);            // stage state U_{st+1}, owned nodes
      }
    }
#pragma unroll
    for (int q = 0; q < WMT; ++q)
      if (own[q]) bad_out |= nonfinite_bit(U[q][0]) | (kq != 0 ? nonfinite_bit(U[q][1]) : 0u);
    put(U, A.out);
  }
  if (RF_BULKOUT && lane == 0) bulk_wait_all();  // every bulk store has left shared memory
  const unsigned bits = (bad_state ? SEM1D_FLAG_STATE_NONFINITE : 0u) | (bad_out ? SEM1D_FLAG_STEP_NONFINITE : 0u);
  const unsigned any = __reduce_or_sync(0xffffffffu, bits);
  if (lane == 0 && any) atomicOr(A.flag, (int)any);
}

}  // namespace sem1d
