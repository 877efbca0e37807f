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
// RF_FWD_X1: the forward step's exchanges in the single-round form of the adjoint step
// (1; A/B against the two-round form, 0)
#ifndef RF_FWD_X1
#define RF_FWD_X1 1
#endif
#ifndef RF_NOCHK
#define RF_NOCHK 0          // timing experiment: no non-finite checks in the adjoint step
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

// RF_EO: F's two contractions on the reflection (even/odd) split.  The GLL nodes and weights
// are symmetric about the element midpoint, so K' = -nu M^-1 K is centrosymmetric
// (K'[7-i][7-j] = K'[i][j]) and Dw' = M^-1 Dw anti-centrosymmetric (Dw'[7-i][7-j] = -Dw'[i][j]);
// with s_j = u_j + u_{7-j}, d_j = u_j - u_{7-j} (j < 4):
//   (K'u)_i = (Ke s)_i + (Ko d)_i,  (K'u)_{7-i} = (Ke s)_i - (Ko d)_i,
//   (Dw'u)_i = (De s)_i + (Do d)_i, (Dw'u)_{7-i} = (Do d)_i - (De s)_i,
// four 4x4 blocks.  K and Dw share the input u, so ONE DMMA m8n8k4 on s gives Ke s and De s
// (output columns 2i and 2i+1) and one on d gives Ko d and Do d: 2 DMMAs per m-tile instead of
// 4, for 6 extra FP64 adds (the DMMA costs 16 sub-partition cycles of the FP64 datapath that
// DADD/DFMA share, a DADD 2).  The blocks are formed from both halves of the matrices
// (symmetrised: the host matrices are centrosymmetric to about one ulp only).
#ifndef RF_EO
#define RF_EO 1
#endif
__device__ __forceinline__ double bfrag_eo(const Consts<7>& C, int par, int lane) {
  const int c = lane >> 2, j = lane & 3, i = c >> 1;
  auto mi = [&](int r) { return C.minv[(r == 0 || r == 7) ? 0 : r]; };
  // exact products summed in double-double and rounded once (eo_block_entry, sem1d_device.cuh)
  if ((c & 1) == 0) {                           // K' blocks
    auto kp = [&](int r, int s) -> DD { return dd_mul(dd_two_prod(-C.nu, mi(r)), C.K[r * 8 + s]); };
    return eo_block_entry(kp, true, par, i, j, 7);
  }
  auto dp = [&](int r, int s) -> DD { return dd_two_prod(C.Dw[r * 8 + s], mi(r)); };   // Dw' blocks
  return eo_block_entry(dp, false, par, i, j, 7);
}
// F at nodes kq / 7-kq of the lane's element from its two node values (RF_EO split); dw0/dw1
// receive Dw'u at the two nodes
__device__ __forceinline__ void f_eo(double u0, double u1, double be, double bo, double& f0, double& f1,
                                     double& dw0, double& dw1) {
  const double s = __dadd_rn(u0, u1), d = __dsub_rn(u0, u1);
  double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
  dmma884(p0, p1, s, be);                       // (Ke s)_kq, (De s)_kq
  dmma884(q0, q1, d, bo);                       // (Ko d)_kq, (Do d)_kq
  dw0 = __dadd_rn(p1, q1);
  dw1 = __dsub_rn(q1, p1);
  f0 = __fma_rn(-u0, dw0, __dadd_rn(p0, q0));
  f1 = __fma_rn(-u1, dw1, __dsub_rn(p0, q0));
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
  double* xF = sout + 2 * PAD;                // [2][8] raw row 7 of each warp's last element
  double* xU = xF + 16;                       // [2][8] raw row 0 of each warp's first element
  uint64_t* full = reinterpret_cast<uint64_t*>(xU + 16);
  uint64_t* empty = full + 2;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  const int e_lane = 8 * WMT * w + WMT * rr;  // tile element of m-tile 0 in this lane
  const int64_t ndof = G.ndof;
  double bk[2], bd[2];
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    bk[kc] = RF_EO ? bfrag_eo(C, kc, lane) : bfrag_rf(C, 0, kc, lane);
    bd[kc] = RF_EO ? 0.0 : bfrag_rf(C, 1, kc, lane);
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
  // tiles k = 0..cnt-1 of the launch are ring tiles (tile_lo + k) mod ntiles (a sharded
  // step launches its interior tiles while the ghost exchange runs, then the edge tiles)
  const int cnt = A.tile_cnt > 0 ? A.tile_cnt : A.ntiles;
  auto tile_of = [&](int k) {
    const int t = A.tile_lo + k;                // < 2 ntiles
    return t >= A.ntiles ? t - A.ntiles : t;
  };
  if (tid == 0 && (int)blockIdx.x < cnt) {
    const TileLoad L = tile_load_plan(tile_of(blockIdx.x), T, H, N, LEN, ndof);
    if (L.bulk) {
      tile_issue(L, LEN, A.u, sbuf, &full[0], 1, nullptr, nullptr);
      pend |= 1u;
    }
  }
  unsigned bad_state = 0u, bad_out = 0u;
  int xpar = 0;                               // exchange-slot parity (one flip per stage)
  int it = 0;
  for (int k = blockIdx.x; k < cnt; k += gridDim.x, ++it) {
    const int t = tile_of(k);
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
    if (tid == 0 && k + (int)gridDim.x < cnt) {
      const TileLoad Ln = tile_load_plan(tile_of(k + gridDim.x), T, H, N, LEN, ndof);
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
      if (RF_EO) {
        double d0, d1;
        f_eo(U[q][0], U[q][1], bk[0], bk[1], F[q][0], F[q][1], d0, d1);
        return;
      }
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
      // the run-ahead form (no checks, no stage stores) keeps the two-round exchange: the
      // single round measured 208.0 against 206.8 us there, 213.7 against 226.8 us with the
      // checks and 268.8 against 271.5 us storing the stages (tools/tile_ab.py)
      if constexpr (!(RF_FWD_X1 && (CHK || STG))) {
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
      } else {
        // (1) the warp's last m-tile first: its raw row 7 is what the right warp waits for
        mtile_F(WMT - 1);
        double left = __shfl_up_sync(0xffffffffu, F[WMT - 1][1], 4);
        if (w < W - 1) {
          if (lane == 28) xF[xpar * 8 + w] = F[WMT - 1][1];
          if (!RF_BAR_NA) __syncwarp();
          nbar_arrive(CF::BAR_F + w, 64);
        }
        // (2) the other m-tiles
#pragma unroll
        for (int q = 0; q + 1 < WMT; ++q) mtile_F(q);
        // (3) ONE pairwise exchange per stage (as in tile_adj_rf_kernel): raw row 7 of the left
        // warp's last element, raw row 0 of the right warp's first; the interface sum of
        // elements e-1 | e (row 7 + row 0, raw, in this order) is formed both by the owner of
        // node 0 of e and by the node-7 replica of e-1, so the replica's next stage state is
        // bitwise the owner's and no exchange of updated states is needed.  Barrier order:
        // arrive BAR_F+w, sync BAR_F+w-1, arrive BAR_U+w-1, sync BAR_U+w (no warp can arrive
        // twice on one barrier generation); slots double-buffered by stage parity.
        double rawr = __shfl_down_sync(0xffffffffu, F[0][0], 4);
        if (w > 0) {
          nbar_sync(CF::BAR_F + w - 1, 64);
          if (lane == 0) left = xF[xpar * 8 + w - 1];
          if (lane == 0) xU[xpar * 8 + w] = F[0][0];
          if (!RF_BAR_NA) __syncwarp();
          nbar_arrive(CF::BAR_U + w - 1, 64);
        } else if (lane == 0) {
          left = 0.0;                             // tile edge: ghost element, left incomplete
        }
        if (kq == 0) {
#pragma unroll
          for (int q = WMT - 1; q > 0; --q) F[q][0] = __dadd_rn(F[q - 1][1], F[q][0]);
          F[0][0] = __dadd_rn(left, F[0][0]);
          if (!last) {                            // replicas inside the lane: the same sums
#pragma unroll
            for (int q = 0; q + 1 < WMT; ++q) F[q][1] = F[q + 1][0];
          }
        }
        // (4) stage update; the last m-tile's replica needs the right warp's raw row 0
#pragma unroll
        for (int q = 0; q + 1 < WMT; ++q) update(q);
        if (w < W - 1) {
          nbar_sync(CF::BAR_U + w, 64);
          if (lane == 28) rawr = xU[xpar * 8 + w + 1];
        }
        if (!last && kq == 0) F[WMT - 1][1] = __dadd_rn(F[WMT - 1][1], rawr);
        update(WMT - 1);
        xpar ^= 1;
        if (!last && STG) put(U, A.stages[st]);   // stage state U_{st+1}, owned nodes
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

// ============================================================================
// Register-resident adjoint step for N = 7 (the transpose of tile_step_rf_kernel's step,
// adjoint.py:54-61 generalised to the tableau):
//   l_i = dt J^T(U_i) (b_i lam + sum_{j>i} a_ji l_j),   lam_n = lam + l_{s-1} + ... + l_0.
// Same lane layout, reflected fragments and pairwise warp exchanges as the forward kernel.
// LD = 0: the stage states are recomputed (forward stages 0..s-2, H = 2s-1 ghost elements per
// side); U_1..U_{s-2} wait in a per-lane shared-memory slot, U_{s-1} stays in registers.
// LD = 1: U_1..U_{s-1} arrive with the tile (stored by the forward step, H = s).
// J^T fragments fold dt and M^-1 (bfrag_adj values; Dw^T negated), so one accumulator
// chain gives term1 - term3 of ops.py:195-212 and l = fma(-z, dt M^-1 Dw u, C).
// Checks (the reference's per-call ones): a non-finite stage state sets the STATE bit, a
// non-finite stage input z the INPUT2 ("cotangent") bit.
// ============================================================================
// The adjoint kernel runs the stage recurrence on w_i = z_i / b_i and l'_i = l_i / b_i:
//   w_i = lam + sum_{j>i} (a_ji b_j / b_i) l'_j,   l'_i = dt J^T(U_i) w_i,   lam_n = lam + sum b_i l'_i,
// which saves the b_i * lam multiply of every node and stage (w_{s-1} = lam).  The ratios are
// exact binary fractions for the three tableaux: RK4 1/2, 1/2, 1; Kutta-3 1/2, 2, -1.
template <int SCH>
struct TabW {
  __host__ __device__ static constexpr double c(int i, int j) {   // coefficient of l'_j in w_i
    return SCH == 2 ? ((i == 2 && j == 3) ? 0.5 : (i == 1 && j == 2) ? 0.5 : (i == 0 && j == 1) ? 1.0 : 0.0)
         : SCH == 1 ? ((i == 1 && j == 2) ? 0.5 : (i == 0 && j == 1) ? 2.0 : (i == 0 && j == 2) ? -1.0 : 0.0)
                    : 0.0;
  }
};

// exponent bits of a double if it may raise a flag (owned node), else 0: max-accumulated,
// the result is non-finite iff it reaches 0x7ff00000 (two integer ops per checked value)
__device__ __forceinline__ unsigned expbits(double x, unsigned mask) {
  return (unsigned)__double2hiint(x) & mask;
}

template <int WMT_ = 4>
struct RfAdjCfg {
  static constexpr int N = 7, W = 8, WMT = WMT_, TE = 8 * W * WMT;
  static constexpr int LEN = TE * N + 1;
  static constexpr int PAD = ((LEN + 2) + 1) & ~1;
  static constexpr int SLOT = W * 32 * WMT * 2;   // doubles of one per-lane stage slot
  // slabs [2 buffers][u, lam (, U_1..U_3)] + per-lane slots (recompute) + exchange + barriers
  // recompute mode: U_1, U_2 and (DR) the stage recompute's M^-1 Dw U_i, i = 0..2, per lane
  template <bool LD, bool DR = false>
  static constexpr size_t smem() {
    return sizeof(double) * ((size_t)2 * (LD ? 5 : 2) * PAD + (LD ? 0 : (DR ? 5 : 2) * (size_t)SLOT) + 32) +
           4 * sizeof(uint64_t);
  }
};

// J^T fragments without dt (the stage recurrence's coefficients carry it): K column j by
// -nu M^-1_j, Dw^T column j by -M^-1_j; the z o (Dw u) term uses the forward kernel's
// M^-1-row-scaled Dw fragment (bfrag_rf mat 1), whose output the stage recompute already has
__device__ __forceinline__ double bfrag_rf_adj(const Consts<7>& C, int mat, int kc, int lane, double dt) {
  const int c = lane >> 2, k = lane & 3;
  const int i = (c & 1) ? 7 - (c >> 1) : (c >> 1);
  const int j = kc == 0 ? k : 7 - k;
  const double mi = C.minv[(i == 0 || i == 7) ? 0 : i];
  const double mj = C.minv[(j == 0 || j == 7) ? 0 : j];
  (void)dt;
  (void)mi;
  if (mat == 0) return __dmul_rn(C.K[i * 8 + j], __dmul_rn(-C.nu, mj));
  return -__dmul_rn(C.Dw[j * 8 + i], mj);
}

__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// DR (recompute mode): J^T(U_i), i < s-1, reuses M^-1 Dw U_i from the stage recompute
// (two of its six DMMAs per m-tile), kept in per-lane shared-memory slots.
// CHK = false (the sweep's run-ahead, check = 0): only the owned outputs lam_n are tested
// (SEM1D_FLAG_STEP_NONFINITE).  A non-finite stage state or cotangent reaches lam_n at its
// element's nodes through every stage term (products with U and w, every b_i != 0), so the
// run-ahead re-runs a flagged step with CHK = true, which classifies its inputs as the
// reference's per-call checks do (state / cotangent bits) and gives bitwise the same lam_n.
template <int SCH, bool LD, int WMT, int MINB, bool DR = false, bool CHK = true>
__global__ void __launch_bounds__(32 * RfAdjCfg<WMT>::W, MINB)
    tile_adj_rf_kernel(const __grid_constant__ Consts<7> C, const Geo G, const TileStepArgs A) {
  using CF = RfAdjCfg<WMT>;
  constexpr int N = 7, W = CF::W, TE = CF::TE, LEN = CF::LEN, PAD = CF::PAD, SLOT = CF::SLOT;
  using TB = TabC<SCH>;
  constexpr int S = TB::s, H = LD ? S : 2 * S - 1, T = TE - 2 * H;
  constexpr int NSLAB = LD ? S + 1 : 2;       // u, lam (, U_1..U_{s-1})
  constexpr int SB = LD ? 5 : 2;              // slabs per buffer in the layout
  extern __shared__ __align__(16) double smem[];
  double* sslab = smem;                       // [2][SB][PAD]
  double* sst = sslab + 2 * SB * PAD;         // [2][SLOT] recompute: U_1, U_2 per lane
  double* sdw = sst + 2 * SLOT;               // [3][SLOT] DR: M^-1 Dw U_0..U_2 per lane
  double* xF = sst + (LD ? 0 : (DR ? 5 : 2) * SLOT);   // [2][8] raw row 7 of each warp's last element
  double* xU = xF + 16;                       // [2][8] raw row 0 of each warp's first element
  uint64_t* full = reinterpret_cast<uint64_t*>(xU + 16);
  uint64_t* empty = full + 2;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int kq = lane & 3, rr = lane >> 2;
  const int e_lane = 8 * WMT * w + WMT * rr;
  const int64_t ndof = G.ndof;
  const double dt = A.dt;
  double bk[2], bd[2], jk[2], jt[2];
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    bk[kc] = RF_EO ? bfrag_eo(C, kc, lane) : bfrag_rf(C, 0, kc, lane);   // (RF_EO: the s / d blocks)
    bd[kc] = bfrag_rf(C, 1, kc, lane);
    jk[kc] = bfrag_rf_adj(C, 0, kc, lane, dt);
    jt[kc] = bfrag_rf_adj(C, 2, kc, lane, dt);
  }
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], W);
    mbar_init(&empty[1], W);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_launch_dependents();
  griddep_wait();
  auto issue = [&](const TileLoad& Lx, int x) {
    const double* srcs[5] = {A.u, A.lam, A.stin[0], A.stin[1], A.stin[2]};
    double* base = sslab + x * SB * PAD;
    double* dsts[5] = {base, base + PAD, base + 2 * PAD, base + 3 * PAD, base + 4 * PAD};
    tile_issue_n(Lx, LEN, srcs, dsts, &full[x], NSLAB);
  };
  uint32_t fphase = 0u, ephase = 0u, pend = 0u;
  int want = -1;                               // tid 0: launch tile k whose prefetch waits for a buffer
  const int cnt = A.tile_cnt > 0 ? A.tile_cnt : A.ntiles;
  auto tile_of = [&](int k) {
    const int t = A.tile_lo + k;                // < 2 ntiles
    return t >= A.ntiles ? t - A.ntiles : t;
  };
  if (tid == 0 && (int)blockIdx.x < cnt) {
    const TileLoad L = tile_load_plan(tile_of(blockIdx.x), T, H, N, LEN, ndof);
    if (L.bulk) {
      issue(L, 0);
      pend |= 1u;
    }
  }
  // tid 0: issue the pending prefetch of tile `want` into buffer x once that buffer's
  // readers (the tile before) are done: polled without blocking at every stage, forced
  // (blocking) at the start of tile `want` itself
  auto try_prefetch = [&](int x, bool block) {
    if (tid != 0 || want < 0) return;
    if (pend & (1u << x)) {
      if (block) {
        while (!mbar_try_wait(&empty[x], (ephase >> x) & 1u)) {
        }
      } else if (!mbar_test_wait(&empty[x], (ephase >> x) & 1u)) {
        return;
      }
      ephase ^= 1u << x;
      pend &= ~(1u << x);
    }
    issue(tile_load_plan(tile_of(want), T, H, N, LEN, ndof), x);
    pend |= 1u << x;
    want = -1;
  };
  unsigned fstate = 0u, fz = 0u, fout = 0u;
  int it = 0;
  for (int k = blockIdx.x; k < cnt; k += gridDim.x, ++it) {
    const int t = tile_of(k);
    const int b = it & 1;
    const TileLoad L = tile_load_plan(t, T, H, N, LEN, ndof);
    // this lane's values of slab s (m-tile q, slot h) at sl[s * PAD + q * N + (h ? 7 - kq : kq)]
    const double* sl = sslab + b * SB * PAD + L.sh + e_lane * N;
    auto val = [&](int sidx, int q, int h) -> double { return sl[sidx * PAD + q * N + (h == 0 ? kq : 7 - kq)]; };
    if (!L.bulk) {
      // the tile wraps around the ring end (at most two per launch): the CTA fills the
      // buffer itself; the barrier also means every warp is done with its previous tiles
      __syncthreads();
      double* dst = sslab + b * SB * PAD;
      for (int k = tid; k < LEN; k += 32 * W) {
        int64_t g = L.g0 + k;
        while (g >= ndof) g -= ndof;
        dst[k] = __ldg(A.u + g);
        dst[PAD + k] = __ldg(A.lam + g);
        if (LD)
          for (int i = 1; i < S; ++i) dst[(1 + i) * PAD + k] = __ldg(A.stin[i - 1] + g);
      }
      __syncthreads();
    }
    if (tid == 0 && want == k) try_prefetch(b, true);   // this tile's load is still owed
    if (L.bulk) {
      while (!mbar_try_wait(&full[b], (fphase >> b) & 1u)) {
      }
      fphase ^= 1u << b;
    }
    if (tid == 0 && k + (int)gridDim.x < cnt) {
      want = tile_load_plan(tile_of(k + gridDim.x), T, H, N, LEN, ndof).bulk ? k + (int)gridDim.x : -1;
      try_prefetch(b ^ 1, false);
    }
    const int64_t e_base = (int64_t)t * T - H;
    bool own[WMT];
    unsigned msk[WMT][2];                        // check masks: owned node, not the node-7 replica
#pragma unroll
    for (int q = 0; q < WMT; ++q) {
      const int e = e_lane + q;
      own[q] = e >= H && e < H + T && e_base + e < G.E;
      msk[q][0] = (!RF_NOCHK && own[q]) ? 0x7ff00000u : 0u;
      msk[q][1] = (!RF_NOCHK && own[q] && kq != 0) ? 0x7ff00000u : 0u;
    }
    double U[WMT][2], F[WMT][2];
    double k0[(SCH == 1) ? WMT : 1][2];
    // Pairwise exchange of a stage result R, ONE round per stage: each warp publishes the raw
    // row 7 of its last element (to the right) and the raw row 0 of its first (to the left),
    // and every interface sum (row 7 of e-1 + row 0 of e) is formed by BOTH lanes that hold
    // the node -- the owner of node 0 of e and the node-7 replica of e-1 -- from the same two
    // raw rows in the same order, so the replica is bitwise the owner's value and no second
    // exchange of updated states is needed.  upd(q) then advances m-tile q (refresh: the
    // replica rows take the full interface value).  Barrier order per warp: arrive BAR_F+w
    // (publish_F), sync BAR_F+w-1, arrive BAR_U+w-1, sync BAR_U+w -- a warp passes its sync
    // on BAR_U+w only after w+1 passed its sync on BAR_F+w, so no barrier generation takes two
    // arrivals of one warp; the slots are double-buffered by exchange parity.
    int xpar = 0;
    auto exchange = [&](double (&R)[WMT][2], auto&& upd, bool refresh) {
      double left = __shfl_up_sync(0xffffffffu, R[WMT - 1][1], 4);
      double rawr = __shfl_down_sync(0xffffffffu, R[0][0], 4);
      if (w > 0) {
        nbar_sync(RfCfg<4>::BAR_F + w - 1, 64);
        if (lane == 0) left = xF[xpar * 8 + w - 1];
        if (lane == 0) xU[xpar * 8 + w] = R[0][0];
        if (!RF_BAR_NA) __syncwarp();
        nbar_arrive(RfCfg<4>::BAR_U + w - 1, 64);
      } else if (lane == 0) {
        left = 0.0;
      }
      if (kq == 0) {
#pragma unroll
        for (int q = WMT - 1; q > 0; --q) R[q][0] = __dadd_rn(R[q - 1][1], R[q][0]);
        R[0][0] = __dadd_rn(left, R[0][0]);
        if (refresh) {                          // replicas inside the lane: the same sums
#pragma unroll
          for (int q = 0; q + 1 < WMT; ++q) R[q][1] = R[q + 1][0];
        }
      }
#pragma unroll
      for (int q = 0; q + 1 < WMT; ++q) upd(q);
      if (w < W - 1) {
        nbar_sync(RfCfg<4>::BAR_U + w, 64);
        if (lane == 28) rawr = xU[xpar * 8 + w + 1];
      }
      if (refresh && kq == 0) R[WMT - 1][1] = __dadd_rn(R[WMT - 1][1], rawr);
      upd(WMT - 1);
      xpar ^= 1;
    };
    auto publish_F = [&](const double (&R)[WMT][2]) {
      if (w < W - 1) {
        if (lane == 28) xF[xpar * 8 + w] = R[WMT - 1][1];
        if (!RF_BAR_NA) __syncwarp();
        nbar_arrive(RfCfg<4>::BAR_F + w, 64);
      }
    };
    // ---- forward recompute of U_1..U_{s-1} (LD = 0) ----
    if constexpr (!LD) {
#pragma unroll
      for (int q = 0; q < WMT; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) U[q][h] = val(0, q, h);
#pragma unroll
      for (int st = 0; st + 1 < S; ++st) {
#pragma unroll
        for (int q = 0; q < WMT; ++q)
          if (CHK) fstate = max(fstate, max(expbits(U[q][0], msk[q][0]), expbits(U[q][1], msk[q][1])));
        auto mtile_F = [&](int q) {
          double da = 0.0, db = 0.0;
          if (RF_EO) {
            f_eo(U[q][0], U[q][1], bk[0], bk[1], F[q][0], F[q][1], da, db);
          } else {
            double ka = 0.0, kb = 0.0;
            dmma884(ka, kb, U[q][0], bk[0]);
            dmma884(da, db, U[q][0], bd[0]);
            dmma884(ka, kb, U[q][1], bk[1]);
            dmma884(da, db, U[q][1], bd[1]);
            F[q][0] = __fma_rn(-U[q][0], da, ka);
            F[q][1] = __fma_rn(-U[q][1], db, kb);
          }
          if (DR) {                               // M^-1 Dw U_st for J^T(U_st)
            sdw[st * SLOT + ((w * WMT + q) * 2 + 0) * 32 + lane] = da;
            sdw[st * SLOT + ((w * WMT + q) * 2 + 1) * 32 + lane] = db;
          }
        };
        mtile_F(WMT - 1);
        publish_F(F);
#pragma unroll
        for (int q = 0; q + 1 < WMT; ++q) mtile_F(q);
        try_prefetch(b ^ 1, false);
        const double c1 = __dmul_rn(dt, TB::a(st + 1, st));
        auto upd = [&](int q) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double k = F[q][h];
            if (TB::nterm(st + 1) == 1) {
              U[q][h] = __fma_rn(c1, k, val(0, q, h));
            } else {
              const double s2 = __fma_rn(TB::a(st + 1, st), k, __dmul_rn(TB::a(st + 1, 0), k0[q][h]));
              U[q][h] = __fma_rn(dt, s2, val(0, q, h));
            }
            if (SCH == 1 && st == 0) k0[q][h] = k;
          }
        };
        exchange(F, upd, true);
        if (st + 2 < S) {                       // U_{st+1} waits in its per-lane slot
          double* slot = sst + st * SLOT;
#pragma unroll
          for (int q = 0; q < WMT; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) slot[((w * WMT + q) * 2 + h) * 32 + lane] = U[q][h];
        }
      }
    }
    // ---- backward: stage-adjoint recurrence ----
    double ln[WMT][2], lacc[WMT][2], l2[(SCH == 1) ? WMT : 1][2];   // l'_{i+1}, sum b l', l'_2
    using TW = TabW<SCH>;
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      // stage state U_i
      if (LD || i + 1 < S || S == 1) {            // (recompute: U_{s-1} is still in registers)
#pragma unroll
        for (int q = 0; q < WMT; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (i == 0) U[q][h] = val(0, q, h);
            else if (LD) U[q][h] = val(1 + i, q, h);
            else U[q][h] = sst[(i - 1) * SLOT + ((w * WMT + q) * 2 + h) * 32 + lane];
          }
      }
      if (LD || i == S - 1) {                    // U_0..U_{s-2} were checked as stage inputs
#pragma unroll
        for (int q = 0; q < WMT; ++q)
          if (CHK) fstate = max(fstate, max(expbits(U[q][0], msk[q][0]), expbits(U[q][1], msk[q][1])));
      }
      double Lr[WMT][2];                         // l'_i / dt (element rows, then assembled)
      // dt rides on the recurrence's coefficients: w_i = lam + c dt l'', lam_n = lam + b dt l''
      const double cdt1 = (i + 1 < S) ? __dmul_rn(TW::c(i, i + 1), dt) : 0.0;
      const double cdt2 = (SCH == 1 && i == 0) ? __dmul_rn(TW::c(0, 2), dt) : 0.0;
      const double bdt = __dmul_rn(TB::b(i), dt);
      auto mtile_L = [&](int q) {
        double z[2], y[2];                       // z = w_i here
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double zz = val(1, q, h);
          if (i + 1 < S && TW::c(i, i + 1) != 0.0) zz = __fma_rn(cdt1, ln[q][h], zz);
          if (SCH == 1 && i == 0) zz = __fma_rn(cdt2, l2[q][h], zz);
          z[h] = zz;
          y[h] = __dmul_rn(U[q][h], zz);
        }
        if (CHK && i + 1 < S) fz = max(fz, max(expbits(z[0], msk[q][0]), expbits(z[1], msk[q][1])));
        double ca = 0.0, cb = 0.0, da = 0.0, db = 0.0;
        dmma884(ca, cb, z[0], jk[0]);
        if (DR && !LD && i + 1 < S) {            // reuse the stage recompute's M^-1 Dw U_i
          da = sdw[i * SLOT + ((w * WMT + q) * 2 + 0) * 32 + lane];
          db = sdw[i * SLOT + ((w * WMT + q) * 2 + 1) * 32 + lane];
        } else {
          dmma884(da, db, U[q][0], bd[0]);
          dmma884(da, db, U[q][1], bd[1]);
        }
        dmma884(ca, cb, z[1], jk[1]);
        dmma884(ca, cb, y[0], jt[0]);
        dmma884(ca, cb, y[1], jt[1]);
        Lr[q][0] = __fma_rn(-z[0], da, ca);
        Lr[q][1] = __fma_rn(-z[1], db, cb);
      };
      if (CHK && i == S - 1) {                   // w_{s-1} = lam: the cotangent input check
#pragma unroll
        for (int q = 0; q < WMT; ++q) fz = max(fz, max(expbits(val(1, q, 0), msk[q][0]), expbits(val(1, q, 1), msk[q][1])));
      }
      mtile_L(WMT - 1);
      publish_F(Lr);
#pragma unroll
      for (int q = 0; q + 1 < WMT; ++q) mtile_L(q);
      try_prefetch(b ^ 1, false);
      auto acc_q = [&](int q) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          lacc[q][h] = (i == S - 1) ? __dmul_rn(bdt, Lr[q][h]) : __fma_rn(bdt, Lr[q][h], lacc[q][h]);
          if (SCH == 1 && i == 1) l2[q][h] = ln[q][h];
          ln[q][h] = Lr[q][h];
        }
      };
      exchange(Lr, acc_q, i > 0);
    }
    // lam_n = lam + (b_{s-1} l'_{s-1} + ... + b_0 l'_0), owned nodes
#pragma unroll
    for (int q = 0; q < WMT; ++q) {
      const double o0 = __dadd_rn(val(1, q, 0), lacc[q][0]), o1 = __dadd_rn(val(1, q, 1), lacc[q][1]);
      if (!CHK) fout = max(fout, max(expbits(o0, msk[q][0]), expbits(o1, msk[q][1])));
      if (!own[q]) continue;
      const int64_t g = (e_base + e_lane + q) * N;
      A.out[g + kq] = o0;
      if (kq != 0) A.out[g + 7 - kq] = o1;
    }
    __syncwarp();
    if (L.bulk && lane == 0) mbar_arrive(&empty[b]);   // this warp is done with the tile's slabs
  }
  const unsigned bits = (fstate == 0x7ff00000u ? SEM1D_FLAG_STATE_NONFINITE : 0u) |
                        (fz == 0x7ff00000u ? SEM1D_FLAG_INPUT2_NONFINITE : 0u) |
                        (fout == 0x7ff00000u ? SEM1D_FLAG_STEP_NONFINITE : 0u);
  const unsigned any = __reduce_or_sync(0xffffffffu, bits);
  if (lane == 0 && any) atomicOr(A.flag, (int)any);
}

}  // namespace sem1d
