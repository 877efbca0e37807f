/*
 * sem1d.h -- C ABI of the B200 (sm_100a) 1D GLL spectral-element Burgers hot path.
 *
 * This is the drop-in boundary.  The reference (semopt 0.1.0, pure Python) has
 * no FFI: its plugin surface is the duck-typed operator object that the time
 * loop and the adjoint sweep call.  Each entry point below
 * replaces one reference call site:
 *
 *   sem1d_plan_create  <- SemOperator.__init__          ops.py:91-124
 *                         (D, Dw, K, M^-1 built on the host, grid.py:126-146)
 *   sem1d_rhs          <- SemOperator.apply_rhs          ops.py:232-236
 *   sem1d_jac          <- SemOperator.apply_jacobian     ops.py:238-244
 *   sem1d_jact         <- SemOperator.apply_jacobian_transpose  ops.py:246-257
 *   sem1d_rk_stage     <- one stage of step_rk3 / rk3_stages  timeloop.py:111-130
 *                         (F apply fused with the stage linear combination)
 *   sem1d_adj_stage    <- one stage of adjoint_step_rk3       adjoint.py:54-61
 *                         (J^T apply fused with the stage-adjoint recurrence)
 *   sem1d_terminal     <- terminal_condition                 adjoint.py:33-47
 *   sem1d_scatter / sem1d_gather <- Grid.scatter / Grid.gather  grid.py:165-182
 *   sem1d_cn_step / sem1d_cn_adjoint_step / sem1d_gmres <- the Crank-Nicolson path
 *                         timeloop.py:133-186, adjoint.py:64-69 (see below)
 *
 * Conventions (mirror the reference contract, ops.py:216-230):
 *  - every array is fp64 in DEVICE memory owned by the caller; inputs are never
 *    written; nothing is allocated inside a compute call except, once per plan
 *    with N+1 % 8 == 0, the tensor-core B-fragment table on its first apply
 *    (freed by sem1d_plan_destroy);
 *  - fields are `batch` consecutive vectors of `ndof` doubles
 *    (ndof = E*N periodic, E*N+1 homogeneous Dirichlet, grid.py:61-63);
 *  - calls are stream ordered (`stream` is a cudaStream_t, NULL = legacy default);
 *    the applies and whole-step kernels use programmatic dependent launch and
 *    wait (griddepcontrol.wait) before reading any global input;
 *  - non-finite inputs do not abort the kernel: they OR a bit into *flag
 *    (device int), which the host maps to NumericFailure / StepFailure;
 *  - return value: 0 ok, SEM1D_EINVAL bad argument, SEM1D_ECUDA launch error
 *    (message via sem1d_last_error()).
 */
#ifndef SEM1D_H
#define SEM1D_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEM1D_OK 0
#define SEM1D_EINVAL (-1)
#define SEM1D_ECUDA (-2)

/* bits OR-ed into *flag */
#define SEM1D_FLAG_STATE_NONFINITE 1   /* first input (state u) had NaN/Inf  -> NumericFailure */
#define SEM1D_FLAG_INPUT2_NONFINITE 2  /* second input (v / z) had NaN/Inf  -> NumericFailure */
#define SEM1D_FLAG_STEP_NONFINITE 4    /* a new RK state is non-finite      -> StepFailure   */

#define SEM1D_MAX_DEGREE 32
#define SEM1D_MAX_TERMS 5

typedef struct sem1d_plan sem1d_plan;

/* Library identity. */
int sem1d_version(void);
/* Kernel-path selection for A/B measurement and tests (process-wide):
 * 0 = automatic (warp-specialised FP64 tensor-core DMMA kernel for N+1 in
 *     {8,16,24,32}, else the TMA-pipelined DFMA kernel for odd N, else the
 *     plain tiled kernel), 1 = never a tensor-core kernel, 2 = plain tiled
 *     kernel only, 3 = the CTA-synchronous tensor-core kernel (A/B reference).
 * Arithmetic: for N+1 in {16, 32} the automatic path contracts on the reflection
 * (even/odd) split of K, Dw and Dw^T (half blocks acting on sums and differences of
 * mirrored nodes; the same products as ops.py:161-212 summed in a different order,
 * within the 1e-12 per-apply tolerance and the smooth-input longdouble bound).  Paths 1
 * and 2 keep the reference's summation order (bit-identical to its numpy result on the
 * inputs tested). */
int sem1d_set_kernel_path(int path);
/* Tile-step kernels for A/B runs: 0 = auto (register-resident kernels for N = 7),
 * 1 = the shared-memory tile kernels for every degree (and the shared-memory ensemble
 * forward sweep at N = 15), 2 = N = 7 register-resident steps on 128-element tiles,
 * 3 = the N = 7 register-resident forward step on 192-element tiles at 3 CTAs/SM. */
int sem1d_set_tile_variant(int variant);
const char* sem1d_last_error(void);
int sem1d_max_degree(void);

/* Operator plan = SemOperator(grid_1d(xa, xb, E, N, bc), PdeCoefficients(nu)).
 * K, Dw: (N+1)x(N+1) row-major host arrays (ops.py:104-106).
 * mass_pattern, minv_pattern: N+2 host doubles each, the assembled mass
 * diagonal (grid.py:128-131) and its reciprocal (ops.py:116) by position:
 *   [0]      element-interface node (local index 0),
 *   [i]      interior local node i, 1 <= i <= N-1,
 *   [N]      first global node of a Dirichlet grid,
 *   [N+1]    last global node of a Dirichlet grid.
 * A uniform mesh needs nothing else; no (ndof,) M^-1 array is ever read.
 * The constants are copied into the plan (kernel-parameter space). */
int sem1d_plan_create(int64_t n_elements, int degree, int periodic, double nu,
                      const double* K, const double* Dw, const double* mass_pattern,
                      const double* minv_pattern, int64_t batch, sem1d_plan** out);
int sem1d_plan_destroy(sem1d_plan* plan);
int64_t sem1d_plan_ndof(const sem1d_plan* plan);
/* Advection kind of the plan (ops.py:44-60, 147-212): 0 Burgers (default), 1 linear with
 * constant speed `speed` (F = M^-1 Q^T(-nu K u - speed Dw u), J v = the same map on v,
 * J^T z = Q^T(-nu K zm - speed Dw^T zm)), 2 none (diffusion only).  Plans of kind 1 / 2
 * run sem1d_rhs / sem1d_jac / sem1d_jact through a generic kernel; the fused stage, step and
 * ensemble entry points accept Burgers plans only (SEM1D_EINVAL otherwise). */
int sem1d_plan_set_advection(sem1d_plan* plan, int mode, double speed);

/* f = M^-1 Q^T F_e(Q u) (masked).  ops.py:232-236 */
int sem1d_rhs(const sem1d_plan* plan, const double* u, double* f, int* flag, void* stream);
/* out = M^-1 Q^T J_e(Qu) Q v (masked).  ops.py:238-244 */
int sem1d_jac(const sem1d_plan* plan, const double* u, const double* v, double* out,
              int* flag, void* stream);
/* out = Q^T J_e^T(Qu) Q mask(M^-1 z) (masked).  ops.py:246-257 */
int sem1d_jact(const sem1d_plan* plan, const double* u, const double* z, double* out,
               int* flag, void* stream);

/* One explicit-RK stage, F fused with its linear combination:
 *   k      = F(U_in)                                  (written to k_out if non-NULL)
 *   Y      = base + dt * sum_j coef[j] * K_j          (association of timeloop.py:114-127:
 *                                                      one term -> base + (dt*coef)*K,
 *                                                      several -> base + dt*((c0 K0 + c1 K1) + ...))
 * where K_j = terms[j], or the freshly computed k when terms[j] == NULL.
 * If check_step != 0 a non-finite Y sets SEM1D_FLAG_STEP_NONFINITE (timeloop.py:100-103,129). */
int sem1d_rk_stage(const sem1d_plan* plan, const double* U_in, double* k_out,
                   const double* base, int nterms, const double* const* terms,
                   const double* coef, double dt, double* Y, int check_step,
                   int* flag, void* stream);

/* One stage of the discrete-adjoint recurrence (adjoint.py:54-61, generalised):
 *   z      = b * lam + sum_j a[j] * l_j                (left to right)
 *   l      = dt * J^T(U) z                             (written to l_out if non-NULL)
 *   lam_out = ((lam + L_0) + L_1) + ...                (only if lam_out != NULL)
 * where L_j = acc_terms[j], or the fresh l when acc_terms[j] == NULL. */
int sem1d_adj_stage(const sem1d_plan* plan, const double* U, const double* lam, double b,
                    int nl, const double* const* l_terms, const double* a,
                    double dt, double* l_out,
                    int nacc, const double* const* acc_terms, double* lam_out,
                    int* flag, void* stream);

/* Ring-resident forward sweep for many small independent problems (BASELINE
 * config 4): one CTA per ring integrates `nsteps` explicit steps of `scheme`
 * (0 euler, 1 rk3, 2 rk4; timeloop.py:106-130) with step sizes dts[0..nsteps)
 * (device), entirely in shared memory, writing state n of problem b to
 * traj[n][b][:] (step-major, so traj[n] is a contiguous batch; traj may be
 * NULL) and the last state to u_final.  flags[b] gets
 * SEM1D_FLAG_STEP_NONFINITE if any new state of problem b was non-finite
 * (the reference's StepFailure, timeloop.py:129; no dt retry in the batched
 * sweep -- the host re-runs failing problems).  Rings must fit one CTA:
 * E*(N+1) <= 1024 (any degree, periodic or Dirichlet; one thread per element
 * row), or periodic with N+1 a multiple of 8 and E a multiple of 8, E <= 256
 * (FP64 tensor-core ring kernel). */
int sem1d_ens_forward(const sem1d_plan* plan, const double* u0, double* traj, double* u_final,
                      const double* dts, int nsteps, int scheme, int* flags, void* stream);

/* Ring-resident backward sweep matching sem1d_ens_forward (adjoint.py:54-61
 * generalised to the tableau): for n = nsteps-1..0 it reloads u_n from the
 * step-major trajectory, recomputes the stage states in shared memory and runs
 * the stage-adjoint recurrence; lam_out[b] = dJ/du0 for the terminal seeds
 * lam_in[b] (sem1d_terminal).  Same ring restrictions as sem1d_ens_forward. */
int sem1d_ens_adjoint(const sem1d_plan* plan, const double* traj, const double* lam_in,
                      double* lam_out, const double* dts, int nsteps, int scheme, int* flags,
                      void* stream);
/* The same sweep with a choice of checks.  check = 1 is sem1d_ens_adjoint: every stage's
 * cotangent is classified (SEM1D_FLAG_INPUT2_NONFINITE).  check = 0 tests only lam_out
 * (SEM1D_FLAG_STEP_NONFINITE; a non-finite cotangent anywhere in the sweep reaches lam_out
 * through the J^T terms): a caller re-runs a flagged problem set with check = 1 to tell a
 * non-finite cotangent (the reference's NumericFailure) from a final overflow. */
int sem1d_ens_adjoint_ex(const sem1d_plan* plan, const double* traj, const double* lam_in,
                         double* lam_out, const double* dts, int nsteps, int scheme, int check,
                         int* flags, void* stream);

/* Temporally blocked steps for large periodic rings (batch 1, N+1 in
 * {8,16,24,32}, at least two 256/128-element tiles): ONE launch per explicit
 * step u -> u_new (all stages of timeloop.py:111-130 in shared memory, 16 B/DOF
 * of HBM traffic) and ONE launch per adjoint step lam -> lam_out (stage states
 * recomputed from u, stage-adjoint chain of adjoint.py:54-61 in shared memory,
 * 24 B/DOF).  Each CTA recomputes s (forward) or 2s-1 (adjoint) ghost elements
 * per side of its tile.  Outputs must not alias inputs.  Flags as for
 * sem1d_rk_stage / sem1d_adj_stage.  sem1d_step_supported(plan) tells whether
 * the plan qualifies. */
int sem1d_step_supported(const sem1d_plan* plan);
/* The same steps with the forward trajectory's stage states held in HBM (north_star item 4):
 * sem1d_rk_step_stages also writes U_1..U_{s-1} of the step to stages[0..s-2] (ndof each);
 * sem1d_adj_step_stages reads them instead of recomputing (s ghost elements per tile
 * instead of 2s-1, no F applies), giving the adjoint of timeloop.py:111-130 /
 * adjoint.py:54-61 with s J^T stages only. */
int sem1d_step_stages_supported(const sem1d_plan* plan);   /* the pair below qualifies */
int sem1d_rk_step_stages(const sem1d_plan* plan, const double* u, double* u_new,
                         double* const* stages, double dt, int scheme, int* flag, void* stream);
int sem1d_adj_step_stages(const sem1d_plan* plan, const double* u, const double* const* stages,
                          const double* lam, double* lam_out, double dt, int scheme, int* flag,
                          void* stream);
int sem1d_rk_step(const sem1d_plan* plan, const double* u, double* u_new, double dt, int scheme,
                  int* flag, void* stream);
int sem1d_adj_step(const sem1d_plan* plan, const double* u, const double* lam, double* lam_out,
                   double dt, int scheme, int* flag, void* stream);
/* One step (timeloop.py:111-130) with a choice of checks; stages may be NULL.  check = 1 is
 * sem1d_rk_step / sem1d_rk_step_stages.  check = 0 tests only the new state: a non-finite
 * stage input then shows as SEM1D_FLAG_STEP_NONFINITE (NaN/Inf reach the new state through
 * every b_i != 0), so a caller that must tell NumericFailure from StepFailure re-runs a
 * flagged step with check = 1 -- bitwise the same state (integrate's run-ahead does). */
int sem1d_rk_step_ex(const sem1d_plan* plan, const double* u, double* u_new, double* const* stages,
                     double dt, int scheme, int check, int tile_lo, int tile_cnt, int* flag, void* stream);
/* The adjoint step (adjoint.py:54-61) with stored stages (may be NULL: recompute), a choice
 * of checks and a tile range.  check = 1 is sem1d_adj_step / sem1d_adj_step_stages: stage
 * states and cotangents are classified (SEM1D_FLAG_STATE_NONFINITE / _INPUT2_NONFINITE).
 * check = 0 (N = 7 kernels; the others always classify) tests only lam_out: a non-finite
 * stage state or cotangent then shows as SEM1D_FLAG_STEP_NONFINITE (it reaches lam_out through
 * every stage term), and a caller that must raise the reference's exception re-runs the
 * flagged step with check = 1 (bitwise the same lam_out; the sweep's run-ahead does).
 * Ranges (N = 7 kernels): the launch covers ring tiles (tile_lo + k) mod ntiles,
 * k < tile_cnt (tile_cnt 0 = all).  A sharded step runs the tiles that read no ghost element
 * while the ghost exchange is in flight, then the rest; sem1d_step_tiling gives the layout:
 * tile t reads elements [t*owned - ghost, (t+1)*owned + ghost) of the ring. */
int sem1d_adj_step_ex(const sem1d_plan* plan, const double* u, const double* const* stages, const double* lam,
                      double* lam_out, double dt, int scheme, int check, int tile_lo, int tile_cnt, int* flag,
                      void* stream);
int sem1d_step_tiling(const sem1d_plan* plan, int kind, int stored, int scheme, int* ntiles, int* owned,
                      int* ghost);

/* Terminal condition (adjoint.py:33-47): d = uN - ud, lam = mask(2 M d),
 * J_out[b] = d^T M d per batch member (deterministic two-level reduction;
 * `work` must hold sem1d_terminal_work_size(plan) doubles). */
int64_t sem1d_terminal_work_size(const sem1d_plan* plan);
int sem1d_terminal(const sem1d_plan* plan, const double* uN, const double* ud, double* lam,
                   double* J_out, double* work, void* stream);

/* Assembly maps (grid.py:165-182): local blocks are (batch, E, N+1). */
int sem1d_scatter(const sem1d_plan* plan, const double* u, double* local, void* stream);
int sem1d_gather(const sem1d_plan* plan, const double* local, double* out, void* stream);

/* ---------------------------------------------------------------------------
 * Implicit path and adaptive Kutta-3 controller.
 *
 *   sem1d_cn_step          <- step_cn          timeloop.py:154-186
 *                             (full Newton, GMRES on I - dt/2 J(v))
 *   sem1d_cn_adjoint_step  <- adjoint_step_cn  adjoint.py:64-69
 *   sem1d_gmres            <- _gmres_solve     timeloop.py:133-151 (scipy 1.18.1
 *                             gmres restated: MGS Arnoldi, Givens, gh-8400 tolerance
 *                             control, one counted matvec per column + per cycle)
 *   sem1d_rk_error_norm    <- controller       timeloop.py:198-218 (reduction part)
 *
 * Batch-1 plans.  `work` is device memory of sem1d_cn_work_size(plan, restart)
 * doubles, ZERO-INITIALISED once before first use (it holds a reduction ticket
 * the kernels leave at zero); a workspace serves one stream at a time.  These
 * calls synchronise `stream` at the reference's decision points (GMRES inner
 * stop test, Newton residual test).  Outcomes are reported in `st` (counters are
 * accumulated, so one stats object can cover a whole sweep). */
#define SEM1D_CN_OK 0
#define SEM1D_CN_GMRES_FAILED 1        /* GMRES did not converge -> StepFailure        */
#define SEM1D_CN_NEWTON_STALLED 2      /* newton_max iterations   -> StepFailure        */
#define SEM1D_CN_RESIDUAL_NONFINITE 3  /* Newton residual NaN/Inf -> StepFailure        */
#define SEM1D_CN_INPUT_NONFINITE 4     /* an operator input NaN/Inf -> NumericFailure   */

typedef struct {
  double newton_tol;   /* TsConfig.newton_tol  (1e-10) */
  int newton_max;      /* TsConfig.newton_max  (25)    */
  double gmres_tol;    /* TsConfig.gmres_tol   (1e-10) */
  int gmres_max;       /* TsConfig.gmres_max   (200)   */
  int gmres_restart;   /* TsConfig.gmres_restart (30), 1..64 */
} sem1d_cn_params;

typedef struct {
  int64_t newton_iters, gmres_iters;              /* the reference's stats counters */
  int64_t rhs_applies, jac_applies, jact_applies; /* SemOperator.counters increments */
  int status;                                     /* SEM1D_CN_* of the last call     */
  int gmres_info;                                 /* scipy info of the failing solve */
  double last_residual;                           /* |r| at the last Newton test     */
} sem1d_cn_stats;

int64_t sem1d_cn_work_size(const sem1d_plan* plan, int restart);
/* v = Crank-Nicolson step of u (v must not alias u). */
int sem1d_cn_step(const sem1d_plan* plan, const double* u, double* v, double dt,
                  const sem1d_cn_params* params, double* work, int* flag, sem1d_cn_stats* st,
                  void* stream);
/* lam_out = transpose of the CN step map between u_n and u_np1, applied to lam. */
int sem1d_cn_adjoint_step(const sem1d_plan* plan, const double* u_n, const double* u_np1,
                          const double* lam, double* lam_out, double dt,
                          const sem1d_cn_params* params, double* work, int* flag,
                          sem1d_cn_stats* st, void* stream);
/* x = GMRES solution of (I + alpha J(p)) x = b, or (I + alpha J(p)^T) x = b if transpose;
 * st->gmres_info = scipy's info (0 converged, else maxiter; -1 non-finite). */
int sem1d_gmres(const sem1d_plan* plan, int transpose, const double* p, double alpha,
                const double* b, double* x, const sem1d_cn_params* params, double* work,
                int* flag, sem1d_cn_stats* st, void* stream);

/* Deterministic reductions; `work` holds sem1d_reduce_work_size() doubles, zeroed once.
 * out[0] = x . y */
int64_t sem1d_reduce_work_size(void);
int sem1d_vec_dot(int64_t n, const double* x, const double* y, double* work, double* out,
                  void* stream);
/* out[0] = sum_i sqrt(r_i) (max_form = 0, the reference's "rms" wlte before /n) or
 * max_i r_i (max_form = 1), r_i = |u_new - u_hat| / (tol_a + max(|u_new|,|u_hat|) tol_r),
 * u_hat = u + dt k2 (timeloop.py:124,205-210). */
int sem1d_rk_error_norm(int64_t n, const double* u_new, const double* u, const double* k2,
                        double dt, double tol_a, double tol_r, int max_form, double* work,
                        double* out, void* stream);

/* ---------------------------------------------------------------------------
 * Stage compositions for operators without fused stage kernels (the 3D path):
 * the same association orders as sem1d_rk_stage / sem1d_adj_stage.
 *   Y   = base + (dt c0) T0  |  base + dt ((c0 T0 + c1 T1) + ...)   (timeloop.py:114-127)
 *   z   = b lam + sum_j a_j l_j                                       (adjoint.py:58-60)
 *   out = ((x + t0) + t1) + ...                                       (adjoint.py:61)
 *   y   = s x
 * `terms` / `coef` are host arrays (of device pointers / values), at most
 * SEM1D_MAX_TERMS entries. */
int sem1d_vec_rk_combine(int64_t n, const double* base, double dt, int nterms,
                         const double* const* terms, const double* coef, double* Y, int check,
                         int* flag, void* stream);
int sem1d_vec_adj_combine(int64_t n, const double* lam, double b, int nl,
                          const double* const* l_terms, const double* a, double* z, void* stream);
int sem1d_vec_accumulate(int64_t n, const double* x, int nt, const double* const* terms,
                         double* out, void* stream);
int sem1d_vec_scale(int64_t n, const double* x, double s, double* y, void* stream);

/* ---------------------------------------------------------------------------
 * 3D periodic boxes: sum-factorised Burgers operators
 *   sem3d_rhs   <- SemOperator.apply_rhs                 ops.py:160-174,232-236 (dim 3)
 *   sem3d_jac   <- SemOperator.apply_jacobian            ops.py:176-193,238-244
 *   sem3d_jact  <- SemOperator.apply_jacobian_transpose  ops.py:195-212,246-257
 *   sem3d_terminal <- terminal_condition                 adjoint.py:33-47
 * Fields: 3 components x P1*P2*P3 scalar nodes, P_a = E_a*N, node (g1,g2,g3) at
 * (g1*P2 + g2)*P3 + g3 (grid.py:118-127).  One degree N (1..12) on all axes.
 * Plan constants (host arrays, copied): K3 = 3 stiffness matrices (n x n, one per
 * axis: ops.py:105-106 with that axis' h), Dw (n x n), T3 = the transverse mass
 * weights (n x n per direction, ops.py:109-115), and the assembled mass diagonal
 * and its reciprocal by position class ((N+1)^3 values, index
 * (c1*(N+1)+c2)*(N+1)+c3 with c = 0 for the wrap node g = 0, g mod N for interior
 * nodes, N for the other element interfaces -- bincount's summation order differs
 * between the two interface kinds, grid.py:131-135).  `work` holds
 * sem3d_work_size(plan) doubles (element-block scratch). */
typedef struct sem3d_plan sem3d_plan;
int sem3d_max_degree(void);
int sem3d_plan_create(const int64_t* elements, int degree, double nu, const double* K3,
                      const double* Dw, const double* T3, const double* minv_pattern,
                      const double* mass_pattern, sem3d_plan** out);
int sem3d_plan_destroy(sem3d_plan* plan);
int64_t sem3d_plan_ndof(const sem3d_plan* plan);
int64_t sem3d_work_size(const sem3d_plan* plan);
int sem3d_rhs(const sem3d_plan* plan, const double* u, double* f, double* work, int* flag,
              void* stream);
int sem3d_jac(const sem3d_plan* plan, const double* u, const double* v, double* out,
              double* work, int* flag, void* stream);
int sem3d_jact(const sem3d_plan* plan, const double* u, const double* z, double* out,
               double* work, int* flag, void* stream);
int sem3d_terminal(const sem3d_plan* plan, const double* uN, const double* ud, double* lam,
                   double* J, double* work, void* stream);
/* Crank-Nicolson on 3D boxes: the sem1d_cn_* drivers over the 3D operators.  `work` holds
 * sem3d_cn_work_size(plan, restart) doubles (Krylov workspace + element scratch), zeroed once. */
int64_t sem3d_cn_work_size(const sem3d_plan* plan, int restart);
int sem3d_cn_step(const sem3d_plan* plan, const double* u, double* v, double dt,
                  const sem1d_cn_params* params, double* work, int* flag, sem1d_cn_stats* st,
                  void* stream);
int sem3d_cn_adjoint_step(const sem3d_plan* plan, const double* u_n, const double* u_np1,
                          const double* lam, double* lam_out, double dt,
                          const sem1d_cn_params* params, double* work, int* flag,
                          sem1d_cn_stats* st, void* stream);
int sem3d_gmres(const sem3d_plan* plan, int transpose, const double* p, double alpha,
                const double* b, double* x, const sem1d_cn_params* params, double* work,
                int* flag, sem1d_cn_stats* st, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SEM1D_H */
