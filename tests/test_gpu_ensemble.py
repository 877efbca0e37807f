"""Ring-resident ensemble sweeps (BASELINE config 4) vs the oracle and vs the
stage-kernel integrator, per problem, within the 1e-9 sweep tolerance."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import configs, timeloop
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scheme", ["rk4", "rk3", "euler"])
@pytest.mark.parametrize("E,N", [(256, 15), (64, 7), (32, 31), (16, 15), (72, 15), (40, 31)])
def test_ensemble_forward_vs_oracle(cuda, scheme, E, N):
    B, steps, dt = 5, 25, 5e-5
    grid = grid_1d(0.0, 20.0, E, N)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0", batch=B)
    u0 = configs.fourier_fields(grid, B, 4, seed=E + N)
    ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=steps * dt, dt=dt)
    fwd = timeloop.integrate_ensemble(op, u0, ts)
    assert fwd.n_steps == steps and not fwd.stats["failed"]
    ref = R.BurgersOracle(R.Mesh1D(0.0, 20.0, E, N, True), 0.01)
    for b in (0, B - 1):
        traj, _ = R.forward(ref, u0[b], 0.0, steps * dt, dt, scheme)
        for n in (1, steps // 2, steps):
            assert rel_err(fwd.snapshots[n][b].cpu().numpy(), traj[n]) <= 1e-12
        assert rel_err(fwd.u_final[b].cpu().numpy(), traj[-1]) <= 1e-12
    # same arithmetic as the stage-kernel integrator, to rounding of the apply order
    fwd2 = timeloop.integrate(op, u0, ts)
    assert float((fwd2.u_final - fwd.u_final).abs().max() / fwd.u_final.abs().max()) <= 1e-12


def test_ensemble_failure_is_reported(cuda):
    grid = grid_1d(0.0, 20.0, 256, 15)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0", batch=3)
    u0 = configs.fourier_fields(grid, 3, 4, seed=1)
    u0[1] *= 1e140
    fwd = timeloop.integrate_ensemble(op, u0, sb.TsConfig(scheme="rk4", t_end=20 * 5e-5, dt=5e-5))
    assert 1 in fwd.stats["failed"] and 0 not in fwd.stats["failed"]


def test_cfg4_batched_gradient_vs_oracle(cuda):
    """config 4 structure at reduced B / steps: batched evaluate() per problem vs oracle."""
    prob = configs.cfg4_problem(B=4, steps=40, device="cuda:0")
    u0 = prob.u_guess
    J, g = prob.evaluate(u0)
    c = configs.CFG4
    ref = R.BurgersOracle(R.Mesh1D(c["xa"], c["xb"], c["E"], c["N"], True), c["nu"])
    target = prob.target().cpu().numpy()
    for b in range(4):
        j_ref, g_ref, _ = R.evaluate(ref, u0[b], target[b], 0.0, 40 * c["dt"], c["dt"], "rk4")
        assert abs(float(J[b]) - j_ref) <= 1e-9 * abs(j_ref)
        assert rel_err(g[b], g_ref) <= 1e-9


@pytest.mark.parametrize("scheme", ["rk4", "rk3", "euler"])
@pytest.mark.parametrize("E,N", [(256, 15), (64, 7), (32, 31), (72, 15), (40, 31)])
def test_ensemble_adjoint_vs_stage_sweep(cuda, scheme, E, N):
    """Ring-resident backward sweep == stage-kernel sweep == oracle (1e-9)."""
    from paper_1806_01422_b200 import adjoint, checkpoint
    B, steps, dt = 3, 12, 5e-5
    grid = grid_1d(0.0, 20.0, E, N)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0", batch=B)
    u0 = configs.fourier_fields(grid, B, 4, seed=3 * E + N)
    ud = configs.fourier_fields(grid, B, 4, seed=7 * E + N)
    ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=steps * dt, dt=dt)
    fwd = timeloop.integrate_ensemble(op, u0, ts)
    J, lam = adjoint.terminal_condition(grid, fwd.u_final, torch.from_numpy(ud).cuda(), op=op)
    g_ens = adjoint.ensemble_sweep(op, ts, fwd, lam)
    g_stage = adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(steps), lam)
    assert float((g_ens - g_stage).abs().max() / g_stage.abs().max()) <= 1e-12
    ref = R.BurgersOracle(R.Mesh1D(0.0, 20.0, E, N, True), 0.01)
    for b in (0, B - 1):
        j_ref, g_ref, _ = R.evaluate(ref, u0[b], ud[b], 0.0, steps * dt, dt, scheme)
        assert abs(float(J[b]) - j_ref) <= 1e-9 * abs(j_ref)
        assert rel_err(g_ens[b].cpu().numpy(), g_ref) <= 1e-9


@pytest.mark.parametrize("scheme", ["rk4", "rk3", "euler"])
@pytest.mark.parametrize("bc", ["periodic", "dirichlet0"])
@pytest.mark.parametrize("E,N", [(16, 9), (5, 2), (40, 12), (3, 31)])
def test_small_ring_sweeps_vs_oracle(cuda, scheme, bc, E, N):
    """Small rings (E*(N+1) <= 1024, any degree / boundary kind): one launch per sweep."""
    from paper_1806_01422_b200 import adjoint
    B, steps, dt = 3, 15, 1e-5       # explicit limit ~3e-5 for E=40, N=12 on [-1, 1]
    grid = grid_1d(-1.0, 1.0, E, N, bc)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0", batch=B)
    rng = np.random.default_rng(E * N)
    x = grid.node_coordinates()[0]
    u0 = np.stack([grid.mask(np.sin(np.pi * x) + 0.05 * rng.standard_normal(grid.nglobal))
                   for _ in range(B)])
    ud = np.stack([grid.mask(np.sin(np.pi * x + 0.3)) for _ in range(B)])
    ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=steps * dt, dt=dt)
    fwd = timeloop.integrate_ensemble(op, u0, ts)
    assert not fwd.stats["failed"]
    J, lam = adjoint.terminal_condition(grid, fwd.u_final, torch.from_numpy(ud).cuda(), op=op)
    g = adjoint.ensemble_sweep(op, ts, fwd, lam)
    ref = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, E, N, bc == "periodic"), 0.01)
    for b in range(B):
        j_ref, g_ref, uf = R.evaluate(ref, u0[b], ud[b], 0.0, steps * dt, dt, scheme)
        assert rel_err(fwd.u_final[b].cpu().numpy(), uf) <= 1e-12
        assert abs(float(J[b]) - j_ref) <= 1e-9 * abs(j_ref)
        assert rel_err(g[b].cpu().numpy(), g_ref) <= 1e-9


def test_cfg4_full_scale_gradients_vs_oracle(cuda):
    """BASELINE config 4 at full size (B = 4096, 1000 RK4 steps, 126 GB trajectory in HBM):
    J and grad J of sampled problems vs the oracle's full 1000-step evaluate (1e-9)."""
    torch.cuda.empty_cache()
    prob = configs.cfg4_problem(device="cuda:0")
    J, g = prob.evaluate(prob.u_guess)
    assert prob.last_forward.trajectory.shape[0] == 1001
    c = configs.CFG4
    ref = R.BurgersOracle(R.Mesh1D(c["xa"], c["xb"], c["E"], c["N"], True), c["nu"])
    target = prob.target().cpu().numpy()
    for b in (0, 2047, 4095):
        j_ref, g_ref, _ = R.evaluate(ref, prob.u_guess[b], target[b], 0.0,
                                     c["steps"] * c["dt"], c["dt"], "rk4")
        assert abs(float(J[b]) - j_ref) <= 1e-9 * abs(j_ref)
        assert rel_err(g[b], g_ref) <= 1e-9
    del prob, J, g
    torch.cuda.empty_cache()


@pytest.mark.parametrize("scheme", ["rk4", "rk3", "euler"])
@pytest.mark.parametrize("E", [256, 32, 96, 160])
def test_register_resident_ensemble_forward_matches_shared_memory_kernel(cuda, scheme, E):
    """N = 15 rings with 32 | E run the register-resident forward sweep (sem1d_ensrf.cuh):
    same flag words as the shared-memory kernel (sem1d_set_tile_variant(1)) and the same
    trajectory and final state to 1e-13 -- the stage arithmetic is the same, and F on the
    reflection (even/odd) split sums the same products in a different order (built with
    ENSRF_EO = 0 the two kernels are bit-identical)."""
    from paper_1806_01422_b200 import _lib
    B, steps, dt = 7, 30, 5e-5
    grid = grid_1d(0.0, 20.0, E, 15)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0", batch=B)
    u0 = configs.fourier_fields(grid, B, 4, seed=E)
    u0[3] *= 1e140                                  # one failing problem: same flag words
    ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=steps * dt, dt=dt)
    lib = _lib.load()
    runs = []
    for variant in (0, 1):
        assert lib.sem1d_set_tile_variant(variant) == 0
        try:
            runs.append(timeloop.integrate_ensemble(op, u0, ts))
        finally:
            lib.sem1d_set_tile_variant(0)
    a, b = runs
    ok = [i for i in range(B) if i != 3]            # (NaN payloads may differ: compare finite runs)
    scale = float(b.trajectory[:, ok].abs().max())
    assert float((a.trajectory[:, ok] - b.trajectory[:, ok]).abs().max()) <= 1e-13 * scale
    assert float((a.u_final[ok] - b.u_final[ok]).abs().max()) <= 1e-13 * scale
    assert a.stats["failed"] == b.stats["failed"] == [3]
    assert not bool(torch.isfinite(a.u_final[3]).all()) and not bool(torch.isfinite(b.u_final[3]).all())


def test_ensemble_adjoint_outputs_only_check_classifies(cuda):
    """The ring-resident adjoint (N = 15) tests only its outputs; a flagged sweep is re-run with
    the per-stage cotangent checks, so a non-finite cotangent still raises NumericFailure with
    unchanged counters, and the gradient of a clean batch equals the classifying kernel's."""
    import torch
    from paper_1806_01422_b200 import adjoint
    grid = grid_1d(0.0, 20.0, 256, 15)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0", batch=3)
    u0 = configs.fourier_fields(grid, 3, 4, seed=9)
    ts = sb.TsConfig(scheme="rk4", t0=0.0, t_end=20 * 5e-5, dt=5e-5)
    fwd = timeloop.integrate_ensemble(op, u0, ts)
    lam = torch.from_numpy(configs.fourier_fields(grid, 3, 4, seed=10)).cuda()
    g = adjoint.ensemble_sweep(op, ts, fwd, lam)
    flags = torch.zeros(3, dtype=torch.int32, device="cuda")
    g1 = op.empty()
    op.launch_ens_adjoint(fwd.trajectory, lam, g1, fwd.dts_device, fwd.n_steps, "rk4", flags, check=True)
    assert torch.equal(g, g1) and int(flags.max()) == 0
    bad = lam.clone()
    bad[1, 17] = float("nan")
    before = dict(op.counters)
    with pytest.raises(sb.NumericFailure, match="cotangent"):
        adjoint.ensemble_sweep(op, ts, fwd, bad)
    assert op.counters == before
