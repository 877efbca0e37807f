"""Forward/adjoint sweep parity on the B200: evaluate() vs the reference fixtures
(RK3 / Euler, periodic / Dirichlet) and vs the RK4 oracle restatement, within 1e-9
relative on u(T), J and grad J (BASELINE north_star); checkpointing transparency;
failure semantics; L-BFGS trajectory."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import adjoint, checkpoint, configs, timeloop
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import golden, rel_err

pytestmark = pytest.mark.gpu
SWEEP_TOL = 1e-9


def _cfg1(bc, scheme, slots=None, t_end=20 * 1e-4, target=None):
    grid = grid_1d(-1.0, 1.0, 16, 9, bc)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0")
    ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=t_end, dt=1e-4)
    return sb.AssimilationProblem(name="cfg1", grid=grid, op=op, ts=ts, u_target=target,
                                  u_guess=None, checkpoint_slots=slots)


@pytest.mark.parametrize("bc", ["periodic", "dirichlet0"])
@pytest.mark.parametrize("scheme", ["rk3", "euler"])
def test_evaluate_vs_reference(cuda, bc, scheme):
    g = golden("sweeps.npz")
    key = f"{bc}_{scheme}"
    prob = _cfg1(bc, scheme, target=g[f"target_{key}"])
    j, grad = prob.evaluate(g[f"u0_{key}"])
    assert abs(j - g[f"J_{key}"][0]) <= SWEEP_TOL * abs(g[f"J_{key}"][0])
    assert rel_err(grad, g[f"grad_{key}"]) <= SWEEP_TOL
    assert rel_err(prob.last_forward.u_final.cpu().numpy(), g[f"ufinal_{key}"]) <= SWEEP_TOL
    assert np.array_equal(prob.last_forward.dts, g[f"dts_{key}"])
    # the fixture's operator also ran the target's forward sweep (20 steps x stages)
    rhs, _, jact = g[f"counters_{key}"]
    stages = {"rk3": 3, "euler": 1}[scheme]
    assert prob.op.counters["rhs"] == rhs - 20 * stages and prob.op.counters["jact"] == jact


def test_binomial_is_bitwise_store_all(cuda):
    g = golden("sweeps.npz")
    a = _cfg1("periodic", "rk3", target=g["target_periodic_rk3"])
    b = _cfg1("periodic", "rk3", slots=4, target=g["target_periodic_rk3"])
    ja, ga = a.evaluate(g["u0_periodic_rk3"])
    jb, gb = b.evaluate(g["u0_periodic_rk3"])
    assert ja == jb and np.array_equal(ga, gb)
    assert b.op.last_sweep_stats["recomputed"] == checkpoint.plan_binomial(20, 4).recomputed


def test_long_clipped_run_with_checkpoints(cuda):
    g = golden("sweeps.npz")
    prob = _cfg1("periodic", "rk3", slots=10, t_end=0.0123, target=g["long_target"])
    j, grad = prob.evaluate(g["u0_periodic_rk3"])
    assert abs(j - g["long_J"][0]) <= SWEEP_TOL * abs(g["long_J"][0])
    assert rel_err(grad, g["long_grad"]) <= SWEEP_TOL
    assert np.array_equal(prob.last_forward.dts, g["long_dts"])


@pytest.mark.parametrize("bc", ["periodic", "dirichlet0"])
def test_rk4_vs_oracle_restatement(cuda, bc):
    """BASELINE config 1 as specified (RK4): vs the oracle's RK4 restatement."""
    prob = configs.cfg1_problem(bc=bc, scheme="rk4", device="cuda:0")
    u0, obs0 = configs.cfg1_inputs(prob.grid)
    m = R.Mesh1D(-1.0, 1.0, 16, 9, bc == "periodic")
    ref = R.BurgersOracle(m, 0.01)
    traj, _ = R.forward(ref, obs0, 0.0, 20e-4, 1e-4, "rk4")
    target_gpu = prob.op.field(prob.u_target)[0].cpu().numpy()
    assert rel_err(target_gpu, traj[-1]) <= SWEEP_TOL
    j, grad = prob.evaluate(u0)
    j_ref, g_ref, uf_ref = R.evaluate(ref, u0, target_gpu, 0.0, 20e-4, 1e-4, "rk4")
    assert abs(j - j_ref) <= SWEEP_TOL * abs(j_ref)
    assert rel_err(grad, g_ref) <= SWEEP_TOL
    assert rel_err(prob.last_forward.u_final.cpu().numpy(), uf_ref) <= SWEEP_TOL


def test_rk4_gradient_matches_finite_differences(cuda):
    prob = configs.cfg1_problem(scheme="rk4", device="cuda:0")
    u0 = configs.cfg1_inputs(prob.grid)[0]
    j, grad = prob.evaluate(u0)
    rng = np.random.default_rng(3)
    for _ in range(5):
        d = rng.standard_normal(u0.size)
        eps = 1e-4
        fd = (prob.evaluate(u0 + eps * d)[0] - prob.evaluate(u0 - eps * d)[0]) / (2 * eps)
        assert abs(fd - grad @ d) <= 1e-6 * max(1.0, abs(fd))


def test_terminal_condition_kats(cuda):
    grid = grid_1d(-1.0, 1.0, 16, 9, "dirichlet0")
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0")
    u = np.random.default_rng(0).standard_normal(grid.nglobal)
    j, lam = adjoint.terminal_condition(grid, u, u, op=op)
    assert j == 0.0 and not lam.any()
    e = np.zeros(grid.nglobal)
    e[40] = 1.0
    j, lam = adjoint.terminal_condition(grid, e, np.zeros_like(e), op=op)
    assert j == grid.mass_scalar[40] and lam[40] == 2 * grid.mass_scalar[40]
    ref = R.terminal(R.Mesh1D(-1.0, 1.0, 16, 9, False), u, 0.5 * u)
    j, lam = adjoint.terminal_condition(grid, u, 0.5 * u, op=op)
    assert abs(j - ref[0]) <= 1e-13 * ref[0] and np.array_equal(lam, ref[1])


def test_step_failure_retry_and_numeric_failure(cuda):
    grid = grid_1d(-1.0, 1.0, 16, 9)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0")
    u0 = np.sin(np.pi * grid.node_coordinates()[0])
    with pytest.raises(sb.NumericFailure, match="initial state"):
        timeloop.integrate(op, np.full(grid.nglobal, np.nan), sb.TsConfig(t_end=1e-3, dt=1e-4))
    # a wildly unstable dt blows up inside a stage -> NumericFailure (not retried),
    # exactly like the reference where the stage apply raises before _check_state
    with pytest.raises(sb.NumericFailure):
        timeloop.integrate(op, 1e150 * u0, sb.TsConfig(scheme="rk4", t_end=1.0, dt=0.5))
    fwd = timeloop.integrate(op, u0, sb.TsConfig(scheme="rk4", t_end=1e-3, dt=1e-4))
    assert fwd.n_steps == 10 and len(fwd.snapshots) == 11


def test_lbfgs_three_iterations_vs_reference(cuda):
    g = golden("sweeps.npz")
    prob = _cfg1("periodic", "rk3", target=None)
    grid = prob.grid
    u0, obs0 = configs.cfg1_inputs(grid)
    prob.u_target = timeloop.integrate(prob.op, obs0, prob.ts, store_steps=None).u_final
    res = sb.minimize(prob.evaluate, torch.from_numpy(u0).to(cuda), sb.OptimConfig(max_iters=3))
    ref = g["opt_log"]
    assert len(res.log) == len(ref)
    for row, rrow in zip(res.log, ref):
        assert row[0] == rrow[0] and row[4] == rrow[4]          # iteration, fevals
        assert abs(row[1] - rrow[1]) <= 1e-8 * abs(rrow[1])     # J
        assert abs(row[2] - rrow[2]) <= 1e-8 * abs(rrow[2])     # |g|
    assert rel_err(res.x.cpu().numpy(), g["opt_x"]) <= 1e-8
