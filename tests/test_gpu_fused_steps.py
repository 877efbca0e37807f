"""Temporally blocked whole-step kernels (sem1d_rk_step / sem1d_adj_step) for large
periodic rings: same trajectory / gradient as the per-stage kernels (to rounding of the
apply order) and as the oracle within the sweep tolerance."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import adjoint, checkpoint, timeloop
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import rel_err

pytestmark = pytest.mark.gpu


def _problem(E, N, nu, dt, steps, scheme, seed):
    g = grid_1d(0.0, 2.0, E, N)
    op = sb.SemOperator(g, sb.PdeCoefficients(nu), device="cuda:0")
    x = g.node_coordinates()[0]
    rng = np.random.default_rng(seed)
    u0 = np.sin(np.pi * x) + 0.3 * np.cos(3 * np.pi * x) + 0.01 * rng.standard_normal(g.nglobal)
    ud = np.sin(np.pi * x + 0.2)
    ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=steps * dt, dt=dt)
    return g, op, u0, ud, ts


@pytest.mark.parametrize("scheme", ["rk4", "rk3", "euler"])
@pytest.mark.parametrize("E,N,dt", [(1061, 7, 2e-6), (301, 15, 2e-7), (260, 31, 1e-8)])
def test_fused_step_sweeps(cuda, scheme, E, N, dt):
    steps = 6
    g, op, u0, ud, ts = _problem(E, N, 1e-3, dt, steps, scheme, E)
    assert op.step_fused_supported()
    fwd = timeloop.integrate(op, u0, ts)
    J, lam = adjoint.terminal_condition(g, fwd.u_final, torch.from_numpy(ud).cuda(), op=op)
    gr = adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(steps), lam)
    # per-stage kernels on the same inputs
    op.use_fused_steps = False
    fwd2 = timeloop.integrate(op, u0, ts)
    J2, lam2 = adjoint.terminal_condition(g, fwd2.u_final, torch.from_numpy(ud).cuda(), op=op)
    gr2 = adjoint.sweep(op, ts, fwd2, checkpoint.plan_store_all(steps), lam2)
    op.use_fused_steps = True
    assert rel_err(fwd.u_final.cpu().numpy(), fwd2.u_final.cpu().numpy()) <= 1e-13
    assert rel_err(gr.cpu().numpy(), gr2.cpu().numpy()) <= 1e-12
    ref = R.BurgersOracle(R.Mesh1D(0.0, 2.0, E, N, True), 1e-3)
    j_ref, g_ref, uf = R.evaluate(ref, u0, ud, 0.0, steps * dt, dt, scheme)
    assert rel_err(fwd.u_final.cpu().numpy(), uf) <= 1e-12
    assert abs(J - j_ref) <= 1e-9 * abs(j_ref)
    assert rel_err(gr.cpu().numpy(), g_ref) <= 1e-9


def test_fused_step_flags(cuda):
    g, op, u0, ud, ts = _problem(1061, 7, 1e-3, 2e-6, 3, "rk4", 1)
    u0[100] = np.nan
    with pytest.raises(sb.NumericFailure):
        timeloop.integrate(op, u0, ts)
    # a blow-up inside the step -> StepFailure retries, then gives up like the reference
    g, op, u0, ud, ts = _problem(1061, 7, 1e-3, 0.5, 3, "rk4", 1)
    with pytest.raises(sb.NumericFailure):
        timeloop.integrate(op, 1e150 * u0, ts)


@pytest.mark.parametrize("scheme,E,N,dt", [("rk4", 1061, 7, 2e-6), ("rk3", 1061, 7, 2e-6),
                                          ("rk4", 301, 15, 2e-7), ("rk4", 260, 31, 1e-8)])
def test_stage_states_in_hbm_match_recompute(cuda, scheme, E, N, dt):
    """integrate(keep_stages=True) + sweep: the adjoint reads the stored stage states instead
    of recomputing them (sem1d_rk_step_stages / sem1d_adj_step_stages); the gradient equals
    the recompute path's and evaluate() picks it for store-all runs."""
    from paper_1806_01422_b200 import adjoint, checkpoint
    g = grid_1d(0.0, 2.0, E, N)
    op = sb.SemOperator(g, sb.PdeCoefficients(1e-3), device="cuda:0")
    assert op.step_fused_supported()
    x = g.node_coordinates()[0]
    u0 = torch.from_numpy(np.sin(np.pi * x) + 0.3 * np.cos(3 * np.pi * x)).cuda()
    ts = timeloop.TsConfig(scheme=scheme, t0=0.0, t_end=12 * dt, dt=dt)
    assert op.step_stages_supported()
    grads = {}
    for keep in (True, False):
        fwd = timeloop.integrate(op, u0, ts, keep_stages=keep)
        assert (len(fwd.stage_snapshots) == fwd.n_steps) == keep
        j, lam = adjoint.terminal_condition(g, fwd.u_final, 0.5 * u0, op=op)
        grads[keep] = adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(fwd.n_steps), lam).cpu().numpy()
    assert rel_err(grads[True], grads[False]) <= 1e-13
    prob = sb.AssimilationProblem(name="ks", grid=g, op=op, ts=ts, u_target=0.5 * u0.cpu().numpy(),
                                  u_guess=u0.cpu().numpy())
    _, ge = prob.evaluate(u0)
    assert len(prob.last_forward.stage_snapshots) == prob.last_forward.n_steps
    assert rel_err(ge.cpu().numpy(), grads[False]) <= 1e-13
