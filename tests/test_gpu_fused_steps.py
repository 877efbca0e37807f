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


def _inject_failures(op, u0, t0, fail_rule):
    """Wrap the fused step launches: a step starting at time T (tracked through the states'
    sums) whose dt exceeds fail_rule[T] reports a non-finite step result through whichever
    flag word it was given -- a deterministic failure, the same whether the step runs ahead
    or is checked at once."""
    from paper_1806_01422_b200 import _lib
    time_of = {float(torch.as_tensor(u0, device="cuda:0").sum()): t0}
    orig_plain, orig_st = op.launch_rk_step, op.launch_rk_step_stages

    def mark(u, u_new, dt, flag):
        t = time_of[float(u.sum())]
        time_of[float(u_new.sum())] = t + dt
        rule = next((v for k, v in fail_rule.items() if abs(k - t) < 1e-12), None)
        if rule is not None and dt > rule:
            if flag is None:
                op._flag.fill_(_lib.SEM1D_FLAG_STEP_NONFINITE)
            else:
                tt = op._flag_slots_t
                tt[(flag - tt.data_ptr()) // 4] = _lib.SEM1D_FLAG_STEP_NONFINITE

    def plain(u, u_new, dt, scheme, flag=None):
        orig_plain(u, u_new, dt, scheme, flag=flag)
        mark(u, u_new, dt, flag)

    def staged(u, u_new, stages, dt, scheme, flag=None):
        orig_st(u, u_new, stages, dt, scheme, flag=flag)
        mark(u, u_new, dt, flag)

    op.launch_rk_step, op.launch_rk_step_stages = plain, staged


@pytest.mark.parametrize("store", ["all", "some"])
@pytest.mark.parametrize("keep", [False, True])
def test_run_ahead_rollback_matches_per_step_checks(cuda, store, keep):
    """integrate() launches fixed-dt fused steps ahead and verifies their per-step flag words
    once per window; a flagged step rolls the run back and is re-run with the per-step check.
    With the same (deterministic) step failures -- the step from t = 1e-5 fails at dt and
    passes at dt/2, the ones from 2e-5 and 3e-5 fail at dt/2 and dt/4 -- the result
    (time grid, trajectory, stage snapshots, counters, retries, log) is identical to the loop
    that checks every step."""
    steps = 40
    out = {}
    for mode in ("ahead", "sync"):
        g, op, u0, ud, ts = _problem(1061, 7, 1e-3, 2e-6, steps, "rk4", 3)
        if mode == "sync":
            op.supports_flag_slots = False
        _inject_failures(op, u0, 0.0, {1e-5: 1.5e-6, 2e-5: 0.75e-6, 3e-5: 0.3e-6})
        st = "all" if store == "all" else [0, 7, 19, 33]
        out[mode] = timeloop.integrate(op, u0, ts, store_steps=st, keep_log=True, keep_stages=keep)
        out[mode + "_counters"] = dict(op.counters)
    a, b = out["ahead"], out["sync"]
    assert out["ahead_counters"] == out["sync_counters"]      # rolled-back steps are not counted
    assert np.array_equal(a.ts, b.ts) and np.array_equal(a.dts, b.dts)
    assert a.stats == b.stats and a.stats["retries"] == 3
    assert a.step_log == b.step_log
    assert sorted(a.snapshots) == sorted(b.snapshots)
    for k in a.snapshots:
        assert torch.equal(a.snapshots[k], b.snapshots[k])
    assert torch.equal(a.u_final, b.u_final)
    assert sorted(a.stage_snapshots) == sorted(b.stage_snapshots)
    for k in a.stage_snapshots:
        for x, y in zip(a.stage_snapshots[k], b.stage_snapshots[k]):
            assert torch.equal(x, y)


def test_run_ahead_raises_like_per_step_checks(cuda):
    """A step that fails at every dt exhausts the halvings: StepFailure from the run-ahead
    loop as from the per-step-checked one."""
    for mode in ("ahead", "sync"):
        g, op, u0, ud, ts = _problem(1061, 7, 1e-3, 2e-6, 30, "rk4", 3)
        if mode == "sync":
            op.supports_flag_slots = False
        _inject_failures(op, u0, 0.0, {9 * 2e-6: 0.0})
        with pytest.raises(sb.StepFailure):
            timeloop.integrate(op, u0, ts)


@pytest.mark.parametrize("keep", [False, True])
@pytest.mark.parametrize("bad_step", [None, 3, 21, 37])
def test_adjoint_run_ahead_matches_per_step_checks(cuda, keep, bad_step):
    """sweep() runs ahead on the fused adjoint-step kernels (per-step flag words, one read
    per window of 16 steps).  Without a failure the gradient is bitwise that of the
    per-step-checked sweep; with a non-finite state planted at step `bad_step` both raise
    the same NumericFailure with the same counters."""
    steps = 40
    out = {}
    for mode in ("ahead", "sync"):
        g, op, u0, ud, ts = _problem(1061, 7, 1e-3, 2e-6, steps, "rk4", 5)
        fwd = timeloop.integrate(op, u0, ts, keep_stages=keep)
        if bad_step is not None:
            nan_state = fwd.snapshots[bad_step].clone()
            nan_state[77] = float("nan")
            fwd.snapshots[bad_step] = nan_state
        J, lam = adjoint.terminal_condition(g, fwd.u_final, torch.from_numpy(ud).cuda(), op=op)
        before = dict(op.counters)
        kw = {} if mode == "ahead" else {"check_every": 1}
        try:
            out[mode] = ("ok", adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(steps), lam, **kw).clone())
        except sb.NumericFailure as exc:
            out[mode] = ("raised", str(exc))
        out[mode + "_counters"] = {k: op.counters[k] - before[k] for k in op.counters}
    assert out["ahead"][0] == out["sync"][0] == ("ok" if bad_step is None else "raised")
    if bad_step is None:
        assert torch.equal(out["ahead"][1], out["sync"][1])
    else:
        assert out["ahead"][1] == out["sync"][1]
    assert out["ahead_counters"] == out["sync_counters"]


def test_adjoint_run_ahead_binomial_and_cotangent_failure(cuda):
    """Run-ahead across recompute Advances (binomial schedule) equals store-all bitwise; a
    NaN terminal cotangent raises 'cotangent' at the first adjoint step in both modes."""
    steps = 35
    g, op, u0, ud, ts = _problem(1061, 7, 1e-3, 2e-6, steps, "rk4", 6)
    fwd = timeloop.integrate(op, u0, ts)
    J, lam = adjoint.terminal_condition(g, fwd.u_final, torch.from_numpy(ud).cuda(), op=op)
    ref = adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(steps), lam, check_every=1).clone()
    sched = checkpoint.plan_binomial(steps, 4)
    fwd_b = timeloop.integrate(op, u0, ts, store_steps=sched.forward_stores.keys())
    got = adjoint.sweep(op, ts, fwd_b, sched, lam)
    assert torch.equal(got, ref)
    bad = lam.clone()
    bad[5] = float("inf")
    for kw in ({}, {"check_every": 1}):
        with pytest.raises(sb.NumericFailure, match="cotangent"):
            adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(steps), bad, **kw)
