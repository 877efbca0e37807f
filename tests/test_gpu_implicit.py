"""Crank-Nicolson (Newton + GMRES) and adaptive Kutta-3 on the
B200, against the reference's own runs (tests/golden/implicit.npz) and the oracle at
larger sizes.  Tolerances: final state 1e-12, objective / gradient 1e-9 (north_star);
iteration counters exact."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import adjoint, problems, timeloop
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import golden, rel_err

pytestmark = pytest.mark.gpu

# key -> (periodic, scheme, adaptive, t_end, dt, TsConfig overrides, checkpoint slots)
CASES = {
    "cn_periodic": (True, "cn", False, 10 * 1e-3, 1e-3, {}, None),
    "cn_dirichlet": (False, "cn", False, 10 * 1e-3, 1e-3, {}, None),
    "cn_binom": (True, "cn", False, 12 * 1e-3, 1e-3, {}, 3),
    "cn_stiff": (True, "cn", False, 4 * 2e-2, 2e-2, {"gmres_restart": 8}, None),
    "ad_rms": (True, "rk3", True, 2e-2, 1e-3, {"tol_a": 1e-7, "tol_r": 1e-7}, None),
    "ad_max": (False, "rk3", True, 2e-2, 5e-4, {"tol_a": 1e-6, "tol_r": 1e-6, "wlte_form": "max"}, 4),
}


def _cfg1(periodic):
    return grid_1d(-1.0, 1.0, 16, 9, "periodic" if periodic else "dirichlet0")


@pytest.mark.parametrize("key", sorted(CASES))
def test_implicit_and_adaptive_match_reference(cuda, key):
    g = golden("implicit.npz")
    per, scheme, adaptive, t_end, dt, kw, slots = CASES[key]
    grid = _cfg1(per)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0")
    ts = timeloop.TsConfig(scheme=scheme, t0=0.0, t_end=t_end, dt=dt, adaptive=adaptive, **kw)
    prob = problems.AssimilationProblem(name=key, grid=grid, op=op, ts=ts,
                                        u_target=g[f"target_{key}"], u_guess=g[f"u0_{key}"],
                                        checkpoint_slots=slots)
    j, gr = prob.evaluate(g[f"u0_{key}"])
    fwd = prob.last_forward
    assert abs(j - g[f"J_{key}"][0]) <= 1e-9 * abs(g[f"J_{key}"][0])
    assert rel_err(gr, g[f"grad_{key}"]) <= 1e-9
    assert rel_err(fwd.u_final.cpu().numpy(), g[f"ufinal_{key}"]) <= 1e-12
    assert len(fwd.dts) == len(g[f"dts_{key}"])
    # adaptive dts: wlte is a device reduction (order differs from numpy's pairwise mean);
    # its last-bit differences feed back through the controller, and the clipped last
    # step is a difference of accumulated times -- 1e-9 relative, not bit-exact
    assert np.max(np.abs(fwd.dts - g[f"dts_{key}"]) / g[f"dts_{key}"]) <= 1e-9
    ref = g[f"fstats_{key}"]
    st = fwd.stats
    assert [st["steps"], st["rejects"], st["retries"]] == list(ref[:3])
    if scheme == "cn":
        assert [st["newton_iters"], st["gmres_iters"]] == list(ref[3:])
        assert op.last_sweep_stats["gmres_iters"] == g[f"sstats_{key}"][1]
        assert op.last_sweep_stats["newton_iters"] == g[f"sstats_{key}"][0]
        assert op.last_sweep_stats["recomputed"] == g[f"sstats_{key}"][2]
    else:
        assert op.last_sweep_stats["recomputed"] == g[f"sstats_{key}"][2]


def test_adaptive_target_run_step_log(cuda):
    """integrate(keep_log=True): accepted / rejected attempts, t, dt and wlte of the
    reference's adaptive run (timeloop.py:296-326)."""
    g = golden("implicit.npz")
    for key in ("ad_rms", "ad_max"):
        per, scheme, adaptive, t_end, dt, kw, _ = CASES[key]
        grid = _cfg1(per)
        op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0")
        ts = timeloop.TsConfig(scheme=scheme, t0=0.0, t_end=t_end, dt=dt, adaptive=adaptive, **kw)
        x = grid.node_coordinates()[0]
        u_obs0 = grid.mask(np.sin(np.pi * x) + 0.5 * np.sin(2.0 * np.pi * x))
        res = timeloop.integrate(op, u_obs0, ts, store_steps=None, keep_log=True)
        log = np.array(res.step_log, dtype=float)
        ref = g[f"tlog_{key}"]
        assert log.shape == ref.shape
        assert np.array_equal(log[:, [0, 4]], ref[:, [0, 4]])          # step index, accepted
        assert np.max(np.abs(log[:, 1:3] - ref[:, 1:3]) / np.abs(ref[:, 1:3]).clip(1e-300)) <= 1e-9
        assert np.max(np.abs(log[:, 3] - ref[:, 3]) / np.abs(ref[:, 3])) <= 1e-9    # wlte
        assert rel_err(res.u_final.cpu().numpy(), R.integrate_general(
            R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 16, 9, per), 0.01), u_obs0, 0.0, t_end, dt, scheme,
            True, kw)[0][-1]) <= 1e-12


@pytest.mark.parametrize("transpose", [False, True])
def test_gmres_matches_scipy(cuda, transpose):
    """sem1d_gmres vs scipy.sparse.linalg.gmres (the reference's solver) on
    (I - h J(p)) x = b at E = 2048, N = 7 (14336 DOF), restart 20: same matvec count,
    solution within the solver tolerance."""
    from paper_1806_01422_b200 import _lib
    E, N, nu, h = 2048, 7, 0.01, 2e-5
    grid = grid_1d(-1.0, 1.0, E, N)
    op = sb.SemOperator(grid, sb.PdeCoefficients(nu), device="cuda:0")
    orc = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, E, N, True), nu)
    p, b, _ = R.seeded_fields(op.ndof, 17)
    ts = timeloop.TsConfig(scheme="cn", gmres_restart=20, gmres_tol=1e-10, gmres_max=400)
    st = _lib.CnStats()
    x = op.empty()
    op.launch_gmres(torch.from_numpy(p).cuda(), -h, torch.from_numpy(b).cuda(), x, ts, st,
                    transpose=transpose)
    torch.cuda.synchronize()
    assert st.status == 0 and st.gmres_info == 0
    stats = {}
    f = orc.jact if transpose else orc.jac
    xr = R.gmres_solve(lambda v: v - h * f(p, v), b, 1e-10, 400, 20, stats)
    assert st.gmres_iters == stats["gmres_iters"]
    assert rel_err(x.cpu().numpy(), xr) <= 1e-9


def test_cn_step_matches_oracle_at_size(cuda):
    """One CN step at E = 4096, N = 7 (28672 DOF): Newton / GMRES counters equal the
    reference algorithm's, state within 1e-12."""
    E, N, nu, dt = 4096, 7, 0.01, 1e-4
    grid = grid_1d(0.0, 2.0, E, N)
    op = sb.SemOperator(grid, sb.PdeCoefficients(nu), device="cuda:0")
    x = grid.node_coordinates()[0]
    u = np.sin(np.pi * x) + 0.3 * np.cos(5 * np.pi * x)
    ts = timeloop.TsConfig(scheme="cn", dt=dt)
    stats = {"newton_iters": 0, "gmres_iters": 0}
    v = timeloop.step_cn(op, u, 0.0, dt, ts, stats)
    orc = R.BurgersOracle(R.Mesh1D(0.0, 2.0, E, N, True), nu)
    rs = {}
    vr = R.cn_step(orc, u, dt, None, rs)
    assert (stats["newton_iters"], stats["gmres_iters"]) == (rs["newton_iters"], rs["gmres_iters"])
    assert rel_err(v, vr) <= 1e-12


def test_cn_gradient_finite_difference(cuda):
    """The CN discrete adjoint is the exact transpose of the CN step map: directional
    derivative of J vs central differences (SURVEY.md 8(c) item 4 methodology)."""
    grid = _cfg1(True)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0")
    g = golden("implicit.npz")
    ts = timeloop.TsConfig(scheme="cn", t0=0.0, t_end=5e-3, dt=1e-3)
    prob = problems.AssimilationProblem(name="fd", grid=grid, op=op, ts=ts,
                                        u_target=g["target_cn_periodic"], u_guess=g["u0_cn_periodic"])
    u0 = g["u0_cn_periodic"]
    _, gr = prob.evaluate(u0)
    d = np.cos(3 * np.pi * grid.node_coordinates()[0])
    eps = 1e-4
    jp, _ = prob.evaluate(u0 + eps * d)
    jm, _ = prob.evaluate(u0 - eps * d)
    fd = (jp - jm) / (2 * eps)
    assert abs(fd - np.dot(gr, d)) <= 1e-7 * abs(fd)


def test_cn_failures_raise_like_reference(cuda):
    """GMRES non-convergence -> StepFailure (retried with halved dt by integrate, then
    raised); NaN input -> NumericFailure; Newton budget exhausted -> StepFailure."""
    grid = _cfg1(True)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0")
    x = grid.node_coordinates()[0]
    u = np.sin(np.pi * x)
    bad = timeloop.TsConfig(scheme="cn", t0=0.0, t_end=2e-2, dt=1e-2, gmres_max=1, gmres_restart=1,
                            gmres_tol=1e-14)
    with pytest.raises(sb.StepFailure):
        timeloop.step_cn(op, u, 0.0, 1e-2, bad)
    with pytest.raises(sb.StepFailure):
        timeloop.integrate(op, u, bad)
    stall = timeloop.TsConfig(scheme="cn", t0=0.0, t_end=1e-2, dt=1e-2, newton_max=0)
    with pytest.raises(sb.StepFailure, match="Newton stalled"):
        timeloop.step_cn(op, u, 0.0, 1e-2, stall)
    un = u.copy()
    un[3] = np.nan
    with pytest.raises(sb.NumericFailure):
        timeloop.step_cn(op, un, 0.0, 1e-3, timeloop.TsConfig(scheme="cn", dt=1e-3))
    # adjoint: a GMRES that cannot converge raises StepFailure (adjoint.py:65-68)
    with pytest.raises(sb.StepFailure):
        adjoint.adjoint_step_cn(op, u, u, np.cos(np.pi * x), 0.0, 1e-2, bad)


@pytest.mark.parametrize("form,tol", [("max", 1e-7), ("rms", 1e-6)])
def test_adaptive_larger_ring_replays_on_oracle(cuda, form, tol):
    """Adaptive Kutta-3 at E = 512, N = 7 (3584 DOF, stability-limited: dozens of rejects).
    Adaptive step sequences are not reproducible bit for bit across implementations --
    the reference itself moves its dt sequence by up to ~1e-1 under a 1e-15 perturbation
    of u0 in this regime, since err = u_new - u_hat is a cancellation at the tolerance
    level.  So every attempt of the GPU run (keep_log) is replayed on the oracle from the
    same state and dt: the oracle's wlte must agree (1e-6), give the same accept / reject
    decision and the same proposed dt, and the accepted states must chain to the GPU's
    final state (1e-11)."""
    E, N, nu = 512, 7, 0.01
    grid = grid_1d(0.0, 4.0, E, N)
    op = sb.SemOperator(grid, sb.PdeCoefficients(nu), device="cuda:0")
    x = grid.node_coordinates()[0]
    u0 = np.sin(np.pi * x) + 0.5 * np.sin(3 * np.pi * x)
    kw = {"tol_a": tol, "tol_r": tol, "wlte_form": form}
    ts = timeloop.TsConfig(scheme="rk3", t0=0.0, t_end=5e-3, dt=1e-3, adaptive=True, **kw)
    res = timeloop.integrate(op, u0, ts, store_steps=None, keep_log=True)
    assert res.stats["rejects"] > 0
    orc = R.BurgersOracle(R.Mesh1D(0.0, 4.0, E, N, True), nu)
    u = u0.copy()
    log = res.step_log
    for i, (n, t, dt, wlte, accepted) in enumerate(log):
        un, uh, err = R.rk3_step_embedded(orc, u, dt)
        acc, prop, w = R.controller(err, un, uh, dt, kw)
        assert abs(w - wlte) <= 1e-6 * abs(wlte)
        assert acc == bool(accepted)
        if i + 1 < len(log):
            # next attempt starts at this row's t (timeloop.py:268-270 clipping rule)
            remaining = ts.t_end - t
            expect = remaining if remaining - prop <= 1e-9 * ts.dt else prop
            assert abs(log[i + 1][2] - expect) <= 1e-6 * expect
        if accepted:
            u = un
    assert rel_err(res.u_final.cpu().numpy(), u) <= 1e-11


# -- LINEAR / NONE advection (ops.py:147-212 branches; problems advdiff1d / diffusion1d) ------

ADV_CASES = [("lin_p", "periodic", "linear", [0.3]), ("lin_d", "dirichlet0", "linear", [-0.7]),
             ("none_p", "periodic", "none", None), ("none_d", "dirichlet0", "none", None)]


@pytest.mark.parametrize("key,bc,kind,speed", ADV_CASES)
def test_advection_kinds_ops_match_reference(cuda, key, bc, kind, speed):
    g = golden("advkinds.npz")
    grid = grid_1d(-1.0, 1.0, 6, 5, bc)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.02, kind, speed=speed), device="cuda:0")
    u, v, w = g[f"u_{key}"], g[f"v_{key}"], g[f"w_{key}"]
    assert rel_err(op.apply_rhs(u), g[f"F_{key}"]) <= 1e-12
    assert rel_err(op.apply_jacobian(u, v), g[f"J_{key}"]) <= 1e-12
    assert rel_err(op.apply_jacobian_transpose(u, w), g[f"JT_{key}"]) <= 1e-12
    bad = u.copy()
    bad[2] = np.inf                     # u is validated even though J does not use it
    with pytest.raises(sb.NumericFailure):
        op.apply_jacobian(bad, v)


@pytest.mark.parametrize("name,kw", [("advdiff1d", {"steps": 20, "horizon": 0.004}),
                                     ("diffusion1d", {"steps": 20, "horizon": 0.01}),
                                     ("advdiff1d_cn", {"steps": 5, "horizon": 0.004, "scheme": "cn"})])
def test_advdiff_and_diffusion_problems_match_reference(cuda, name, kw):
    g = golden("advkinds.npz")
    prob = problems.make_problem(name.split("_")[0], device="cuda:0", **kw)
    assert rel_err(prob.u_target, g[f"{name}_target"]) <= 1e-15
    assert rel_err(prob.u_exact_ic, g[f"{name}_exact_ic"]) <= 1e-15
    j, gr = prob.evaluate(g[f"{name}_u0"])
    assert abs(j - g[f"{name}_J"][0]) <= 1e-9 * abs(g[f"{name}_J"][0])
    assert rel_err(gr, g[f"{name}_grad"]) <= 1e-9
    assert rel_err(prob.last_forward.u_final.cpu().numpy(), g[f"{name}_ufinal"]) <= 1e-12
