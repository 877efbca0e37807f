"""The drop-in, executed: INTEGRATION.md's reference-side binding (integration/semopt_b200.py,
a SemOperator subclass calling libsemb200.so) plugged into the UNMODIFIED reference package
(semopt 0.1.0, installed into baseline/_ref) and driven by the reference's own
timeloop.integrate / adjoint.sweep / AssimilationProblem.evaluate / optimize.minimize
(problems.py:184-199, timeloop.py:237-329, adjoint.py:72-158, optimize.py:210-265).
Objective and gradient must match stock semopt's own to 1e-9 (BASELINE north_star)."""

import importlib
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def semopt(cuda):
    if not os.path.isdir(os.path.join(REF, "semopt")):
        pytest.skip("baseline/_ref (stock semopt) is not installed on this box; see DESIGN.md section 9")
    sys.path.insert(0, REF)
    mods = {m: importlib.import_module(f"semopt.{m}") for m in
            ("grid", "ops", "timeloop", "adjoint", "problems", "optimize", "errors", "checkpoint")}
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    mods["b200"] = importlib.import_module("semopt_b200")
    return mods


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _swap(prob, S):
    twin = S["problems"].AssimilationProblem(**{k: getattr(prob, k) for k in (
        "name", "grid", "op", "ts", "u_target", "u_guess", "u_exact_ic", "exact_solution",
        "checkpoint_slots")})
    twin.op = S["b200"].B200SemOperator(prob.grid, prob.op.coef)
    return twin


@pytest.mark.parametrize("slots", [None, 7])
def test_stock_burgers1d_evaluate(semopt, slots):
    """The reference's own burgers1d problem (Dirichlet0, E = 5, N = 8, Kutta-3, 400 steps),
    store-all and binomial checkpointing."""
    S = semopt
    prob = S["problems"].burgers1d_problem(checkpoint_slots=slots)
    j_ref, g_ref = prob.evaluate(prob.u_guess)
    twin = _swap(prob, S)
    j, g = twin.evaluate(prob.u_guess)
    assert abs(j - j_ref) <= 1e-9 * abs(j_ref)
    assert rel(g, g_ref) <= 1e-9
    assert twin.op.counters["rhs"] == prob.op.counters["rhs"] > 0
    assert twin.op.counters["jact"] == prob.op.counters["jact"] > 0


def test_stock_periodic_config1_evaluate_and_minimize(semopt):
    """BASELINE config 1's ring (periodic, E = 16, N = 9, nu = 0.01, 20 Kutta-3 steps of 1e-4)
    through stock AssimilationProblem.evaluate and three stock L-BFGS iterations."""
    S = semopt
    g = S["grid"].grid_1d(-1.0, 1.0, 16, 9)
    coef = S["ops"].PdeCoefficients(0.01)
    x = g.node_coordinates()[0]
    rng = np.random.default_rng(1806)
    u0 = np.sin(np.pi * x) + 0.01 * rng.standard_normal(x.size)
    ts = S["timeloop"].TsConfig(scheme="rk3", t0=0.0, t_end=20 * 1e-4, dt=1e-4)
    op_ref = S["ops"].SemOperator(g, coef)
    target = S["timeloop"].integrate(op_ref, np.sin(np.pi * x) + 0.5 * np.sin(2 * np.pi * x), ts).u_final
    mk = S["problems"].AssimilationProblem
    prob = mk(name="cfg1", grid=g, op=op_ref, ts=ts, u_target=target, u_guess=u0)
    twin = mk(name="cfg1", grid=g, op=S["b200"].B200SemOperator(g, coef), ts=ts, u_target=target,
              u_guess=u0)
    j_ref, g_ref = prob.evaluate(u0)
    j, gr = twin.evaluate(u0)
    assert abs(j - j_ref) <= 1e-9 * abs(j_ref) and rel(gr, g_ref) <= 1e-9
    cfg = S["optimize"].OptimConfig(max_iters=3, gtol=0.0)
    r_ref = S["optimize"].minimize(prob.evaluate, u0, cfg)
    r = S["optimize"].minimize(twin.evaluate, u0, cfg)
    assert r.iterations == r_ref.iterations and r.fevals == r_ref.fevals and r.status == r_ref.status
    for a, b in zip(r.log, r_ref.log):
        assert a[0] == b[0] and a[4] == b[4]
        assert abs(a[1] - b[1]) <= 1e-9 * abs(b[1]) and abs(a[2] - b[2]) <= 1e-8 * abs(b[2])
    assert rel(r.x, r_ref.x) <= 1e-9


def test_stock_error_semantics(semopt):
    """ValidationError on a wrong shape and NumericFailure on NaN, raised from inside the stock
    time loop exactly as with the stock operator (ops.py:216-224)."""
    S = semopt
    g = S["grid"].grid_1d(-1.0, 1.0, 16, 9)
    op = S["b200"].B200SemOperator(g, S["ops"].PdeCoefficients(0.01))
    with pytest.raises(S["errors"].ValidationError):
        op.apply_rhs(np.zeros(g.nglobal + 1))
    bad = np.zeros(g.nglobal)
    bad[3] = np.nan
    ts = S["timeloop"].TsConfig(scheme="rk3", t0=0.0, t_end=1e-3, dt=1e-4)
    with pytest.raises(S["errors"].NumericFailure):
        S["timeloop"].integrate(S["ops"].SemOperator(g, S["ops"].PdeCoefficients(0.01)), bad, ts)
    with pytest.raises(S["errors"].NumericFailure):
        S["timeloop"].integrate(op, bad, ts)
    assert np.array_equal(op.apply_rhs(np.zeros(g.nglobal)), np.zeros(g.nglobal))   # flag cleared
