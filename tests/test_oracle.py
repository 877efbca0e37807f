"""The oracle (oracle/semref.py) pinned against fixtures made by the REAL reference
(tests/golden/make_golden.py), plus the SPEC.md known-answer tests."""

import numpy as np
import pytest

from oracle import semref as R
from semtest_util import golden

DEGREES = list(range(1, 33)) + [48, 64]


@pytest.mark.parametrize("n", DEGREES)
def test_basis_bit_exact(n):
    g = golden("basis.npz")
    x, w = R.gll_nodes_weights(n)
    assert np.array_equal(x, g[f"nodes_{n}"])
    assert np.array_equal(w, g[f"weights_{n}"])
    assert np.array_equal(R.diff_matrix(x), g[f"diff_{n}"])
    op = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 16, n), 0.01)
    assert np.array_equal(op.K, g[f"K_{n}"])
    assert np.array_equal(op.Dw, g[f"Dw_{n}"])


def test_basis_kats():
    # SPEC.md:43-45,52-54
    x, w = R.gll_nodes_weights(1)
    assert np.allclose(x, [-1, 1]) and np.allclose(w, [1, 1])
    x, w = R.gll_nodes_weights(2)
    assert np.allclose(x, [-1, 0, 1], atol=1e-15) and np.allclose(w, [1 / 3, 4 / 3, 1 / 3])
    assert np.allclose(R.diff_matrix(R.gll_nodes_weights(1)[0]), [[-0.5, 0.5], [-0.5, 0.5]])
    x, w = R.gll_nodes_weights(8)
    assert abs(np.sum(w * x ** 14) - 2.0 / 15.0) <= 1e-14
    for n in range(1, 17):
        x, w = R.gll_nodes_weights(n)
        for k in range(2 * n):
            exact = 0.0 if k % 2 else 2.0 / (k + 1)
            assert abs(np.sum(w * x ** k) - exact) <= 1e-12
        d = R.diff_matrix(x)
        for k in range(1, n + 1):
            assert np.max(np.abs(d @ x ** k - k * x ** (k - 1))) <= 1e-10


def _mesh_from_case(c):
    xa, xb, e, n, per = c[:5]
    return R.Mesh1D(xa, xb, int(e), int(n), bool(per))


def test_maps_bit_exact():
    g = golden("maps.npz")
    k = 0
    while f"case_{k}" in g:
        m = _mesh_from_case(g[f"case_{k}"])
        assert np.array_equal(m.table, g[f"table_{k}"])
        assert np.array_equal(m.multiplicity, g[f"mult_{k}"])
        assert np.array_equal(m.mass, g[f"mass_{k}"])
        assert np.array_equal(m.maskv, g[f"mask_{k}"])
        assert np.array_equal(m.coordinates(), g[f"coords_{k}"])
        k += 1
    assert k >= 10


def test_ops_bit_exact():
    g = golden("ops.npz")
    k = 0
    while f"case_{k}" in g:
        c = g[f"case_{k}"]
        op = R.BurgersOracle(_mesh_from_case(c), c[5])
        u, v, w = g[f"u_{k}"], g[f"v_{k}"], g[f"w_{k}"]
        assert np.array_equal(op.rhs(u), g[f"f_{k}"])
        assert np.array_equal(op.jac(u, v), g[f"jv_{k}"])
        assert np.array_equal(op.jact(u, w), g[f"jtw_{k}"])
        k += 1


@pytest.mark.parametrize("bc", ["periodic", "dirichlet0"])
@pytest.mark.parametrize("scheme", ["rk3", "euler"])
def test_sweep_bit_exact(bc, scheme):
    g = golden("sweeps.npz")
    key = f"{bc}_{scheme}"
    op = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 16, 9, bc == "periodic"), 0.01)
    j, grad, uf = R.evaluate(op, g[f"u0_{key}"], g[f"target_{key}"], 0.0, 20 * 1e-4, 1e-4, scheme)
    assert j == g[f"J_{key}"][0]
    assert np.array_equal(grad, g[f"grad_{key}"])
    assert np.array_equal(uf, g[f"ufinal_{key}"])
    _, dts = R.step_sizes(0.0, 20 * 1e-4, 1e-4)
    assert np.array_equal(dts, g[f"dts_{key}"])
    # binomial checkpointing replays identical arithmetic
    assert np.array_equal(grad, g[f"gradbinom_{key}"])


def test_long_sweep_clipped_last_step():
    g = golden("sweeps.npz")
    op = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 16, 9, True), 0.01)
    u0 = g["u0_periodic_rk3"]
    j, grad, _ = R.evaluate(op, u0, g["long_target"], 0.0, 0.0123, 1e-4, "rk3")
    assert j == g["long_J"][0]
    assert np.array_equal(grad, g["long_grad"])
    _, dts = R.step_sizes(0.0, 0.0123, 1e-4)
    assert np.array_equal(dts, g["long_dts"])


def test_rk4_restatement_matches_finite_differences():
    """RK4 is absent from the reference: pin its adjoint by central FD."""
    g = golden("sweeps.npz")
    op = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 16, 9, True), 0.01)
    u0, tgt = g["u0_periodic_rk3"], g["target_periodic_rk3"]
    j, grad, _ = R.evaluate(op, u0, tgt, 0.0, 20 * 1e-4, 1e-4, "rk4")
    rng = np.random.default_rng(7)
    for _ in range(3):
        d = rng.standard_normal(u0.size)

        def fun(u):
            return R.evaluate(op, u, tgt, 0.0, 20 * 1e-4, 1e-4, "rk4")[0]

        fd = R.finite_difference_gradient(fun, u0, d, eps=1e-4)
        assert abs(fd - grad @ d) <= 1e-7 * max(1.0, abs(fd))


def test_rk3_scalar_kat():
    """u' = -u, dt = 0.1, u0 = 1 -> 0.9048375 (scalar surrogate of the tableau)."""

    class Scalar:
        def rhs(self, u):
            return -u

    # SPEC.md:266 quotes 0.9048375 with the bound |u' - e^-0.1| <= 5e-6; Kutta-3 gives
    # 1 - 0.1 + 0.005 - 1/6000 = 0.904833..., and 0.9048375 is the RK4 value exactly.
    u = R.rk_step(Scalar(), np.array([1.0]), 0.1, "rk3")
    assert abs(u[0] - np.exp(-0.1)) <= 5e-6
    assert abs(u[0] - (1 - 0.1 + 0.005 - 0.1 ** 3 / 6)) < 1e-15
    u4 = R.rk_step(Scalar(), np.array([1.0]), 0.1, "rk4")
    assert abs(u4[0] - 0.9048375) < 1e-15


def test_dot_product_identity_oracle():
    rng = np.random.default_rng(3)
    for per in (True, False):
        op = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 3, 4, per), 0.01)
        for _ in range(50):
            # Dirichlet tangent/cotangent fields keep zero boundary entries (SPEC.md ops Field)
            u, w, z = (op.mesh.apply_mask(rng.standard_normal(op.mesh.ndof)) for _ in range(3))
            lhs = op.jac(u, w) @ z
            rhs = w @ op.jact(u, z)
            assert abs(lhs - rhs) / (np.linalg.norm(w) * np.linalg.norm(z)) <= 1e-13


def test_binomial_dp_matches_reference_counts():
    s = golden("schedules.npz")
    for m, slots in [(10, 3), (20, 4), (30, 5), (100, 10), (57, 7)]:
        assert R.binomial_recompute_table(m, slots) - m == s[f"meta_{m}_{slots}"][0]


# Crank-Nicolson / adaptive Kutta-3 cases of tests/golden/make_golden.py (IMPLICIT_CASES):
# key -> (periodic, scheme, adaptive, t_end, dt, TsConfig overrides)
IMPLICIT = {
    "cn_periodic": (True, "cn", False, 10 * 1e-3, 1e-3, {}),
    "cn_dirichlet": (False, "cn", False, 10 * 1e-3, 1e-3, {}),
    "cn_stiff": (True, "cn", False, 4 * 2e-2, 2e-2, {"gmres_restart": 8}),
    "ad_rms": (True, "rk3", True, 2e-2, 1e-3, {"tol_a": 1e-7, "tol_r": 1e-7}),
    "ad_max": (False, "rk3", True, 2e-2, 5e-4, {"tol_a": 1e-6, "tol_r": 1e-6, "wlte_form": "max"}),
}


@pytest.mark.parametrize("key", sorted(IMPLICIT))
def test_implicit_and_adaptive_bit_exact(key):
    """CN (Newton + scipy GMRES, timeloop.py:154-186, adjoint.py:64-69) and adaptive RK3
    (controller timeloop.py:198-218): objective, gradient, final state, accepted dt
    sequence and the Newton / GMRES / reject counters equal the reference's."""
    g = golden("implicit.npz")
    per, scheme, adaptive, t_end, dt, cfg = IMPLICIT[key]
    op = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 16, 9, per), 0.01)
    j, gr, uf, fs, ss = R.evaluate_general(op, g[f"u0_{key}"], g[f"target_{key}"], 0.0, t_end,
                                           dt, scheme, adaptive, cfg)
    assert j == g[f"J_{key}"][0]
    assert np.array_equal(gr, g[f"grad_{key}"])
    assert np.array_equal(uf, g[f"ufinal_{key}"])
    assert [fs[k] for k in ("steps", "rejects", "retries", "newton_iters", "gmres_iters")] == \
        list(g[f"fstats_{key}"])
    if scheme == "cn" and key != "cn_binom":
        assert ss["gmres_iters"] == g[f"sstats_{key}"][1]
    # the target run's step log (accepted and rejected attempts)
    _, dts, _, _, log = R.integrate_general(op, _target_ic(per), 0.0, t_end, dt, scheme,
                                            adaptive, cfg)
    assert np.array_equal(dts, g[f"tdts_{key}"])
    assert np.array_equal(np.array(log, dtype=float).reshape(-1, 5), g[f"tlog_{key}"])


def _target_ic(periodic):
    """u_obs0 of make_golden.cfg1_inputs (sin pi x + 0.5 sin 2 pi x, masked)."""
    mesh = R.Mesh1D(-1.0, 1.0, 16, 9, periodic)
    x = mesh.coordinates()
    return mesh.apply_mask(np.sin(np.pi * x) + 0.5 * np.sin(2.0 * np.pi * x))


def _mesh3d_case(g, k):
    c = g[f"case_{k}"]
    ext = [(c[0], c[1]), (c[2], c[3]), (c[4], c[5])]
    return R.Mesh3D(ext, [int(x) for x in c[6:9]], int(c[9]))


@pytest.mark.parametrize("k", [0, 1, 2])
def test_3d_maps_and_ops_bit_exact(k):
    """3D periodic boxes (grid.py:112-146) and the sum-factorised F, J, J^T
    (ops.py:63-81,160-257), incl. an anisotropic box with different E per axis."""
    g = golden("grid3d.npz")
    m = _mesh3d_case(g, k)
    o = R.BurgersOracle3D(m, 0.05)
    assert np.array_equal(m.table, g[f"table_{k}"])
    assert np.array_equal(m.mass_scalar, g[f"mass_{k}"])
    assert np.array_equal(np.concatenate(m.coordinates()), g[f"coords_{k}"])
    u, v, w = g[f"u_{k}"], g[f"v_{k}"], g[f"w_{k}"]
    assert np.array_equal(o.rhs(u), g[f"F_{k}"])
    assert np.array_equal(o.jac(u, v), g[f"J_{k}"])
    assert np.array_equal(o.jact(u, w), g[f"JT_{k}"])
    # discrete-adjoint identity <J v, w>_ = <v, M^-1-weighted J^T ...>: the transpose is exact
    lhs = np.dot(o.jac(u, v), w)
    rhs = np.dot(v, o.jact(u, w))
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), 1.0)


@pytest.mark.parametrize("scheme", ["rk3", "cn"])
def test_burgers3d_evaluate_bit_exact(scheme):
    """problems.burgers3d (elements=2, degree=3, 6 steps): J, gradient, final state and
    Newton / GMRES counters equal the reference's."""
    g = golden("grid3d.npz")
    m = R.Mesh3D([(-2.0, 2.0)] * 3, [2, 2, 2], 3)
    o = R.BurgersOracle3D(m, 0.001)
    j, gr, uf, fs, ss = R.evaluate_general(o, g[f"b3d_{scheme}_guess"], g[f"b3d_{scheme}_target"],
                                           0.0, 0.03, 0.03 / 6, scheme)
    assert j == g[f"b3d_{scheme}_J"][0]
    assert np.array_equal(gr, g[f"b3d_{scheme}_grad"])
    assert np.array_equal(uf, g[f"b3d_{scheme}_ufinal"])
    assert [fs["steps"], fs["newton_iters"], fs["gmres_iters"], ss["gmres_iters"]] == \
        list(g[f"b3d_{scheme}_stats"])


@pytest.mark.parametrize("key,periodic,kind,speed", [("lin_p", True, "linear", [0.3]),
                                                     ("lin_d", False, "linear", [-0.7]),
                                                     ("none_p", True, "none", None),
                                                     ("none_d", False, "none", None)])
def test_advection_kinds_bit_exact(key, periodic, kind, speed):
    """LINEAR / NONE branches of ops.py:147-212 restated (AdvectionOracle)."""
    g = golden("advkinds.npz")
    o = R.AdvectionOracle(R.Mesh1D(-1.0, 1.0, 6, 5, periodic), 0.02, kind, speed)
    u, v, w = g[f"u_{key}"], g[f"v_{key}"], g[f"w_{key}"]
    assert np.array_equal(o.rhs(u), g[f"F_{key}"])
    assert np.array_equal(o.jac(u, v), g[f"J_{key}"])
    assert np.array_equal(o.jact(u, w), g[f"JT_{key}"])


@pytest.mark.parametrize("name,kind,speed,nu,E,t_end,steps,scheme", [
    ("advdiff1d", "linear", [0.1], 1e-5, 8, 0.004, 20, "rk3"),
    ("diffusion1d", "none", None, 1e-3, 5, 0.01, 20, "rk3"),
    ("advdiff1d_cn", "linear", [0.1], 1e-5, 8, 0.004, 5, "cn")])
def test_advdiff_diffusion_problems_bit_exact(name, kind, speed, nu, E, t_end, steps, scheme):
    g = golden("advkinds.npz")
    o = R.AdvectionOracle(R.Mesh1D(0.0, 1.0, E, 8, True), nu, kind, speed)
    j, gr, uf, _, _ = R.evaluate_general(o, g[f"{name}_u0"], g[f"{name}_target"], 0.0, t_end,
                                         t_end / steps, scheme)
    assert j == g[f"{name}_J"][0]
    assert np.array_equal(gr, g[f"{name}_grad"]) and np.array_equal(uf, g[f"{name}_ufinal"])


@pytest.mark.parametrize("N,per", [(7, True), (15, True), (31, True), (9, False)])
def test_longdouble_restatement(N, per):
    """The longdouble restatement of ops.py:161-212 (the yard stick of the smooth-input
    bound) agrees with the fp64 oracle to rounding on rough inputs,
    its RK4 step / adjoint step to the fp64 restatement, and its own J^T is the transpose of
    its J (dot-product identity in longdouble)."""
    m = R.Mesh1D(-1.0, 1.0, 24, N, per)
    o = R.BurgersOracle(m, 0.01)
    L = R.LongDoubleBurgers(o)
    u, v, w = R.seeded_fields(m.ndof, N)
    for a, b in ((o.rhs(u), L.rhs(u)), (o.jac(u, v), L.jac(u, v)), (o.jact(u, w), L.jact(u, w))):
        assert b.dtype == np.longdouble
        assert float(np.max(np.abs(a - b)) / np.max(np.abs(a))) <= 1e-14
    mask = m.maskv
    lhs = np.dot(L.jac(u, v * mask), (w * mask).astype(np.longdouble))
    rhs = np.dot((v * mask).astype(np.longdouble), L.jact(u, w * mask))
    assert abs(float(lhs - rhs)) <= 1e-16 * float(np.linalg.norm(L.jac(u, v * mask)) * np.linalg.norm(w))
    if per:
        dt = 1e-9
        s = R.rk_step(o, u, dt, "rk4")
        assert float(np.max(np.abs(s - L.rk_step(u, dt, "rk4")))) <= 1e-14
        a = R.adjoint_rk_step(o, u, w, dt, "rk4")
        assert float(np.max(np.abs(a - L.adjoint_rk_step(u, w, dt, "rk4")))) <= 1e-13 * float(np.max(np.abs(a)))


def test_smooth_fields_and_bound_helper():
    m = R.Mesh1D(0.0, 64.0, 4096, 7, True)
    u, v, w = R.smooth_fields(m, 7)
    assert u.shape == (m.ndof,) and np.all(np.isfinite(u)) and np.max(np.abs(u)) <= 3.0
    # smooth: neighbouring nodes differ by far less than the amplitude
    assert np.max(np.abs(np.diff(u))) <= 0.05
    err, bound = R.ld_bound(u + 1e-13, u, u.astype(np.longdouble))
    assert err > 0 and bound >= 1e-12 * np.max(np.abs(u))
