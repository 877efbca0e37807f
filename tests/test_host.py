"""Host-side product logic on CPU: constants and maps bit-exact against the reference
fixtures, schedules action-for-action, time-step bookkeeping, L-BFGS control flow."""

import numpy as np
import pytest

import paper_1806_01422_b200 as sb
from paper_1806_01422_b200 import checkpoint as C
from paper_1806_01422_b200 import timeloop as T
from paper_1806_01422_b200.grid import grid_1d
from oracle import semref as R
from semtest_util import golden

DEGREES = list(range(1, 33)) + [48, 64]


@pytest.mark.parametrize("n", DEGREES)
def test_product_basis_bit_exact(n):
    g = golden("basis.npz")
    b = sb.gll_rule(n)
    assert np.array_equal(b.nodes, g[f"nodes_{n}"])
    assert np.array_equal(b.weights, g[f"weights_{n}"])
    assert np.array_equal(b.diff, g[f"diff_{n}"])
    # the operator constants shipped to the device (ops.py:103-107)
    grid = grid_1d(-1.0, 1.0, 16, n)
    w = b.weights
    k = (2.0 / grid.axis.element_length) * (b.diff.T * w) @ b.diff
    assert np.array_equal(0.5 * (k + k.T), g[f"K_{n}"])
    assert np.array_equal(b.diff * w[:, None], g[f"Dw_{n}"])
    eo = sb.element_operators(b, 2.0 / 16)
    assert np.array_equal(eo.stiffness, g[f"K_{n}"])


def test_grid_closed_forms_bit_exact():
    g = golden("maps.npz")
    k = 0
    while f"case_{k}" in g:
        xa, xb, e, n, per = g[f"case_{k}"]
        grid = grid_1d(xa, xb, int(e), int(n), "periodic" if per else "dirichlet0")
        assert np.array_equal(grid.table, g[f"table_{k}"])
        assert np.array_equal(grid.multiplicity, g[f"mult_{k}"])
        assert np.array_equal(grid.mass_scalar, g[f"mass_{k}"])
        assert np.array_equal(grid.mask_scalar, g[f"mask_{k}"])
        assert np.array_equal(grid.node_coordinates()[0], g[f"coords_{k}"])
        # the per-position M^-1 pattern the kernels use == 1/mass everywhere it is read
        minv_full = 1.0 / g[f"mass_{k}"]
        loc = np.arange(grid.nglobal) % int(n)
        expanded = grid.minv_pattern[loc]
        if not per:
            expanded[0] = grid.minv_pattern[int(n)]
            expanded[-1] = grid.minv_pattern[int(n) + 1]
        assert np.array_equal(expanded, minv_full)
        k += 1


def test_grid_kats_and_validation():
    g = grid_1d(0.0, 1.0, 2, 2)
    assert g.nglobal == 4 and list(g.multiplicity) == [2, 1, 2, 1]
    assert grid_1d(-1.0, 1.0, 1, 4, "dirichlet0").nglobal == 5
    assert list(grid_1d(0.0, 1.0, 2, 1).node_coordinates()[0]) == [0.0, 0.5]
    with pytest.raises(sb.ValidationError):
        grid_1d(0.0, 1.0, 1, 1)
    with pytest.raises(sb.ValidationError):
        grid_1d(1.0, 0.0, 4, 4)
    g3 = sb.grid_3d((-2.0, 2.0), 2, 4)            # 3D periodic box
    assert g3.nglobal == 3 * 8 ** 3 and g3.ncomp == 3 and not g3.has_mask
    with pytest.raises(sb.ValidationError):       # 3D grids require periodic axes (grid.py:97-101)
        sb.build_grid([sb.Axis(-1.0, 1.0, 2, 3, "dirichlet0")] * 3)
    with pytest.raises(sb.ValidationError):       # one degree on all axes (kernel constraint)
        sb.build_grid([sb.Axis(-1.0, 1.0, 2, 3), sb.Axis(-1.0, 1.0, 2, 4), sb.Axis(-1.0, 1.0, 2, 3)])
    with pytest.raises(sb.ValidationError):
        sb.PdeCoefficients(-1.0)
    assert sb.PdeCoefficients(0.1, "linear", speed=[1.0]).speed.tolist() == [1.0]   # ops.py:44-60
    with pytest.raises(sb.ValidationError):
        sb.PdeCoefficients(0.1, "linear")            # linear advection needs a speed
    with pytest.raises(sb.ValidationError):
        sb.PdeCoefficients(0.1, "upwind")
    big = grid_1d(-1.0, 1.0, 1 << 25, 7)  # config 5 size: no O(ndof) host arrays built
    assert big.nglobal == (1 << 25) * 7 and "table" not in big.__dict__


SCHED = [(1, 1), (3, 3), (5, 2), (10, 3), (20, 4), (30, 5), (100, 10), (57, 7), (500, 64)]
KIND = {C.Store: 0, C.Restore: 1, C.Advance: 2, C.AdjointStep: 3, C.Done: 4}


def _rows(sch):
    out = []
    for a in sch.actions:
        k = KIND[type(a)]
        if k in (0, 1):
            out.append((k, a.slot, a.step))
        elif k == 2:
            out.append((k, a.start, a.stop))
        elif k == 3:
            out.append((k, a.step, -1))
        else:
            out.append((k, -1, -1))
    return np.array(out, dtype=np.int64)


@pytest.mark.parametrize("m,s", SCHED)
def test_binomial_schedule_matches_reference(m, s):
    g = golden("schedules.npz")
    sch = C.plan_binomial(m, s)
    assert np.array_equal(_rows(sch), g[f"actions_{m}_{s}"])
    assert [sch.recomputed, sch.backward_start, sch.slots] == list(g[f"meta_{m}_{s}"])
    assert np.array_equal(np.array(sorted(sch.forward_stores.items())), g[f"stores_{m}_{s}"])
    rep = C.simulate_schedule(sch)
    assert rep.forward_evals == m + sch.recomputed and rep.max_live <= s


def test_schedule_properties():
    rng = np.random.default_rng(0)
    for _ in range(200):  # SPEC: high-water mark <= s for randomized (m, s)
        m, s = int(rng.integers(1, 80)), int(rng.integers(1, 12))
        sch = C.plan_binomial(m, s)
        assert C.simulate_schedule(sch).max_live <= s
    sch = C.plan_store_all(3)
    assert sch.recomputed == 0 and C.simulate_schedule(sch).forward_evals == 3
    bad = C.plan_binomial(10, 3)
    acts = list(bad.actions)
    acts[3], acts[4] = acts[4], acts[3]
    with pytest.raises(sb.ScheduleError):
        C.simulate_schedule(C.Schedule(bad.n_steps, bad.slots, acts, bad.recomputed))
    with pytest.raises(sb.ValidationError):
        C.plan_binomial(5, 0)


def test_tsconfig_and_step_counts():
    cfg = T.TsConfig(scheme="rk4", t0=0.0, t_end=20 * 1e-4, dt=1e-4)
    assert T.count_steps(cfg) == 20
    g = golden("sweeps.npz")
    assert T.count_steps(T.TsConfig(scheme="rk3", t_end=0.0123, dt=1e-4)) == len(g["long_dts"])
    with pytest.raises(sb.ValidationError):
        T.TsConfig(scheme="rk5")
    with pytest.raises(sb.ValidationError):
        T.TsConfig(scheme="rk4", adaptive=True)


def test_tableau_engine_planning():
    """Which slopes the fused stage kernels keep in HBM (no GPU needed)."""

    class FakeOp:
        counters = {"rhs": 0}

    e3 = T.StepEngine(FakeOp(), "rk3")
    assert e3.stored_k == [0, 1] and e3.stored_k_recompute == [0]
    e4 = T.StepEngine(FakeOp(), "rk4")
    assert e4.stored_k == [0, 1, 2] and e4.stored_k_recompute == []
    assert e4.rows[1] == [(1, 0.5)] and e4.rows[2] == [(2, 1.0)]
    e1 = T.StepEngine(FakeOp(), "euler")
    assert e1.rows == [[(0, 1.0)]]


def test_lbfgs_quadratic_and_reference_log_shape():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((20, 20))
    H = A @ A.T + 20 * np.eye(20)
    b = rng.standard_normal(20)

    def fun(x):
        return 0.5 * x @ H @ x - b @ x, H @ x - b

    res = sb.minimize(fun, np.zeros(20), sb.OptimConfig(max_iters=200, gtol=1e-10))
    assert res.status == "gtol"
    assert np.allclose(res.x, np.linalg.solve(H, b), atol=1e-8)
    js = [r[1] for r in res.log]
    assert all(b2 <= a2 for a2, b2 in zip(js, js[1:]))  # monotone (Wolfe decrease)
    with pytest.raises(sb.LineSearchError):
        sb.line_search(lambda t: (0.0, 0.0, None), 0.0, 1.0)

@pytest.mark.parametrize("n", [7, 15, 31])
def test_reflection_symmetry_behind_the_split_kernels(n):
    """The reflection (even/odd) split of the DMMA kernels (bfrag_eo_value in
    csrc/sem1d_device.cuh) relies on K being centrosymmetric and Dw anti-centrosymmetric, which
    holds for the reference's own matrices (ops.py:103-107) to a few ulp, and on the mass
    pattern being symmetric.  The half blocks formed as the kernels form them (from both
    halves of each matrix) reproduce the full products on the sums and differences of
    mirrored nodes to rounding."""
    g = golden("basis.npz")
    K, Dw, w = g[f"K_{n}"], g[f"Dw_{n}"], g[f"weights_{n}"]
    flip = lambda a: a[::-1, ::-1]
    assert np.max(np.abs(K - flip(K))) <= 64 * np.finfo(float).eps * np.max(np.abs(K))
    assert np.max(np.abs(Dw + flip(Dw))) <= 64 * np.finfo(float).eps * np.max(np.abs(Dw))
    assert np.array_equal(w, w[::-1]) or np.max(np.abs(w - w[::-1])) <= 4 * np.finfo(float).eps
    h = (n + 1) // 2
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n + 1)
    s, d = x[:h] + x[::-1][:h], x[:h] - x[::-1][:h]
    for M, centro in ((K, True), (Dw, False), (Dw.T.copy(), False)):
        sg = 1.0 if centro else -1.0
        a = M[:h, :h] + sg * flip(M)[:h, :h]                 # M[i][j] +- M[N-i][N-j]
        b = M[:h, ::-1][:, :h] + sg * flip(M)[:h, ::-1][:, :h]   # M[i][N-j] +- M[N-i][j]
        Me, Mo = 0.25 * (a + b), 0.25 * (a - b)
        lo = Me @ s + Mo @ d
        hi = sg * (Me @ s - Mo @ d)
        y = M @ x
        tol = 1e-13 * np.max(np.abs(M)) * np.max(np.abs(x)) * (n + 1)
        assert np.max(np.abs(lo - y[:h])) <= tol and np.max(np.abs(hi - y[::-1][:h])) <= tol



@pytest.mark.parametrize("k", [0, 1, 2])
def test_grid3d_maps_bit_exact(k):
    """Grid3D: table, coordinates and the mass diagonal built from (N+1)^3 position
    classes equal the reference's bincount arrays bit for bit (grid.py:112-146)."""
    g = golden("grid3d.npz")
    c = g[f"case_{k}"]
    ext = [(c[0], c[1]), (c[2], c[3]), (c[4], c[5])]
    grid = sb.build_grid([sb.Axis(e[0], e[1], int(E), int(c[9])) for e, E in zip(ext, c[6:9])])
    assert np.array_equal(grid.table, g[f"table_{k}"])
    assert np.array_equal(grid.mass_scalar, g[f"mass_{k}"])
    assert np.array_equal(np.concatenate(grid.node_coordinates()), g[f"coords_{k}"])
    u = g[f"u_{k}"]
    assert np.array_equal(grid.gather(grid.scatter(u)), R.Mesh3D(ext, [int(x) for x in c[6:9]],
                                                                 int(c[9])).gather(grid.scatter(u)))


@pytest.mark.parametrize("key,bc,E,N,ext", [("burgers", "dirichlet0", 5, 8, (-2.0, 2.0)),
                                           ("smooth", "periodic", 6, 10, (0.0, 1.0)),
                                           ("rough", "periodic", 4, 6, (0.0, 1.0))])
def test_spectral_error_estimate_matches_reference(key, bc, E, N, ext):
    """problems.spectral_error_estimate (problems.py:106-155): the vectorised closed-form fits
    equal the reference's per-element np.polyfit to rounding."""
    from paper_1806_01422_b200.problems import spectral_error_estimate
    g = golden("spectral.npz")
    rep = spectral_error_estimate(g[f"{key}_values"], grid_1d(ext[0], ext[1], E, N, bc))
    for f in ("resolved", "under_resolved"):
        assert np.array_equal(getattr(rep, f), g[f"{key}_{f}"])
    for f in ("sigma", "scale", "a_top", "eps"):
        ref = g[f"{key}_{f}"]
        assert np.allclose(getattr(rep, f), ref, rtol=1e-9, atol=1e-300), f
