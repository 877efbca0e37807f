"""3D periodic boxes: sum-factorised F, J, J^T and the burgers3d
evaluation on the B200 vs the reference's fixtures (tests/golden/grid3d.npz) and the
oracle restatement at larger sizes.  Tolerances: 1e-12 per apply, 1e-9 J / gradient."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import problems, timeloop
from paper_1806_01422_b200.grid import Axis, build_grid, grid_3d
from paper_1806_01422_b200.ops3d import SemOperator3D
from semtest_util import golden, rel_err

pytestmark = pytest.mark.gpu


def _case(g, k):
    c = g[f"case_{k}"]
    ext = [(c[0], c[1]), (c[2], c[3]), (c[4], c[5])]
    els = [int(x) for x in c[6:9]]
    return ext, els, int(c[9])


@pytest.mark.parametrize("k", [0, 1, 2])
def test_3d_ops_match_reference(cuda, k):
    g = golden("grid3d.npz")
    ext, els, N = _case(g, k)
    grid = build_grid([Axis(e[0], e[1], E, N, "periodic") for e, E in zip(ext, els)])
    op = SemOperator3D(grid, sb.PdeCoefficients(0.05), device="cuda:0")
    u, v, w = g[f"u_{k}"], g[f"v_{k}"], g[f"w_{k}"]
    assert rel_err(op.apply_rhs(u), g[f"F_{k}"]) <= 1e-12
    assert rel_err(op.apply_jacobian(u, v), g[f"J_{k}"]) <= 1e-12
    assert rel_err(op.apply_jacobian_transpose(u, w), g[f"JT_{k}"]) <= 1e-12
    assert op.counters == {"rhs": 1, "jac": 1, "jact": 1}


@pytest.mark.parametrize("N", [3, 7, 8])
def test_3d_ops_match_oracle_at_size(cuda, N):
    """E = 4 per axis (N = 7: 28^3 x 3 = 65,856 DOF), anisotropic extents."""
    ext = [(0.0, 1.0), (-1.0, 1.0), (0.0, 3.0)]
    grid = build_grid([Axis(a, b, 4, N, "periodic") for a, b in ext])
    op = SemOperator3D(grid, sb.PdeCoefficients(0.02), device="cuda:0")
    orc = R.BurgersOracle3D(R.Mesh3D(ext, [4, 4, 4], N), 0.02)
    u, v, w = R.seeded_fields(grid.nglobal, 40 + N)
    ud, vd, wd = (torch.from_numpy(a).cuda() for a in (u, v, w))
    assert rel_err(op.apply_rhs(ud).cpu().numpy(), orc.rhs(u)) <= 1e-12
    assert rel_err(op.apply_jacobian(ud, vd).cpu().numpy(), orc.jac(u, v)) <= 1e-12
    assert rel_err(op.apply_jacobian_transpose(ud, wd).cpu().numpy(), orc.jact(u, w)) <= 1e-12
    # discrete transpose identity <J v, w> = <v, J^T w> (ops.py:246-257)
    a = float(torch.dot(op.apply_jacobian(ud, vd), wd))
    b = float(torch.dot(vd, op.apply_jacobian_transpose(ud, wd)))
    assert abs(a - b) <= 1e-11 * max(abs(a), 1.0)


def test_3d_dense_jacobian_matches_oracle(cuda):
    grid = grid_3d((-2.0, 2.0), 1, 2)                 # 8 nodes x 3 components
    op = SemOperator3D(grid, sb.PdeCoefficients(0.1), device="cuda:0")
    orc = R.BurgersOracle3D(R.Mesh3D([(-2.0, 2.0)] * 3, [1, 1, 1], 2), 0.1)
    u = np.sin(np.arange(grid.nglobal) * 0.37)
    d = op.densify(u)
    e = np.eye(grid.nglobal)
    dref = np.stack([orc.jac(u, e[k]) for k in range(grid.nglobal)], axis=1)
    assert rel_err(d, dref) <= 1e-12


@pytest.mark.parametrize("scheme", ["rk3", "cn"])
def test_burgers3d_evaluate_matches_reference(cuda, scheme):
    g = golden("grid3d.npz")
    prob = problems.make_problem("burgers3d", elements=2, degree=3, steps=6, horizon=0.03,
                                 scheme=scheme, device="cuda:0")
    assert np.array_equal(prob.u_guess, g[f"b3d_{scheme}_guess"])
    assert rel_err(prob.u_target, g[f"b3d_{scheme}_target"]) <= 1e-15
    j, gr = prob.evaluate(prob.u_guess)
    assert abs(j - g[f"b3d_{scheme}_J"][0]) <= 1e-9 * abs(g[f"b3d_{scheme}_J"][0])
    assert rel_err(gr, g[f"b3d_{scheme}_grad"]) <= 1e-9
    assert rel_err(prob.last_forward.u_final.cpu().numpy(), g[f"b3d_{scheme}_ufinal"]) <= 1e-12
    st = prob.last_forward.stats
    assert [st["steps"], st["newton_iters"], st["gmres_iters"], prob.op.last_sweep_stats["gmres_iters"]] == \
        list(g[f"b3d_{scheme}_stats"])


def test_burgers3d_gradient_finite_difference_and_binomial(cuda):
    prob = problems.make_problem("burgers3d", elements=2, degree=4, steps=8, horizon=0.04, scheme="rk4",
                                 device="cuda:0")
    u0 = prob.u_guess
    _, gr = prob.evaluate(u0)
    d = np.cos(np.arange(prob.grid.nglobal) * 0.11)
    eps = 1e-4
    jp, _ = prob.evaluate(u0 + eps * d)
    jm, _ = prob.evaluate(u0 - eps * d)
    fd = (jp - jm) / (2 * eps)
    assert abs(fd - np.dot(gr, d)) <= 1e-7 * abs(fd)
    prob.checkpoint_slots = 3                       # binomial schedule: recompute path
    _, gb = prob.evaluate(u0)
    assert rel_err(gb, gr) <= 1e-13


def test_3d_nonfinite_inputs_raise(cuda):
    grid = grid_3d((-1.0, 1.0), 2, 3)
    op = SemOperator3D(grid, sb.PdeCoefficients(0.01), device="cuda:0")
    u = np.sin(np.arange(grid.nglobal) * 0.1)
    bad = u.copy()
    bad[5] = np.nan
    with pytest.raises(sb.NumericFailure):
        op.apply_rhs(bad)
    with pytest.raises(sb.NumericFailure):
        op.apply_jacobian_transpose(u, bad)
    with pytest.raises(sb.ValidationError):
        op.apply_rhs(u[:-1])


def test_3d_tensor_core_and_cuda_core_paths_agree(cuda):
    """N = 7 runs the DMMA element kernel by default; kernel path 1 forces the DFMA one."""
    from paper_1806_01422_b200 import _lib
    ext = [(0.0, 1.0), (-1.0, 1.0), (0.0, 3.0)]
    grid = build_grid([Axis(a, b, 3, 7, "periodic") for a, b in ext])
    op = SemOperator3D(grid, sb.PdeCoefficients(0.02), device="cuda:0")
    u, v, w = (torch.from_numpy(a).cuda() for a in R.seeded_fields(grid.nglobal, 77))
    outs = {}
    lib = _lib.load()
    try:
        for path in (0, 1):
            lib.sem1d_set_kernel_path(path)
            outs[path] = [op.apply_rhs(u), op.apply_jacobian(u, v), op.apply_jacobian_transpose(u, w)]
    finally:
        lib.sem1d_set_kernel_path(0)
    for a, b in zip(outs[0], outs[1]):
        assert rel_err(a.cpu().numpy(), b.cpu().numpy()) <= 1e-13


def test_semoperator_dispatches_3d_grids(cuda):
    """The reference's single SemOperator class serves 3D grids (ops.py:84-124)."""
    grid = grid_3d((-2.0, 2.0), 2, 3)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.05), device="cuda:0")
    assert isinstance(op, SemOperator3D)
    g = golden("grid3d.npz")
    assert rel_err(op.apply_rhs(g["u_0"]), g["F_0"]) <= 1e-12
