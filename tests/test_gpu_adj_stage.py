"""The per-stage adjoint kernel (sem1d_adj_stage, adjoint.py:54-61) on the FP64 tensor-core
path: for N + 1 in {8, 16, 24, 32} it runs the warp-specialised DMMA kernel with the
z = b lam + sum_j a_j l_j prologue formed from staged lam / l_j slabs and the l / lam_out
epilogue.  These are the stages Dirichlet rings, batched rings and the non-fused path run.
Checked against the oracle's adjoint step (1e-12 relative, like an apply) and against the
thread-per-element DFMA kernel (kernel path 2) on the same inputs."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import _lib, adjoint
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import rel_err

pytestmark = pytest.mark.gpu


def _setup(E, N, periodic, batch, seed):
    g = grid_1d(-1.0, 1.0, E, N, "periodic" if periodic else "dirichlet0")
    op = sb.SemOperator(g, sb.PdeCoefficients(1e-2), device="cuda:0", batch=batch)
    op.use_fused_steps = False             # the per-stage kernels, also on periodic rings
    x = g.node_coordinates()[0]
    rng = np.random.default_rng(seed)
    u = np.stack([np.sin(np.pi * x + b) + 0.01 * rng.standard_normal(g.nglobal) for b in range(batch)])
    lam = rng.standard_normal((batch, g.nglobal))
    if not periodic:
        u[:, 0] = u[:, -1] = 0.0
    ref = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, E, N, periodic), 1e-2)
    return op, u, lam, ref


def _step(op, u, lam, dt, scheme):
    sh = op.shape
    ud = torch.from_numpy(u.reshape(sh).copy()).cuda()
    ld = torch.from_numpy(lam.reshape(sh).copy()).cuda()
    out = adjoint.adjoint_step(op, ud, ld, 0.0, dt, scheme)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(u.shape)


@pytest.mark.parametrize("scheme", ["rk4", "rk3", "euler"])
@pytest.mark.parametrize("N,E", [(7, 1061), (15, 301), (23, 150), (31, 260), (7, 37), (31, 5)])
@pytest.mark.parametrize("periodic", [False, True])
def test_adjoint_stage_dmma_vs_oracle(cuda, scheme, N, E, periodic):
    dt = 1e-5
    op, u, lam, ref = _setup(E, N, periodic, 1, E + N)
    got = _step(op, u, lam, dt, scheme)
    want = R.adjoint_rk_step(ref, u[0], lam[0], dt, scheme)
    assert rel_err(got[0], want) <= 1e-12
    # the thread-per-element DFMA kernel on the same inputs
    lib = _lib.load()
    assert lib.sem1d_set_kernel_path(2) == 0
    try:
        plain = _step(op, u, lam, dt, scheme)
    finally:
        lib.sem1d_set_kernel_path(0)
    assert rel_err(got, plain) <= 1e-13
    assert op.counters["jact"] == 2 * len(R.TABLEAUX[scheme][1])


@pytest.mark.parametrize("N", [7, 31])
def test_adjoint_stage_dmma_batched(cuda, N):
    E, batch, dt = 203, 3, 1e-5
    op, u, lam, ref = _setup(E, N, False, batch, 7)
    got = _step(op, u, lam, dt, "rk4")
    for b in range(batch):
        assert rel_err(got[b], R.adjoint_rk_step(ref, u[b], lam[b], dt, "rk4")) <= 1e-12, b


@pytest.mark.parametrize("N", [7, 15, 31])
def test_adjoint_stage_dmma_flags(cuda, N):
    op, u, lam, _ = _setup(300, N, False, 1, 3)
    bad = lam.copy()
    bad[0, 77] = np.nan
    with pytest.raises(sb.NumericFailure, match="cotangent"):
        _step(op, u, bad, 1e-5, "rk4")
    bad = u.copy()
    bad[0, 123] = np.inf
    with pytest.raises(sb.NumericFailure, match="state"):
        _step(op, bad, lam, 1e-5, "rk4")
