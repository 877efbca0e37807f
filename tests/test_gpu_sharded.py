"""The sharded geometry on the GPU kernels: for every rank of a P-way partition, the
local apply on the extended chain (ghosts filled from the global field, exactly what
HaloExchange delivers) reproduces the owned part of the single-GPU apply.  The
exchange itself is covered by tests/test_dist_gloo.py on CPU ranks."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import dist as sd
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import rel_err

pytestmark = pytest.mark.gpu


def _ext(part, glob):
    """Extended local array of a partition cut from a global (ring) array."""
    n = glob.size
    idx = (part.g_lo - part.gl * part.N + np.arange(part.ext_ndof))
    if part.periodic:
        idx %= n
    else:
        idx = np.clip(idx, 0, n - 1)
    return glob[idx]


@pytest.mark.parametrize("E,N,P,bc", [(4096, 7, 4, "periodic"), (4096, 7, 3, "dirichlet0"),
                                      (1024, 15, 8, "periodic"), (512, 31, 2, "dirichlet0"),
                                      (600, 9, 5, "periodic")])
def test_sharded_local_applies_match_global(cuda, E, N, P, bc):
    g = grid_1d(-1.0, 1.0, E, N, bc)
    glob_op = sb.SemOperator(g, sb.PdeCoefficients(0.01), device="cuda:0")
    u, v, w = R.seeded_fields(g.nglobal, E + N)
    F, JV, JT = glob_op.apply_rhs(u), glob_op.apply_jacobian(u, v), glob_op.apply_jacobian_transpose(u, w)
    ref = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, E, N, bc == "periodic"), 0.01)
    Fr = ref.rhs(u)
    for rank in range(P):
        op = sd.ShardedOperator(g, sb.PdeCoefficients(0.01), rank, P, device="cuda:0")
        part = op.part
        ue, ve, we = (torch.from_numpy(_ext(part, a)).cuda() for a in (u, v, w))
        outs = [op.empty() for _ in range(3)]
        op.local.launch_rhs(ue, outs[0])
        op.local.launch_jac(ue, ve, outs[1])
        op.local.launch_jact(ue, we, outs[2])
        assert op.local.flags() == 0
        sl = slice(part.g_lo, part.g_lo + part.n_own)
        for got, full in zip(outs, (F, JV, JT)):
            own = op.public(got).cpu().numpy()
            assert rel_err(own, full[sl]) <= 1e-14
        assert rel_err(op.public(outs[0]).cpu().numpy(), Fr[sl]) <= 1e-12


def test_single_rank_sharded_is_global(cuda):
    g = grid_1d(-1.0, 1.0, 300, 7)
    op = sd.ShardedOperator(g, sb.PdeCoefficients(0.01), 0, 1, device="cuda:0")
    glob = sb.SemOperator(g, sb.PdeCoefficients(0.01), device="cuda:0")
    u, _, w = R.seeded_fields(g.nglobal, 1)
    assert np.array_equal(op.apply_rhs(u), glob.apply_rhs(u))
    assert np.array_equal(op.apply_jacobian_transpose(u, w), glob.apply_jacobian_transpose(u, w))
