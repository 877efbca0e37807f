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


@pytest.mark.parametrize("scheme", ["rk4", "rk3"])
def test_sharded_fused_steps_match_global(cuda, scheme):
    """Ghost-zone mode (periodic rings): every rank's single-launch RK step and adjoint
    step on its periodic extended chain reproduce the owned part of the global step."""
    E, N, P, dt = 4400, 7, 4, 2e-6
    g = grid_1d(0.0, 2.0, E, N)
    glob = sb.SemOperator(g, sb.PdeCoefficients(1e-3), device="cuda:0")
    assert glob.step_fused_supported()
    x = g.node_coordinates()[0]
    u = np.sin(np.pi * x) + 0.2 * np.cos(3 * np.pi * x)
    lam = np.cos(2 * np.pi * x)
    ud, ld = torch.from_numpy(u).cuda(), torch.from_numpy(lam).cuda()
    un_g, ln_g = glob.empty(), glob.empty()
    glob.launch_rk_step(ud, un_g, dt, scheme)
    glob.launch_adj_step(ud, ld, ln_g, dt, scheme)
    assert glob.flags() == 0
    for rank in range(P):
        op = sd.ShardedOperator(g, sb.PdeCoefficients(1e-3), rank, P, device="cuda:0")
        assert op.part.zone == 8 and op.step_fused_supported()
        ue, le = (torch.from_numpy(_ext(op.part, a)).cuda() for a in (u, lam))
        un, ln = op.empty(), op.empty()
        op.local.launch_rk_step(ue, un, dt, scheme)
        op.local.launch_adj_step(ue, le, ln, dt, scheme)
        assert op.local.flags() == 0
        sl = slice(op.part.g_lo, op.part.g_lo + op.part.n_own)
        assert rel_err(op.public(un).cpu().numpy(), un_g[sl].cpu().numpy()) <= 1e-14
        assert rel_err(op.public(ln).cpu().numpy(), ln_g[sl].cpu().numpy()) <= 1e-13


def test_bench_two_ranks_json_line(cuda, tmp_path):
    """bench.py under torchrun with 2 ranks (the driver's N > 1 launch), here on one GPU with
    --same-device and a gloo exchange (no kernel waits on another rank): one JSON line from
    rank 0 with the whole-job value, n_gpus = 2 and the sharded parallelism."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-sweep",
           "--cfg5-steps", "2", "--same-device", "--dist-backend", "gloo"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert "sharded" in d["config"]["parallelism"]
    st = d["strong_scaling_cfg5"]          # config 5's ring strong-scaled over the 2 ranks
    assert st["n_gpus"] == 2 and st["dof"] == 7 * 2 ** 25 and st["n1_reference"]["n_gpus"] == 1
    assert st["efficiency_vs_n1"] > 0 and st["forward_ms"] > 0 and st["adjoint_ms"] > 0


def test_sharded_evaluate_two_ranks_matches_single(cuda):
    """Config-5 tool at small size: L-BFGS on evaluate() (run-ahead fused forward steps with
    per-step flag words verified by a cross-rank max, binomial checkpointing, fused adjoint
    steps) on 2 element-sharded ranks (one GPU, gloo exchange) gives the objective and
    gradient-norm history of the single-GPU run."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tool = os.path.join(root, "tools", "bench_cfg5.py")
    args = ["--E", "16384", "--steps", "24", "--slots", "4", "--iters", "2", "--band", "80,160", "--amp", "0.015625"]
    one = subprocess.run([sys.executable, tool] + args, cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    env = dict(os.environ, SEM1D_DIST_BACKEND="gloo", SEM1D_SAME_DEVICE="1")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                          "29541", tool] + args, cwd=root, capture_output=True, text=True,
                         timeout=600, env=env)
    assert two.returncode == 0, two.stderr[-2000:]
    a, b = (json.loads([ln for ln in o.stdout.splitlines() if ln.startswith("{")][-1]) for o in (one, two))
    assert b["n_gpus"] == 2
    assert len(a["J_log"]) == len(b["J_log"]) >= 2
    for x, y in zip(a["J_log"] + a["gnorm_log"], b["J_log"] + b["gnorm_log"]):
        assert abs(x - y) <= 1e-9 * max(abs(x), 1e-300)
