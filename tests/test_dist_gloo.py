"""Element-sharded path on CPU ranks (gloo, world size 2 and 3): a sharded apply is
bit-identical to the single-process oracle apply (the interface sums have the same
two terms), and a sharded forward/adjoint evaluate() matches the global one."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, bc, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _work(rank, world, bc, q)
    except Exception as exc:  # report instead of dying silently (the parent would time out)
        import traceback
        q.put((rank, {"exception: " + "".join(traceback.format_exception(exc))[-1500:]: False}))
    finally:
        dist.destroy_process_group()


def _work(rank, world, bc, q):
    if True:
        from cpu_local_op import CpuLocalOp
        from oracle import semref as R
        import paper_1806_01422_b200 as sb
        from paper_1806_01422_b200 import dist as sd, timeloop
        from paper_1806_01422_b200.grid import grid_1d

        E, N, nu = 24, 9, 0.01   # >= 8 elements (one ghost zone) per rank up to world 3
        g = grid_1d(-1.0, 1.0, E, N, bc)
        op = sd.ShardedOperator(g, sb.PdeCoefficients(nu), rank, world,
                                local_factory=CpuLocalOp)
        ref = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, E, N, bc == "periodic"), nu)
        u, v, w = R.seeded_fields(ref.mesh.ndof, 5)
        sl = slice(op.part.g_lo, op.part.g_lo + op.part.n_own)
        res = {}
        res["rhs"] = np.array_equal(op.apply_rhs(u[sl]), ref.rhs(u)[sl])
        res["jac"] = np.array_equal(op.apply_jacobian(u[sl], v[sl]), ref.jac(u, v)[sl])
        res["jact"] = np.array_equal(op.apply_jacobian_transpose(u[sl], w[sl]), ref.jact(u, w)[sl])
        # full forward + adjoint evaluate, RK3, sharded vs global oracle
        x = g.node_coordinates()[0]
        u0 = g.mask(np.sin(np.pi * x) + 0.01 * np.random.default_rng(1).standard_normal(g.nglobal))
        ud = g.mask(np.sin(np.pi * x) + 0.5 * np.sin(2 * np.pi * x))
        ts = sb.TsConfig(scheme="rk3", t0=0.0, t_end=12 * 1e-4, dt=1e-4)
        prob = sb.AssimilationProblem(name="shard", grid=op.grid, op=op, ts=ts,
                                      u_target=ud[sl], u_guess=u0[sl])
        J, grad = prob.evaluate(u0[sl])
        j_ref, g_ref, _ = R.evaluate(ref, u0, ud, 0.0, 12 * 1e-4, 1e-4, "rk3")
        res["J"] = abs(J - j_ref) <= 1e-13 * abs(j_ref)
        res["grad"] = float(np.max(np.abs(grad - g_ref[sl]))) <= 1e-13 * float(np.max(np.abs(g_ref)))
        # binomial checkpointing through the sharded engine: bitwise equal to store-all
        prob_b = sb.AssimilationProblem(name="shardb", grid=op.grid, op=op, ts=ts,
                                        u_target=ud[sl], u_guess=u0[sl], checkpoint_slots=3)
        Jb, gb = prob_b.evaluate(u0[sl])
        res["binomial"] = bool(np.array_equal(gb, grad)) and Jb == J
        # sharded dot == global dot (all-reduced owned parts)
        ue, _ = op.field(u[sl])
        we, _ = op.field(w[sl])
        res["dot"] = abs(op.dot(ue, we) - float(u @ w)) <= 1e-12 * abs(float(u @ w))
        # one batched ghost refresh of (u, v, w), then the applies without their own refresh
        ve, _ = op.field(v[sl])
        o1, o2 = op.empty(), op.empty()
        op.launch_jact(ue, we, o1)
        ue2, _ = op.field(u[sl])
        ve2, _ = op.field(v[sl])
        we2, _ = op.field(w[sl])
        op.refresh([ue2, ve2, we2])
        op.launch_jact(ue2, we2, o2, refresh=False)
        o3, o4 = op.empty(), op.empty()
        op.launch_jac(ue, ve, o3)
        op.launch_jac(ue2, ve2, o4, refresh=False)
        res["batched_refresh"] = bool(np.array_equal(np.asarray(o1), np.asarray(o2))
                                      and np.array_equal(np.asarray(o3), np.asarray(o4)))
        # step-count / time grid identical on every rank
        res["steps"] = prob.last_forward.n_steps == timeloop.count_steps(ts)
        q.put((rank, res))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("bc", ["periodic", "dirichlet0"])
def test_sharded_matches_global(world, bc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bc, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, res in sorted(out):
        for k, ok in res.items():
            assert ok, f"rank {rank}: {k}"


def test_partition_covers_every_node_once():
    from paper_1806_01422_b200.dist import Partition
    for E, N, P, per in [(16, 9, 2, True), (17, 7, 3, False), (64, 3, 8, True), (20, 1, 4, False)]:
        owned = []
        for r in range(P):
            p = Partition(E, N, P, r, per)
            owned.extend(range(p.g_lo, p.g_lo + p.n_own))
            assert p.ext_ndof == p.E_ext * N + 1
            assert (p.left is None) == (not per and r == 0) or P == 1
        assert owned == list(range(E * N + (0 if per else 1)))


def test_sharded_tile_split_covers_every_tile_once():
    """ShardedOperator._tile_split: the interior launch (run while the ghost exchange is in
    flight) reads no ghost element; interior + edge launches cover every ring tile once."""
    from paper_1806_01422_b200 import dist as sd
    from paper_1806_01422_b200.grid import grid_1d

    class FakeLocal:
        device = "cpu"
        counters = {}
        max_matrix_dim = 8

        def __init__(self, g, c):
            self.g = g

        def step_tiling(self, kind, stored, scheme):
            H = 4 if kind == 0 else 7
            T = 256 - 2 * H
            E = self.g.axis.elements
            return (E + T - 1) // T, T, H

    for E, P in ((1 << 14, 2), (1 << 14, 8), (3000, 3)):
        g = grid_1d(0.0, 1.0, E, 7)
        for rank in range(P):
            op = sd.ShardedOperator(g, None, rank, P, local_factory=FakeLocal)
            for kind in (0, 1):
                split = op._tile_split(kind, "rk4")
                nt, T, H = op.local.step_tiling(kind, False, "rk4")
                assert split is not None
                (a0, ac), (b0, bc) = split
                assert ac + bc == nt
                tiles = [(a0 + k) % nt for k in range(ac)] + [(b0 + k) % nt for k in range(bc)]
                assert sorted(tiles) == list(range(nt))
                z, Ee = op.part.zone, op.part.E_ext
                for k in range(ac):
                    t = a0 + k
                    assert t * T - H >= z and (t + 1) * T + H <= Ee - z
