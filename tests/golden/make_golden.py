"""Generate the golden fixtures from the REAL reference (semopt 0.1.0).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``semopt`` from /root/reference/pkg/src and writes small .npz files
next to this script.  The fixtures travel with the repo; nothing on the GPU box
reads /root/reference.  Inputs are seeded numpy PCG64 draws per global node in
node order.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import semopt  # noqa: F401
    from semopt import adjoint, checkpoint, grid, ops, optimize, problems, timeloop
    return semopt, grid, ops, timeloop, adjoint, checkpoint, problems, optimize


def basis_fixture(semopt, ops, grid):
    out = {}
    for n in list(range(1, 33)) + [48, 64]:
        b = semopt.gll_rule(n)
        out[f"nodes_{n}"] = b.nodes
        out[f"weights_{n}"] = b.weights
        out[f"diff_{n}"] = b.diff
        g = grid.grid_1d(-1.0, 1.0, 16, n)
        op = ops.SemOperator(g, ops.PdeCoefficients(0.01))
        out[f"K_{n}"] = op._kmat[0]
        out[f"Dw_{n}"] = op._dw[0]
    return out


MAP_CASES = [
    (0.0, 1.0, 2, 2, "periodic"), (-1.0, 1.0, 1, 4, "dirichlet0"), (0.0, 1.0, 2, 1, "periodic"),
    (-1.0, 1.0, 3, 4, "periodic"), (-1.0, 1.0, 16, 9, "periodic"), (-1.0, 1.0, 16, 9, "dirichlet0"),
    (-2.0, 2.0, 5, 8, "dirichlet0"), (-1.0, 1.0, 4, 31, "periodic"), (0.0, 20.0, 256, 15, "periodic"),
    (-1.0, 1.0, 1, 3, "periodic"), (-1.0, 1.0, 7, 1, "dirichlet0"),
]


def maps_fixture(grid):
    out = {}
    for k, (xa, xb, e, n, bc) in enumerate(MAP_CASES):
        g = grid.grid_1d(xa, xb, e, n, bc)
        out[f"case_{k}"] = np.array([xa, xb, e, n, bc == "periodic"], dtype=float)
        out[f"table_{k}"] = g.table
        out[f"mult_{k}"] = g.multiplicity
        out[f"mass_{k}"] = g.mass_scalar
        out[f"mask_{k}"] = g.mask_scalar
        out[f"coords_{k}"] = g.node_coordinates()[0]
    return out


# (xa, xb, E, N, bc, nu, seed)
OP_CASES = [
    (-1.0, 1.0, 16, 9, "periodic", 0.01, 0),
    (-1.0, 1.0, 16, 9, "dirichlet0", 0.01, 1),
    (-1.0, 1.0, 3, 4, "periodic", 0.01, 2),
    (-1.0, 1.0, 64, 7, "periodic", 0.01, 3),
    (-1.0, 1.0, 64, 7, "dirichlet0", 0.01, 4),
    (0.0, 20.0, 32, 15, "periodic", 0.01, 5),
    (-1.0, 1.0, 8, 31, "periodic", 1e-3, 6),
    (-1.0, 1.0, 1, 5, "periodic", 0.05, 7),
    (-1.0, 1.0, 2, 1, "periodic", 0.1, 8),
    (-1.0, 1.0, 5, 2, "dirichlet0", 0.1, 9),
    (-1.0, 1.0, 300, 3, "periodic", 0.02, 10),
    (-1.0, 1.0, 40, 12, "dirichlet0", 0.005, 11),
]


def ops_fixture(grid, ops):
    out = {}
    for k, (xa, xb, e, n, bc, nu, seed) in enumerate(OP_CASES):
        g = grid.grid_1d(xa, xb, e, n, bc)
        op = ops.SemOperator(g, ops.PdeCoefficients(nu))
        rng = np.random.default_rng(seed)
        u = rng.uniform(-1.0, 1.0, g.nglobal)
        v = rng.standard_normal(g.nglobal)
        w = rng.standard_normal(g.nglobal)
        out[f"case_{k}"] = np.array([xa, xb, e, n, bc == "periodic", nu, seed], dtype=float)
        out[f"u_{k}"], out[f"v_{k}"], out[f"w_{k}"] = u, v, w
        out[f"f_{k}"] = op.apply_rhs(u)
        out[f"jv_{k}"] = op.apply_jacobian(u, v)
        out[f"jtw_{k}"] = op.apply_jacobian_transpose(u, w)
    return out


def cfg1_inputs(grid, bc):
    """BASELINE config 1: E=16, N=9, nu=0.01 on [-1,1]; u0 = sin(pi x) + 0.01 N(0,1)."""
    g = grid.grid_1d(-1.0, 1.0, 16, 9, bc)
    x = g.node_coordinates()[0]
    rng = np.random.default_rng(1806)
    u0 = g.mask(np.sin(np.pi * x) + 0.01 * rng.standard_normal(g.nglobal))
    u_obs0 = g.mask(np.sin(np.pi * x) + 0.5 * np.sin(2.0 * np.pi * x))
    return g, u0, u_obs0


def sweep_fixture(grid, ops, timeloop, adjoint, checkpoint, problems, optimize):
    out = {}
    for bc in ("periodic", "dirichlet0"):
        for scheme in ("rk3", "euler"):
            g, u0, uo0 = cfg1_inputs(grid, bc)
            op = ops.SemOperator(g, ops.PdeCoefficients(0.01))
            ts = timeloop.TsConfig(scheme=scheme, t0=0.0, t_end=20 * 1e-4, dt=1e-4)
            target = timeloop.integrate(op, uo0, ts, store_steps=None).u_final
            prob = problems.AssimilationProblem(name="cfg1", grid=g, op=op, ts=ts,
                                                u_target=target, u_guess=u0)
            j, gr = prob.evaluate(u0)
            key = f"{bc}_{scheme}"
            out[f"u0_{key}"], out[f"target_{key}"] = u0, target
            out[f"J_{key}"] = np.array([j])
            out[f"grad_{key}"] = gr
            out[f"ufinal_{key}"] = prob.last_forward.u_final
            out[f"dts_{key}"] = prob.last_forward.dts
            out[f"counters_{key}"] = np.array([op.counters["rhs"], op.counters["jac"],
                                               op.counters["jact"]])
            # binomial checkpointing must give the same gradient
            prob_b = problems.AssimilationProblem(name="cfg1b", grid=g, op=op, ts=ts,
                                                  u_target=target, u_guess=u0,
                                                  checkpoint_slots=4)
            jb, gb = prob_b.evaluate(u0)
            out[f"gradbinom_{key}"] = gb
    # a longer RK3 periodic run (m=100) for schedule transparency
    g, u0, uo0 = cfg1_inputs(grid, "periodic")
    op = ops.SemOperator(g, ops.PdeCoefficients(0.01))
    ts = timeloop.TsConfig(scheme="rk3", t0=0.0, t_end=0.0123, dt=1e-4)  # clipped last step
    target = timeloop.integrate(op, uo0, ts, store_steps=None).u_final
    prob = problems.AssimilationProblem(name="cfg1l", grid=g, op=op, ts=ts,
                                        u_target=target, u_guess=u0, checkpoint_slots=10)
    j, gr = prob.evaluate(u0)
    out["long_target"], out["long_J"], out["long_grad"] = target, np.array([j]), gr
    out["long_dts"] = prob.last_forward.dts
    # three L-BFGS iterations on cfg1 periodic RK3
    g, u0, uo0 = cfg1_inputs(grid, "periodic")
    op = ops.SemOperator(g, ops.PdeCoefficients(0.01))
    ts = timeloop.TsConfig(scheme="rk3", t0=0.0, t_end=20 * 1e-4, dt=1e-4)
    target = timeloop.integrate(op, uo0, ts, store_steps=None).u_final
    prob = problems.AssimilationProblem(name="cfg1o", grid=g, op=op, ts=ts,
                                        u_target=target, u_guess=u0)
    res = optimize.minimize(prob.evaluate, u0, optimize.OptimConfig(max_iters=3))
    out["opt_log"] = np.array([[r[0], r[1], r[2], r[3], r[4]] for r in res.log])
    out["opt_x"] = res.x
    return out


IMPLICIT_CASES = [
    # (key, bc, scheme, adaptive, t_end, dt, extra TsConfig kwargs, checkpoint slots)
    ("cn_periodic", "periodic", "cn", False, 10 * 1e-3, 1e-3, {}, None),
    ("cn_dirichlet", "dirichlet0", "cn", False, 10 * 1e-3, 1e-3, {}, None),
    ("cn_binom", "periodic", "cn", False, 12 * 1e-3, 1e-3, {}, 3),
    ("cn_stiff", "periodic", "cn", False, 4 * 2e-2, 2e-2, {"gmres_restart": 8}, None),
    ("ad_rms", "periodic", "rk3", True, 2e-2, 1e-3, {"tol_a": 1e-7, "tol_r": 1e-7}, None),
    ("ad_max", "dirichlet0", "rk3", True, 2e-2, 5e-4, {"tol_a": 1e-6, "tol_r": 1e-6,
                                                      "wlte_form": "max"}, 4),
]


def implicit_fixture(grid, ops, timeloop, problems):
    """Crank-Nicolson (Newton + scipy GMRES, timeloop.py:154-186 / adjoint.py:64-69) and
    adaptive Kutta-3 (controller timeloop.py:198-218) runs on config-1 inputs."""
    out = {}
    for key, bc, scheme, adaptive, t_end, dt, kw, slots in IMPLICIT_CASES:
        g, u0, uo0 = cfg1_inputs(grid, bc)
        op = ops.SemOperator(g, ops.PdeCoefficients(0.01))
        ts = timeloop.TsConfig(scheme=scheme, t0=0.0, t_end=t_end, dt=dt, adaptive=adaptive, **kw)
        tgt_run = timeloop.integrate(op, uo0, ts, store_steps=None, keep_log=True)
        target = tgt_run.u_final
        prob = problems.AssimilationProblem(name=key, grid=g, op=op, ts=ts, u_target=target,
                                            u_guess=u0, checkpoint_slots=slots)
        j, gr = prob.evaluate(u0)
        fwd = prob.last_forward
        out[f"u0_{key}"], out[f"target_{key}"] = u0, target
        out[f"J_{key}"], out[f"grad_{key}"] = np.array([j]), gr
        out[f"ufinal_{key}"], out[f"dts_{key}"], out[f"ts_{key}"] = fwd.u_final, fwd.dts, fwd.ts
        st = fwd.stats
        out[f"fstats_{key}"] = np.array([st["steps"], st["rejects"], st["retries"],
                                         st["newton_iters"], st["gmres_iters"]])
        sw = op.last_sweep_stats
        out[f"sstats_{key}"] = np.array([sw["newton_iters"], sw["gmres_iters"], sw["recomputed"]])
        out[f"tlog_{key}"] = np.array(tgt_run.step_log, dtype=float).reshape(-1, 5)
        out[f"tdts_{key}"] = tgt_run.dts
    return out


CLI_RUNS = {
    # name -> argv of the reference CLI (outputs land in a temp dir)
    "schedule": ["schedule", "--steps", "30", "--checkpoint-slots", "5", "--output", "{d}/sched.csv"],
    "forward": ["forward", "--problem", "burgers1d", "--elements", "5", "--degree", "8", "--steps",
                "40", "--horizon", "0.4", "--output", "{d}/fwd"],
    "forward_cn": ["forward", "--problem", "burgers1d", "--elements", "5", "--degree", "8", "--steps",
                   "8", "--horizon", "0.4", "--scheme", "cn", "--output", "{d}/fwdcn"],
    "gradcheck": ["gradcheck", "--problem", "burgers1d", "--elements", "4", "--degree", "6",
                  "--steps", "20", "--horizon", "0.2", "--ndirs", "2", "--eps", "1e-4,1e-5",
                  "--output", "{d}/gc.csv"],
}


def cli_fixture(semopt, grid):
    """Outputs of the reference CLI (cli.py:208-401) and one snapshot file
    (grid.py:253-270), as raw bytes."""
    import tempfile
    from semopt import cli
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, argv in CLI_RUNS.items():
            rc = cli.main([a.format(d=d) for a in argv])
            out[f"rc_{name}"] = np.array([rc])
        for name, fname in (("schedule", "sched.csv"), ("forward_csv", "fwd.csv"),
                            ("forward_field", "fwd.field"), ("forward_cn_csv", "fwdcn.csv"),
                            ("forward_cn_field", "fwdcn.field"), ("gradcheck", "gc.csv")):
            with open(os.path.join(d, fname), "rb") as fh:
                out[name] = np.frombuffer(fh.read(), dtype=np.uint8)
        g = grid.grid_1d(-1.0, 1.0, 3, 4, "dirichlet0")
        vals = np.sin(np.arange(g.nglobal) * 0.7) * 1e3
        grid.save_field(os.path.join(d, "snap.field"), g, vals)
        with open(os.path.join(d, "snap.field"), "rb") as fh:
            out["snapshot"] = np.frombuffer(fh.read(), dtype=np.uint8)
        out["snapshot_values"] = vals
    return out


GRID3D_CASES = [
    # (extents per axis, elements per axis, degree)
    (((-2.0, 2.0),) * 3, (2, 2, 2), 3),
    (((0.0, 1.0), (-1.0, 2.0), (0.0, 2.5)), (2, 3, 2), 4),
    (((-2.0, 2.0),) * 3, (1, 2, 1), 2),
]


def grid3d_fixture(grid, ops, problems, timeloop):
    """3D sum-factorised operators (ops.py:71-81,109-115,141-150,160-212) and maps
    (grid.py:112-146) on small periodic boxes, plus a short burgers3d evaluation."""
    out = {}
    for k, (ext, els, deg) in enumerate(GRID3D_CASES):
        axes = [grid.Axis(e[0], e[1], n, deg, "periodic") for e, n in zip(ext, els)]
        g = grid.build_grid(axes)
        op = ops.SemOperator(g, ops.PdeCoefficients(0.05))
        rng = np.random.default_rng(300 + k)
        u = rng.uniform(-1.0, 1.0, g.nglobal)
        v = rng.standard_normal(g.nglobal)
        w = rng.standard_normal(g.nglobal)
        out[f"case_{k}"] = np.array([*[x for e in ext for x in e], *els, deg], dtype=float)
        out[f"table_{k}"] = g.table
        out[f"mass_{k}"] = g.mass_scalar
        out[f"u_{k}"], out[f"v_{k}"], out[f"w_{k}"] = u, v, w
        out[f"F_{k}"] = op.apply_rhs(u)
        out[f"J_{k}"] = op.apply_jacobian(u, v)
        out[f"JT_{k}"] = op.apply_jacobian_transpose(u, w)
        out[f"coords_{k}"] = np.concatenate(g.node_coordinates())
    for scheme in ("rk3", "cn"):
        prob = problems.make_problem("burgers3d", elements=2, degree=3, steps=6, horizon=0.03,
                                     scheme=scheme)
        j, gr = prob.evaluate(prob.u_guess)
        out[f"b3d_{scheme}_J"] = np.array([j])
        out[f"b3d_{scheme}_grad"] = gr
        out[f"b3d_{scheme}_ufinal"] = prob.last_forward.u_final
        out[f"b3d_{scheme}_guess"] = prob.u_guess
        out[f"b3d_{scheme}_target"] = prob.u_target
        st = prob.last_forward.stats
        out[f"b3d_{scheme}_stats"] = np.array([st["steps"], st["newton_iters"], st["gmres_iters"],
                                               prob.op.last_sweep_stats["gmres_iters"]])
    return out


def advkinds_fixture(grid, ops, problems):
    """LINEAR / NONE advection (ops.py:147-212 branches) on 1D grids, and the reference's
    advdiff1d / diffusion1d problems (problems.py:235-290)."""
    out = {}
    cases = [("lin_p", "periodic", ops.LINEAR, [0.3]), ("lin_d", "dirichlet0", ops.LINEAR, [-0.7]),
             ("none_p", "periodic", ops.NONE, None), ("none_d", "dirichlet0", ops.NONE, None)]
    for key, bc, kind, speed in cases:
        g = grid.grid_1d(-1.0, 1.0, 6, 5, bc)
        op = ops.SemOperator(g, ops.PdeCoefficients(0.02, kind, speed=speed))
        rng = np.random.default_rng(len(key) * 7 + (1 if bc == "periodic" else 2))
        u, v, w = (rng.standard_normal(g.nglobal) for _ in range(3))
        if bc == "dirichlet0":
            u, v = g.mask(u), g.mask(v)
        out[f"u_{key}"], out[f"v_{key}"], out[f"w_{key}"] = u, v, w
        out[f"F_{key}"] = op.apply_rhs(u)
        out[f"J_{key}"] = op.apply_jacobian(u, v)
        out[f"JT_{key}"] = op.apply_jacobian_transpose(u, w)
    for name, kw in (("advdiff1d", {"steps": 20, "horizon": 0.004}),
                     ("diffusion1d", {"steps": 20, "horizon": 0.01}),
                     ("advdiff1d_cn", {"steps": 5, "horizon": 0.004, "scheme": "cn"})):
        kind = name.split("_")[0]
        prob = problems.make_problem(kind, **kw)
        u0 = 1.1 * prob.u_guess            # diffusion1d's guess is the exact IC (J ~ 1e-20)
        j, gr = prob.evaluate(u0)
        out[f"{name}_u0"] = u0
        out[f"{name}_J"], out[f"{name}_grad"] = np.array([j]), gr
        out[f"{name}_ufinal"] = prob.last_forward.u_final
        out[f"{name}_guess"], out[f"{name}_target"] = prob.u_guess, prob.u_target
        out[f"{name}_exact_ic"] = prob.u_exact_ic
    return out


def spectral_fixture(grid, problems):
    """problems.spectral_error_estimate (problems.py:106-155) on three fields."""
    out = {}
    cases = {
        "burgers": (grid.grid_1d(-2.0, 2.0, 5, 8, "dirichlet0"), None),
        "smooth": (grid.grid_1d(0.0, 1.0, 6, 10, "periodic"), lambda x: np.sin(2 * np.pi * x) + 0.2 * np.cos(6 * np.pi * x)),
        "rough": (grid.grid_1d(0.0, 1.0, 4, 6, "periodic"), lambda x: np.abs(np.sin(3 * np.pi * x)) ** 0.5),
    }
    for key, (g, fn) in cases.items():
        if fn is None:
            vals = problems.make_problem("burgers1d").u_target
        else:
            vals = fn(g.node_coordinates()[0])
        rep = problems.spectral_error_estimate(vals, g)
        out[f"{key}_values"] = vals
        for f in ("eps", "sigma", "scale", "a_top", "resolved", "under_resolved"):
            out[f"{key}_{f}"] = np.asarray(getattr(rep, f))
    return out


SCHED_CASES = [(1, 1), (3, 3), (5, 2), (10, 3), (20, 4), (30, 5), (100, 10), (57, 7), (500, 64)]


def schedules_fixture(checkpoint):
    out = {}
    kinds = {"Store": 0, "Restore": 1, "Advance": 2, "AdjointStep": 3, "Done": 4}
    for m, s in SCHED_CASES:
        sch = checkpoint.plan_binomial(m, s)
        rows = []
        for a in sch.actions:
            name = type(a).__name__
            if name in ("Store", "Restore"):
                rows.append((kinds[name], a.slot, a.step))
            elif name == "Advance":
                rows.append((kinds[name], a.start, a.stop))
            elif name == "AdjointStep":
                rows.append((kinds[name], a.step, -1))
            else:
                rows.append((kinds[name], -1, -1))
        out[f"actions_{m}_{s}"] = np.array(rows, dtype=np.int64)
        out[f"meta_{m}_{s}"] = np.array([sch.recomputed, sch.backward_start, sch.slots])
        out[f"stores_{m}_{s}"] = np.array(sorted(sch.forward_stores.items()), dtype=np.int64)
    return out


def main():
    semopt, grid, ops, timeloop, adjoint, checkpoint, problems, optimize = _ref()
    np.savez_compressed(os.path.join(HERE, "basis.npz"), **basis_fixture(semopt, ops, grid))
    np.savez_compressed(os.path.join(HERE, "maps.npz"), **maps_fixture(grid))
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ops_fixture(grid, ops))
    np.savez_compressed(os.path.join(HERE, "sweeps.npz"),
                        **sweep_fixture(grid, ops, timeloop, adjoint, checkpoint, problems, optimize))
    np.savez_compressed(os.path.join(HERE, "schedules.npz"), **schedules_fixture(checkpoint))
    np.savez_compressed(os.path.join(HERE, "implicit.npz"),
                        **implicit_fixture(grid, ops, timeloop, problems))
    np.savez_compressed(os.path.join(HERE, "cli.npz"), **cli_fixture(semopt, grid))
    np.savez_compressed(os.path.join(HERE, "grid3d.npz"), **grid3d_fixture(grid, ops, problems, timeloop))
    np.savez_compressed(os.path.join(HERE, "advkinds.npz"), **advkinds_fixture(grid, ops, problems))
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), **spectral_fixture(grid, problems))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
