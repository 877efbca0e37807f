"""Crank-Nicolson forward + adjoint sweep on one B200 vs the
reference algorithm on the host CPU.

Workload: config-5 physics (h = 1/64, N = 7, nu = 1e-3, smooth 32-mode Fourier IC) on a
config-2-size ring (E = 2^22, 29.4 M DOF), CN with dt = 1e-3 (5x the explicit RK4 step of
config 5), 10 steps, store-all forward then the discrete-adjoint sweep (GMRES with J^T only,
adjoint.py:64-69).  CPU baseline: oracle/semref.py (numpy + scipy GMRES, the reference's
arithmetic) on E = 2^16 with the same physics, reported per DOF-step.

    python tools/bench_cn.py [--E 4194304] [--steps 10] [--cpu-E 8192]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1806_01422_b200 import adjoint, configs, timeloop  # noqa: E402
from paper_1806_01422_b200.grid import PERIODIC, grid_1d  # noqa: E402
from paper_1806_01422_b200.ops import PdeCoefficients, SemOperator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=1 << 22)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--dt", type=float, default=1e-3)
    ap.add_argument("--cpu-E", type=int, default=1 << 16)
    ap.add_argument("--cpu-steps", type=int, default=3)
    args = ap.parse_args()
    c = configs.CFG5
    E, N, h, nu = args.E, c["N"], c["h"], c["nu"]
    grid = grid_1d(0.0, E * h, E, N, PERIODIC)
    op = SemOperator(grid, PdeCoefficients(nu), device="cuda:0")
    ts = timeloop.TsConfig(scheme="cn", t0=0.0, t_end=args.steps * args.dt, dt=args.dt)
    u0 = configs.fourier_field_device(grid, c["modes"], c["seed"], op.device) / 8.0
    ud = configs.fourier_field_device(grid, c["modes"], c["seed"] + 77, op.device) / 40.0 + u0

    # warm-up (one step + one adjoint step: plans, workspace, kernels)
    w = timeloop.integrate(op, u0, timeloop.TsConfig(scheme="cn", t0=0.0, t_end=args.dt, dt=args.dt))
    adjoint.adjoint_step_cn(op, u0, w.u_final, u0, 0.0, args.dt, ts)
    torch.cuda.synchronize()

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    fwd = timeloop.integrate(op, u0, ts, store_steps="all")
    ev[1].record()
    j, lam = adjoint.terminal_condition(grid, fwd.u_final, ud, op=op)
    from paper_1806_01422_b200 import checkpoint
    g = adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(fwd.n_steps), lam)
    ev[2].record()
    torch.cuda.synchronize()
    t_fwd, t_adj = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    ndof = op.ndof
    m = fwd.n_steps
    res = {
        "workload": f"CN forward + adjoint sweep, E={E} N={N} (DOF {ndof}), h=1/64, nu={nu}, "
                    f"dt={args.dt}, {m} steps, store-all",
        "gpu": {"forward_ms": t_fwd, "adjoint_ms": t_adj, "ms_per_forward_step": t_fwd / m,
                "ms_per_adjoint_step": t_adj / m,
                "newton_iters": fwd.stats["newton_iters"], "gmres_iters_forward": fwd.stats["gmres_iters"],
                "gmres_iters_adjoint": op.last_sweep_stats["gmres_iters"],
                "dof_steps_per_s_forward": ndof * m / (t_fwd * 1e-3),
                "dof_steps_per_s_adjoint": ndof * m / (t_adj * 1e-3),
                "J": float(j), "grad_norm": float(torch.linalg.norm(g))},
    }
    del fwd, g, lam
    torch.cuda.empty_cache()

    # CPU: the reference algorithm (oracle: numpy + scipy GMRES) on a bounded sample
    from oracle import semref as R
    Ec = args.cpu_E
    orc = R.BurgersOracle(R.Mesh1D(0.0, Ec * h, Ec, N, True), nu)
    gc = grid_1d(0.0, Ec * h, Ec, N, PERIODIC)
    u0c = configs.fourier_field_device(gc, c["modes"], c["seed"], "cpu").numpy() / 8.0
    udc = configs.fourier_field_device(gc, c["modes"], c["seed"] + 77, "cpu").numpy() / 40.0 + u0c
    R.cn_step(R.BurgersOracle(R.Mesh1D(0.0, 8 * h, 8, N, True), nu),
              np.sin(np.arange(56.0)), args.dt)            # warm-up: scipy import, BLAS threads
    t0 = time.perf_counter()
    traj, dts, _, fst, _ = R.integrate_general(orc, u0c, 0.0, args.cpu_steps * args.dt, args.dt, "cn")
    t1 = time.perf_counter()
    _, lamc = R.terminal(orc.mesh, traj[-1], udc)
    sst = {}
    for n in range(len(dts) - 1, -1, -1):
        lamc = R.adjoint_cn_step(orc, traj[n], traj[n + 1], lamc, dts[n], None, sst)
    t2 = time.perf_counter()
    dsc = orc.mesh.ndof * len(dts)
    res["cpu_reference_algorithm"] = {
        "sample": f"E={Ec} (DOF {orc.mesh.ndof}), {len(dts)} CN steps, same h/nu/dt",
        "threads": os.cpu_count(), "forward_s": t1 - t0, "adjoint_s": t2 - t1,
        "newton_iters": fst["newton_iters"], "gmres_iters_forward": fst["gmres_iters"],
        "gmres_iters_adjoint": sst.get("gmres_iters", 0),
        "dof_steps_per_s_forward": dsc / (t1 - t0), "dof_steps_per_s_adjoint": dsc / (t2 - t1)}
    res["speedup_forward"] = res["gpu"]["dof_steps_per_s_forward"] / res["cpu_reference_algorithm"][
        "dof_steps_per_s_forward"]
    res["speedup_adjoint"] = res["gpu"]["dof_steps_per_s_adjoint"] / res["cpu_reference_algorithm"][
        "dof_steps_per_s_adjoint"]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
