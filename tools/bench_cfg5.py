"""BASELINE config 5: E = 2^25 elements (N = 7, 235M DOF), 500 RK4 steps per gradient with
binomial checkpointing (s slots in HBM), L-BFGS on device vectors.  One GPU, or element-
sharded under torchrun (ghost-zone mode: one NCCL exchange per step, all-reduced dots).

  python tools/bench_cfg5.py [--E 33554432] [--steps 500] [--slots 40] [--iters 10] [--gtol 1e-8]
                             [--band KMIN,KMAX]
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/bench_cfg5.py ...
--band draws the 32 Fourier modes of u0 and of its perturbation from a wavenumber band on
the element scale (viscosity then damps them within the 500-step horizon, so recovering the
perturbation is an ill-conditioned problem that needs many L-BFGS iterations; with the
default lowest modes the forward map is close to the identity and L-BFGS converges in 2).
Prints one JSON line (rank 0): per-evaluate time (max over ranks) and the optimisation log."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_01422_b200 as sb  # noqa: E402
from paper_1806_01422_b200 import configs, timeloop  # noqa: E402


def main(E=None, steps=None, slots=None, iters=None, gtol=1e-8, band=None, amp=1.0 / 8.0):
    import torch.distributed as dist

    from paper_1806_01422_b200 import dist as sd
    from paper_1806_01422_b200.grid import grid_1d
    c = configs.CFG5
    E = int(E or c["E"])
    steps = int(steps or c["steps"])
    slots = int(slots or c["slots"])
    iters = int(iters if iters is not None else c["lbfgs_iters"])
    backend = os.environ.get("SEM1D_DIST_BACKEND")
    rank, world, local = sd.init_from_env(backend)
    if os.environ.get("SEM1D_SAME_DEVICE"):
        local = 0
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    t0 = time.perf_counter()
    g = grid_1d(0.0, E * c["h"], E, c["N"])
    coef = sb.PdeCoefficients(c["nu"])
    if world == 1:
        prob = configs.cfg5_problem(E=E, steps=steps, slots=slots, device=dev, band=band, amp=amp)
        op = prob.op
        dot = sb.optimize.default_dot
    else:
        op = sd.ShardedOperator(g, coef, rank, world, device=dev)
        ts = timeloop.TsConfig(scheme="rk4", t0=0.0, t_end=steps * c["dt"], dt=c["dt"])
        sl = slice(op.part.g_lo, op.part.g_lo + op.part.n_own)
        u0 = configs.fourier_field_device(g, c["modes"], c["seed"], dev, band)[sl] * amp
        pert = configs.fourier_field_device(g, c["modes"], c["seed"] + 77, dev, band)[sl] * (amp / 5.0)
        target = timeloop.integrate(op, op.field(u0 + pert)[0], ts, store_steps=None).u_final
        prob = sb.AssimilationProblem(name="cfg5-sharded", grid=op.grid, op=op, ts=ts,
                                      u_target=target, u_guess=op.field(u0)[0],
                                      checkpoint_slots=slots)
        dot = op.dot
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    times = []

    def fun(x):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a = time.perf_counter()
        j, gr = prob.evaluate(x)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - a], dtype=torch.float64,
                         device=dev if backend != "gloo" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
        return j, gr

    t0 = time.perf_counter()
    res = sb.minimize(fun, prob.u_guess, sb.OptimConfig(max_iters=iters, gtol=gtol), dot=dot)
    torch.cuda.synchronize()
    opt_s = time.perf_counter() - t0
    if rank == 0:
        out = {"workload": "BASELINE config 5", "n_gpus": world, "E": E, "N": c["N"],
               "dof": E * c["N"], "steps": steps, "slots": slots,
               "recomputed_steps": prob.schedule_for(steps).recomputed, "setup_s": setup_s,
               "lbfgs_iterations": res.iterations, "status": res.status,
               "evaluations": len(times), "evaluate_s_min": min(times),
               "evaluate_s_mean": sum(times) / len(times), "optimize_s": opt_s,
               "dof_steps_per_s_forward_equiv": E * c["N"] * steps / min(times),
               "J_log": [r[1] for r in res.log], "gnorm_log": [r[2] for r in res.log],
               "kernels": "fused whole-step" if op.step_fused_supported() else "per-stage",
               "gtol": gtol, "band": band, "amp": amp, "optimize_wall_s": opt_s,
               "sharding": "single GPU" if world == 1 else
                           f"{world} ranks, ghost zones of {op.part.zone} elements"}
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int)
    ap.add_argument("--steps", type=int)
    ap.add_argument("--slots", type=int)
    ap.add_argument("--iters", type=int)
    ap.add_argument("--gtol", type=float, default=1e-8)
    ap.add_argument("--band", type=lambda v: tuple(float(x) for x in v.split(",")))
    ap.add_argument("--amp", type=float, default=1.0 / 8.0)
    a = ap.parse_args()
    main(a.E, a.steps, a.slots, a.iters, a.gtol, a.band, a.amp)
