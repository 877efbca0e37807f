"""BASELINE config 4 at full size: B=4096 rings (E=256, N=15), 1000 RK4 steps forward with
the full trajectory in HBM, terminal condition, backward sweep.  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import adjoint, configs, timeloop  # noqa: E402


def main(B=4096, steps=1000, cpu_sample=2):
    B, steps, cpu_sample = int(B), int(steps), int(cpu_sample)
    prob = configs.cfg4_problem(B=B, steps=steps, device="cuda:0")
    op = prob.op
    u0 = torch.from_numpy(prob.u_guess).cuda()
    target = prob.target()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    # warm-up on a few steps
    ts_w = timeloop.TsConfig(scheme="rk4", t0=0.0, t_end=2 * 5e-5, dt=5e-5)
    fw = timeloop.integrate_ensemble(op, u0, ts_w)
    _, lam = adjoint.terminal_condition(prob.grid, fw.u_final, target, op=op)
    adjoint.ensemble_sweep(op, ts_w, fw, lam)
    del fw
    # the trajectory block (126 GB at full size) into torch's caching allocator before the timed
    # region: a cold cudaMalloc of that size once measured 120 ms inside the forward time
    warm = torch.empty((steps + 1) * B * prob.grid.nglobal, dtype=torch.float64, device="cuda:0")
    del warm
    torch.cuda.synchronize()
    ev[0].record()
    fwd = timeloop.integrate_ensemble(op, u0, prob.ts)
    ev[1].record()
    J, lam = adjoint.terminal_condition(prob.grid, fwd.u_final, target, op=op)
    ev[2].record()
    g = adjoint.ensemble_sweep(op, prob.ts, fwd, lam)
    ev[3].record()
    torch.cuda.synchronize()
    f_ms, t_ms, a_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])
    ndof = prob.grid.nglobal
    E, N = configs.CFG4["E"], configs.CFG4["N"]
    n = N + 1
    f_flop = (4 * n * n + 3 * n + N + 1) * E          # per ring per F
    jt_flop = (6 * n * n + 5 * n + N + 1) * E
    fwd_flops = 4 * f_flop * B * steps
    adj_flops = (3 * f_flop + 4 * jt_flop) * B * steps
    out = {"workload": "BASELINE config 4", "B": B, "E": E, "N": N, "steps": steps,
           "dof_per_problem": ndof, "forward_ms": f_ms, "terminal_ms": t_ms, "adjoint_ms": a_ms,
           "evaluate_ms": f_ms + t_ms + a_ms, "adjoint_over_forward": a_ms / f_ms,
           "forward_fp64_tflops": fwd_flops / (f_ms * 1e-3) / 1e12,
           "adjoint_fp64_tflops": adj_flops / (a_ms * 1e-3) / 1e12,
           "gradients_per_s": B / ((f_ms + t_ms + a_ms) * 1e-3),
           "traj_GB": fwd.trajectory.numel() * 8 / 1e9,
           "J_mean": float(J.mean()), "g_finite": bool(torch.isfinite(g).all()),
           "fp64_tflops_count": "the reference algorithm's flops (full n x n contractions); the kernels run "
                                "the reflection split and execute about half of them"}
    if cpu_sample:
        from oracle import semref as R
        c = configs.CFG4
        ref = R.BurgersOracle(R.Mesh1D(c["xa"], c["xb"], E, N, True), c["nu"])
        tg = target.cpu().numpy()
        t0 = time.perf_counter()
        for b in range(int(cpu_sample)):
            R.evaluate(ref, prob.u_guess[b], tg[b], 0.0, steps * c["dt"], c["dt"], "rk4")
        per = (time.perf_counter() - t0) / int(cpu_sample)
        out["cpu_oracle_s_per_problem"] = per
        out["cpu_gradients_per_s"] = 1.0 / per
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
