"""Profiling driver: a short RK4 forward + adjoint sweep on the config-2 field."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1806_01422_b200 import adjoint, checkpoint, configs, timeloop  # noqa: E402


def main(steps=2, mode="recompute"):
    op = configs.cfg_operator(configs.CFG2, device="cuda:0")
    dt = 1e-14
    ts = timeloop.TsConfig(scheme="rk4", t0=0.0, t_end=steps * dt, dt=dt)
    u0 = torch.sin(torch.linspace(0, 6.283185307179586, op.ndof, dtype=torch.float64, device="cuda:0"))
    fwd = timeloop.integrate(op, u0, ts, keep_stages=mode != "recompute")
    j, lam = adjoint.terminal_condition(op.grid, fwd.u_final, 0.5 * u0, op=op)
    adjoint.sweep(op, ts, fwd, checkpoint.plan_store_all(fwd.n_steps), lam)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2, sys.argv[2] if len(sys.argv) > 2 else "recompute")
