"""Config-4 ensemble sweep on a reduced batch (B rings, a few steps) for ncu captures of
ens_forward_kernel / ens_adjoint_kernel.

    python tools/ens_prof.py [B] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import adjoint, configs, timeloop  # noqa: E402


def main(B=296, steps=20):
    prob = configs.cfg4_problem(B=int(B), steps=int(steps), device="cuda:0")
    op = prob.op
    u0 = torch.from_numpy(prob.u_guess).cuda()
    fwd = timeloop.integrate_ensemble(op, u0, prob.ts)
    _, lam = adjoint.terminal_condition(prob.grid, fwd.u_final, prob.target(), op=op)
    g = adjoint.ensemble_sweep(op, prob.ts, fwd, lam)
    torch.cuda.synchronize()
    print("ok", bool(torch.isfinite(g).all()))


if __name__ == "__main__":
    main(*sys.argv[1:])
