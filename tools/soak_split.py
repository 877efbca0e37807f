"""Randomised parity soak of the reflection-split kernels (N = 15, 31; plus N = 7 and 23 as the
unsplit controls): random ring sizes, both boundary kinds, batches, F / J v / J^T w against the
oracle at 1e-12, and one fused RK4 step + adjoint step per case where the fused kernels apply
(increments of the state and of the cotangent at 1e-9).  python tools/soak_split.py [cases] [seed]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1806_01422_b200 as sb  # noqa: E402
from oracle import semref as R  # noqa: E402
from paper_1806_01422_b200.grid import grid_1d  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(float(np.max(np.abs(b))), 1e-300))


def main(cases=150, seed=0):
    rng = np.random.default_rng(int(seed))
    worst = {"F": 0.0, "J": 0.0, "JT": 0.0, "step": 0.0, "adj": 0.0}
    fails = []
    for c in range(int(cases)):
        N = int(rng.choice([15, 31, 31, 15, 7, 23]))
        E = int(rng.choice([rng.integers(1, 20), rng.integers(20, 300), rng.integers(300, 1500)]))
        per = bool(rng.integers(0, 2))
        B = int(rng.choice([1, 1, 2, 3]))
        nu = float(rng.choice([1e-3, 1e-2, 0.1]))
        L = float(rng.uniform(0.5, 30.0))
        g = grid_1d(0.0, L, E, N, "periodic" if per else "dirichlet0")
        op = sb.SemOperator(g, sb.PdeCoefficients(nu), device="cuda:0", batch=B)
        ref = R.BurgersOracle(R.Mesh1D(0.0, L, E, N, per), nu)
        U = rng.uniform(-1, 1, (B, ref.mesh.ndof))
        V = rng.standard_normal((B, ref.mesh.ndof))
        W = rng.standard_normal((B, ref.mesh.ndof))
        sq = (lambda x: x) if B > 1 else (lambda x: x[0])
        F, JV, JT = op.apply_rhs(sq(U)), op.apply_jacobian(sq(U), sq(V)), op.apply_jacobian_transpose(sq(U), sq(W))
        for b in range(B):
            e = {"F": rel((F[b] if B > 1 else F), ref.rhs(U[b])),
                 "J": rel((JV[b] if B > 1 else JV), ref.jac(U[b], V[b])),
                 "JT": rel((JT[b] if B > 1 else JT), ref.jact(U[b], W[b]))}
            for k, v in e.items():
                worst[k] = max(worst[k], v)
                if not v <= 1e-12:
                    fails.append((c, N, E, per, B, k, v))
        if B == 1 and per and op.step_fused_supported():
            u = 0.3 * np.sin(2 * np.pi * np.arange(ref.mesh.ndof) / ref.mesh.ndof) + 0.01 * U[0]
            lam = W[0]
            h = L / E
            dt = 0.05 * h * h / (N ** 4 * nu + 1.0)
            ud, ld = torch.from_numpy(u).cuda(), torch.from_numpy(lam).cuda()
            un, lo = op.empty(), op.empty()
            op.launch_rk_step(ud, un, dt, "rk4")
            op.launch_adj_step(ud, ld, lo, dt, "rk4")
            torch.cuda.synchronize()
            if op.flags() == 0:
                # the INCREMENTS of the step and of the adjoint step (the states themselves move by
                # ~dt and would hide an error in the stage arithmetic)
                es = rel(un.cpu().numpy() - u, R.rk_step(ref, u, dt, "rk4") - u)
                ea = rel(lo.cpu().numpy() - lam, R.adjoint_rk_step(ref, u, lam, dt, "rk4") - lam)
                worst["step"], worst["adj"] = max(worst["step"], es), max(worst["adj"], ea)
                if not es <= 1e-9:
                    fails.append((c, N, E, per, B, "step", es))
                if not ea <= 1e-9:
                    fails.append((c, N, E, per, B, "adj", ea))
        del op
    print(json.dumps({"cases": int(cases), "seed": int(seed), "worst_rel_err": worst, "failures": fails[:20]}))
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main(*sys.argv[1:]))
