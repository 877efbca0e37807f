"""Randomised parity soak of the ring-resident ensemble sweeps (N = 15 on the reflection split;
N = 7 and 9 as controls): random ring sizes, batch sizes and schemes; objective and gradient of
every problem against the oracle's evaluate at 1e-9.  python tools/soak_ensemble.py [cases] [seed]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1806_01422_b200 as sb  # noqa: E402
from oracle import semref as R  # noqa: E402
from paper_1806_01422_b200 import adjoint, configs, timeloop  # noqa: E402
from paper_1806_01422_b200.grid import grid_1d  # noqa: E402


def main(cases=40, seed=0):
    rng = np.random.default_rng(int(seed))
    worst = {"J": 0.0, "g": 0.0}
    fails = []
    for c in range(int(cases)):
        N = int(rng.choice([15, 15, 15, 7, 9]))
        E = int(rng.choice([8, 16, 24, 32, 40, 64, 96, 104, 160, 256])) if N != 9 else int(rng.integers(4, 40))
        B = int(rng.integers(2, 6))
        scheme = str(rng.choice(["rk4", "rk3", "euler"]))
        steps = int(rng.integers(3, 25))
        L = 20.0 * E / 256.0
        dt = 5e-5 if scheme != "euler" else 1e-5
        g = grid_1d(0.0, L, E, N)
        op = sb.SemOperator(g, sb.PdeCoefficients(0.01), device="cuda:0", batch=B)
        u0 = configs.fourier_fields(g, B, 4, seed=1000 * int(seed) + c)
        tgt = configs.fourier_fields(g, B, 4, seed=5000 + 1000 * int(seed) + c)
        ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=steps * dt, dt=dt)
        fwd = timeloop.integrate_ensemble(op, u0, ts)
        J, lam = adjoint.terminal_condition(g, fwd.u_final, torch.from_numpy(tgt).cuda(), op=op)
        grad = adjoint.ensemble_sweep(op, ts, fwd, lam).cpu().numpy()
        ref = R.BurgersOracle(R.Mesh1D(0.0, L, E, N, True), 0.01)
        for b in range(B):
            j_ref, g_ref, _ = R.evaluate(ref, u0[b], tgt[b], 0.0, steps * dt, dt, scheme)
            ej = abs(float(J[b]) - j_ref) / abs(j_ref)
            eg = float(np.max(np.abs(grad[b] - g_ref)) / np.max(np.abs(g_ref)))
            worst["J"], worst["g"] = max(worst["J"], ej), max(worst["g"], eg)
            if not (ej <= 1e-9 and eg <= 1e-9):
                fails.append((c, N, E, B, scheme, steps, ej, eg))
        del op
    print(json.dumps({"cases": int(cases), "seed": int(seed), "worst_rel_err": worst, "failures": fails[:20]}))
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main(*sys.argv[1:]))
