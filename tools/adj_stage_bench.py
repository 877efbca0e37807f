"""Per-stage adjoint kernels (sem1d_adj_stage) on a Dirichlet ring: one RK4 adjoint step
(stage recompute + 4 adjoint stages) and the adjoint stages alone, DMMA ws kernel (path 0)
against the thread-per-element DFMA kernel (path 2).
  python tools/adj_stage_bench.py [N] [log2 E]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_01422_b200 as sb  # noqa: E402
from paper_1806_01422_b200 import _lib, adjoint  # noqa: E402
from paper_1806_01422_b200.grid import grid_1d  # noqa: E402


def main(N=7, lg=22, reps=20):
    N, E = int(N), 1 << int(lg)
    g = grid_1d(-1.0, 1.0, E, N, "dirichlet0")
    op = sb.SemOperator(g, sb.PdeCoefficients(1e-2), device="cuda:0")
    x = torch.linspace(-1, 1, op.ndof, dtype=torch.float64, device="cuda")
    u = torch.sin(torch.pi * x)
    u[0] = u[-1] = 0.0
    lam = torch.cos(3 * x)
    eng = adjoint.adjoint_engine_for(op, "rk4")
    out = op.empty()
    Us = eng.fwd.stages(u, 1e-5, eng.U)
    res = {"N": N, "E": E}
    lib = _lib.load()
    for path, name in ((0, "dmma_ws"), (2, "dfma")):
        lib.sem1d_set_kernel_path(path)
        L = eng.L

        def stages():
            for i in range(3, -1, -1):
                lts = [L[j] for j, _ in eng.zterms[i]]
                acs = [a for _, a in eng.zterms[i]]
                if i > 0:
                    op.launch_adj_stage(Us[i], lam, eng.b[i], lts, acs, 1e-5, L[i], None, None)
                else:
                    op.launch_adj_stage(Us[0], lam, eng.b[0], lts, acs, 1e-5, None, [None, L[1], L[2], L[3]], out)

        for fn, key in ((stages, "adj_stages_us"), (lambda: eng.step(u, lam, 1e-5, out), "adj_step_us")):
            for _ in range(3):
                fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(reps):
                fn()
            e.record()
            torch.cuda.synchronize()
            res.setdefault(name, {})[key] = round(1e3 * s.elapsed_time(e) / reps, 2)
        assert op.flags() == 0
    lib.sem1d_set_kernel_path(0)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:])
