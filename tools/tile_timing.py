"""Fused RK4 step / adjoint step timings (recompute and stored-stage variants) for N = 7, 15, 23, 31."""
import json, sys, torch
sys.path.insert(0, '.')
import paper_1806_01422_b200 as sb
from paper_1806_01422_b200.grid import grid_1d
for N, E in ((7, 1 << 20), (15, 1 << 19), (23, 1 << 18), (31, 1 << 18)):
    g = grid_1d(0.0, E / 64.0, E, N)
    op = sb.SemOperator(g, sb.PdeCoefficients(1e-3), device="cuda:0")
    u = torch.sin(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device="cuda"))
    lam = torch.cos(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device="cuda"))
    o = op.empty()
    st = [op.empty() for _ in range(3)]
    def t(fn, reps=10):
        for _ in range(2): fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps): fn()
        e.record(); torch.cuda.synchronize()
        return s.elapsed_time(e) / reps
    r = {"N": N, "E": E, "fwd": t(lambda: op.launch_rk_step(u, o, 1e-5, "rk4")),
         "adj": t(lambda: op.launch_adj_step(u, lam, o, 1e-5, "rk4")),
         "fwd_st": t(lambda: op.launch_rk_step_stages(u, o, st, 1e-5, "rk4")) if op.step_stages_supported() else None,
         "adj_st": t(lambda: op.launch_adj_step_stages(u, st, lam, o, 1e-5, "rk4")) if op.step_stages_supported() else None,
         "stages_supported": op.step_stages_supported()}
    print(json.dumps(r), flush=True)
