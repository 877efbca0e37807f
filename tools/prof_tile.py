"""Profiling driver: a few fused RK4 steps / adjoint steps on the config-2 field.
  python tools/prof_tile.py [fwd|fwd_st|adj|adj_st] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1806_01422_b200 import configs  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "fwd"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
op = configs.cfg_operator(configs.CFG2, device="cuda:0")
u = torch.sin(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device="cuda"))
lam = torch.cos(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device="cuda"))
o = op.empty()
st = [op.empty() for _ in range(3)]
slots = op.flag_slots(1)
dt = 1e-14
for _ in range(reps):
    if kind == "fwd":
        op.launch_rk_step(u, o, dt, "rk4", flag=slots.data_ptr())
    elif kind == "fwd_st":
        op.launch_rk_step_stages(u, o, st, dt, "rk4")
    elif kind == "adj":
        op.launch_adj_step(u, lam, o, dt, "rk4")
    else:
        op.launch_adj_step_stages(u, st, lam, o, dt, "rk4")
torch.cuda.synchronize()
print("ok", kind)
