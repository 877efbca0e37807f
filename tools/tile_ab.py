"""A/B of the fused RK4 step / adjoint-step kernels on the config-2 field (E = 2^22, N = 7):
tile variant 0 (auto: register-resident N = 7 kernels) vs 1 (shared-memory tile kernels).
Kernel times from CUDA events around `reps` back-to-back launches (PDL overlap kept)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1806_01422_b200 as sb  # noqa: E402
from paper_1806_01422_b200 import _lib, configs  # noqa: E402

lib = _lib.load()
E = int(sys.argv[1]) if len(sys.argv) > 1 else configs.CFG2["E"]
op = configs.cfg_operator(dict(configs.CFG2, E=E), device="cuda:0")
u = torch.sin(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device="cuda"))
lam = torch.cos(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device="cuda"))
o = op.empty()
st = [op.empty() for _ in range(3)]
dt = 1e-14
slots = op.flag_slots(1)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return 1e3 * s.elapsed_time(e) / reps


for variant in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("1", "0", "2"))]:
    assert lib.sem1d_set_tile_variant(variant) == 0
    r = {"variant": variant, "E": E,
         "fwd_us": t(lambda: op.launch_rk_step(u, o, dt, "rk4")),
         "fwd_fast_us": t(lambda: op.launch_rk_step(u, o, dt, "rk4", flag=slots.data_ptr())),
         "fwd_st_us": t(lambda: op.launch_rk_step_stages(u, o, st, dt, "rk4")),
         "fwd_st_fast_us": t(lambda: op.launch_rk_step_stages(u, o, st, dt, "rk4", flag=slots.data_ptr())),
         "adj_us": t(lambda: op.launch_adj_step(u, lam, o, dt, "rk4")),
         "adj_fast_us": t(lambda: op.launch_adj_step(u, lam, o, dt, "rk4", flag=slots.data_ptr())),
         "adj_st_fast_us": t(lambda: op.launch_adj_step_stages(u, st, lam, o, dt, "rk4", flag=slots.data_ptr())),
         "adj_st_us": t(lambda: op.launch_adj_step_stages(u, st, lam, o, dt, "rk4"))}
    op.launch_rk_step(u, o, 1e-3 * 2.0 / E, "rk4")       # a physical dt: compare the states
    ref = ref if variant != 1 and "ref" in dir() else o.clone()
    r["max_rel_diff_vs_first"] = float((o - ref).abs().max() / ref.abs().max())
    print(json.dumps(r), flush=True)
lib.sem1d_set_tile_variant(0)
assert op.flags() == 0 and int(slots[0]) == 0
