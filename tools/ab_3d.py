import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1806_01422_b200 import PdeCoefficients
from paper_1806_01422_b200.grid import grid_3d
from paper_1806_01422_b200.ops3d import SemOperator3D
def timed(fn, reps=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps * 1e3, 1)
grid = grid_3d((-2.0, 2.0), 32, 7)
op = SemOperator3D(grid, PdeCoefficients(0.01), device="cuda:0")
rng = np.random.default_rng(7)
u, v, w = (torch.from_numpy(a).cuda() for a in (rng.uniform(-1, 1, grid.nglobal), rng.standard_normal(grid.nglobal), rng.standard_normal(grid.nglobal)))
o = op.empty()
print(json.dumps({"lib": os.environ.get("SEM1D_LIB", "default")[-8:], "F": timed(lambda: op.launch_rhs(u, o)), "J": timed(lambda: op.launch_jac(u, v, o)), "JT": timed(lambda: op.launch_jact(u, w, o))}))
