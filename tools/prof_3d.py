"""Profiling driver: 3D N = 7, E = 32^3 F / J / J^T applies (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1806_01422_b200 import PdeCoefficients  # noqa: E402
from paper_1806_01422_b200.grid import grid_3d  # noqa: E402
from paper_1806_01422_b200.ops3d import SemOperator3D  # noqa: E402


def main(reps=2):
    grid = grid_3d((-2.0, 2.0), 32, 7)
    op = SemOperator3D(grid, PdeCoefficients(0.01), device="cuda:0")
    rng = np.random.default_rng(7)
    u, v, w = (torch.from_numpy(a).cuda() for a in (rng.uniform(-1, 1, grid.nglobal),
                                                   rng.standard_normal(grid.nglobal),
                                                   rng.standard_normal(grid.nglobal)))
    o = op.empty()
    for _ in range(reps):
        op.launch_rhs(u, o)
        op.launch_jac(u, v, o)
        op.launch_jact(u, w, o)
    torch.cuda.synchronize()
    assert op.flags() == 0
    print("ok")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
