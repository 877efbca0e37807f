"""Profiling driver: config-2 F, J, J^T applies (for ncu launch lists / --set full)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1806_01422_b200 import configs  # noqa: E402


def main(reps=3, cfg="2"):
    c = {"2": configs.CFG2, "3": configs.CFG3}[cfg]
    op = configs.cfg_operator(c, device="cuda:0")
    u, v, w = configs.operator_inputs(op.ndof, c["seed"])
    ud, vd, wd = (torch.from_numpy(a).cuda() for a in (u, v, w))
    o = op.empty()
    for _ in range(reps):
        op.launch_rhs(ud, o)
        op.launch_jac(ud, vd, o)
        op.launch_jact(ud, wd, o)
    torch.cuda.synchronize()
    assert op.flags() == 0
    print("ok")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3, sys.argv[2] if len(sys.argv) > 2 else "2")
