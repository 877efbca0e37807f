"""A/B of the config-2-field RK4 sweep (bench.sweep_ratio) for one library build (SEM1D_LIB=...)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1806_01422_b200 import configs  # noqa: E402


def main(reps=3):
    op = configs.cfg_operator(configs.CFG2, device="cuda:0")
    best = None
    for _ in range(reps):
        r = bench.sweep_ratio(op, torch)
        if best is None or r["ms_per_adjoint_step"] + r["ms_per_forward_step"] < \
                best["ms_per_adjoint_step"] + best["ms_per_forward_step"]:
            best = r
    print(json.dumps({"lib": os.environ.get("SEM1D_LIB", "default"), "sweep": best}))


if __name__ == "__main__":
    main()
