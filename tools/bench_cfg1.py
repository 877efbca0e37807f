"""BASELINE config 1 (E=16, N=9, 20 RK4 steps): wall time of one evaluate() on the GPU
path vs the oracle port on the host (the reference algorithm), same inputs."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import semref as R  # noqa: E402
from paper_1806_01422_b200 import configs  # noqa: E402


def main(reps=20):
    out = {}
    for scheme in ("rk4", "rk3"):
        prob = configs.cfg1_problem(scheme=scheme, device="cuda:0")
        u0 = torch.from_numpy(configs.cfg1_inputs(prob.grid)[0]).cuda()
        for _ in range(3):
            prob.evaluate(u0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            j, g = prob.evaluate(u0)
        torch.cuda.synchronize()
        gpu_ms = (time.perf_counter() - t0) / reps * 1e3
        c = configs.CFG1
        ref = R.BurgersOracle(R.Mesh1D(c["xa"], c["xb"], c["E"], c["N"], True), c["nu"])
        tg = prob.target().cpu().numpy()
        u0h = u0.cpu().numpy()
        t0 = time.perf_counter()
        for _ in range(reps):
            R.evaluate(ref, u0h, tg, 0.0, c["steps"] * c["dt"], c["dt"], scheme)
        cpu_ms = (time.perf_counter() - t0) / reps * 1e3
        out[scheme] = {"gpu_evaluate_ms": gpu_ms, "cpu_oracle_evaluate_ms": cpu_ms,
                       "launches_per_evaluate": None}
    print(json.dumps({"workload": "BASELINE config 1", **out}))


if __name__ == "__main__":
    main()
