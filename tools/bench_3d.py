"""3D sum-factorised Burgers applies on one B200 vs the reference
algorithm on the host CPU.

Boxes: N = 7 with E = 32 per axis, N = 8 with E = 28 (P = 224 nodes per axis, 33.7 M DOF,
270 MB per 3-component field).  Per apply: CUDA-event average of 20 launches, FP64
throughput from the algorithmic flop count of the sum-factorised contractions (2 n^4 per
axis contraction per element: F 18, J / J^T 27 contractions per element) against the
measured DFMA peak, and HBM throughput from the algorithmic bytes (fields read once,
result written once).  CPU: oracle/semref.py (the reference's numpy arithmetic, all
host threads) on E = 8 per axis.

    python tools/bench_3d.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1806_01422_b200 import PdeCoefficients  # noqa: E402
from paper_1806_01422_b200.grid import grid_3d  # noqa: E402
from paper_1806_01422_b200.ops3d import SemOperator3D  # noqa: E402

DFMA_PEAK_TF = 34.4      # measured FP64 FMA peak on this pool's B200 (profiles/r1_membench_ceilings.jsonl)
HBM_GBS = 6550.7         # MEASURED_PEAKS.json hbm_gbs


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3      # us


def main():
    res = {"workload": "3D periodic Burgers box on [-2,2]^3, nu=0.01, u ~ U(-1,1), v, w ~ N(0,1)"}
    for N, E in ((7, 32), (8, 28)):
        grid = grid_3d((-2.0, 2.0), E, N)
        op = SemOperator3D(grid, PdeCoefficients(0.01), device="cuda:0")
        rng = np.random.default_rng(N)
        u = torch.from_numpy(rng.uniform(-1, 1, grid.nglobal)).cuda()
        v = torch.from_numpy(rng.standard_normal(grid.nglobal)).cuda()
        w = torch.from_numpy(rng.standard_normal(grid.nglobal)).cuda()
        o = op.empty()
        n = N + 1
        nel = grid.nelem
        t = {"F": timed(lambda: op.launch_rhs(u, o)), "J": timed(lambda: op.launch_jac(u, v, o)),
             "JT": timed(lambda: op.launch_jact(u, w, o))}
        assert op.flags() == 0
        flops = {"F": 18 * 2 * n ** 4 * nel, "J": 27 * 2 * n ** 4 * nel, "JT": 27 * 2 * n ** 4 * nel}
        byts = {"F": 2 * 8 * grid.nglobal, "J": 3 * 8 * grid.nglobal, "JT": 3 * 8 * grid.nglobal}
        res[f"N{N}"] = {
            "E_per_axis": E, "dof": grid.nglobal, "elements": nel,
            "us": {k: round(x, 1) for k, x in t.items()},
            "dof_per_s": {k: grid.nglobal / (x * 1e-6) for k, x in t.items()},
            "fp64_tflops": {k: flops[k] / (t[k] * 1e-6) / 1e12 for k in t},
            "fp64_frac_of_dfma_peak": {k: flops[k] / (t[k] * 1e-6) / 1e12 / DFMA_PEAK_TF for k in t},
            "algorithmic_hbm_gbs": {k: byts[k] / (t[k] * 1e-6) / 1e9 for k in t},
        }
        del op, u, v, w, o
        torch.cuda.empty_cache()
    # CPU: the reference algorithm (numpy, all host threads) on E = 8 per axis
    from oracle import semref as R
    for N in (7, 8):
        m = R.Mesh3D([(-2.0, 2.0)] * 3, [8, 8, 8], N)
        orc = R.BurgersOracle3D(m, 0.01)
        rng = np.random.default_rng(N)
        u, v, w = rng.uniform(-1, 1, m.ndof), rng.standard_normal(m.ndof), rng.standard_normal(m.ndof)
        best = {}
        for k, fn in (("F", lambda: orc.rhs(u)), ("J", lambda: orc.jac(u, v)), ("JT", lambda: orc.jact(u, w))):
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            best[k] = min(ts)
        res[f"cpu_N{N}"] = {"sample": f"E=8 per axis, N={N} ({m.ndof} DOF), min of 3", "threads": os.cpu_count(),
                            "dof_per_s": {k: m.ndof / x for k, x in best.items()}}
        res[f"speedup_N{N}"] = {k: res[f"N{N}"]["dof_per_s"][k] / res[f"cpu_N{N}"]["dof_per_s"][k] for k in best}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
