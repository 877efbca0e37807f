"""Per-launch fixed cost of the apply kernels, free of host launch overhead: 20 launches
captured in a CUDA graph and replayed, at ring sizes of 1, 2, 4, 8 and 13.84 tiles per SM
(config 3, N = 31, or config 2, N = 7).  time(E) = fixed + slope * E separates the
prologue / pipeline fill / drain / last-wave cost from the steady state.
  python tools/launch_overhead.py [3|2]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import configs  # noqa: E402


def graph_time(fn, reps=20, iters=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, 1e3 * a.elapsed_time(b) / reps)
    return best


def main(cfg="3"):
    base = {"2": configs.CFG2, "3": configs.CFG3}[cfg]
    per_tile = 128 if cfg == "3" else 256
    rows = []
    for E in (148 * per_tile, 2 * 148 * per_tile, 4 * 148 * per_tile, 8 * 148 * per_tile, base["E"]):
        c = dict(base, E=E)
        op = configs.cfg_operator(c, device="cuda:0")
        u, v, w = configs.operator_inputs(op.ndof, c["seed"])
        ud, vd, wd = (torch.from_numpy(a).cuda() for a in (u, v, w))
        o = op.empty()
        t = {"F": graph_time(lambda: op.launch_rhs(ud, o)), "J": graph_time(lambda: op.launch_jac(ud, vd, o)),
             "JT": graph_time(lambda: op.launch_jact(ud, wd, o))}
        assert op.flags() == 0
        rows.append({"E": E, "us": {k: round(x, 2) for k, x in t.items()}})
        print(json.dumps(rows[-1]), flush=True)
        del ud, vd, wd, o, op
        torch.cuda.empty_cache()
    # least-squares fixed + slope over the sizes
    import numpy as np
    Es = np.array([r["E"] for r in rows], dtype=float)
    fit = {}
    for k in ("F", "J", "JT"):
        y = np.array([r["us"][k] for r in rows])
        slope, fixed = np.polyfit(Es, y, 1)
        fit[k] = {"fixed_us": round(float(fixed), 2), "us_per_1M_elements": round(float(slope) * 2 ** 20, 2)}
    print(json.dumps({"cfg": cfg, "fit": fit}))


if __name__ == "__main__":
    main(*sys.argv[1:])
