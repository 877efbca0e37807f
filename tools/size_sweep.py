"""F / J / J^T time vs ring size (config 2, N = 7, or config 3, N = 31: size_sweep.py 3): separates the fixed per-launch cost
(prologue, last-wave tail) from the steady-state bandwidth.  Also times a plain
torch copy of the same bytes for the ceiling at each size."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import configs  # noqa: E402


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return 1e3 * s.elapsed_time(e) / reps


def main(cfg="2"):
    base = {"2": configs.CFG2, "3": configs.CFG3}[cfg]
    lgs = (18, 19, 20, 21, 22, 23, 24) if cfg == "2" else (15, 16, 17, 18, 19, 20, 21)
    for lg in lgs:
        c = dict(base, E=1 << lg)
        op = configs.cfg_operator(c, device="cuda:0")
        u, v, w = configs.operator_inputs(op.ndof, c["seed"])
        ud, vd, wd = (torch.from_numpy(a).cuda() for a in (u, v, w))
        o = op.empty()
        t = {"F": timed(lambda: op.launch_rhs(ud, o)), "J": timed(lambda: op.launch_jac(ud, vd, o)),
             "JT": timed(lambda: op.launch_jact(ud, wd, o)), "copy": timed(lambda: o.copy_(ud))}
        gbs = {k: (16 if k in ("F", "copy") else 24) * op.ndof / (t[k] * 1e3) for k in t}
        print(json.dumps({"E": 1 << lg, "ndof": op.ndof, "us": {k: round(x, 2) for k, x in t.items()},
                          "GBs": {k: round(x) for k, x in gbs.items()}}), flush=True)
        del ud, vd, wd, o, op
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(*sys.argv[1:])
