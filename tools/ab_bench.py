"""A/B timing of F, J, J^T on config 2 for one library build (SEM1D_LIB=...)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import configs  # noqa: E402


def main(cfg="2", reps=20):
    from paper_1806_01422_b200 import _lib
    path = int(os.environ.get("SEM1D_PATH", "0"))   # 0 auto (DMMA), 1 DFMA/TMA, 2 plain
    _lib.load().sem1d_set_kernel_path(path)
    c = {"2": configs.CFG2, "3": configs.CFG3}[cfg]
    op = configs.cfg_operator(c, device="cuda:0")
    u, v, w = configs.operator_inputs(op.ndof, c["seed"])
    ud, vd, wd = (torch.from_numpy(a).cuda() for a in (u, v, w))
    o = op.empty()
    res = {}
    for name, fn in (("F", lambda: op.launch_rhs(ud, o)), ("J", lambda: op.launch_jac(ud, vd, o)),
                     ("JT", lambda: op.launch_jact(ud, wd, o))):
        for _ in range(3):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(int(reps)):
            fn()
        e.record()
        torch.cuda.synchronize()
        res[name] = round(1e3 * s.elapsed_time(e) / int(reps), 2)
    assert op.flags() == 0
    print(json.dumps({"lib": os.path.basename(os.environ.get("SEM1D_LIB", "default")), "cfg": cfg,
                      "path": {0: "dmma-ws", 1: "dfma-tma", 2: "plain-dfma"}[path], "us": res}))


if __name__ == "__main__":
    main(*sys.argv[1:])
