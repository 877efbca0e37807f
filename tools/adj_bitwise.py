"""Save / compare SHA-256 digests of the register-resident step kernels' outputs (N = 7) on
a few rings, for bitwise A/B of kernel restructurings that must not change results.
  python tools/adj_bitwise.py save|check <file.json>"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import configs  # noqa: E402


def digest(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()


def outputs():
    res = {}
    for E in (65536, 70001):
        op = configs.cfg_operator(dict(configs.CFG2, E=E), device="cuda:0")
        x = torch.linspace(0, 50, op.ndof, dtype=torch.float64, device="cuda")
        u = torch.sin(x) + 0.1 * torch.cos(7 * x)
        lam = torch.cos(x) + 0.2 * torch.sin(3 * x)
        dt = 1e-3 * 2.0 / E
        slot = op.flag_slots(1)
        for scheme in ("rk4", "rk3", "euler"):
            o = op.empty()
            st = [op.empty() for _ in range(3)]
            op.launch_rk_step(u, o, dt, scheme)
            res[f"fwd_{E}_{scheme}"] = digest(o)
            op.launch_rk_step(u, o, dt, scheme, flag=slot.data_ptr())
            res[f"fwdfast_{E}_{scheme}"] = digest(o)
            for check in (True, False):
                kw = {} if check else {"flag": slot.data_ptr()}
                op.launch_adj_step(u, lam, o, dt, scheme, **kw)
                res[f"adj_{E}_{scheme}_{check}"] = digest(o)
                if scheme != "euler":
                    op.launch_rk_step_stages(u, o, st, dt, scheme)
                    op.launch_adj_step_stages(u, st, lam, o, dt, scheme, **kw)
                    res[f"adjst_{E}_{scheme}_{check}"] = digest(o)
        assert op.flags() == 0 and int(slot[0]) == 0
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    r = outputs()
    if mode == "save":
        json.dump(r, open(path, "w"), indent=0)
        print("saved", len(r))
    else:
        ref = json.load(open(path))
        bad = [k for k in ref if ref[k] != r.get(k)]
        print("bitwise equal" if not bad else f"DIFFER: {bad}", len(ref))
