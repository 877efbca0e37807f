"""Slot / chunk-count sweep of SemOperator.apply_host on config 2, plus raw PCIe H2D / D2H / duplex."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import configs  # noqa: E402


def t_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    c = configs.CFG2
    op = configs.cfg_operator(c, device="cuda:0")
    u, v, w = configs.operator_inputs(op.ndof, c["seed"])
    uh, vh, wh = (torch.from_numpy(a).pin_memory() for a in (u, v, w))
    d = torch.empty(op.ndof, dtype=torch.float64, device="cuda")
    h = torch.empty(op.ndof, dtype=torch.float64).pin_memory()
    res = {"h2d_GBs": op.ndof * 8 / t_ms(lambda: d.copy_(uh, non_blocking=True)) / 1e6,
           "d2h_GBs": op.ndof * 8 / t_ms(lambda: h.copy_(d, non_blocking=True)) / 1e6}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    d2 = torch.empty_like(d)

    def duplex():
        with torch.cuda.stream(s1):
            d.copy_(uh, non_blocking=True)
        with torch.cuda.stream(s2):
            h.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    res["duplex_GBs_each_way"] = op.ndof * 8 / t_ms(duplex) / 1e6
    outs = {k: torch.empty(op.ndof, dtype=torch.float64).pin_memory() for k in ("rhs", "jac", "jact")}
    for sl in (2, 3):
        for ch in (4, 6, 8, 12):
            ms = t_ms(lambda: op.apply_host(uh, vh, wh, chunks=ch, slots=sl, out=outs), reps=3)
            res[f"apply_host_slots{sl}_chunks{ch}_ms"] = ms
    ms = t_ms(lambda: op.apply_host(uh, vh, wh), reps=3)
    res["apply_host_default_fresh_outputs_ms"] = ms
    print(json.dumps(res))


if __name__ == "__main__":
    main()
