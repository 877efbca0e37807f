"""Duplex PCIe rates for the streamer's copy pattern (24 x 29.4 MB each way), without
kernels or cross-stream dependencies, vs one large copy each way.  Diagnostic only."""
import json

import torch


def main():
    n = 29360128 // 8 + 1000      # ~ one chunk's field (config 2, 8 chunks)
    k = 24
    hin = [torch.empty(n * 8, dtype=torch.float64).pin_memory().fill_(1.0) for _ in range(3)]
    hout = [torch.empty(n * 8, dtype=torch.float64).pin_memory().fill_(0.0) for _ in range(3)]
    din = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    dout = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for label, sizes, distinct in (("warmup", n, False), ("same_src", n, False), ("distinct_src", n, True),
                                   ("same_src_again", n, False), ("distinct_src_again", n, True)):
        for mode in ("both",):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            reps = k * n // sizes
            torch.cuda.synchronize()
            ev[0].record(s1)
            ev[2].record(s2)
            for i in range(reps):
                if mode != "d2h_only":
                    with torch.cuda.stream(s1):
                        jj = (i // 3) % 8 if distinct else 0
                        din[i % 3][:sizes].copy_(hin[i % 3][jj * n:jj * n + sizes], non_blocking=True)
                if mode != "h2d_only":
                    with torch.cuda.stream(s2):
                        j = (i // 3) % 8
                        hout[i % 3][j * n:j * n + sizes].copy_(dout[i % 3][:sizes], non_blocking=True)
            ev[1].record(s1)
            ev[3].record(s2)
            torch.cuda.synchronize()
            b = reps * sizes * 8 / 1e6
            res[f"{label}_{mode}"] = {"h2d_GBs": round(b / ev[0].elapsed_time(ev[1]), 1) if mode != "d2h_only" else None,
                                      "d2h_GBs": round(b / ev[2].elapsed_time(ev[3]), 1) if mode != "h2d_only" else None}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
