"""PCIe H2D / D2H / duplex rates with pinned buffers first-touched from (a) the default
CPU set and (b) the GPU's local CPUs (NVML affinity).  Diagnostic only."""
import json
import os
import sys

import torch


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


def rates(n):
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty_like(d)
    hu = torch.empty(n, dtype=torch.float64).pin_memory()
    hu.fill_(1.0)
    ho = torch.empty(n, dtype=torch.float64).pin_memory()
    ho.fill_(0.0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def duplex():
        with torch.cuda.stream(s1):
            d.copy_(hu, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    # duplex with per-direction timing
    ea = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def duplex_split():
        torch.cuda.synchronize()
        ea[0].record(s1)
        with torch.cuda.stream(s1):
            d.copy_(hu, non_blocking=True)
        ea[1].record(s1)
        ea[2].record(s2)
        with torch.cuda.stream(s2):
            ho.copy_(d2, non_blocking=True)
        ea[3].record(s2)
        torch.cuda.synchronize()
        return ea[0].elapsed_time(ea[1]), ea[2].elapsed_time(ea[3])

    duplex_split()
    h, o = duplex_split()
    b = n * 8 / 1e6
    return {"h2d": b / t_ms(lambda: d.copy_(hu, non_blocking=True)),
            "d2h": b / t_ms(lambda: ho.copy_(d, non_blocking=True)),
            "duplex_each": b / t_ms(duplex), "duplex_h2d_alone_timed": b / h, "duplex_d2h_alone_timed": b / o}


def main():
    import pynvml
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    words = pynvml.nvmlDeviceGetCpuAffinity(hd, 16)
    cpus = [64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1]
    out = {"ncpu": os.cpu_count(), "default_affinity": len(os.sched_getaffinity(0)),
           "gpu_local_cpus": f"{cpus[0]}-{cpus[-1]} ({len(cpus)})" if cpus else None}
    try:
        out["numa_of_gpu"] = open(f"/sys/bus/pci/devices/{pynvml.nvmlDeviceGetPciInfo(hd).busId.lower()[4:] if False else ''}numa_node").read().strip()
    except Exception:
        pass
    n = 29360128
    out["default"] = rates(n)
    if cpus:
        os.sched_setaffinity(0, cpus)
        torch.set_num_threads(min(16, len(cpus)))
        out["gpu_local"] = rates(n)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
