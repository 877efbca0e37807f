"""Summarise ncu captures into profiles/ (text + JSON), read here without a GPU.

  python tools/ncu_summary.py full <report.ncu-rep> <out.txt>
  python tools/ncu_summary.py launches <launches.csv> <out.txt> [traffic.json]
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_write_MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak", 1),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct", 1),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct", 1),
    # FP64 tensor core (DMMA) issue utilisation; it shares the FP64 datapath with DFMA
    # (tools/fp64_pipes.cu), so dmma_pipe_pct + fp64_pipe_pct is the datapath's busy share
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_pipe_pct", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem_B", 1),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_pipe_pct", 1),
]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "math_pipe_throttle", "wait",
          "mio_throttle", "branch_resolving", "no_instructions", "selected", "not_selected",
          "dispatch_stall", "lg_throttle", "membar", "sleeping"]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    lines = [f"# ncu --set full summary of {rep}", ""]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        lines.append(f"## {name[:110]}")
        for m, label, _ in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"  {label:18s} {r[i]} {units[i]}")
        tot = 0
        st = {}
        for s in STALLS:
            k = "smsp__pcsamp_warps_issue_stalled_" + s
            if k in hdr:
                st[s] = int(float(r[hdr.index(k)].replace(",", "") or 0))
                tot += st[s]
        if tot:
            top = sorted(st.items(), key=lambda x: -x[1])[:6]
            lines.append("  stalls(sampled)   " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
        lines.append("")
    open(out, "w").write("\n".join(lines))
    print("\n".join(lines))


def launches(path, out, traffic=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    k = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        key = (int(r[hdr["ID"]]), r[hdr["Kernel Name"]])
        k.setdefault(key, {})[r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
    lines = [f"# ncu launch list ({path}); cold-cache, serialised: compare shares, not absolutes", "",
             f"{'id':>4} {'us':>9} {'read MB':>9} {'write MB':>9}  kernel"]
    tot = sum(m.get("gpu__time_duration.sum", 0) for m in k.values())
    per = {}
    for (i, n), m in k.items():
        t = m.get("gpu__time_duration.sum", 0) / 1e3
        lines.append(f"{i:>4} {t:9.1f} {m.get('dram__bytes_read.sum', 0) / 1e6:9.1f} "
                     f"{m.get('dram__bytes_write.sum', 0) / 1e6:9.1f}  {n[:90]}")
        if "apply" in n:
            op = {"0": "rhs", "1": "jac", "2": "jact"}.get(n.split("<")[1].split(",")[1].strip()[-1:], None) \
                if "<" in n else None
            if op:
                per.setdefault(op, []).append((t, m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)))
    lines.append("")
    lines.append(f"total {tot / 1e3:.1f} us")
    open(out, "w").write("\n".join(lines))
    print("\n".join(lines))
    if traffic:
        # the bench's config-2 launches only (the small sweep-size launches of the same
        # kernels are a fraction of the longest one)
        res = {}
        for op, v in per.items():
            big = [b for t, b in v if t >= 0.5 * max(t for t, _ in v)]
            res[op] = sum(big) / len(big)
        json.dump(res, open(traffic, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3])
    else:
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
