"""FP64 pipe accounting of EVERY launch in one ncu --set full capture (read here, no GPU): DMMA
and FP64 pipe shares, issue, occupancy, DRAM bytes, the top stall reasons, and stalls by SASS
opcode per launch.  python tools/ncu_pipes_all.py <rep.ncu-rep> [label ...]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]


def by_opcode(rep, skip):
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(skip),
            "--launch-count", "1"]
    src = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
    hdr, data = None, []
    for r in src:
        if r and r[0] == "Address":
            if hdr is not None:
                break
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(r)
    if not hdr:
        return {}, {}
    cols = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
    ops, stalls, ins = collections.Counter(), collections.defaultdict(collections.Counter), collections.Counter()
    for r in data:
        t = r[1].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ins[op] += int(r[hdr.index("Instructions Executed")] or 0)
        for c in cols:
            v = int(r[hdr.index(c)] or 0)
            stalls[op][c[6:]] += v
            ops[op] += v
    tot = sum(ops.values()) or 1
    return ({op: {"pct": round(100 * s / tot, 1), "top": {k: round(100 * v / tot, 1) for k, v in stalls[op].most_common(3)}}
             for op, s in ops.most_common(8)}, dict(ins.most_common(12)))


def main(rep, *labels):
    rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv",
                                                        "--kernel-name-base", "demangled"],
                                                       capture_output=True, text=True).stdout)))
    hdr = rows[0]
    for n, r in enumerate(rows[2:]):
        name = labels[n] if n < len(labels) else r[hdr.index("Kernel Name")][:70]
        print(f"== launch {n}: {name}")
        for k in KEYS:
            if k in hdr:
                print(f"{k:84s} {r[hdr.index(k)]}")
        st = [(float(r[i].replace(",", "") or 0), h) for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in h]
        tot = sum(v for v, _ in st) or 1
        print("stalls:", ", ".join(f"{h[33:]} {100 * v / tot:.1f}%" for v, h in sorted(st, reverse=True)[:7]))
        so, ins = by_opcode(rep, n)
        print("stall_by_opcode", so)
        print("inst_executed", ins)
        print()


if __name__ == "__main__":
    main(*sys.argv[1:])
