"""FP64 pipe accounting of one ncu --set full capture (read here, no GPU):
DMMA subpipe and FP64 (DFMA/DMUL/DADD) pipe activity, issue, occupancy, DRAM, and the
top stall reasons by SASS opcode.  python tools/ncu_pipes.py <rep.ncu-rep> [kernel-regex]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "sm__cycles_active.avg": "sm_cycles_active",
    "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg": "dmma_subpipe_cycles",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_inst_pct_of_peak",
    "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_cycles_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct_of_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "launch__grid_size": "grid",
}


def main(rep, kregex=None):
    args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kregex:
        args += ["-k", f"regex:{kregex}"]
    rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
    hdr = rows[0]
    out = {}
    for r in rows[2:3]:
        for k, name in KEYS.items():
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                try:
                    out[name] = float(v)
                except ValueError:
                    out[name] = v
    if "dmma_subpipe_cycles" in out and "sm_cycles_active" in out:
        out["dmma_subpipe_frac"] = out["dmma_subpipe_cycles"] / out["sm_cycles_active"]
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kregex:
        args += ["-k", f"regex:{kregex}"]
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
    ops, stalls, ins = collections.Counter(), collections.defaultdict(collections.Counter), collections.Counter()
    cols = [h for h in hdr if h.startswith("stall_") and "Not" not in h] if hdr else []
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
    out["stall_by_opcode"] = {op: {"pct": round(100 * s / tot, 1),
                                   "top": {k: round(100 * v / tot, 1) for k, v in stalls[op].most_common(3)}}
                              for op, s in ops.most_common(10)}
    out["inst_executed"] = dict(ins.most_common(14))
    for k, v in out.items():
        print(f"{k:24s} {v}")


if __name__ == "__main__":
    main(*sys.argv[1:])
