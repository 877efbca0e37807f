"""Opcode mix and stall samples per SASS opcode from `ncu -i R --page source --csv --print-source sass`."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    cnt, st = collections.Counter(), collections.Counter()
    hdr = None
    for r in rows:
        if "Source" in r and "Instructions Executed" in r:
            hdr = r
            i_src, i_ex = r.index("Source"), r.index("Instructions Executed")
            i_s = r.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) <= i_ex or not r[i_ex].isdigit():
            continue
        op = r[i_src].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        cnt[o.split(".")[0]] += int(r[i_ex])
        st[o.split(".")[0]] += int(r[i_s] or 0)
    tot, stot = sum(cnt.values()), max(1, sum(st.values()))
    print("total warp instructions", tot)
    for o, n in cnt.most_common(top):
        print(f"{o:10s} {n:12d} {100 * n / tot:5.1f}%  stall samples {100 * st[o] / stot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
