"""Attribute ncu per-SASS samples/instructions to source lines (needs a -lineinfo cubin)."""
import collections
import csv
import re
import subprocess
import sys


def main(rep, cubin_sass, kernel_match, mangled, col="stall"):
    sass = open(cubin_sass).read().split("\n")
    offs, infun, cur = {}, False, None
    for l in sass:
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            infun = m.group(1) == mangled
            continue
        if not infun:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m:
            offs[int(m.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, base, agg, n = None, None, collections.Counter(), 0
    idx = 2 if col == "stall" else 5
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = r[1]
            base = None
            continue
        if not cur or kernel_match not in cur or len(r) < 6 or r[0] == "Address":
            continue
        a = int(r[0], 16)
        base = a if base is None else base
        try:
            v = int(r[idx])
        except ValueError:
            continue
        agg[offs.get(a - base)] += v
        n += v
    src = {}
    for li, c in agg.most_common(30):
        if li is None:
            print(f"{100 * c / n:5.1f}  ?")
            continue
        if li[0] not in src:
            try:
                src[li[0]] = open(f"paper_1806_01422_b200/csrc/{li[0]}").read().split("\n")
            except OSError:
                src[li[0]] = []
        txt = src[li[0]][li[1] - 1].strip()[:90] if len(src[li[0]]) >= li[1] else ""
        print(f"{100 * c / n:5.1f}  {li[0]}:{li[1]}  {txt}")


if __name__ == "__main__":
    main(*sys.argv[1:])
