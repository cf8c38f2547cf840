#!/usr/bin/env python
"""Executed-instruction mix of a kernel from an ncu report's source page.

    python tools/sass_exec.py gpurun_out/x.ncu-rep [--cells N] [--top K]
    python tools/sass_exec.py gpurun_out/x_source.csv ...   (an exported source page)

Groups `Instructions Executed` (warp-level) by opcode (first mnemonic
component), prints totals per 32 cells, and the K hottest instructions by
stall samples.
"""
import argparse
import csv
import io
import subprocess
from collections import Counter


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--cells", type=float, default=0)
    ap.add_argument("--top", type=int, default=0)
    a = ap.parse_args()
    if a.rep.endswith(".csv"):
        out = open(a.rep).read()
    else:
        out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    ops, total, hot = Counter(), 0, []
    for r in rows[1:]:
        if len(r) <= ie or not r[ie].isdigit():
            continue
        n = int(r[ie])
        ins = r[src].strip()
        if ins.startswith("@"):
            ins = ins.split(None, 1)[1] if " " in ins else ins
        op = ins.split()[0].split(".")[0] if ins else "?"
        ops[op] += n
        total += n
        hot.append((int(r[st] or 0), n, r[src].strip()))
    warps = a.cells / 32 if a.cells else 0
    print(f"total warp instructions {total:.4g}" + (f" = {total / warps:.1f} per warp of 32 cells" if warps else ""))
    for op, n in ops.most_common():
        print(f"  {op:10s} {n:14d} {100 * n / total:6.2f} %" + (f"  {n / warps:7.2f}/warp" if warps else ""))
    if a.top:
        print("hottest by stall samples:")
        for s, n, ins in sorted(hot, reverse=True)[:a.top]:
            print(f"  {s:8d} {n:12d}  {ins}")


if __name__ == "__main__":
    main()
