#!/usr/bin/env python
"""Per-kernel SASS instruction counts of the built library (cuobjdump).

    python tools/sass_stats.py [regex]

Prints, for each matching kernel, the number of global loads/stores,
local-memory (spill) accesses and FP64 instructions - the quick check that a
kernel is spill-free and what its instruction mix looks like before spending
GPU time.
"""
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_1909_13772_b200" / "_lbm_b200.so"
OPS = ["LDG", "STG", "LDL", "STL", "LDS", "DADD", "DMUL", "DFMA", "F2F", "IMAD", "BRA", "SHFL"]


def main():
    pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else "k_fused")
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    cur, counts = None, {}
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = {k: 0 for k in OPS}
            counts[cur]["total"] = 0
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(1).split(".")[0]
            counts[cur]["total"] += 1
            if op in counts[cur]:
                counts[cur][op] += 1
    for fn, c in counts.items():
        if pat.search(fn):
            print(fn[:90], " ".join(f"{k}={v}" for k, v in c.items() if v))


if __name__ == "__main__":
    main()
