#!/usr/bin/env python
"""Summarise an ncu capture of the fused kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv \
        profiles/ncu_c4_f64  --cells 134217728 --bytes-per-cell 304

Writes <stem>.json (the numbers bench.py reads: dram bytes per launch, ...)
and <stem>.txt (human-readable: SOL, occupancy, stall reasons, launch list
shares).
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "sm__cycles_elapsed.avg",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            d[h] = (r[i], units[i])
        launches.append(d)
    return launches


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}.get(unit, 1)
    x = num(v)
    return None if x is None else x * f


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launches")
    ap.add_argument("stem")
    ap.add_argument("--cells", type=float, required=True)
    ap.add_argument("--bytes-per-cell", type=float, required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    L = raw(a.rep)[0]
    name = L.get("Kernel Name", ("?", ""))[0]
    m = {k: L[k] for k in KEYS if k in L}
    t = scale(*m["gpu__time_duration.sum"])
    rd = scale(*m["dram__bytes_read.sum"])
    wr = scale(*m["dram__bytes_write.sum"])
    alg = a.cells * a.bytes_per_cell
    summary = {
        "kernel": name, "note": a.note,
        "duration_ms": t * 1e3, "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": alg,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "dram_bytes_per_cell": (rd + wr) / a.cells,
        "achieved_dram_GBps": (rd + wr) / t / 1e9, "algorithmic_GBps": alg / t / 1e9,
        "metrics": {k: f"{v[0]} {v[1]}".strip() for k, v in m.items()},
    }
    stalls = {k: num(v[0]) for k, v in L.items()
              if k.startswith("smsp__average_warps_issue_stalled") and k.endswith(".ratio")}
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", ""): v for k, v in stalls.items() if v and v > 0.05}
    summary["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    # launch list shares
    shares = defaultdict(float)
    total = 0.0
    with open(a.launches) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    if rows:
        hdr = rows[0]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        for r in rows[1:]:
            d = scale(r[vi], r[ui]) or 0.0
            shares[r[ki].split("(")[0]] += d
            total += d
    summary["launch_list"] = {k: {"total_ms": v * 1e3, "share": v / total}
                              for k, v in sorted(shares.items(), key=lambda kv: -kv[1])}
    with open(a.stem + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    with open(a.stem + ".txt", "w") as fh:
        fh.write(f"{name}\n{a.note}\n")
        fh.write(f"duration {t*1e3:.3f} ms; DRAM read {rd/1e9:.2f} GB write {wr/1e9:.2f} GB "
                 f"-> {(rd+wr)/a.cells:.1f} B/cell (algorithmic {a.bytes_per_cell:.0f}); "
                 f"{(rd+wr)/t/1e9:.0f} GB/s DRAM, {alg/t/1e9:.0f} GB/s algorithmic\n")
        for k, v in m.items():
            fh.write(f"  {k:70s} {v[0]} {v[1]}\n")
        fh.write("stalls per issued instruction:\n")
        for k, v in summary["stalls_per_issue"].items():
            fh.write(f"  {k:40s} {v:.3f}\n")
        fh.write("launch list (cold-cache, serialised; shares):\n")
        for k, v in summary["launch_list"].items():
            fh.write(f"  {k:60s} {v['total_ms']:10.3f} ms  {100*v['share']:5.1f} %\n")
    print(open(a.stem + ".txt").read())


if __name__ == "__main__":
    main()
