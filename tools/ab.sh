#!/bin/bash
# A/B of run-time kernel selections on one box (under gpurun, from the repo root):
#   bash tools/ab.sh "CFG DT" "ENV1" "ENV2" ...    e.g. "c4 f64" "LBM_B200_ZM=0" ""
# Each variant runs the device-resident bench only (no e2e / CPU leg), twice,
# interleaved, so box drift shows up as spread.  Lines go to gpurun_out/ab.log.
set -u
mkdir -p gpurun_out
spec=$1; shift
read cfg dt <<< "$spec"
for rep in 1 2; do
  for v in "$@"; do
    line=$(env $v timeout 600 python bench.py --config $cfg --dtype $dt --steps ${AB_STEPS:-60} --warmup 5 \
           --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
    python - "$cfg $dt [$v] rep$rep" "$line" <<'PY' | tee -a gpurun_out/ab.log
import json, sys
tag, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    c = d.get("clocks", {})
    print(f"{tag:48s} {d['value']:9.1f} MLUPS frac {d['roofline']['frac']:.4f} "
          f"{d['ms_per_step']:.4f} ms  sm {c.get('sm_mhz')} {','.join(c.get('reasons', []))}")
except Exception as e:
    print(f"{tag:48s} FAILED {line[:200]}")
PY
  done
done
