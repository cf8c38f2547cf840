#!/bin/bash
# One launcher for the GPU-box measurements (run under gpurun from the repo root):
#
#   bash tools/gpu.sh test                  pytest -m gpu (+ smoke), logs in gpurun_out/
#   bash tools/gpu.sh bench CFG DT [K]      bench.py line for one config / dtype
#   bash tools/gpu.sh prof CFG DT TAG       launch list + one ncu --set full capture of
#                                           k_fused, summarised to gpurun_out/ncu_TAG.*
#   bash tools/gpu.sh final                 every bench config, the reference arm and the
#                                           profiles of the headline kernels
# Outputs go to gpurun_out/ (merged back by gpurun); copy what is judged to profiles/.
set -u
mkdir -p gpurun_out
cells_of() { case $1 in c4|c3) echo 134217728;; c1) echo 2097152;; c2) echo 16777216;; c0) echo 262144;; esac; }
bpc_of() { case "$1 $2" in "c2 f32") echo 216;; "c2 f64") echo 432;; *" f32") echo 152;; *) echo 304;; esac; }

bench() {   # cfg dtype steps
  timeout 900 python bench.py --config $1 --dtype $2 --steps ${3:-100} --warmup 5 \
      > gpurun_out/bench_$1_$2.log 2>&1; echo bench_$1_$2=$?
  tail -1 gpurun_out/bench_$1_$2.log | cut -c1-400
}

prof() {    # cfg dtype tag
  local CMD="python bench.py --config $1 --dtype $2 --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/$3_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/$3_plain.log; return 1; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$3.csv $CMD > /dev/null 2>&1; echo launches=$?
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 \
      -o gpurun_out/$3 $CMD > gpurun_out/$3_ncu.log 2>&1; echo ncu=$?
  python tools/ncu_summary.py gpurun_out/$3.ncu-rep gpurun_out/launches_$3.csv gpurun_out/ncu_$3 \
      --cells $(cells_of $1) --bytes-per-cell $(bpc_of $1 $2) --note "round 2: $1 $2" > /dev/null 2>&1
  echo summary=$?
  ncu -i gpurun_out/$3.ncu-rep --page source --csv > gpurun_out/$3_source.csv 2>/dev/null
  rm -f gpurun_out/$3.ncu-rep
}

case ${1:-test} in
  test)
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
    timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1
    echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log ;;
  bench) bench $2 $3 ${4:-100} ;;
  prof) prof $2 $3 $4 ;;
  final)
    timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_default=$?
    tail -1 gpurun_out/bench_default.log | cut -c1-400
    for spec in "c4 f32" "c3 f64" "c1 f64" "c2 f32" "c0 f64"; do bench $spec 100; done
    timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
    echo reference=$?
    for spec in "c4 f64 c4_f64" "c4 f32 c4_f32" "c2 f32 c2_f32" "c3 f64 c3_f64"; do prof $spec; done
    du -sh gpurun_out ;;
  *) echo "usage: tools/gpu.sh test|bench CFG DT [K]|prof CFG DT TAG|final"; exit 2 ;;
esac
