mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "config0 or config1 or golden or rank_invariance_bitwise" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for zc in ${ZCS:-0 8 16 32}; do
  LBM_ZCHUNK=$zc timeout 600 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_zc$zc.log 2>&1
  echo zc=$zc $(python -c "import json;d=json.loads(open('gpurun_out/bench_zc$zc.log').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'])")
done
