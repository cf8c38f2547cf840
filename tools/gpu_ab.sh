mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "config1 or golden or flat" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset LBM_B200_LIB; else export LBM_B200_LIB=$PWD/paper_1909_13772_b200/_lbm_b200_$v.so; fi
  timeout 600 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$v.log 2>&1
  echo v=$v $(python -c "import json;d=json.loads(open('gpurun_out/bench_$v.log').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['ms_per_step'])" 2>&1 | tail -1)
done
