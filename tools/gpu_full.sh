mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_default.log | cut -c1-400
for extra in "--dtype f32" "--config c1" "--config c3" "--config c2" "--config c0"; do
  tag=$(echo $extra | tr -d ' -')
  timeout 900 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline $extra > gpurun_out/bench_$tag.log 2>&1
  echo $tag $(python -c "import json;d=json.loads(open('gpurun_out/bench_$tag.log').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['dtype'])" 2>&1 | tail -1)
done
