# Parity subset + bench sweep over tuning-variant libraries.
#   K="pytest -k expr"  VARIANTS="default f32minb6 ..."  BENCHES="--dtype f32;--config c2"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
IFS=';' read -ra BL <<< "${BENCHES:---dtype f32}"
for v in ${VARIANTS:-default}; do
  lib=""; [ "$v" != default ] && lib=paper_1909_13772_b200/_lbm_b200_$v.so
  for b in "${BL[@]}"; do
    tag=$(echo "$v$b" | tr -d ' -')
    LBM_B200_LIB=$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $b > gpurun_out/bench_$tag.log 2>&1
    echo "$v [$b]" $(python -c "import json;d=json.loads(open('gpurun_out/bench_$tag.log').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['dtype'])" 2>&1 | tail -1)
  done
done
