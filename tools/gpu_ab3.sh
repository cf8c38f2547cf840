# A/B of library variants over a list of configs (CFGLIST entries separated by ';')
mkdir -p gpurun_out
IFS=';' read -ra CL <<< "${CFGLIST:---config c4}"
for rep in ${REPS:-1}; do
 for cfg in "${CL[@]}"; do
  for v in ${VARIANTS:-default}; do
    unset LBM_B200_LIB
    [ "$v" != default ] && export LBM_B200_LIB=$PWD/paper_1909_13772_b200/_lbm_b200_$v.so
    tag=$(echo "$cfg" | tr -d ' -')_${v}_$rep
    timeout 600 python bench.py --steps ${STEPS:-40} --warmup 5 --no-e2e --no-cpu-baseline $cfg > gpurun_out/ab_$tag.log 2>&1
    echo "$cfg" v=$v $(python -c "import json;d=json.loads(open('gpurun_out/ab_$tag.log').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['clocks']['reasons'])" 2>&1 | tail -1)
  done
 done
done
