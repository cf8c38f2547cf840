# A/B of library variants (LBM_B200_LIB) across configs, variants interleaved
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "config1 or golden or rank_invariance or fused_peer" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-"--config c4" "--config c4 --dtype f32" "--config c2"}; do
 for rep in ${REPS:-1}; do
  for v in ${VARIANTS:-default}; do
    unset LBM_B200_LIB LBM_B200_FUSED LBM_B200_VEC
    case "$v" in
      default) ;;
      fused=*) export LBM_B200_FUSED=${v#fused=} ;;
      vec=*) export LBM_B200_VEC=${v#vec=} ;;
      vec+*) export LBM_B200_VEC=1 LBM_B200_LIB=$PWD/paper_1909_13772_b200/_lbm_b200_${v#vec+}.so ;;
      *) export LBM_B200_LIB=$PWD/paper_1909_13772_b200/_lbm_b200_$v.so ;;
    esac
    tag=$(echo "$cfg" | tr -d ' -')_$(echo $v | tr -d '=')
    timeout 600 python bench.py --steps ${STEPS:-40} --warmup 5 --no-e2e --no-cpu-baseline $cfg > gpurun_out/ab_$tag.log 2>&1
    echo "$cfg" v=$v $(python -c "import json;d=json.loads(open('gpurun_out/ab_$tag.log').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)
  done
 done
done
