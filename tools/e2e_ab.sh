# e2e (run_arrays wavefront) schedule A/B at the driver's K = 20: bash tools/e2e_ab.sh
# each line: LBM_B200_JOB_RAMP / LBM_B200_JOB_TAIL / LBM_B200_JOB_CHUNK, device value, e2e
run() {  # ramp tail chunk
  LBM_B200_JOB_RAMP="$1" LBM_B200_JOB_TAIL=$2 LBM_B200_JOB_CHUNK=$3 timeout 600 python bench.py \
      --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('ramp=$1 tail=$2 chunk=$3', d['value'], d['e2e']['value'], d['e2e']['seconds'])"
}
for rep in 1 2; do
  run "" 0 32
  run "4,4,8,16" 4 32
  run "2,2,4,8,16" 2 32
  run "4,4,8,16" 8 32
  run "4,4,8,16,32" 4 64
done
