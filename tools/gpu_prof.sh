mkdir -p gpurun_out
CMD="python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/prof_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
tail -3 gpurun_out/ncu_full.log
