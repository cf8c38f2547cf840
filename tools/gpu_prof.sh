# ncu launch list + one full capture of k_fused for BENCH_ARGS; outputs tagged by TAG.
mkdir -p gpurun_out
TAG=${TAG:-prof}
CMD="python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/${TAG}_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo ncu=$?
tail -2 gpurun_out/${TAG}_ncu_full.log
