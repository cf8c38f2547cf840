# ncu summary of the fused kernel at 128^3 (config 1), summarised on the box
mkdir -p gpurun_out
CMD="python bench.py --config c1 --profile --steps 3 --warmup 4 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/c1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -o gpurun_out/c1_f64 $CMD > gpurun_out/c1_ncu.log 2>&1
echo ncu=$?
python tools/ncu_summary.py gpurun_out/c1_f64.ncu-rep gpurun_out/c1_launches.csv gpurun_out/ncu_c1_f64 --cells 2097152 --bytes-per-cell 304 --note "round 1 final: config 1 fp64 128^3 (25 % spheres), k_fused" > /dev/null 2>&1; echo sum=$?
rm -f gpurun_out/c1_f64.ncu-rep
