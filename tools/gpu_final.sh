# Round-end measurement: smoke, GPU parity suite, every bench config, the
# reference arm, and the ncu launch list + one full capture of the default
# (config 4 fp64) and config 3 fused kernels.  Outputs in gpurun_out/final_*.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/final_pytest.log
timeout 900 python bench.py > gpurun_out/final_bench_c4_f64.log 2>&1; echo bench_default=$?
tail -1 gpurun_out/final_bench_c4_f64.log | cut -c1-300
for spec in "c4 f32" "c3 f64" "c1 f64" "c2 f32" "c0 f64"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --dtype $2 --steps 100 --warmup 5 > gpurun_out/final_bench_$1_$2.log 2>&1; echo bench_$1_$2=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_reference.log 2>&1; echo ref=$?
[ -n "$BENCH_ONLY" ] && exit 0
CMD="python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/final_plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c4_f64.csv $CMD > /dev/null 2>&1; echo launches=$?
$CMD > gpurun_out/final_plain_c4b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/final_c4_f64 $CMD > gpurun_out/final_ncu_c4.log 2>&1; echo ncu_c4=$?
CMD3="python bench.py --config c3 --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD3 > gpurun_out/final_plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/final_c3_f64 $CMD3 > gpurun_out/final_ncu_c3.log 2>&1; echo ncu_c3=$?
# summarise on the box (a full report is ~60 MB; gpurun copies back <= 64 MiB)
python tools/ncu_summary.py gpurun_out/final_c4_f64.ncu-rep gpurun_out/final_launches_c4_f64.csv \
    gpurun_out/ncu_c4_f64 --cells 134217728 --bytes-per-cell 304 \
    --note "round 1 final: config 4 fp64, k_fused (LDG), bitwise" > /dev/null 2>&1; echo sum_c4=$?
ncu -i gpurun_out/final_c4_f64.ncu-rep --page source --csv > gpurun_out/final_c4_f64_source.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/final_c3_f64.ncu-rep gpurun_out/final_launches_c4_f64.csv \
    gpurun_out/ncu_c3_f64 --cells 134217728 --bytes-per-cell 304 \
    --note "round 1 final: config 3 fp64 (periodic, NULL cell mask), k_fused" > /dev/null 2>&1; echo sum_c3=$?
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
