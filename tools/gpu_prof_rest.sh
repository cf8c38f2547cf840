# ncu summaries + executed SASS mixes of the fp32 config-4, config-2 and the
# default config-4 fp64 fused kernels (summarised on the box; reports deleted)
mkdir -p gpurun_out
run() {  # tag bench-args cells bytes note
  CMD="python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $2"
  $CMD > gpurun_out/$1_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$1_launches.csv $CMD > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/$1 $CMD > gpurun_out/$1_ncu.log 2>&1
  echo $1 ncu=$?
  python tools/ncu_summary.py gpurun_out/$1.ncu-rep gpurun_out/$1_launches.csv gpurun_out/ncu_$1 --cells $3 --bytes-per-cell $4 --note "$5" > /dev/null 2>&1
  python tools/sass_exec.py gpurun_out/$1.ncu-rep --cells $3 > gpurun_out/sass_mix_$1.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
run c4_f32 "--config c4 --dtype f32" 134217728 152 "round 1 final: config 4 fp32 storage"
run c2_f32 "--config c2" 16777216 216 "round 1 final: config 2 D3Q27 raw-moment MRT fp32"
run c4_f64 "--config c4" 134217728 304 "round 1 final: config 4 fp64 (keep-in-L2 link hint)"
du -sh gpurun_out
