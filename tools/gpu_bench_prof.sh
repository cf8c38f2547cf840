mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log
bash tools/gpu_prof.sh
