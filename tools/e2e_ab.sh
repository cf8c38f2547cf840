for rep in 1 2; do for c in 8 16 32 64; do
  LBM_B200_JOB_CHUNK=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk $c', d['value'], d['e2e']['value'], d['e2e']['seconds'])"
done; done
