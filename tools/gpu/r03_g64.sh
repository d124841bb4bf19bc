timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gram" > gpurun_out/pt_g64.log 2>&1; tail -2 gpurun_out/pt_g64.log
for v in new old; do
  if [ $v = old ]; then export CQR_GRAM_NO64=1; fi
  python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c3', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['stage_ms'].items()})"
done
