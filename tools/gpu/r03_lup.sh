timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "lu or config or singular" 2>&1 | tail -3
for v in new old; do
  if [ $v = old ]; then export CQR_LU_NO_PERSIST=1; fi
  timeout 300 python bench.py --workload c4 --steps 5 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c4', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['stage_ms'].items()})"
done
