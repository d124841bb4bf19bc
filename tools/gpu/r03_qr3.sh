timeout 800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_acceptance.py -q -x -k "qr or config or c1 or c2" 2>&1 | tail -2
timeout 300 python bench.py --workload c2 --steps 4 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['stage_ms'].items()}, d['check'])"
