timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "trisolve" 2>&1 | tail -2
CQR_TRISOLVE_VARIANT=2 CQR_TRISOLVE_NO_PANELS=1 python tools/tri_ab.py 1000000 512
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 512
timeout 300 python bench.py --workload c4 --steps 4 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['stage_ms'].items()})"
