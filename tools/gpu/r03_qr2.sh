timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "qr or config" 2>&1 | tail -2
timeout 300 python bench.py --workload c2 --steps 4 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['stage_ms'].items()})"
python tools/prof_one.py c2 > /dev/null 2>&1 && ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"qr_blocked" -s 2 -c 1 -o gpurun_out/qr_c2b python tools/prof_one.py c2 > gpurun_out/ncu_qr2.log 2>&1; tail -1 gpurun_out/ncu_qr2.log
