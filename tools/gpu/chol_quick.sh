# Cholesky A/B: bitwise tests, then the c1/c3 Cholesky stage with the register kernel and the blocked/legacy ones
python -m pytest -q -x tests/test_gpu_parity.py -k "cholesky or cholqr or scholqr or identity or retry or cond" 2>&1 | tail -2
for env in "" "CQR_CHOL_LEGACY=1"; do
  for w in c1 c3; do
    env $env python bench.py --workload $w --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', '$w', round(d['ms_per_step'],3), 'chol', round(d['stage_ms']['cholesky'],4))"
  done
done
