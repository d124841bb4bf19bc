for v in base c4as3; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  for w in c2 c4; do CQR_LIB=$L timeout 200 python bench.py --workload $w --steps 4 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3))" 2>/dev/null || echo "$v $w failed"; done
done
for w in c1 c3; do timeout 120 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('base', '$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3), d['check'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "sketch or config or gaussian" 2>&1 | tail -2
