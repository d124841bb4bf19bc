for v in base nosl sl20; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  for w in c2 c4; do CQR_LIB=$L timeout 300 python bench.py --workload $w --steps 4 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3))" 2>/dev/null || echo "$v $w failed"; done
done
