for v in base t2_8; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  CQR_LIB=$L python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c1', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3))"
done
for v in base t4_8 t4_2; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  for w in c2 c4; do CQR_LIB=$L python bench.py --workload $w --steps 4 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3))"; done
done
