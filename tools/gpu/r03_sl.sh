for v in base sl8g12 sl8g16; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  for w in c1 c3; do CQR_LIB=$L timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3), d['check']['orth'])" 2>/dev/null || echo "$v $w failed"; done
done
