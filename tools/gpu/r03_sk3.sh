for v in s4pf16 s4pf0 s2pf0 s2pf24; do
  L=tools/gpu/libcqr_$v.so
  for w in c1 c3; do CQR_LIB=$L python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3))"; done
done
