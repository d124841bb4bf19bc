for v in base ch64 ch16; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  CQR_LIB=$L python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c3', round(d['ms_per_step'],3), round(d['stage_ms']['gram'],3))"
done
