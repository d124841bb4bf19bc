for v in base qrt256 qrt1024; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  CQR_LIB=$L timeout 300 python bench.py --workload c2 --steps 4 --warmup 2 --no-cpu --no-compare 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c2', round(d['ms_per_step'],3), round(d['stage_ms']['precondition'],3), d['check']['orth'])" 2>/dev/null || echo "$v failed"
done
