for v in base nocomp; do
  if [ $v = base ]; then L=paper_2111_11148_b200/libcqr.so; else L=tools/gpu/libcqr_$v.so; fi
  for w in c2 c4; do CQR_DEBUG_PLAN=1 CQR_LIB=$L timeout 300 python bench.py --workload $w --steps 4 --warmup 2 --no-cpu --no-compare 2>gpurun_out/comp_$v_$w.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3), d['check'])" 2>/dev/null || echo "$v $w failed"; grep -m1 sketch_i8_plan gpurun_out/comp_$v_$w.err; done
done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -2
