for w in c1 c2 c3 c4; do CQR_DEBUG_PLAN=1 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu --no-compare 2>gpurun_out/sk8_$w.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), 'sketch', round(d['stage_ms']['sketch'],3), d['check'])"; grep -m1 sketch_i8_plan gpurun_out/sk8_$w.err; done
