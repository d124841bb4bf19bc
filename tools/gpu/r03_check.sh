# full GPU suite + c1/c2 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt_check.log 2>&1; tail -2 gpurun_out/pt_check.log
python bench.py --no-cpu > gpurun_out/bench_check_c1.json 2> gpurun_out/bench_check_c1.err
python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_check_c2.json 2> gpurun_out/bench_check_c2.err
python -c "
import json
for w in ('c1','c2'):
    d = json.load(open('gpurun_out/bench_check_%s.json' % w)); print(w, round(d['ms_per_step'], 3), round(d['value'], 2), {k: round(v, 3) for k, v in d['stage_ms'].items()})
"
