# new sketch (in-kernel exponent scan): GPU suite + c1/c3 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt_sk.log 2>&1; tail -5 gpurun_out/pt_sk.log
for w in c1 c3; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-compare > gpurun_out/bench_sk_$w.json 2> gpurun_out/bench_sk_$w.err; done
python -c "
import json
for w in ('c1','c3'):
    d = json.load(open('gpurun_out/bench_sk_%s.json' % w)); print(w, round(d['ms_per_step'], 3), round(d['value'], 2), {k: round(v, 3) for k, v in d['stage_ms'].items()}, d['check'])
"
