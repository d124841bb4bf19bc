# Round capture: GPU tests, smoke, bench lines c1-c4, c1 launch list + ncu --set full of the top kernels
tag=${1:-r01j}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${tag}.log 2>&1; tail -2 gpurun_out/pytest_gpu_${tag}.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; tail -1 gpurun_out/smoke_${tag}.log
for w in c2 c3 c4; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_${tag}_$w.json 2> gpurun_out/bench_${tag}_$w.err; done
bash tools/profile_round.sh ${tag}
python -c "
import json
for f in ['gpurun_out/bench_${tag}.json'] + ['gpurun_out/bench_${tag}_%s.json' % w for w in ('c2','c3','c4')]:
    d = json.load(open(f)); print(f, round(d['ms_per_step'], 3), round(d['value'], 2), {k: round(v, 3) for k, v in d['stage_ms'].items()})
"
