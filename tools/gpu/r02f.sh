timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pt_r02f.log 2>&1; tail -3 gpurun_out/pt_r02f.log; grep -E "^FAILED" gpurun_out/pt_r02f.log | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02f.log 2>&1; tail -1 gpurun_out/smoke_r02f.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r02f.json')); print(d['ms_per_step'], d['value'], d['check'], d['e2e']['ms_per_step'], d['comparison'])"
