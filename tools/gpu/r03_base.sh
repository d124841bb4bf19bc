# Session start check: GPU tests, smoke, c1 bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt_base.log 2>&1; tail -2 gpurun_out/pt_base.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --no-cpu > gpurun_out/bench_base_c1.json 2> gpurun_out/bench_base_c1.err; cut -c1-400 gpurun_out/bench_base_c1.json
