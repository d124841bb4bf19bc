timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pt_r02e.log 2>&1; tail -3 gpurun_out/pt_r02e.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02e.log 2>&1; tail -1 gpurun_out/smoke_r02e.log
python bench.py > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err; tail -c 1500 gpurun_out/bench_r02e.json; tail -3 gpurun_out/bench_r02e.err
