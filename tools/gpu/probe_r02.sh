# Round-2 first call: probe the box for Eigen, record the host CPU, run GPU tests + default bench
mkdir -p gpurun_out
{ echo "== eigen"; ls -d /usr/include/eigen3 /usr/local/include/eigen3 2>&1; find / -name Core -path '*Eigen*' -not -path '/proc/*' 2>/dev/null | head;
  echo "== cpu"; lscpu | head -20; nproc; echo "== gpu"; nvidia-smi -L; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/probe_r02.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02a.log 2>&1; tail -2 gpurun_out/pytest_gpu_r02a.log
python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; tail -c 600 gpurun_out/bench_r02a.json
