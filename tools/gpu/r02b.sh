# new parity tests at the config shapes, acceptance criteria, full-size c4 orth vs the oracle
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_acceptance.py -m gpu -x -q -s > gpurun_out/pt_r02b.log 2>&1; tail -3 gpurun_out/pt_r02b.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scholqr3 or invalid or counters" > gpurun_out/pt_r02b2.log 2>&1; tail -2 gpurun_out/pt_r02b2.log
timeout 900 python tools/gpu/c4_orth.py > gpurun_out/c4_orth.json 2> gpurun_out/c4_orth.err; tail -c 800 gpurun_out/c4_orth.json; tail -3 gpurun_out/c4_orth.err
