PROF_M=4194304 PROF_N=64 PROF_KAPPA=1e15 PROF_METHODS=rlu python tools/bench_kernels.py > gpurun_out/plain.log 2>&1 && \
PROF_M=4194304 PROF_N=64 PROF_KAPPA=1e15 PROF_METHODS=rlu ncu --set full --clock-control none --import-source on -k regex:sketch_i8 -s 2 -c 1 -o gpurun_out/i8c3 python tools/bench_kernels.py > gpurun_out/ncu_i8.log 2>&1; tail -2 gpurun_out/ncu_i8.log
