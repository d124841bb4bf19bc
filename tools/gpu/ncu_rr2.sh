python tools/tri_ab.py 1000000 128 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:trisolve_rr -s 2 -c 1 -o gpurun_out/rr128b python tools/tri_ab.py 1000000 128 > gpurun_out/ncu_rr.log 2>&1; tail -1 gpurun_out/ncu_rr.log
