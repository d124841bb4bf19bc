python tools/sk_time.py 1000000 512 768 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_i8 -s 1 -c 1 -o gpurun_out/i8c4 python tools/sk_time.py 1000000 512 768 > gpurun_out/ncu_i8.log 2>&1; tail -1 gpurun_out/ncu_i8.log
