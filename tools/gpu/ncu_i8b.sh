CQR_LIB=tools/gpu/libcqr_nogen.so python tools/sk_time.py 1000000 128 256 > gpurun_out/plain.log 2>&1 && \
CQR_LIB=tools/gpu/libcqr_nogen.so ncu --set full --clock-control none --import-source on -k regex:sketch_i8 -s 2 -c 1 -o gpurun_out/i8nogen python tools/sk_time.py 1000000 128 256 > gpurun_out/ncu_i8.log 2>&1; tail -1 gpurun_out/ncu_i8.log
