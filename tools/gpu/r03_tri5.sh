CQR_LIB=tools/gpu/libcqr_tm8w12.so PROF_N=128 PROF_REPS=1 ncu --set full --clock-control none --import-source on -k regex:"trisolve_(sb|tma)" -c 1 \
  -o gpurun_out/tri_128_tm python tools/prof_tri.py > gpurun_out/tri_ncu_128_tm.log 2>&1; tail -2 gpurun_out/tri_ncu_128_tm.log
