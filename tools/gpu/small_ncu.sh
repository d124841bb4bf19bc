# ncu --set full of the small factorization kernels on the c1 path
PROF_REPS=1 ncu --set full --clock-control none --import-source on \
  -k regex:"lu_reg|lu_blocked|cholesky_kernel|cholesky_blocked" --launch-skip 4 -c 2 \
  -o gpurun_out/small python tools/prof_c1.py > gpurun_out/small_ncu.log 2>&1; tail -2 gpurun_out/small_ncu.log
