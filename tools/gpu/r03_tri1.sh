# trisolve n=128: stagger A/B + ncu full capture with stall sampling
CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 128
for s in 2000 8000 26000; do CQR_LIB=tools/gpu/libcqr_st$s.so CQR_TRISOLVE_VARIANT=st$s python tools/tri_ab.py 1000000 128; done
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 128
PROF_N=128 PROF_REPS=1 ncu --set full --clock-control none --import-source on -k regex:"trisolve_(sb|tma)" -c 1 \
  -o gpurun_out/tri_128 python tools/prof_tri.py > gpurun_out/tri_ncu_128.log 2>&1; tail -2 gpurun_out/tri_ncu_128.log
