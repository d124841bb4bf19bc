# ncu --set full of the default trisolve kernel at the c1 shape (n from $1, default 128)
n=${1:-128}
PROF_N=$n python tools/prof_tri.py && \
PROF_N=$n PROF_REPS=1 ncu --set full --clock-control none --import-source on -k regex:"trisolve_(sb|tma)" -c 1 \
  -o gpurun_out/tri_$n python tools/prof_tri.py > gpurun_out/tri_ncu_$n.log 2>&1; tail -2 gpurun_out/tri_ncu_$n.log
