./tools/probe/warpid_probe
PROF_N=128 PROF_REPS=1 ncu --set full --clock-control none --import-source on -k regex:"trisolve_split" -c 1 -o gpurun_out/tri_split python tools/prof_tri.py > gpurun_out/tri_split.log 2>&1; tail -1 gpurun_out/tri_split.log
