#!/bin/bash
# Round profile capture on a GPU box (run under gpurun from the repo root):
# plain bench, launch list of one c1 factorization, ncu --set full of the top kernels.
set -u
mkdir -p gpurun_out
tag=${1:-r01}
python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python tools/prof_c1.py > gpurun_out/prof_plain_${tag}.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
    python tools/prof_c1.py > /dev/null 2>&1
PROF_REPS=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"sketch_ws_kernel|trisolve_tma|gram_leaf|lu_rot|lu_blocked|cholesky_blocked" -c 7 \
    -o gpurun_out/full_${tag} python tools/prof_c1.py > gpurun_out/ncu_full_${tag}.log 2>&1
tail -2 gpurun_out/ncu_full_${tag}.log
