timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt_tri.log 2>&1; tail -3 gpurun_out/pt_tri.log
for v in ${VARIANTS:-0 7}; do for n in ${NS:-64 128 256 512}; do CQR_TRISOLVE_VARIANT=$v PROF_N=$n timeout 120 python tools/prof_tri.py 2>&1 | tail -1 | sed "s/^/v$v /"; done; done
