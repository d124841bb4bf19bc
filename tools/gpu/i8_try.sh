timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sketch or gaussian or smoke or launch" > gpurun_out/pt_i8.log 2>&1; tail -3 gpurun_out/pt_i8.log; grep -E "^E " gpurun_out/pt_i8.log | head -5
for w in "1000000 128 1e14" "4194304 64 1e15"; do set -- $w
  PROF_M=$1 PROF_N=$2 PROF_KAPPA=$3 PROF_METHODS=rlu,rqr timeout 300 python tools/bench_kernels.py
  CQR_SKETCH_DMMA=1 PROF_M=$1 PROF_N=$2 PROF_KAPPA=$3 PROF_METHODS=rlu timeout 300 python tools/bench_kernels.py
done
