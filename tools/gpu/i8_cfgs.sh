for w in "1000000 128 1e14" "4000000 256 1e12" "4194304 64 1e15" "1000000 512 two-segment"; do set -- $w
  m=rlu; [ $2 = 256 -o $2 = 64 ] && m=rqr
  PROF_M=$1 PROF_N=$2 PROF_KAPPA=$3 PROF_METHODS=$m PROF_RATE=$([ $2 = 512 ] && echo 1.5 || echo 2.0) timeout 600 python tools/bench_kernels.py
  CQR_SKETCH_DMMA=1 PROF_M=$1 PROF_N=$2 PROF_KAPPA=$3 PROF_METHODS=$m PROF_RATE=$([ $2 = 512 ] && echo 1.5 || echo 2.0) timeout 600 python tools/bench_kernels.py
done
