for lib in paper_2111_11148_b200/libcqr.so tools/gpu/libcqr_g24.so tools/gpu/libcqr_g8.so; do
for w in "1000000 128 1e14" "4194304 64 1e15"; do set -- $w
  echo $lib; CQR_LIB=$lib PROF_M=$1 PROF_N=$2 PROF_KAPPA=$3 PROF_METHODS=rlu timeout 300 python tools/bench_kernels.py
done; done
