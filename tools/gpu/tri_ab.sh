for mn in "1000000 128" "4194304 64" "1000003 100" "777 40"; do
  CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py $mn; CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py $mn
done
for w in c1 c3; do
  n=$([ $w = c1 ] && echo 128 || echo 64); m=$([ $w = c1 ] && echo 1000000 || echo 4194304)
  PROF_M=$m PROF_N=$n PROF_METHODS=rlu,rqr python tools/bench_kernels.py
done
