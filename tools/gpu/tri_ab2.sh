for mn in "1000000 128" "4194304 64"; do
  CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py $mn; CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py $mn
  CQR_LIB=tools/gpu/libcqr_rr64w8.so CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py $mn
done
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000003 100; CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 777 40
