CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 128
for v in tm8w12 sync2 sync2n; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v timeout 60 python tools/tri_ab.py 1000000 128; done
