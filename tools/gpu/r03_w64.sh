CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 128
for v in w64a w64b; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v timeout 60 python tools/tri_ab.py 1000000 128; done
CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 100003 128
for v in w64a; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v timeout 60 python tools/tri_ab.py 100003 128; done
