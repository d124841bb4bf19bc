CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 128
for v in tm8w8 tm8w10 tm8w12; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v python tools/tri_ab.py 1000000 128; done
CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 100003 128
for v in tm8w8 tm8w12; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v python tools/tri_ab.py 100003 128; done
CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 256
CQR_LIB=tools/gpu/libcqr_tm4w16n256.so CQR_TRISOLVE_VARIANT=tm4 python tools/tri_ab.py 1000000 256
