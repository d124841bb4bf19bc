CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 4194304 64
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 4194304 64
for v in rw16w16 rw16w12; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v python tools/tri_ab.py 4194304 64; done
