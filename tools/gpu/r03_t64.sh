CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 4194304 64
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 4194304 64
for v in t64tm12 t64tm16; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 4194304 64 2>&1 | head -1; done
