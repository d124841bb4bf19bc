for v in NOBW NOBWLL NOBOTH; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v python tools/tri_ab.py 1000000 128 2>/dev/null | head -1; done
for v in NOBW NOBWLL; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v python tools/tri_ab.py 1000000 512 2>/dev/null | head -1; done
