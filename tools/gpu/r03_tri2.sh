# trisolve phase bounds at n=128 (probe builds; not bitwise)
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 128
for v in NOLL NODIAG NOBOTH; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v python tools/tri_ab.py 1000000 128 2>/dev/null | head -1; done
for v in NOLL NODIAG NOBOTH; do CQR_LIB=tools/gpu/libcqr_$v.so CQR_TRISOLVE_VARIANT=$v python tools/tri_ab.py 1000000 512 2>/dev/null | head -1; done
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 512
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 256
