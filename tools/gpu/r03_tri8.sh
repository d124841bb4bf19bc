for i in 1 2; do
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 128
CQR_LIB=tools/gpu/libcqr_late.so CQR_TRISOLVE_VARIANT=late python tools/tri_ab.py 1000000 128 | head -1
done
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 256
CQR_LIB=tools/gpu/libcqr_late.so CQR_TRISOLVE_VARIANT=late python tools/tri_ab.py 1000000 256 | head -1
