CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 128
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 128
CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 256
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 256
