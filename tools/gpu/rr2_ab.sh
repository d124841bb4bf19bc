# n = 128 trisolve: bitwise against the left-looking kernel, times of the pair kernel / single-warp rr / left-looking
CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 128
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 1000000 128
CQR_RR128_SINGLE=1 CQR_TRISOLVE_VARIANT=1x python tools/tri_ab.py 1000000 128 2>&1 | head -1
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 100003 128
CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 100003 128
CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py 100003 128
