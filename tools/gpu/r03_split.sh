CQR_TRISOLVE_VARIANT=2 CQR_TRI_NO_SPLIT=1 python tools/tri_ab.py 1000000 128
CQR_TRISOLVE_VARIANT=0 timeout 60 python tools/tri_ab.py 1000000 128
CQR_TRI_NO_SPLIT=1 CQR_TRISOLVE_VARIANT=nosplit python tools/tri_ab.py 1000000 128
CQR_TRISOLVE_VARIANT=2 CQR_TRI_NO_SPLIT=1 python tools/tri_ab.py 100003 128
CQR_TRISOLVE_VARIANT=0 timeout 60 python tools/tri_ab.py 100003 128
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "trisolve" 2>&1 | tail -2
