for lib in paper_2111_11148_b200/libcqr.so tools/gpu/libcqr_w8a.so tools/gpu/libcqr_w8b.so tools/gpu/libcqr_w8c.so; do
  echo $lib; CQR_LIB=$lib CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 128; CQR_LIB=$lib CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 512; CQR_LIB=$lib CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py 1000000 256
done
