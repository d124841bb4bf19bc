for lib in paper_2111_11148_b200/libcqr.so tools/gpu/libcqr_st2a6.so tools/gpu/libcqr_a2.so tools/gpu/libcqr_g8.so tools/gpu/libcqr_sl4.so tools/gpu/libcqr_g12.so; do
  CQR_LIB=$lib python tools/sk_time.py 1000000 128 256; CQR_LIB=$lib python tools/sk_time.py 1000000 512 768; CQR_LIB=$lib python tools/sk_time.py 4194304 64 128
done
