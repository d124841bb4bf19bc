for v in g_s4 g_ns g_s2; do
  L=tools/gpu/libcqr_$v.so
  CQR_LIB=$L python tools/sk_time.py 1000000 128 256 2>&1 | tail -1; CQR_LIB=$L python tools/sk_time.py 4194304 64 128 2>&1 | tail -1
done
