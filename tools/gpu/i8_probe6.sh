for lib in paper_2111_11148_b200/libcqr.so tools/gpu/libcqr_g24s2.so tools/gpu/libcqr_g20s4.so tools/gpu/libcqr_g24s4.so tools/gpu/libcqr_g12s4.so; do
for a in "1000000 128 256" "4000000 256 512" "4194304 64 128" "1000000 512 768"; do CQR_LIB=$lib python tools/sk_time.py $a; done; done
