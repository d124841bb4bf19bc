timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sketch or gaussian" > gpurun_out/pt_i8.log 2>&1; tail -1 gpurun_out/pt_i8.log
for lib in paper_2111_11148_b200/libcqr.so tools/gpu/libcqr_nogen.so tools/gpu/libcqr_ngnsnm.so; do
  CQR_LIB=$lib python tools/sk_time.py 1000000 128 256; CQR_LIB=$lib python tools/sk_time.py 1000000 512 768; CQR_LIB=$lib python tools/sk_time.py 4194304 64 128
done
python tools/sk_time.py 4000000 256 512
