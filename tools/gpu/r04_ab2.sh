# same-call A/B: main vs the slicer with one exact scaling and no row select (om), alternating, two rounds; parity tests on om
for r in 1 2; do
  for cfg in "1000000 128 256" "4194304 64 128" "4000000 256 512" "1000000 512 768"; do
    timeout 120 python tools/sk_time.py $cfg; CQR_LIB=tools/gpu/libcqr_om.so timeout 120 python tools/sk_time.py $cfg
  done
done 2>&1 | grep "sketch\|rror" | tee gpurun_out/r04_ab2.txt
CQR_LIB=tools/gpu/libcqr_om.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -k "sketch or config_shape or gaussian or non_finite or sweep" 2>&1 | tail -3 | tee -a gpurun_out/r04_ab2.txt
