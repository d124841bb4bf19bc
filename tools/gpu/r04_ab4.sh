# same-call A/B: main (candidate) vs prev, two rounds; sketch tests on main
for r in 1 2; do
  for cfg in "1000000 128 256" "4194304 64 128" "4000000 256 512" "1000000 512 768"; do
    timeout 120 python tools/sk_time.py $cfg; CQR_LIB=tools/gpu/libcqr_prev.so timeout 120 python tools/sk_time.py $cfg
  done
done 2>&1 | grep "sketch\|rror" | tee gpurun_out/r04_ab4.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -k "sketch or config_shape or gaussian or box_muller or rng" 2>&1 | tail -3 | tee -a gpurun_out/r04_ab4.txt
